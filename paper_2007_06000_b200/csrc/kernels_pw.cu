// Pointwise-conv GEMM kernel for sm_100a (see pw_params.hpp): 1x1 convs as
// one GEMM over all pixels of the launch (rows = images x H x W, K = input
// channels, N = output channels), tcgen05 with the fp32 accumulator in TMEM.
//   warp 4  producer: the channel group's packed weights once (resident),
//           then 128-row x 128-byte A chunks through a 4-stage TMA ring
//           (SWIZZLE_128B), M tile after M tile;
//   warp 5  MMA issuer (one thread): per M tile, every K step of every chunk
//           into accumulator set j & 1 (two sets: tile j+1's MMAs run while
//           tile j drains);
//   warps 0-3 epilogue: thread t = TMEM lane t = row t of the M tile: bias +
//           ReLU, then an NHWC store, or the global-average-pool reduction.
// The GAP epilogue sums each warp's 32 rows per column with a shuffle
// transpose-reduction, split at the (at most one) image boundary inside the
// warp, into part[warp][segment][channel]; pw_gap_finish adds an image's
// warps in order (deterministic) and scales.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "pw_params.hpp"
#include "umma.cuh"

namespace xlf {

namespace {

using namespace umma;

constexpr int kPwEpi = 256;  // two epilogue warp groups: lanes = rows, 32-column chunks alternate between the groups
constexpr int kPwThreads = kPwEpi + 64;
constexpr int kPwProd = kPwEpi / 32, kPwMma = kPwEpi / 32 + 1;  // role warps
constexpr int kStageBytes = 128 * 128;

template <class T>
struct PwElem;
template <>
struct PwElem<__nv_bfloat16> {
    static constexpr uint32_t idesc(int N) { return idesc_bf16(128, N); }
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_bf16(t, a, b, id, acc); }
    __device__ static void store8(void* dst, const float* v) {
        uint4 u;
        __nv_bfloat162 h;
        h = __floats2bfloat162_rn(v[0], v[1]), u.x = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[2], v[3]), u.y = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[4], v[5]), u.z = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[6], v[7]), u.w = *reinterpret_cast<uint32_t*>(&h);
        *reinterpret_cast<uint4*>(dst) = u;
    }
    static constexpr int cpc = 8;
};
template <>
struct PwElem<float> {
    static constexpr uint32_t idesc(int N) { return idesc_tf32(128, N); }
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_tf32(t, a, b, id, acc); }
    __device__ static void store8(void* dst, const float* v) {
        float4* d = reinterpret_cast<float4*>(dst);
        d[0] = make_float4(round_tf32(v[0]), round_tf32(v[1]), round_tf32(v[2]), round_tf32(v[3]));
        d[1] = make_float4(round_tf32(v[4]), round_tf32(v[5]), round_tf32(v[6]), round_tf32(v[7]));
    }
    static constexpr int cpc = 4;
};

__device__ __forceinline__ void tma_2d(void* smem, const void* desc, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(smem)),
        "l"(desc), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// lane l returns the sum over the warp's 32 rows of column l (v: this lane's row)
__device__ __forceinline__ float colsum32(float* v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < off; ++j) {
            const float send = upper ? v[j] : v[j + off];
            const float keep = upper ? v[j + off] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

template <class T>
__global__ void __launch_bounds__(kPwThreads, 1) pw_kernel(const __grid_constant__ PwParams P, int n0, int count) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[kPwStages], empty[kPwStages], accf[2], acce[2], wbar;  // acce: one arrival per epilogue warp
    __shared__ uint32_t tmem_slot;
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int rows = count * P.HW, mtiles = (rows + 127) / 128;
    const int row0 = n0 * P.HW;
    const int g = blockIdx.y, gch = P.gch;
    // cluster multicast (mc > 1): the mc channel groups of one M tile form a
    // cluster; rank 0 loads each A chunk once and multicasts it to all of
    // them, and frees a stage only when every CTA released it
    const int mc = P.mc > 1 ? P.mc : 1;
    const uint32_t rank = mc > 1 ? cluster_rank() : 0u;
    const uint16_t all = uint16_t((1u << mc) - 1u), rel = uint16_t((1u << rank) | 1u);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPwStages; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], rank == 0 ? uint32_t(mc) : 1u);
        for (int a = 0; a < 2; ++a) mbar_init(&accf[a], 1), mbar_init(&acce[a], kPwEpi / 32);
        mbar_init(&wbar, 1);
        mbar_fence_init();
    }
    if (warp == kPwMma) tmem_alloc(&tmem_slot, uint32_t(P.tmem_cols));
    fence_before();
    __syncthreads();
    if (mc > 1) cluster_sync();  // peers' barriers initialised before any multicast / remote arrival
    fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t ring = smem_u32(smem + P.ring_off), wsm = smem_u32(smem + P.w_off);

    if (warp == kPwProd) {
        if (lane == 0) {
            const uint32_t wb = uint32_t(P.ksteps) * uint32_t(gch) * 32u;
            mbar_expect_tx(&wbar, wb);
            const uint8_t* src = P.wmma + P.gwb * g;
            for (uint32_t o = 0; o < wb; o += 65536) bulk_g2s(smem + P.w_off + o, src + o, min(65536u, wb - o), &wbar);
            asm volatile("griddepcontrol.wait;" ::: "memory");  // A is the previous step's output
            const int kc_elems = 128 / P.es;
            int it = 0;
            for (int m = blockIdx.x; m < mtiles; m += gridDim.x)
                for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                    const int s = it % kPwStages;
                    if (it >= kPwStages) mbar_sleep_wait(&empty[s], uint32_t(it / kPwStages - 1) & 1u);
                    mbar_expect_tx(&full[s], kStageBytes);
                    if (mc == 1) tma_2d(smem + P.ring_off + s * kStageBytes, &P.amap, P.coff_in + kc * kc_elems, row0 + m * 128, &full[s]);
                    else if (rank == 0)
                        tma_load_2d_mc(smem + P.ring_off + s * kStageBytes, &P.amap, P.coff_in + kc * kc_elems, row0 + m * 128, &full[s], all);
                }
            // the leader consumes every stage's last release (remote arrivals) before it may exit
            if (mc > 1 && rank == 0)
                for (int k = max(0, it - kPwStages); k < it; ++k) mbar_sleep_wait(&empty[k % kPwStages], uint32_t(k / kPwStages) & 1u);
        }
    } else if (warp == kPwMma) {
        if (elect_one()) {
            mbar_sleep_wait(&wbar, 0);
            const uint32_t idesc = PwElem<T>::idesc(gch);
            const uint64_t bdesc0 = sdesc(wsm, uint32_t(gch) * 16u, 128u, kNoSwizzle);
            const uint32_t bstep = (uint32_t(gch) * 32u) >> 4;  // one K step of B, 16-byte units
            int it = 0, j = 0;
            for (int m = blockIdx.x; m < mtiles; m += gridDim.x, ++j) {
                const int a = j & 1;
                if (j >= 2) mbar_wait(&acce[a], uint32_t((j >> 1) - 1) & 1u);
                fence_after();
                const uint32_t d = tmem + uint32_t(a * gch);
                uint32_t acc = 0;
                uint64_t bd = bdesc0;
                for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                    const int s = it % kPwStages;
                    mbar_wait(&full[s], uint32_t(it / kPwStages) & 1u);
                    fence_after();
                    const int steps = min(4, P.ksteps - kc * 4);
                    const uint64_t ad = sdesc(ring + uint32_t(s * kStageBytes), 16u, 1024u, kSW128);
                    for (int k = 0; k < steps; ++k) {
                        PwElem<T>::mma(d, ad + uint64_t(k * 2), bd, idesc, acc);  // +32 bytes inside the 128-byte swizzle row
                        acc = 1;
                        bd += bstep;
                    }
                    if (mc == 1) commit(&empty[s]);
                    else commit_mc(&empty[s], rel);  // own stage (pacing this CTA's expect_tx) + the leader's
                }
                commit(&accf[a]);
            }
        }
        __syncwarp();
    } else {
        const int t = threadIdx.x & 127, half = threadIdx.x >> 7;  // TMEM lane / row; column-chunk parity
        float* bias = reinterpret_cast<float*>(smem + P.bias_off);
        for (int k = threadIdx.x; k < gch; k += kPwEpi) bias[k] = g * gch + k < P.cout ? __ldg(P.bias + g * gch + k) : 0.0f;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("bar.sync 1, %0;\n" ::"n"(kPwEpi) : "memory");
        constexpr int cpc = PwElem<T>::cpc;
        const int cend = min(gch, (P.cout + cpc - 1) / cpc * cpc - g * gch);  // channels of this group to store
        const int ntot = P.nsplit * gch;
        const uint32_t tl = uint32_t(t & ~31) << 16;
        const uint32_t bias_s = smem_u32(bias);
        int j = 0;
        for (int m = blockIdx.x; m < mtiles; m += gridDim.x, ++j) {
            const int a = j & 1;
            mbar_sleep_wait(&accf[a], uint32_t(j >> 1) & 1u);
            fence_after();
            const int r = m * 128 + t;  // launch-relative row
            const bool valid = r < rows;
            // GAP: the warp's rows [rw, rw + 32) split at the image boundary (warp-uniform)
            const int rw = m * 128 + (t & ~31);
            const int bnd = P.gap ? (rw / P.HW + 1) * P.HW - rw : 32;  // lanes < bnd: the first image
            T* dst = static_cast<T*>(P.out) + size_t(row0 + r) * P.out_cstride + P.out_coff + g * gch;
            for (int c0 = 32 * half; c0 < gch; c0 += 64) {
                float v[32];
                const int nc = min(32, gch - c0);
                if (nc == 32) tmem_ld32(tmem + tl + uint32_t(a * gch + c0), v);
                else {
                    tmem_ld16(tmem + tl + uint32_t(a * gch + c0), v);
#pragma unroll
                    for (int k = 16; k < 32; ++k) v[k] = 0.0f;
                }
#pragma unroll
                for (int k = 0; k < 32; k += 4) {
                    float4 b4;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(b4.x), "=f"(b4.y), "=f"(b4.z), "=f"(b4.w)
                                 : "r"(bias_s + uint32_t(min(c0 + k, gch - 4)) * 4u));
                    v[k] += b4.x, v[k + 1] += b4.y, v[k + 2] += b4.z, v[k + 3] += b4.w;
                }
                if (P.relu)
#pragma unroll
                    for (int k = 0; k < 32; ++k) v[k] = fmaxf(v[k], 0.0f);
                if (!P.gap) {
                    if (valid)
#pragma unroll
                        for (int k = 0; k < 32; k += 8)
                            if (c0 + k < cend) PwElem<T>::store8(dst + c0 + k, v + k);
                } else {
                    float* pp = P.gap_part + size_t(rw / 32) * 2 * ntot + g * gch + c0 + lane;
                    if (bnd >= 32) {  // the whole warp inside one image
#pragma unroll
                        for (int k = 0; k < 32; ++k) v[k] = valid && k < nc ? v[k] : 0.0f;
                        const float s0 = colsum32(v);
                        if (lane < nc) pp[0] = s0, pp[ntot] = 0.0f;
                    } else {
                        float v1[32];
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            const bool in = valid && k < nc;
                            v1[k] = in && lane >= bnd ? v[k] : 0.0f;
                            v[k] = in && lane < bnd ? v[k] : 0.0f;
                        }
                        const float s0 = colsum32(v), s1 = colsum32(v1);
                        if (lane < nc) pp[0] = s0, pp[ntot] = s1;
                    }
                }
            }
            fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acce[a]);
        }
    }
    fence_before();
    __syncthreads();
    if (mc > 1) cluster_sync();
    fence_after();
    if (warp == kPwMma) tmem_free(tmem, uint32_t(P.tmem_cols));
}

// out[n][coff + c] = scale * sum of image n's warp partials (launch-relative
// warps (n*HW)/32 .. ((n+1)*HW-1)/32, segment 0 when the warp starts inside n)
template <class T>
__global__ void pw_gap_finish(const float* __restrict__ part, int HW, int ntot, int C, float scale, T* __restrict__ out, int cs, int coff,
                              int n0, int count) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (long long)count * C; i += (long long)gridDim.x * blockDim.x) {
        const int n = int(i / C), c = int(i % C);
        const int w0 = n * HW / 32, w1 = ((n + 1) * HW - 1) / 32;
        float acc = 0.0f;
        for (int w = w0; w <= w1; ++w) acc += part[(size_t(w) * 2 + ((w * 32) / HW == n ? 0 : 1)) * ntot + c];
        const float y = acc * scale;
        if constexpr (sizeof(T) == 2) out[size_t(n0 + n) * cs + coff + c] = __float2bfloat16(y);
        else out[size_t(n0 + n) * cs + coff + c] = round_tf32(y);
    }
}

template <class T>
cudaError_t launch_t(const PwParams& P, int n0, int count, cudaStream_t st) {
    static bool init = false;
    if (!init) {
        cudaError_t e = cudaFuncSetAttribute(pw_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 - 2048);
        if (e != cudaSuccess) return e;
        init = true;
    }
    const int mtiles = (count * P.HW + 127) / 128;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int gx = std::max(1, std::min(mtiles, sms * std::max(1, P.ctas_per_sm) / std::max(1, P.nsplit)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(gx), unsigned(std::max(1, P.nsplit)), 1u), cfg.blockDim = dim3(kPwThreads);
    cfg.dynamicSmemBytes = size_t(P.smem_bytes), cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = P.pdl ? 1 : 0;
    cfg.attrs = attr, cfg.numAttrs = 1;
    if (P.mc > 1) {  // the channel groups of an M tile as one cluster; as many clusters as can be resident
        attr[1].id = cudaLaunchAttributeClusterDimension;
        attr[1].val.clusterDim.x = 1, attr[1].val.clusterDim.y = unsigned(P.mc), attr[1].val.clusterDim.z = 1;
        cfg.numAttrs = 2;
        static int max_clusters = 0;
        if (!max_clusters) {
            cudaLaunchConfig_t q = cfg;
            q.gridDim = dim3(unsigned(sms), unsigned(P.mc), 1u);
            if (cudaOccupancyMaxActiveClusters(&max_clusters, pw_kernel<T>, &q) != cudaSuccess || max_clusters < 1) max_clusters = 1;
        }
        gx = std::max(1, std::min(mtiles, max_clusters));
        cfg.gridDim.x = unsigned(gx);
    }
    cudaLaunchKernelEx(&cfg, pw_kernel<T>, P, n0, count);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_pw(const PwParams& P, int n0, int count, cudaStream_t st) {
    return P.es == 4 ? launch_t<float>(P, n0, count, st) : launch_t<__nv_bfloat16>(P, n0, count, st);
}

cudaError_t launch_pw_gap_finish(const PwParams& P, int C, float scale, void* out, int cs, int coff, int n0, int count, cudaStream_t st) {
    const long long work = (long long)count * C;
    const int grid = int(std::min<long long>((work + 255) / 256, 148 * 8));
    if (P.es == 4)
        pw_gap_finish<float><<<grid, 256, 0, st>>>(P.gap_part, P.HW, P.nsplit * P.gch, C, scale, static_cast<float*>(out), cs, coff, n0, count);
    else
        pw_gap_finish<__nv_bfloat16><<<grid, 256, 0, st>>>(P.gap_part, P.HW, P.nsplit * P.gch, C, scale, static_cast<__nv_bfloat16*>(out), cs,
                                                           coff, n0, count);
    return cudaGetLastError();
}

}  // namespace xlf
