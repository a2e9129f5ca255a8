// "Stem" kernel for sm_100a: the first conv of a network (stride 2 on the
// image, rewritten by the engine as a stride-1 conv on the space-to-depth
// input) -> bias -> ReLU -> 3x3/2 max-pool (zero pad 0), one kernel, the conv
// output never leaves the SM (SqueezeNet conv1 + pool1: 111x111x64 per image).
//
// Why its own kernel: the generic fused-block kernel (kernels_tc.cu) stages
// the conv output of a 2-D tile in shared memory and runs the pool as a SIMT
// loop over it; for this layer that is ~0.5 M warp instructions per image
// (ncu: issue-bound, tensor pipe 7 %, DRAM 8 %).  Here the GEMM's M dimension
// is ONE conv output row (TMEM lane t = conv column t, <= 128 columns), so
//   * the vertical half of the pool is a register max over consecutive conv
//     rows held by the same thread (rows 2i, 2i+1, 2i+2 -> pooled row i; the
//     shared even row is reused, never recomputed),
//   * only the finished vertical maxima (one row per pooled row) go through
//     shared memory, where the horizontal 3/2 max + bias + ReLU run chunk-wise
//     (16-byte chunks) with 128-byte coalesced NHWC stores,
//   * max commutes with the monotone per-channel bias + ReLU and with the
//     round-to-bf16, so bias and ReLU are applied once per POOLED value.
// Input rows stream through a TMA ring (the engine stores the space-to-depth
// input row-planar, so one row's 16-byte channel planes are one contiguous run
// and one 2-D box); weights and bias are resident.  Lanes past the conv width
// read past their row's planes (garbage, never stored).  Warps: 0-3 epilogue (128 threads
// = 128 TMEM lanes), 4 TMA producer, 5 MMA issuer (one elected thread).
// Work unit = (image, band of pooled rows); persistent CTAs walk units.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>

#include "stem_params.hpp"
#include "umma.cuh"

namespace xlf {

namespace {

using namespace umma;

__device__ __forceinline__ void tma_load_2d(void* smem, const void* desc, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(smem)),
        "l"(desc), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <class T>
struct SElem;

template <>
struct SElem<__nv_bfloat16> {
    static constexpr int cpc = 8;
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_bf16(t, a, b, id, acc); }
    static constexpr uint32_t idesc(int N) { return idesc_bf16(128, N); }
    __device__ static uint32_t pack2(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    __device__ static float2 unpack2(uint32_t u) { return __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u)); }
    __device__ static uint32_t max2(uint32_t a, uint32_t b) {
        __nv_bfloat162 m = __hmax2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
        return *reinterpret_cast<uint32_t*>(&m);
    }
};

template <>
struct SElem<float> {
    static constexpr int cpc = 4;
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_tf32(t, a, b, id, acc); }
    static constexpr uint32_t idesc(int N) { return idesc_tf32(128, N); }
    __device__ static uint32_t max2(uint32_t a, uint32_t b) { return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b))); }
};

constexpr int kEpiThreads = 128;
constexpr int kStemThreads = kEpiThreads + 64;  // + producer warp + MMA warp

__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kEpiThreads) : "memory"); }

__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// Band u of the persistent walk: image n, pooled rows [i0, i1).
struct Band {
    int n, i0, i1;
};
__device__ __forceinline__ Band band_of(const StemParams& P, int u, int n0) {
    Band b;
    const int img = u / P.bands, k = u - img * P.bands;
    b.n = n0 + img;
    b.i0 = k * P.band_rows;
    b.i1 = min(b.i0 + P.band_rows, P.Hp);
    return b;
}
// conv rows of a band: 2*i0 .. 2*i1 (inclusive), input rows 2*i0 .. 2*i1 + kh - 1
__device__ __forceinline__ int conv_rows(const Band& b) { return 2 * (b.i1 - b.i0) + 1; }

// Vertical maxima of one pooled row (per thread: one conv column; columns
// [32h, 32h+32) of the accumulator, as T) -> stage buffer (16-byte chunks rotated by the column so the
// per-thread 16-byte stores of a warp spread over all banks).
template <class T, int NCH>
__device__ __forceinline__ void stage_part(uint32_t stage, int t, int h, const float* w) {
    constexpr int cpc = SElem<T>::cpc, chunks = NCH * 32 / cpc, per = 32 / cpc;
    const uint32_t row = stage + uint32_t(t) * chunks * 16u;
#pragma unroll
    for (int q = 0; q < per; ++q) {
        const int c = h * per + q;
        uint4 u;
        if constexpr (cpc == 8) {
            u.x = SElem<T>::pack2(w[q * 8 + 0], w[q * 8 + 1]), u.y = SElem<T>::pack2(w[q * 8 + 2], w[q * 8 + 3]);
            u.z = SElem<T>::pack2(w[q * 8 + 4], w[q * 8 + 5]), u.w = SElem<T>::pack2(w[q * 8 + 6], w[q * 8 + 7]);
        } else {
            u = make_uint4(__float_as_uint(w[q * 4]), __float_as_uint(w[q * 4 + 1]), __float_as_uint(w[q * 4 + 2]),
                           __float_as_uint(w[q * 4 + 3]));
        }
        sts128(row + uint32_t(((c + t) % chunks) * 16), u);
    }
}

// Horizontal 3/2 max of the staged row + bias + ReLU -> NHWC pooled row.
// Thread t owns chunk c = t % chunks of pooled columns j = t / chunks + k *
// (128 / chunks) (chunks | 128: c and its bias are fixed per thread); `out`
// points at the pooled row's pixel 0, channel 0 (concat offset applied).
template <class T, int NCH>
__device__ __forceinline__ void emit_row(const StemParams& P, uint32_t stage, const float* bias, int c, T* out) {
    constexpr int cpc = SElem<T>::cpc, chunks = NCH * 32 / cpc, jstep = kEpiThreads / chunks;
    static_assert(kEpiThreads % chunks == 0, "chunks per pixel must divide 128");
    const int t = threadIdx.x;
    const int cend = (P.cout + cpc - 1) / cpc;  // chunks holding real channels (+ their zero padding)
    if (c >= cend) return;
    const int cs = P.out_cstride;
    for (int j = t / chunks; j < P.Wp; j += jstep) {
        const int x0 = 2 * j;
        const uint32_t r0 = stage + uint32_t(x0 * chunks) * 16u;
        const uint4 a = lds128(r0 + uint32_t((c + x0) % chunks) * 16u);
        const uint4 b = lds128(r0 + uint32_t(chunks + (c + x0 + 1) % chunks) * 16u);
        const uint4 d = lds128(r0 + uint32_t(2 * chunks + (c + x0 + 2) % chunks) * 16u);
        uint4 m;
        m.x = SElem<T>::max2(SElem<T>::max2(a.x, b.x), d.x), m.y = SElem<T>::max2(SElem<T>::max2(a.y, b.y), d.y);
        m.z = SElem<T>::max2(SElem<T>::max2(a.z, b.z), d.z), m.w = SElem<T>::max2(SElem<T>::max2(a.w, b.w), d.w);
        uint4 o;
        if constexpr (cpc == 8) {
            float2 p;
            p = SElem<T>::unpack2(m.x), o.x = SElem<T>::pack2(fmaxf(p.x + bias[0], 0.0f), fmaxf(p.y + bias[1], 0.0f));
            p = SElem<T>::unpack2(m.y), o.y = SElem<T>::pack2(fmaxf(p.x + bias[2], 0.0f), fmaxf(p.y + bias[3], 0.0f));
            p = SElem<T>::unpack2(m.z), o.z = SElem<T>::pack2(fmaxf(p.x + bias[4], 0.0f), fmaxf(p.y + bias[5], 0.0f));
            p = SElem<T>::unpack2(m.w), o.w = SElem<T>::pack2(fmaxf(p.x + bias[6], 0.0f), fmaxf(p.y + bias[7], 0.0f));
        } else {
            o.x = __float_as_uint(round_tf32(fmaxf(__uint_as_float(m.x) + bias[0], 0.0f)));
            o.y = __float_as_uint(round_tf32(fmaxf(__uint_as_float(m.y) + bias[1], 0.0f)));
            o.z = __float_as_uint(round_tf32(fmaxf(__uint_as_float(m.z) + bias[2], 0.0f)));
            o.w = __float_as_uint(round_tf32(fmaxf(__uint_as_float(m.w) + bias[3], 0.0f)));
        }
        *reinterpret_cast<uint4*>(out + size_t(j) * cs + c * cpc) = o;
    }
}

#ifdef XLF_STEM_PROF
#define PROF_T0 long long _t0 = clock64();
#define PROF_ADD(v) v += clock64() - _t0;
#else
#define PROF_T0
#define PROF_ADD(v)
#endif

template <class T, int NCH>
__global__ void __launch_bounds__(kStemThreads, 2) stem_kernel(const __grid_constant__ StemParams P, int batch, int n0) {
    constexpr int N = NCH * 32;  // accumulator columns per conv row (npad)
    // ring / accumulator depths are compile-time powers of two: slot and
    // phase of the k-th use are a mask and a shift, not a division
    constexpr int S = kStemSlots, SL = 3, Acc = NCH == 2 ? 4 : 2, AccL = NCH == 2 ? 2 : 1;
    static_assert((1 << SL) == S && (1 << AccL) == Acc, "powers of two");
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[kStemMaxSlots], empty[kStemMaxSlots], accf[kStemMaxAcc], acce[kStemMaxAcc], wbar;
    __shared__ uint32_t tmem_slot;
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int units = batch * P.bands;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
        for (int a = 0; a < Acc; ++a) mbar_init(&accf[a], 1), mbar_init(&acce[a], kEpiThreads / 32);
        mbar_init(&wbar, 1);
        mbar_fence_init();
    }
    if (warp == 5) tmem_alloc(&tmem_slot, uint32_t(P.tmem_cols));
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t sbase = smem_u32(smem);
#ifdef XLF_STEM_PROF
    long long w_empty = 0, w_full = 0, w_acce = 0, w_accf = 0, w_sync = 0;
    const long long t_start = clock64();
#endif
    const uint32_t ring = sbase + uint32_t(P.ring_off), wsm = sbase + uint32_t(P.w_off);
    const uint32_t stage0 = sbase + uint32_t(P.stage_off);

    if (warp == 4) {
        // ---------------------------------------------------------------- TMA producer
        if (lane == 0) {
            mbar_expect_tx(&wbar, uint32_t(P.w_bytes));
            for (int o = 0; o < P.w_bytes; o += 32768) bulk_g2s(smem + P.w_off + o, P.wmma + o, uint32_t(min(32768, P.w_bytes - o)), &wbar);
            asm volatile("griddepcontrol.wait;" ::: "memory");  // the input is the previous step's output
            const uint32_t row_bytes = uint32_t(P.planes) * uint32_t(P.Win) * 16u;
            int q = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const Band b = band_of(P, u, n0);
                const int rows = conv_rows(b) + P.kh - 1;
                for (int r = 0; r < rows; ++r, ++q) {
                    const int s = q & (S - 1);
                    PROF_T0
                    if (q >= S) mbar_wait(&empty[s], uint32_t((q >> SL) - 1) & 1u);
                    PROF_ADD(w_empty)
                    mbar_expect_tx(&full[s], row_bytes);
                    tma_load_2d(smem + P.ring_off + s * P.slot_bytes, &P.xmap, 0, ((b.n * P.Hin) + 2 * b.i0 + r) * P.row_lines, &full[s]);
                }
            }
        }
    } else if (warp == 5) {
        // ---------------------------------------------------------------- MMA issuer
        if (elect_one()) {
            mbar_wait(&wbar, 0);
            const uint32_t idesc = SElem<T>::idesc(N);
            const int kpt = P.planes / 2;  // 32-byte K steps per tap
            const uint64_t bdesc0 = sdesc(0, uint32_t(N) * 16u, 128u, kNoSwizzle);
            int q = 0, c = 0;  // input rows loaded so far (ring position of this band's first row), conv rows issued
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const Band b = band_of(P, u, n0);
                const int nconv = conv_rows(b);
                for (int lr = 0; lr < nconv; ++lr, ++c) {
                    // input rows lr .. lr + kh - 1 of the band; the newest one (or all, first row) must have landed
                    for (int ty = lr == 0 ? 0 : P.kh - 1; ty < P.kh; ++ty) {
                        const int qq = q + lr + ty;
                        PROF_T0
                        mbar_wait(&full[qq & (S - 1)], uint32_t(qq >> SL) & 1u);
                        PROF_ADD(w_full)
                    }
                    const int a = c & (Acc - 1);
                    { PROF_T0
                    if (c >= Acc) mbar_wait(&acce[a], uint32_t((c >> AccL) - 1) & 1u);
                    PROF_ADD(w_acce) }
                    fence_after();
                    PROF_T0
                    const uint32_t d = tmem + uint32_t(a * N);
                    uint32_t acc = 0;
                    for (int ty = 0; ty < P.kh; ++ty) {
                        const uint32_t rowbase = ring + uint32_t(((q + lr + ty) & (S - 1)) * P.slot_bytes);
                        for (int tx = 0; tx < P.kw; ++tx)
                            for (int k = 0; k < kpt; ++k) {
                                // A: 128 consecutive pixels from column tx, chunks 2k, 2k+1 (planes)
                                const uint64_t ad = sdesc(rowbase + uint32_t(tx * 16 + 2 * k * P.plane_bytes), uint32_t(P.plane_bytes), 128u, kNoSwizzle);
                                const uint32_t boff = uint32_t(((ty * P.kw + tx) * P.planes + 2 * k) * N * 16);
                                SElem<T>::mma(d, ad, bdesc0 + ((wsm + boff) >> 4), idesc, acc);
                                acc = 1;
                            }
                    }
                    PROF_ADD(w_sync)
                    { PROF_T0
                    commit(&accf[a]);
                    commit(&empty[(q + lr) & (S - 1)]);  // input row lr: no later conv row of the band reads it
                    PROF_ADD(w_empty) }
                }
                for (int r = nconv; r < nconv + P.kh - 1; ++r) commit(&empty[(q + r) & (S - 1)]);
                q += nconv + P.kh - 1;
            }
        }
        __syncwarp();
    } else {
        // ---------------------------------------------------------------- epilogue (thread t = conv column t)
        const int t = threadIdx.x;
        constexpr int cpc = SElem<T>::cpc, chunks = N / cpc;
        const int cown = t % chunks;  // the output chunk this thread stores (emit_row)
        float bias[cpc];
#pragma unroll
        for (int k = 0; k < cpc; ++k) bias[k] = cown * cpc + k < P.cout ? __ldg(P.bias + cown * cpc + k) : 0.0f;
        asm volatile("griddepcontrol.wait;" ::: "memory");
        const uint32_t trow = tmem + (uint32_t(t & ~31) << 16);
        // vm = the pooled row being built (vertical max so far, fp32).  Odd conv
        // rows are max-ed into it; an even conv row closes it (max -> stage)
        // and becomes the next one.  Every accumulator is read from TMEM once:
        // TMEM reads (~64 B/cycle/SM) bound this kernel, not the registers
        // copies.
        float vm[N];
        int c = 0, emitted = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            const Band b = band_of(P, u, n0);
            const int nconv = conv_rows(b);
            T* orow = static_cast<T*>(P.out) + (size_t(b.n) * P.Hp + b.i0) * P.Wp * P.out_cstride + P.out_coff;
            const size_t orow_step = size_t(P.Wp) * P.out_cstride;
            for (int lr = 0; lr < nconv; ++lr, ++c) {
                const int a = c & (Acc - 1);
                PROF_T0
                mbar_sleep_wait(&accf[a], uint32_t(c >> AccL) & 1u);  // suspended, not spinning: the other CTA's warps issue
                PROF_ADD(w_accf)
                fence_after();
                const uint32_t ta = trow + uint32_t(a * N);
                const bool closes = lr > 0 && !(lr & 1);
                const uint32_t stage = (emitted & 1) ? stage0 + uint32_t(P.stage_bytes) : stage0;
                if constexpr (NCH <= 2) {
                    // every chunk of the row in flight at once (TMEM reads are
                    // latency-bound per warp), one wait
                    uint32_t rv[NCH][32];
#pragma unroll
                    for (int h = 0; h < NCH; ++h) tmem_ld32_issue(ta + uint32_t(h * 32), rv[h]);
#pragma unroll
                    for (int h = 0; h < NCH; ++h) tmem_ld_wait32(rv[h]);
                    if (lr == 0) {
#pragma unroll
                        for (int h = 0; h < NCH; ++h)
#pragma unroll
                            for (int k = 0; k < 32; ++k) vm[h * 32 + k] = __uint_as_float(rv[h][k]);
                    } else if (!closes) {
#pragma unroll
                        for (int h = 0; h < NCH; ++h)
#pragma unroll
                            for (int k = 0; k < 32; ++k) vm[h * 32 + k] = fmaxf(vm[h * 32 + k], __uint_as_float(rv[h][k]));
                    } else {
#pragma unroll
                        for (int h = 0; h < NCH; ++h) {
                            // the pooled maxima replace the row's values in rv (no third 32-register array)
#pragma unroll
                            for (int k = 0; k < 32; ++k) {
                                const float v = __uint_as_float(rv[h][k]);
                                rv[h][k] = __float_as_uint(fmaxf(vm[h * 32 + k], v)), vm[h * 32 + k] = v;
                            }
                            stage_part<T, NCH>(stage, t, h, reinterpret_cast<const float*>(rv[h]));
                        }
                    }
                } else {
                if (lr == 0) {
#pragma unroll
                    for (int h = 0; h < NCH; ++h) tmem_ld32(ta + uint32_t(h * 32), vm + h * 32);
                } else if (!closes) {
#pragma unroll
                    for (int h = 0; h < NCH; ++h) {
                        float v[32];
                        tmem_ld32(ta + uint32_t(h * 32), v);
#pragma unroll
                        for (int k = 0; k < 32; ++k) vm[h * 32 + k] = fmaxf(vm[h * 32 + k], v[k]);
                    }
                } else {
#pragma unroll
                    for (int h = 0; h < NCH; ++h) {
                        float v[32];
                        tmem_ld32(ta + uint32_t(h * 32), v);
                        float m[32];
#pragma unroll
                        for (int k = 0; k < 32; ++k) m[k] = fmaxf(vm[h * 32 + k], v[k]), vm[h * 32 + k] = v[k];
                        stage_part<T, NCH>(stage, t, h, m);
                    }
                }
                }
                fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acce[a]);  // TMEM slot free for conv row c + Acc
                if (closes) {
                    PROF_T0
                    epi_sync();
                    PROF_ADD(w_sync)
                    emit_row<T, NCH>(P, stage, bias, cown, orow);
                    orow += orow_step;
                    ++emitted;
                }
            }
        }
    }
#ifdef XLF_STEM_PROF
    if (blockIdx.x < 3 && (threadIdx.x == 0 || threadIdx.x == 64 || (warp == 4 && lane == 0) || (warp == 5 && w_full + w_acce > 0)))
        printf("cta %d thread %d: total %lld empty %lld full %lld acce %lld accf %lld sync %lld\n", blockIdx.x, threadIdx.x,
               clock64() - t_start, w_empty, w_full, w_acce, w_accf, w_sync);
#endif
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 5) tmem_free(tmem, uint32_t(P.tmem_cols));
}

template <class T, int NCH>
cudaError_t launch_nch(const StemParams& P, int batch, cudaStream_t st, int n0) {
    static bool init = false;
    if (!init) {
        cudaError_t e = cudaFuncSetAttribute(stem_kernel<T, NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, kStemSmemMax);
        if (e != cudaSuccess) return e;
        init = true;
    }
    const int units = batch * P.bands;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = std::min(units, sms * std::max(1, P.ctas_per_sm));
    if (grid < 1) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid)), cfg.blockDim = dim3(kStemThreads), cfg.dynamicSmemBytes = size_t(P.smem_bytes), cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = P.pdl ? 1 : 0;
    cfg.attrs = attr, cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, stem_kernel<T, NCH>, P, batch, n0);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_stem(const StemParams& P, int batch, cudaStream_t st, int n0) {
    const int nch = P.npad / 32;
    if (P.es == 2) {
        if (nch == 2) return launch_nch<__nv_bfloat16, 2>(P, batch, st, n0);
        if (nch == 4) return launch_nch<__nv_bfloat16, 4>(P, batch, st, n0);
    } else {
        if (nch == 2) return launch_nch<float, 2>(P, batch, st, n0);
        if (nch == 4) return launch_nch<float, 4>(P, batch, st, n0);
    }
    return cudaErrorInvalidValue;
}

}  // namespace xlf
