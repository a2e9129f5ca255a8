// Probe: tcgen05.mma rate for the fire kernel's expand issue loop -- A = a
// "plane" (K-major SWIZZLE_NONE, 16-byte cells, LBO = plane stride) read at
// per-tap shifted starts, B = packed weights advancing per MMA, descriptors
// advanced by deltas exactly as kernels_fire.cu -- alone, and with 256
// threads concurrently (a) polling an mbarrier, (b) reading TMEM,
// (c) storing to global memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2007_06000_b200/csrc fire_mma_rate.cu -o fire_mma_rate
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "umma.cuh"
using namespace xlf::umma;

__global__ void k(int jobs, int N, int nks, int busy, float* gout, unsigned long long* out, int dcol0 = 0, int dstep = 256) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, never;
    __shared__ uint32_t slot;
    __shared__ volatile int done;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u * (i & 1);
    if (threadIdx.x == 0) mbar_init(&bar, 1), mbar_init(&never, 1), mbar_fence_init(), done = 0;
    if (warp == 0) tmem_alloc(&slot, 512);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = slot;
    const int Wp = 56;
    const uint32_t PS = 1024 * 16;
    if (warp == 0) {
        if (elect_one()) {
            const uint32_t sb = smem_u32(smem);
            const uint32_t idesc = idesc_bf16(128, N);
            const uint64_t aplane = sdesc(sb + uint32_t(1 + Wp) * 16u, PS, 128, kNoSwizzle);
            const uint64_t b0 = sdesc(sb + 4 * PS, uint32_t(N * 16), 128, kNoSwizzle);
            const uint32_t da = (2u * PS) >> 4, db = 2u * uint32_t(N);
            long long t0 = clock64();
            for (int j = 0; j < jobs; ++j) {
                const uint64_t ajob = aplane + uint64_t((j & 3) * 128);
                uint64_t arow = ajob + uint64_t(int64_t(-Wp - 1));
                uint64_t bd = b0;
                uint32_t acc = 0;
                for (int ky = 0; ky < 3; ++ky, arow += uint64_t(Wp)) {
                    uint64_t atap = arow;
                    for (int kx = 0; kx < 3; ++kx, ++atap) {
                        uint64_t ad = atap;
                        for (int kk = 0; kk < nks; ++kk) {
                            mma_bf16(tmem + uint32_t(dcol0 + (j & 1) * dstep), ad, bd, idesc, acc);
                            acc = 1;
                            ad += da;
                            bd += db;
                        }
                    }
                }
            }
            long long t1 = clock64();
            commit(&bar);
            mbar_wait(&bar, 0);
            long long t2 = clock64();
            out[0] = t1 - t0, out[1] = t2 - t0;
            done = 1;
        }
        __syncwarp();
    } else if (busy == 1) {  // poll a barrier that never completes (suspend hint, as the epilogue waits)
        while (!done) {
            uint32_t ok;
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0, 1000000;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                         : "=r"(ok) : "r"(smem_u32(&never)) : "memory");
        }
    } else if (busy == 2) {  // TMEM readers on other columns
        float acc = 0.f;
        const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16);
        int r = 0;
        while (!done) {
            float v[32];
            tmem_ld32(base + 512 - 32 - ((r++ * 32) & 127), v);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += v[i];
        }
        if (acc == 1.2345f) gout[0] = acc;
    } else if (busy == 4) {  // shared-memory stores + loads (plane writes / staging)
        const int t = threadIdx.x - 32;
        uint32_t base = smem_u32(smem) + 150 * 1024 + (t % 128) * 16;
        uint32_t acc = 0;
        while (!done) {
            asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base), "r"(acc) : "memory");
            uint32_t v;
            asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(base + 4096) : "memory");
            acc += v;
        }
        if (acc == 12345) gout[1] = float(acc);
    } else if (busy == 3) {  // scattered 16-byte global stores (the epilogue's pattern)
        const int t = threadIdx.x - 32;
        int r = 0;
        while (!done) {
            float4* p = reinterpret_cast<float4*>(gout + (size_t((r++ & 1023) * 224 + t) * 64));
            p[0] = make_float4(1.f, 2.f, 3.f, 4.f);
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0) tmem_free(tmem, 512);
}

// The fire kernel's round: a squeeze tile (4 MMAs, N = 16, A in a SWIZZLE_128B
// stage) + commit, then an expand tile (e1: 1 MMA, e3: 9 shifted MMAs, N = 64)
// + commit, with the kernel's shared-memory placement (plane stride 16256 B).
__device__ __forceinline__ bool lane_is0() { return (threadIdx.x & 31) == 0; }
__device__ __forceinline__ void tma2d(void* smem, const void* desc, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(smem)),
        "l"(desc), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__global__ void kround(int jobs, int with_sq, unsigned long long* out, int fence_mode = 0, const __grid_constant__ CUtensorMap tmap = CUtensorMap{}, int tma = 0) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, jb;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u * (i & 1);
    if (threadIdx.x == 0) mbar_init(&bar, 1), mbar_init(&jb, 1), mbar_fence_init();
    if (warp == 0) tmem_alloc(&slot, 512);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = slot;
    __shared__ volatile int stop;
    __shared__ uint64_t tb;
    if (threadIdx.x == 0) stop = 0, mbar_init(&tb, 1), mbar_fence_init();
    __syncthreads();
    if (warp == 1) {  // concurrent TMA: 16 KB boxes into a separate region, back to back
        if (tma && lane_is0()) {
            uint32_t ph = 0;
            int r = 0;
            while (!stop) {
                mbar_expect_tx(&tb, 16384);
                tma2d(smem + 176 * 1024, &tmap, 0, (r++ * 128) & 65535, &tb);
                mbar_wait(&tb, ph);
                ph ^= 1;
            }
        }
    } else if (warp == 0 && elect_one()) {
        const uint32_t sb = smem_u32(smem);
        const int Wp = 56;
        const uint32_t PS = 1016 * 16;
        const uint32_t plane = sb + 120 * 1024, wex = sb + 96 * 1024 + 2048, wsq = sb + 96 * 1024;
        const uint64_t aplane = sdesc(plane + uint32_t(1 + Wp) * 16u, PS, 128, kNoSwizzle);
        const uint64_t ring0 = sdesc(sb, 16u, 1024u, kSW128);
        const uint64_t bsq = sdesc(wsq, 16 * 16, 128, kNoSwizzle);
        const uint32_t idsq = idesc_bf16(128, 16), idex = idesc_bf16(128, 64);
        long long t0 = clock64();
        __shared__ uint64_t done_bar;
        mbar_init(&done_bar, 1);
        mbar_fence_init();
        mbar_arrive(&done_bar);  // phase 0 complete: waits on parity 0 return at once
        for (int j = 0; j < jobs; ++j) {
            if (fence_mode & 1) fence_after();
            if (fence_mode & 2) mbar_wait(&done_bar, 0);
            if (fence_mode & 4) fence_before();
            if (with_sq) {
                uint64_t ad = ring0 + uint64_t((j % 6) * 1024), bd = bsq;
                for (int kk = 0; kk < 4; ++kk) mma_bf16(tmem + 0 + (j & 1) * 32, ad, bd, idsq, kk > 0), ad += 2, bd += 32;
                commit(&jb);
            }
            const uint64_t ajob = aplane + uint64_t((j % 7) * 128);
            const uint32_t d = tmem + 64 + uint32_t((j % 3) * 128);
            mma_bf16(d, ajob, sdesc(wex, 64 * 16, 128, kNoSwizzle), idex, 0);
            uint64_t arow = ajob + uint64_t(int64_t(-Wp - 1)), bd = sdesc(wex + 2048, 64 * 16, 128, kNoSwizzle);
            uint32_t acc = 0;
            for (int ky = 0; ky < 3; ++ky, arow += uint64_t(Wp)) {
                uint64_t atap = arow;
                for (int kx = 0; kx < 3; ++kx, ++atap) {
                    mma_bf16(d + 64, atap, bd, idex, acc);
                    acc = 1;
                    bd += 128;
                }
            }
            commit(&jb);
        }
        long long t1 = clock64();
        commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        out[0] = t1 - t0, out[1] = t2 - t0;
        stop = 1;
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0) tmem_free(tmem, 512);
}

int main() {
    unsigned long long* d;
    float* g;
    cudaMalloc(&d, 16);
    cudaMalloc(&g, size_t(1024) * 224 * 64 * 4 + 1024 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"alone", "+256 pollers", "+256 TMEM readers", "+256 scattered stores", "+256 smem st/ld"};
    for (int busy = 0; busy < 1; ++busy)
        for (int N : {64, 128})
            for (int nks : {1, 2}) {
                unsigned long long h[2];
                const int jobs = 200;
                k<<<1, busy ? 288 : 32, 200 * 1024>>>(jobs, N, nks, busy, g, d);
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                const double n = jobs * 9.0 * nks;
                printf("%-22s N=%3d nks=%d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", names[busy], N, nks, h[0] / n, h[1] / n);
            }
    for (int dc : {0, 32, 64, 96})
        for (int ds : {128, 256}) {
            unsigned long long h[2];
            k<<<1, 32, 200 * 1024>>>(200, 64, 1, 0, g, d, dc, ds);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("dcol %3d step %3d N=64 nks=1: %.1f cyc/mma\n", dc, ds, h[1] / 1800.0);
        }
    cudaFuncSetAttribute(kround, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    // a 2-D tensor {64 bf16 channels, 65536 rows} for the concurrent TMA loads
    void* gsrc;
    cudaMalloc(&gsrc, size_t(65536) * 128);
    CUtensorMap tm;
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
    const cuuint64_t dims[2] = {64, 65536};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, gsrc, dims, strides, box, es,
                                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int tma : {0, 1})
        for (int sq : {0, 1}) {
            unsigned long long h[2];
            kround<<<1, 64, 210 * 1024>>>(200, sq, d, 0, tm, tma);
            cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
            printf("kernel round (squeeze %d, concurrent TMA %d): %.0f cycles per round\n", sq, tma, h[1] / 200.0);
        }
    for (int tma : {0, 1}) {  // all SMs at once
        unsigned long long h[2];
        kround<<<148, 64, 210 * 1024>>>(200, 1, d, 0, tm, tma);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("148 CTAs, kernel round (squeeze 1, concurrent TMA %d): %.0f cycles per round\n", tma, h[1] / 200.0);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
