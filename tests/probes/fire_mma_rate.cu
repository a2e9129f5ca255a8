// Probe: tcgen05.mma rate for the fire kernel's expand issue loop -- A = a
// "plane" (K-major SWIZZLE_NONE, 16-byte cells, LBO = plane stride) read at
// per-tap shifted starts, B = packed weights advancing per MMA, descriptors
// advanced by deltas exactly as kernels_fire.cu -- alone, and with 256
// threads concurrently (a) polling an mbarrier, (b) reading TMEM,
// (c) storing to global memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2007_06000_b200/csrc fire_mma_rate.cu -o fire_mma_rate
#include <cstdio>
#include <cstdint>
#include "umma.cuh"
using namespace xlf::umma;

__global__ void k(int jobs, int N, int nks, int busy, float* gout, unsigned long long* out) {
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
                            mma_bf16(tmem + uint32_t((j & 1) * 256), ad, bd, idesc, acc);
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

int main() {
    unsigned long long* d;
    float* g;
    cudaMalloc(&d, 16);
    cudaMalloc(&g, size_t(1024) * 224 * 64 * 4 + 1024 * 1024);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char* names[] = {"alone", "+256 pollers", "+256 TMEM readers", "+256 scattered stores"};
    for (int busy = 0; busy < 4; ++busy)
        for (int N : {64, 128, 256})
            for (int nks : {1, 4}) {
                unsigned long long h[2];
                const int jobs = 200;
                k<<<1, busy ? 288 : 32, 200 * 1024>>>(jobs, N, nks, busy, g, d);
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                const double n = jobs * 9.0 * nks;
                printf("%-22s N=%3d nks=%d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", names[busy], N, nks, h[0] / n, h[1] / n);
            }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
