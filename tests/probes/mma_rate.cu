// Probe: tcgen05.mma issue/execution rate for the shapes the stem / fused
// kernels use (kind::f16 bf16, A and B K-major from shared memory).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2007_06000_b200/csrc mma_rate.cu -o mma_rate -lcuda
#include <cstdio>
#include <cstdint>
#include "umma.cuh"
using namespace xlf::umma;

__global__ void k(int iters, int N, int mode, int lbo_a, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u * (i & 1);
    if (threadIdx.x == 0) mbar_init(&bar, 1), mbar_fence_init();
    if (warp == 0) tmem_alloc(&slot, 512);
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = slot;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (warp >= 4 && mode == 4) {  // concurrent TMEM readers (the epilogue) on other columns
        float acc = 0.f;
        const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + 256;
        int r = 0;
        while (!done) {
            float v[32];
            tmem_ld32(base + ((r++ * 32) & 255), v);
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += v[i];
        }
        if (acc == 1.2345f) out[2] = 1;
    }
    if (warp == 0 && elect_one()) {
        const uint32_t sb = smem_u32(smem);
        const uint32_t idesc = idesc_bf16(128, N);
        uint64_t a = mode == 1 ? sdesc(sb, 16, 256, kSW32) : sdesc(sb, uint32_t(lbo_a), 128, kNoSwizzle);
        const uint64_t b = sdesc(sb + 32768, uint32_t(N * 16), 128, kNoSwizzle);
        long long t0 = clock64();
        if (mode >= 6) {  // groups of 4 MMAs + 2 commits (the stem's issue pattern); mode 7 waits each group
            __shared__ uint64_t gb[2];
            mbar_init(&gb[0], 1), mbar_init(&gb[1], 1);
            mbar_fence_init();
            for (int i = 0; i < iters / 4; ++i) {
                const uint32_t d = tmem + uint32_t((i & 3) * N);
                for (int j = 0; j < 4; ++j) mma_bf16(d, a, b, idesc, j > 0);
                commit(&gb[0]);
                commit(&gb[1]);
                if (mode == 7) mbar_wait(&gb[0], uint32_t(i & 1));
            }
        } else
        for (int i = 0; i < iters; ++i) {
            const uint32_t d = tmem + uint32_t(mode == 2 ? (i & 3) * N : 0);
            mma_bf16(d, a + (mode == 3 ? uint64_t(i & 3) : 0), b, idesc, i > 0);
        }
        long long t1 = clock64();
        commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        out[0] = t1 - t0, out[1] = t2 - t0;
        done = 1;
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0) tmem_free(tmem, 512);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    const char* names[] = {"noswz", "sw32", "noswz,4 acc", "noswz,shifted A", "noswz+4 tmem readers", "noswz+8 tmem readers",
                           "4mma+2commit", "4mma+2commit+wait"};
    for (int mode = 0; mode < 8; ++mode)
        for (int N : {64, 128})
            for (int lbo : {1792}) {
                unsigned long long h[2];
                k<<<1, mode == 5 ? 384 : mode == 4 ? 256 : 128, 65536>>>(2000, N, mode == 5 ? 4 : mode, lbo, d);
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                printf("%-16s N=%3d lbo_a=%4d: issue %.1f cyc/mma, complete %.1f cyc/mma\n", names[mode], N, lbo, h[0] / 2000.0, h[1] / 2000.0);
            }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
