// Throughput probe: R back-to-back tcgen05.mma (M=128, K=16, bf16) from one
// thread, timed with clock64 until the commit lands.  Layout variants for A/B.
#include <cstdio>
#include <cuda_bf16.h>

#include "../../paper_2007_06000_b200/csrc/umma.cuh"

using namespace xlf::umma;

__global__ void rate(int N, int alayout, int blayout, int reps, long long* out, int spin) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, never;
    __shared__ uint32_t slot;
    __shared__ int stop;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
    fence_async_smem();
    if (threadIdx.x == 0) mbar_init(&bar, 1), mbar_init(&never, 1), stop = 0, mbar_fence_init();
    if (threadIdx.x < 32) tmem_alloc(&slot, 256);
    fence_before();
    __syncthreads();
    fence_after();
    if (spin == 2 && threadIdx.x < 32) {  // kernel-like: whole warp, elected lane, varying descriptors
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
        const uint64_t ad0 = sdesc(0, 16, 1024, kSW128), bd0 = sdesc(0, N * 16, 128, kNoSwizzle);
        const uint32_t idesc = idesc_bf16(128, N);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const int s = r >> 1, mt = r & 1;
            if (elect_one()) mma_bf16(slot + mt * N, ad0 + ((a0 + (s & 3) * 32 + mt * 16384) >> 4), bd0 + ((b0 + (s & 7) * N * 32) >> 4), idesc, s > 0);
            __syncwarp();
        }
        long long t1 = clock64();
        if (elect_one()) commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (threadIdx.x == 0) out[0] = t1 - t0, out[1] = t2 - t0, mbar_arrive(&never);
    } else if (spin == 3 && threadIdx.x < 32) {  // elected lane runs the whole loop, varying descriptors
        if (elect_one()) {
            const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
            const uint64_t ad0 = sdesc(0, 16, 1024, kSW128), bd0 = sdesc(0, N * 16, 128, kNoSwizzle);
            const uint32_t idesc = idesc_bf16(128, N);
            long long t0 = clock64();
            for (int r = 0; r < reps; ++r) {
                const int s = r >> 1, mt = r & 1;
                mma_bf16(slot + mt * N, ad0 + ((a0 + (s & 3) * 32 + mt * 16384) >> 4), bd0 + ((b0 + (s & 7) * N * 32) >> 4), idesc, s > 0);
            }
            long long t1 = clock64();
            commit(&bar);
            mbar_wait(&bar, 0);
            long long t2 = clock64();
            out[0] = t1 - t0, out[1] = t2 - t0, mbar_arrive(&never);
        }
        __syncwarp();
    } else if (spin == 4 && threadIdx.x < 32) {  // whole warp loop, elect per MMA, no __syncwarp
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
        const uint64_t ad0 = sdesc(0, 16, 1024, kSW128), bd0 = sdesc(0, N * 16, 128, kNoSwizzle);
        const uint32_t idesc = idesc_bf16(128, N);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const int s = r >> 1, mt = r & 1;
            if (elect_one()) mma_bf16(slot + mt * N, ad0 + ((a0 + (s & 3) * 32 + mt * 16384) >> 4), bd0 + ((b0 + (s & 7) * N * 32) >> 4), idesc, s > 0);
        }
        long long t1 = clock64();
        if (elect_one()) commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        if (threadIdx.x == 0) out[0] = t1 - t0, out[1] = t2 - t0, mbar_arrive(&never);
    } else if (spin != 2 && threadIdx.x == 0) {
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 32768);
        const uint64_t ad = alayout == 2 ? sdesc(a0, 16, 1024, kSW128) : sdesc(a0, 4096, 128, kNoSwizzle);
        const uint64_t bd = blayout == 2 ? sdesc(b0, 16, 1024, kSW128) : sdesc(b0, N * 16, 128, kNoSwizzle);
        const uint32_t idesc = idesc_bf16(128, N);
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) mma_bf16(slot, ad, bd, idesc, r > 0);
        long long t1 = clock64();
        commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        out[0] = t1 - t0;
        out[1] = t2 - t0;
        mbar_arrive(&never);
    } else if (spin && threadIdx.x >= 32 && (threadIdx.x & 31) == 0) {
        mbar_wait(&never, 0);  // spinning waiters, as in the fused kernel
    }
    fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_free(slot, 256);
}

int main() {
    long long* d;
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int spin : {0, 2, 3, 4})
    for (int al : {2})
        for (int bl : {0})
            for (int N : {16, 64}) {
                for (int reps : {64}) {
                    rate<<<1, 128, 64 * 1024>>>(N, al, bl, reps, d, spin);
                    long long h[2];
                    cudaError_t e = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
                    printf("spin=%d A%s B%s N=%3d reps=%3d issue=%6lld cyc total=%7lld cyc  per-mma=%.1f\n", spin, al ? "sw128" : "none ",
                           bl ? "sw128" : "none ", N, reps, h[0], h[1], double(h[1]) / reps);
                }
            }
    return 0;
}
