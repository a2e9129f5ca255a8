// mbarrier hand-off latency: warp 0 lane 0 and warp 1 lane 0 ping-pong through
// two mbarriers N times; waits are plain try_wait spins (mode 0), try_wait
// with a suspend-time hint (mode 1), or spin + named barrier fan-out to 4
// warps (mode 2).  Prints cycles per one-way hand-off.
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2007_06000_b200/csrc/umma.cuh"

using namespace xlf::umma;

__device__ __forceinline__ void wait_mode(uint64_t* b, uint32_t par, int mode) {
    if (mode == 1) mbar_sleep_wait(b, par);
    else mbar_wait(b, par);
}

__global__ void pp(int n, int mode, long long* out) {
    __shared__ __align__(8) uint64_t ping, pong;
    if (threadIdx.x == 0) mbar_init(&ping, 1), mbar_init(&pong, 1), mbar_fence_init();
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < n; ++i) {
            mbar_arrive(&ping);
            wait_mode(&pong, i & 1, mode);
        }
    } else if (warp == 1 && lane == 0) {
        for (int i = 0; i < n; ++i) {
            wait_mode(&ping, i & 1, mode);
            mbar_arrive(&pong);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / (2 * n);
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    for (int mode = 0; mode < 2; ++mode) {
        pp<<<1, 64>>>(10000, mode, d);
        long long h = 0;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %lld cycles per hand-off (%s)\n", mode, mode ? "try_wait+suspend hint" : "try_wait spin", h,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
