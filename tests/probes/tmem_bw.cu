// Probe: TMEM -> register read bandwidth (tcgen05.ld.32x32b.x32 / .x64, one
// warp per lane quadrant and more) on one SM, cycles per KB.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2007_06000_b200/csrc tmem_bw.cu -o tmem_bw
#include <cstdio>
#include <cstdint>
#include "umma.cuh"
using namespace xlf::umma;

__global__ void k(int iters, int split_wait, unsigned long long* out, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) tmem_alloc(&slot, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = slot;
    const uint32_t base = tmem + (uint32_t((warp & 3) * 32) << 16) + uint32_t((warp >> 2) * 64);
    float acc = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (split_wait) {
            uint32_t r0[32], r1[32];
            tmem_ld32_issue(base + uint32_t((i & 1) * 256), r0);
            tmem_ld32_issue(base + uint32_t((i & 1) * 256) + 32, r1);
            tmem_ld_wait32(r0);
            tmem_ld_wait32(r1);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += __uint_as_float(r0[j]) + __uint_as_float(r1[j]);
        } else {
            float v[32];
            tmem_ld32(base + uint32_t((i & 1) * 256), v);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc += v[j];
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (acc == 1.2345f) sink[0] = acc;
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 0) tmem_free(tmem, 512);
}

int main() {
    unsigned long long* d;
    float* s;
    cudaMalloc(&d, 8);
    cudaMalloc(&s, 8);
    for (int sw : {0, 1})
        for (int warps : {4, 8, 16}) {
            const int iters = 1000;
            k<<<1, warps * 32>>>(iters, sw, d, s);
            unsigned long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            const double bytes = double(iters) * warps * 32 * 32 * 4 * (sw ? 2 : 1);
            printf("warps %2d %s: %.1f bytes/cycle\n", warps, sw ? "2 loads, one wait" : "load+wait      ", bytes / double(h));
        }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
