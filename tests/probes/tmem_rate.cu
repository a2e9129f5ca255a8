// TMEM read-rate probe: W warps per CTA, C CTAs per SM (grid = 148*C), each
// warp repeatedly tcgen05.ld 32x32b.x32 from its lane quadrant; reports
// bytes per SM-cycle.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_rate tmem_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../../paper_2007_06000_b200/csrc/umma.cuh"

using namespace xlf::umma;

__global__ void rd(int reps, long long* cyc, float* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc(&slot, 256);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t base = slot + (uint32_t((warp & 3) * 32) << 16);
    float acc = 0.f;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        float v[32];
        tmem_ld32(base + ((r * 32 + (warp >> 2) * 64) & 255), v);
#pragma unroll
        for (int i = 0; i < 32; ++i) acc += v[i];
    }
    long long t1 = clock64();
    fence_before();
    __syncthreads();
    if (warp == 0) tmem_free(slot, 256);
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[0] = acc;
}

int main() {
    long long* cyc;
    float* sink;
    cudaMalloc(&cyc, 148 * 4 * 8);
    cudaMalloc(&sink, 4);
    const int reps = 4096;
    for (int ctas = 1; ctas <= 2; ++ctas)
        for (int warps = 4; warps <= 16; warps *= 2) {
            rd<<<148 * ctas, warps * 32>>>(reps, cyc, sink);
            cudaDeviceSynchronize();
            long long h[148 * 4];
            cudaMemcpy(h, cyc, 148 * ctas * 8, cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int i = 0; i < 148 * ctas; ++i) mx = h[i] > mx ? h[i] : mx;
            const double bytes = double(ctas) * warps * reps * 4096.0;  // per SM
            printf("ctas/SM %d warps %2d: %.1f B/cycle/SM (%.0f cycles) %s\n", ctas, warps, bytes / mx, mx,
                   cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
