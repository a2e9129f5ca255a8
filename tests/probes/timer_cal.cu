// %globaltimer vs clock64 calibration: spin a known number of SM cycles and
// compare the two clocks (ns per cycle should be ~1/f_sm).
#include <cstdio>
__global__ void k(long long spin, unsigned long long* out) {
    unsigned long long g0, g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    long long c0 = clock64();
    while (clock64() - c0 < spin) {}
    long long c1 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    out[0] = g1 - g0, out[1] = c1 - c0;
}
int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    for (long long spin : {1000LL, 10000LL, 100000LL, 1000000LL}) {
        k<<<1, 1>>>(spin, d);
        unsigned long long h[2];
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("spin %lld cycles: globaltimer %llu ns, clock64 %llu -> %.3f GHz\n", spin, h[0], h[1], double(h[1]) / double(h[0]));
    }
}
