// Hardware probe of the tcgen05 descriptor conventions the bf16 kernels rely
// on (run on a B200 via gpurun; prints PASS/FAIL per case).
//   mode 0: SWIZZLE_NONE planes, contiguous rows, start shifted by `shift` rows
//   mode 1: SWIZZLE_NONE planes, M-groups strided by 10 rows (SBO = 160 B):
//           the shifted-window trick of the fused 3x3 consumers
//   mode 2: SWIZZLE_128B, start shifted by `shift` 128-B rows, base_offset = boff
// A: 256 x 64 bf16, B: 64 x 64 bf16 (small integers: products/sums exact).
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>
#include <vector>

#include "../../paper_2007_06000_b200/csrc/umma.cuh"

using namespace xlf::umma;

__host__ __device__ inline float aval(int m, int k) { return float(((m * 7 + k * 3) % 9) - 4); }
__host__ __device__ inline float bval(int n, int k) { return float(((n * 5 + k) % 7) - 3); }

__device__ inline uint32_t a_off(int mode, int m, int k) {
    if (mode == 2) return (m / 8) * 1024 + (m % 8) * 128 + (((k / 8) ^ (m % 8)) * 16) + (k % 8) * 2;
    return (k / 8) * (256 * 16) + m * 16 + (k % 8) * 2;
}
__device__ inline uint32_t b_off(int mode, int n, int k) {
    if (mode == 2) return (n / 8) * 1024 + (n % 8) * 128 + (((k / 8) ^ (n % 8)) * 16) + (k % 8) * 2;
    return (k / 8) * (64 * 16) + n * 16 + (k % 8) * 2;
}

__global__ void probe(int mode, int shift, int boff, float* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* A = sm;
    uint8_t* B = sm + 32768;
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    for (int i = threadIdx.x; i < 256 * 64; i += blockDim.x) {
        int m = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(A + a_off(mode, m, k)) = __float2bfloat16(aval(m, k));
    }
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
        int n = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16*>(B + b_off(mode, n, k)) = __float2bfloat16(bval(n, k));
    }
    fence_async_smem();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_fence_init();
    }
    if (threadIdx.x < 32) tmem_alloc(&slot, 64);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tm = slot;
    if (threadIdx.x == 0) {
        const uint32_t idesc = idesc_bf16(128, 64);
        const uint32_t a0 = smem_u32(A), b0 = smem_u32(B);
        for (int ks = 0; ks < 4; ++ks) {
            uint64_t ad, bd;
            if (mode == 0) {
                ad = sdesc(a0 + shift * 16 + ks * 2 * 4096, 4096, 128, kNoSwizzle);
                bd = sdesc(b0 + ks * 2 * 1024, 1024, 128, kNoSwizzle);
            } else if (mode == 1) {
                ad = sdesc(a0 + shift * 16 + ks * 2 * 4096, 4096, 160, kNoSwizzle);
                bd = sdesc(b0 + ks * 2 * 1024, 1024, 128, kNoSwizzle);
            } else {
                ad = sdesc(a0 + shift * 128 + ks * 32, 16, 1024, kSW128, boff);
                bd = sdesc(b0 + ks * 32, 16, 1024, kSW128, 0);
            }
            mma_bf16(tm, ad, bd, idesc, ks > 0);
        }
        commit(&bar);
    }
    mbar_wait(&bar, 0);
    fence_after();
    const int w = threadIdx.x / 32;
    float v[32];
    for (int c = 0; c < 64; c += 32) {
        tmem_ld32(tm + ((uint32_t)(32 * w) << 16) + c, v);
        for (int j = 0; j < 32; ++j) out[threadIdx.x * 64 + c + j] = v[j];
    }
    fence_before();
    __syncthreads();
    if (threadIdx.x < 32) tmem_free(tm, 64);
}

int main() {
    float* d;
    cudaMalloc(&d, 128 * 64 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    struct Case { int mode, shift, boff; };
    std::vector<Case> cases = {{0, 0, 0}, {0, 1, 0}, {0, 5, 0}, {1, 0, 0}, {1, 11, 0}, {1, 22, 0},
                               {2, 0, 0}, {2, 1, 0}, {2, 1, 1}, {2, 3, 0}, {2, 3, 3}, {2, 8, 0}};
    int fails = 0;
    for (const Case& c : cases) {
        cudaMemset(d, 0, 128 * 64 * 4);
        probe<<<1, 128, 48 * 1024>>>(c.mode, c.shift, c.boff, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("case mode=%d shift=%d boff=%d: CUDA error %s\n", c.mode, c.shift, c.boff, cudaGetErrorString(e));
            return 1;
        }
        std::vector<float> h(128 * 64);
        cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int m = 0; m < 128; ++m) {
            int row = c.mode == 1 ? c.shift + (m / 8) * 10 + m % 8 : c.shift + m;
            for (int n = 0; n < 64; ++n) {
                float ref = 0;
                for (int k = 0; k < 64; ++k) ref += aval(row, k) * bval(n, k);
                if (h[m * 64 + n] != ref) ++bad;
            }
        }
        printf("%s mode=%d shift=%d boff=%d mismatches=%d\n", bad ? "FAIL" : "PASS", c.mode, c.shift, c.boff, bad);
        fails += bad != 0;
    }
    return 0;
}
