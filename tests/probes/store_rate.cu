// HBM store-pattern probe for the epilogue: each thread owns one "cell" and
// 64 bf16 channels (128 B) of an NHWC tensor with a 256 B pixel stride (the
// fire concat), i.e. the pattern of a 32x32b TMEM load.  Variants:
//   0: 8 x st.global.v4 (16 B) per thread, warp instruction = 32 cells   (current)
//   1: 4 x st.global.v8 (32 B) per thread
//   2: transpose through shared memory, each warp instruction writes 4 cells x 128 B
//      contiguous (full lines)
// Reports GB/s of useful bytes over a 256 MB tensor.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void st16(uint4* out, long long cells, int pitch16) {
    for (long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x; cell < cells; cell += (long long)gridDim.x * blockDim.x) {
        uint4* p = out + cell * pitch16;
        uint4 v = make_uint4(uint32_t(cell), 1, 2, 3);
#pragma unroll
        for (int j = 0; j < 8; ++j) p[j] = v;
    }
}

__global__ void st32(uint4* out, long long cells, int pitch16) {
    for (long long cell = blockIdx.x * (long long)blockDim.x + threadIdx.x; cell < cells; cell += (long long)gridDim.x * blockDim.x) {
        uint4* p = out + cell * pitch16;
        const uint32_t a = uint32_t(cell);
#pragma unroll
        for (int j = 0; j < 8; j += 2)
            asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p + j), "r"(a), "r"(1u), "r"(2u), "r"(3u), "r"(a),
                         "r"(1u), "r"(2u), "r"(3u)
                         : "memory");
    }
}

__global__ void stsmem(uint4* out, long long cells, int pitch16) {
    __shared__ uint4 stage[8][32 * 8 + 8];  // per warp: 32 cells x 8 chunks (+pad)
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (long long base = (blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31)); base < cells; base += (long long)gridDim.x * blockDim.x) {
        const long long cell = base + lane;
        uint4 v = make_uint4(uint32_t(cell), 1, 2, 3);
#pragma unroll
        for (int j = 0; j < 8; ++j) stage[w][lane * 8 + ((j + lane) & 7)] = v;  // rotated: conflict-free
        __syncwarp();
        // 8 rounds: lanes 0..31 write cells (4 per round) x 8 chunks
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const int c = r * 4 + (lane >> 3), j = lane & 7;
            if (base + c < cells) out[(base + c) * pitch16 + j] = stage[w][c * 8 + ((j + c) & 7)];
        }
        __syncwarp();
    }
}

int main() {
    const long long bytes = 256ll << 20, pitch16 = 16;  // 256 B pixel stride, 128 B written per pixel
    const long long cells = bytes / (pitch16 * 16);
    uint4* out;
    cudaMalloc(&out, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a), cudaEventCreate(&b);
    for (int v = 0; v < 3; ++v) {
        for (int it = 0; it < 2; ++it) {
            cudaEventRecord(a);
            if (v == 0) st16<<<148 * 8, 256>>>(out, cells, int(pitch16));
            if (v == 1) st32<<<148 * 8, 256>>>(out, cells, int(pitch16));
            if (v == 2) stsmem<<<148 * 8, 256>>>(out, cells, int(pitch16));
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("variant %d: %.0f GB/s useful (%.3f ms) %s\n", v, cells * 128.0 / (ms * 1e6), ms, cudaGetErrorString(cudaGetLastError()));
    }
}
