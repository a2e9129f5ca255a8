// Depthwise (+ pointwise) kernel for sm_100a (see dw_params.hpp): the paper's
// a.2 block, depthwise kh x kw conv -> 1x1 conv, channel-parallel SIMT.
//
// CTA = one tile_h x tile_w output tile of one image, one thread per output
// pixel.  The input tile (+ halo) is staged in shared memory as fp32
// [row][col][channel] (zero outside the image = the conv padding); each
// thread accumulates every depthwise channel of its pixel in registers
// (float4 shared loads over channels, the weights broadcast), applies bias /
// ReLU, then -- without leaving registers -- the 1x1 conv over those channels
// and stores NHWC (16-byte vectors).  Arithmetic in fp32; in EXACT mode with
// separate multiply / add in the reference's order (ic -> kh -> kw,
// reference.cpp:16-57; a zero-padded tap adds a +-0 product, which leaves
// the sum unchanged), so fp32_exact reproduces run_reference bit for bit.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "dw_params.hpp"

namespace xlf {

namespace {

template <bool EXACT>
__device__ __forceinline__ float mac(float acc, float a, float b) {
    if constexpr (EXACT) return __fadd_rn(acc, __fmul_rn(a, b));
    else return fmaf(a, b, acc);
}
template <bool EXACT>
__device__ __forceinline__ float add(float a, float b) {
    if constexpr (EXACT) return __fadd_rn(a, b);
    else return a + b;
}

__device__ __forceinline__ float4 load4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 load4(const __nv_bfloat16* p) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(&u.x), b = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
    const float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
    return make_float4(fa.x, fa.y, fb.x, fb.y);
}

__device__ __forceinline__ float tf32r(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// 4 consecutive channels of one pixel -> HBM (channels >= valid skipped)
__device__ __forceinline__ void store4(float* p, float4 v, int valid, bool tf32) {
    if (tf32) v = make_float4(tf32r(v.x), tf32r(v.y), tf32r(v.z), tf32r(v.w));
    if (valid >= 4) {
        *reinterpret_cast<float4*>(p) = v;
    } else {
        p[0] = v.x;
        if (valid > 1) p[1] = v.y;
        if (valid > 2) p[2] = v.z;
    }
}
__device__ __forceinline__ void store4(__nv_bfloat16* p, float4 v, int valid, bool) {
    if (valid >= 4) {
        uint2 u;
        __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
        u.x = *reinterpret_cast<uint32_t*>(&a), u.y = *reinterpret_cast<uint32_t*>(&b);
        *reinterpret_cast<uint2*>(p) = u;
    } else {
        p[0] = __float2bfloat16(v.x);
        if (valid > 1) p[1] = __float2bfloat16(v.y);
        if (valid > 2) p[2] = __float2bfloat16(v.z);
    }
}

// PX output pixels per thread along a row (stride 1: 2, sharing the weight
// loads and the overlapping input columns; stride 2: 1).  (4 pixels per
// thread measured slower: 100 registers, 92 KB tiles, 2 CTAs per SM.)
template <class T, bool EXACT, int PX>
__global__ void __launch_bounds__(kDwThreads) dw_kernel(const __grid_constant__ DwParams P, int n0) {
    extern __shared__ __align__(16) float sm[];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    constexpr int CM = PX == 1 ? kDwMaxC : kDwMaxC / 2;  // channels held per pixel
    const int C = P.C, cp = P.cp, taps = P.kh * P.kw;
    float* xs = sm;                                            // [cin_h][cin_w][cp]
    float* wd = xs + P.cin_h * P.cin_w * cp;                   // [taps][cw]
    float* bd = wd + taps * P.cw;                              // [cw]
    float* wp = bd + P.cw;                                     // [C][cpw]
    float* bp = wp + (P.pw ? C * P.cpw : 0);                   // [cpw]
    // weights (constant: before waiting on the previous step)
    for (int i = threadIdx.x; i < taps * P.cw; i += kDwThreads) wd[i] = P.wdw[i];
    for (int i = threadIdx.x; i < P.cw; i += kDwThreads) bd[i] = P.bdw && i < C ? P.bdw[i] : 0.0f;
    if (P.pw) {
        for (int i = threadIdx.x; i < C * P.cpw; i += kDwThreads) wp[i] = P.wpw[i];
        for (int i = threadIdx.x; i < P.cpw; i += kDwThreads) bp[i] = P.bpw && i < P.cout ? P.bpw[i] : 0.0f;
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int tiles_w = (P.Wo + P.tile_w - 1) / P.tile_w;
    const int ty0 = (blockIdx.x / tiles_w) * P.tile_h, tx0 = (blockIdx.x % tiles_w) * P.tile_w;
    const int n = n0 + blockIdx.y;
    const int iy0 = ty0 * P.stride - P.pad, ix0 = tx0 * P.stride - P.pad;
    const T* in = static_cast<const T*>(P.in) + size_t(n) * P.H * P.W * P.in_cstride + P.in_coff;
    // stage the input tile: thread -> (cell, 4-channel chunk q), q fastest;
    // cells advance by a fixed step, (row, col) tracked without division
    const int c4 = (C + 3) / 4, cells = P.cin_h * P.cin_w;
    if (kDwThreads % c4 == 0) {
        const int q = threadIdx.x % c4, step = kDwThreads / c4;
        int cell = threadIdx.x / c4, r = cell / P.cin_w, c = cell - r * P.cin_w;
        const int dr = step / P.cin_w, dc = step - dr * P.cin_w;
        for (; cell < cells; cell += step) {
            const int iy = iy0 + r, ix = ix0 + c;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (iy >= 0 && iy < P.H && ix >= 0 && ix < P.W) v = load4(in + (size_t(iy) * P.W + ix) * P.in_cstride + q * 4);
            *reinterpret_cast<float4*>(xs + cell * cp + q * 4) = v;
            r += dr, c += dc;
            if (c >= P.cin_w) c -= P.cin_w, ++r;
        }
    } else {
        for (int i = threadIdx.x; i < cells * c4; i += kDwThreads) {
            const int q = i % c4, cell = i / c4, r = cell / P.cin_w, c = cell % P.cin_w;
            const int iy = iy0 + r, ix = ix0 + c;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (iy >= 0 && iy < P.H && ix >= 0 && ix < P.W) v = load4(in + (size_t(iy) * P.W + ix) * P.in_cstride + q * 4);
            *reinterpret_cast<float4*>(xs + cell * cp + q * 4) = v;
        }
    }
    __syncthreads();
    const int tpr = P.tile_w / PX;  // threads per tile row
    const int ty = threadIdx.x / tpr, tx = (threadIdx.x % tpr) * PX;
    const int oy = ty0 + ty, ox = tx0 + tx;
    if (oy >= P.Ho || ox >= P.Wo) return;
    // depthwise: every channel of PX pixels, taps in kh -> kw order per pixel
    float d[PX][CM];
#pragma unroll
    for (int p = 0; p < PX; ++p)
#pragma unroll
        for (int c = 0; c < CM; ++c) d[p][c] = 0.0f;
    for (int ky = 0; ky < P.kh; ++ky) {
        const float* xrow = xs + ((ty * P.stride + ky) * P.cin_w + tx * P.stride) * cp;
        for (int kx = 0; kx < P.kw; ++kx) {
            const float* wt = wd + (ky * P.kw + kx) * P.cw;
#pragma unroll
            for (int c = 0; c < CM; c += 4) {
                if (c >= C) break;
                const float4 w4 = load4(wt + c);
#pragma unroll
                for (int p = 0; p < PX; ++p) {
                    const float4 x4 = load4(xrow + ((p * P.stride + kx) * cp) + c);
                    d[p][c] = mac<EXACT>(d[p][c], w4.x, x4.x), d[p][c + 1] = mac<EXACT>(d[p][c + 1], w4.y, x4.y);
                    d[p][c + 2] = mac<EXACT>(d[p][c + 2], w4.z, x4.z), d[p][c + 3] = mac<EXACT>(d[p][c + 3], w4.w, x4.w);
                }
            }
        }
    }
#pragma unroll
    for (int c = 0; c < CM; ++c) {
        if (c >= C) break;
        const float b = bd[c];
#pragma unroll
        for (int p = 0; p < PX; ++p) {
            float y = add<EXACT>(d[p][c], b);
            if (P.relu_dw) y = y < 0.0f ? 0.0f : y;
            d[p][c] = y;
        }
    }
    T* out0 = static_cast<T*>(P.out) + (size_t(n) * P.Ho * P.Wo + size_t(oy) * P.Wo + ox) * P.out_cstride + P.out_coff;
    const int npx = min(PX, P.Wo - ox);
    if (!P.pw) {
#pragma unroll
        for (int p = 0; p < PX; ++p) {
            if (p >= npx) break;
#pragma unroll
            for (int c = 0; c < CM; c += 4) {
                if (c >= C) break;
                store4(out0 + p * P.out_cstride + c, make_float4(d[p][c], d[p][c + 1], d[p][c + 2], d[p][c + 3]), C - c, P.tf32);
            }
        }
        return;
    }
    // pointwise over the depthwise channels (ic order), 4 outputs at a time
    for (int oc = 0; oc < P.cout; oc += 4) {
        float a[PX][4];
#pragma unroll
        for (int p = 0; p < PX; ++p) a[p][0] = a[p][1] = a[p][2] = a[p][3] = 0.0f;
#pragma unroll
        for (int ic = 0; ic < CM; ++ic) {
            if (ic >= C) break;
            const float4 w4 = load4(wp + ic * P.cpw + oc);
#pragma unroll
            for (int p = 0; p < PX; ++p) {
                a[p][0] = mac<EXACT>(a[p][0], w4.x, d[p][ic]), a[p][1] = mac<EXACT>(a[p][1], w4.y, d[p][ic]);
                a[p][2] = mac<EXACT>(a[p][2], w4.z, d[p][ic]), a[p][3] = mac<EXACT>(a[p][3], w4.w, d[p][ic]);
            }
        }
        const float4 b4 = load4(bp + oc);
#pragma unroll
        for (int p = 0; p < PX; ++p) {
            if (p >= npx) break;
            float y[4] = {add<EXACT>(a[p][0], b4.x), add<EXACT>(a[p][1], b4.y), add<EXACT>(a[p][2], b4.z), add<EXACT>(a[p][3], b4.w)};
            if (P.relu_pw)
#pragma unroll
                for (int j = 0; j < 4; ++j) y[j] = y[j] < 0.0f ? 0.0f : y[j];
            store4(out0 + p * P.out_cstride + oc, make_float4(y[0], y[1], y[2], y[3]), P.cout - oc, P.tf32);
        }
    }
}

template <class T, bool EXACT, int PX>
cudaError_t launch_t(const DwParams& P, int n0, int count, cudaStream_t st) {
    static bool init = false;
    if (!init) {
        cudaError_t e = cudaFuncSetAttribute(dw_kernel<T, EXACT, PX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        init = true;
    }
    const int tiles = ((P.Ho + P.tile_h - 1) / P.tile_h) * ((P.Wo + P.tile_w - 1) / P.tile_w);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(tiles), unsigned(count), 1u), cfg.blockDim = dim3(kDwThreads);
    cfg.dynamicSmemBytes = size_t(P.smem_bytes), cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = P.pdl ? 1 : 0;
    cfg.attrs = attr, cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, dw_kernel<T, EXACT, PX>, P, n0);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dw(const DwParams& P, int n0, int count, cudaStream_t st) {
    if (P.px == 2) {
        if (P.es == 2) return launch_t<__nv_bfloat16, false, 2>(P, n0, count, st);
        return P.exact ? launch_t<float, true, 2>(P, n0, count, st) : launch_t<float, false, 2>(P, n0, count, st);
    }
    if (P.es == 2) return launch_t<__nv_bfloat16, false, 1>(P, n0, count, st);
    return P.exact ? launch_t<float, true, 1>(P, n0, count, st) : launch_t<float, false, 1>(P, n0, count, st);
}

}  // namespace xlf
