// Launch descriptor of the depthwise kernel (kernels_dw.cu): a depthwise
// kh x kw conv (groups == channels, multiplier 1) optionally followed by a
// 1x1 pointwise conv reading only its output -- the paper's a.2 block
// (MobileNet's depthwise-separable unit).  Channel-parallel
// SIMT: one thread per output pixel holds every depthwise channel in
// registers, so the depthwise output never leaves the SM.
#pragma once

namespace xlf {

constexpr int kDwMaxC = 32;     // depthwise channels held per thread
constexpr int kDwMaxTaps = 25;  // kh * kw
constexpr int kDwThreads = 256;

struct DwParams {
    int es;                 // HBM element bytes: 2 bf16, 4 fp32 (fp32 / fp32_exact / TF32 storage)
    int exact;              // 1: reference order, separate mul / add (fp32_exact, bit for bit); 0: FFMA
    int tf32;               // 1: outputs rounded to TF32 (the TF32 path's producer rounding)
    int H, W, C, Ho, Wo;    // input map, depthwise channels, output map
    int kh, kw, pad, stride;
    const void* in;         // NHWC, channel pitch in_cstride, first channel in_coff
    int in_cstride, in_coff;
    const float* wdw;       // packed fp32 [tap][C_pad4] (pack_weights: [ic/g][kh][kw][oc_pad4] with ic/g = 1)
    const float* bdw;       // C (nullptr: no bias)
    int relu_dw;
    int pw;                 // 1: a 1x1 conv follows
    int cout;               // pointwise outputs
    const float* wpw;       // packed fp32 [C][cout_pad4]
    const float* bpw;
    int relu_pw;
    void* out;              // NHWC (the pointwise output, else the depthwise output)
    int out_cstride, out_coff, out_c;  // out_c: channels written
    int px;                 // output pixels per thread along a row (2: stride 1, C <= 16; else 1)
    int tile_h, tile_w;     // output pixels per CTA (tile_h * tile_w == px * kDwThreads)
    int cin_h, cin_w, cp;   // staged input tile (rows, cols), channel pitch in shared memory (floats)
    int cw, cpw;            // padded weight pitches: C_pad4, cout_pad4
    int smem_bytes;
    int pdl;
};

}  // namespace xlf
