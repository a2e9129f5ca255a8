// Launch descriptor of the pointwise-conv GEMM kernel (kernels_pw.cu): a 1x1,
// stride-1, pad-0 conv over NHWC is a GEMM with one row per pixel, so the
// pixels of ALL images of a launch form one M dimension (M tiles of 128 rows
// cross image boundaries: no per-image tile waste on 13x13 / 27x27 maps).
// Output channels may be split into `nsplit` groups over the grid's y
// dimension, each CTA keeping its group's weights resident.  Epilogue: bias +
// ReLU + NHWC store, or (gap = 1) a global-average-pool reduction whose
// per-warp, per-image partial column sums a finish kernel adds in a fixed order.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace xlf {

constexpr int kPwStages = 4;  // A-tile ring (K chunks of 128 bytes per row)

struct PwParams {
    CUtensorMap amap;     // A: 2-D {cstride, rows = max_batch * HW}, box {128 bytes of channels, 128 rows}, SWIZZLE_128B
    int es;               // element bytes (2 bf16 / 4 TF32)
    int HW;               // pixels per image
    int coff_in;          // first channel of the input inside its allocation (concat view)
    int kchunks;          // 128-byte K chunks per row (input channels rounded up)
    int ksteps;           // 32-byte MMA K steps (= 4 per chunk, the last chunk may hold fewer)
    int cout, gch, nsplit;  // output channels; channels per group (16 | gch <= 256); groups
    const uint8_t* wmma;  // packed B [group][ksteps][gch][cpc] (nb = gch, one block per group)
    long long gwb;        // packed bytes per group
    const float* bias;    // >= cout fp32
    int relu;
    void* out;            // NHWC (gap = 0)
    int out_cstride, out_coff;
    int gap;              // 1: global average pool epilogue into gap_part
    float* gap_part;      // [warp of the launch][2 image segments][nsplit * gch]
    int smem_bytes, ring_off, w_off, bias_off;
    int tmem_cols;        // 2 accumulator sets x gch (power of two)
    int ctas_per_sm, pdl;
    int mc;               // > 1: the nsplit channel groups of an M tile run as one cluster, A chunks multicast (TMA .multicast::cluster)
};

}  // namespace xlf
