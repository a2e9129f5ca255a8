// Launch descriptor of the stem kernel (kernels_stem.cu): space-to-depth
// input (NHWC, `planes` 16-byte channel planes per pixel) -> stride-1 kh x kw
// conv (tensor cores, fp32 accumulate) -> bias -> ReLU -> 3x3/2 max-pool, pad 0.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace xlf {

constexpr int kStemSlots = 8;      // input-row ring
constexpr int kStemMaxSlots = kStemSlots;
constexpr int kStemMaxAcc = 4;     // TMEM conv-row accumulators (4 at 64 columns, else 2)
constexpr int kStemSmemMax = 227 * 1024 - 1024;

struct StemParams {
    CUtensorMap xmap;           // row-planar input as 2-D {inner, N*Hin*row_lines}; box = one input row
    int row_lines;              // box lines per input row
    int es;                     // element bytes: 2 bf16 (kind::f16), 4 fp32/TF32 (kind::tf32)
    int Hin, Win, planes;       // input rows / pixels per row / 16-byte planes per pixel
    int kh, kw;                 // conv taps (stride 1 on the input)
    int Hc, Wc;                 // conv output (Wc <= 128: one M tile per row)
    int cout, npad;             // output channels; accumulator columns (64 or 128) = packed N
    int Hp, Wp;                 // pooled output
    const uint8_t* wmma;        // packed B operand [tap][plane][npad][cpc] (pack_weights_tc, one N block)
    int w_bytes;
    const float* bias;          // >= cout fp32
    void* out;                  // NHWC pooled output
    int out_cstride, out_coff;
    int bands, band_rows;       // work unit = (image, band of band_rows pooled rows)
    int slots, acc_slots, tmem_cols;
    int plane_bytes, slot_bytes;  // plane = Win * 16 bytes (contiguous planes); slot = one input row
    int ring_off, w_off, stage_off, stage_bytes, bias_off, smem_bytes;
    int ctas_per_sm, pdl;
};

}  // namespace xlf
