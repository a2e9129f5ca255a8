// Launch descriptor of the fire kernel (kernels_fire.cu): a split-mode fused
// block -- one 1x1 "squeeze" conv whose output feeds several stride-1
// "same"-padded expand convs (SqueezeNet fire module: squeeze 1x1 -> expand
// 1x1 + expand 3x3 -> concat; reference fused_exec.cpp:116-280) -- with the
// squeeze output kept in shared memory as a zero-bordered "plane".
//
// Plane geometry.  A unit of work is G whole images (R == H) or one band of
// R output rows of one image (G == 1).  Its squeeze output is laid out as
// rows of Wp = W + 1 cells: cell 0 of every row is the zero column (it is
// both the left pad of its row and the right pad of the previous one), and
// rows are image rows r0-1 .. r0+R of each image with one row between images
// (zero: rows -1 / H).  In this flattened form a kh x kw expand tap is a
// constant shift of the cell index, so every tap of every expand op is a
// plain K-major GEMM operand read at a shifted start address (no im2col):
// the MMA M dimension is the plane's cell index.  Cells that are not output
// pixels (the zero column, rows between images) are computed and dropped.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace xlf {

constexpr int kFireStages = 6;     // max squeeze-input ring stages (128 px x 128 or 64 B each)
constexpr int kFireMaxOps = 4;     // expand ops
constexpr int kFireMaxExSlots = 8; // expand accumulator slots in TMEM
constexpr int kFireSmemMax = 227 * 1024 - 1024;
constexpr int kFireSmemMax2 = 111 * 1024;  // per CTA with two CTAs per SM (228 KB per SM less 1 KB reserved + 2 KB static per CTA)
constexpr int kFireTraceN = 1024;  // trace events per role (option trace=1)

struct FireOp {
    int kh, kw, pad;      // stride 1, pad = (k - 1) / 2
    int cout;             // output channels of the whole layer
    void* out;            // NHWC allocation (a concat view: out_cstride / out_coff)
    int out_cstride, out_coff;
    const uint8_t* w;     // packed B [group][tap][S / cpc][gch][cpc], group stride gwb bytes
    long long gwb;
    const float* bias;    // >= cout fp32
    int relu;
    int w_off;            // shared-memory byte offset of this group's packed weights
    int bias_off;         // shared-memory byte offset of this group's bias (gch fp32)
};

struct FireParams {
    CUtensorMap amap;     // squeeze A: 2-D {cstride_in, max_batch * H * W}, box {cb bytes of channels, 128 pixels}, SWIZZLE_128B / 64B
    int cps;              // CTAs per SM: 1 (8 epilogue warps, 512 TMEM columns) or 2 (4 epilogue warps, 256 columns, <= kFireSmemMax2 bytes each)
    int cb;               // input chunk bytes per pixel per stage: 128 (SWIZZLE_128B) or 64 (SWIZZLE_64B)
    int es;               // element bytes (2 bf16 kind::f16 / 4 TF32 kind::tf32)
    int H, W, HW, Wp;     // Wp = W + 1
    int coff_in;          // first input channel inside its allocation (concat view)
    int kchunks, ksteps;  // squeeze K: cb-byte chunks / 32-byte MMA steps
    int S, schunks;       // squeeze channels (multiple of 16) / 16-byte chunks per plane cell
    const uint8_t* wsq;   // squeeze packed B [ksteps * 2][S][cpc]
    const float* sq_bias;
    int sq_relu;
    int G, R, bands;      // unit = G images x R rows (G > 1: R == H); bands = ceil(H / R)
    int Ts, Te;           // squeeze / expand M tiles per unit
    int nops;
    FireOp op[kFireMaxOps];
    int gch, nsplit;      // channels per group of every expand op; groups (grid y)
    int nst;              // ring stages
    int stage_bytes;      // ring stage: 128 x cb-byte input chunk (+ that K chunk's squeeze weights when sq_stream)
    int sq_stream;        // squeeze weights streamed through the ring per K chunk instead of resident
    int nplane;           // squeeze planes (2: the next unit's squeeze overlaps this unit's expand)
    int plane_cells;      // cells per plane, incl. one leading slack cell
    int plane_bytes;      // plane_cells * 16 * schunks
    int sq_cols;          // TMEM columns per squeeze accumulator (two of them)
    int nexslots;         // expand accumulators (nops * gch columns each: every op of one M tile; gch with per_op)
    int per_op;           // one expand job per (M tile, op) instead of per M tile (two whole-tile accumulators would not fit TMEM)
    int seg;              // expand store segment: channels of one op per warp pass (64 bf16 if gch % 64 == 0, else 32)
    int ring_off, wsq_off, plane_off, sqbias_off, stage_off, smem_bytes;  // stage: 8 epilogue warps x 4 KB store staging (-1: direct stores)
    int pdl;
    int st32;             // every op's output pixel / channel offsets are 32-byte aligned: 256-bit stores
    unsigned long long* trace;  // option trace=1: 3 roles x kFireTraceN x (code, globaltimer) of CTA (0, 0)
    int stage_mode;             // host planning only: 0 direct stores, 1 staged through shared memory (option fire_stage)
    int cps_mode;               // host planning only: 0 either, else 1 / 2 CTAs per SM (option fire_cps)
    int cb_mode;                // host planning only: chunk width 128 (0: default) or 64 (option fire_cb)
    int sq_stream_mode;         // host planning only: 0 either, 1 streamed squeeze weights only, 2 resident only (option fire_sqs)
};

}  // namespace xlf
