// Plain-old-data launch descriptor of one fused block, shared by the host
// planner (device_plan.cpp) and the sm_100a kernels.  It is the B200
// successor of the reference's TilingPlan + emitted kernel text
// (tiling.hpp:103-122, codegen.cpp:77-404): instead of generating CUDA source
// per block, one templated kernel family interprets this descriptor.
//
// Execution model of one CTA = (image n, output tile (ty, tx)):
//   stage X   : the block input region needed by every stage-1 op is copied
//               from NHWC global memory into shared memory (zero outside the
//               image = the producers' conv padding, reference.cpp:38-44);
//   stage 1   : ops reading X.  Each either keeps its result on chip in a
//               shared buffer (cells outside its tensor are 0 = the consumer's
//               padding, fused_exec.cpp:129-139) and/or stores it to global;
//   barrier   : (fused_exec.cpp:212)
//   stage 2   : ops reading stage-1 buffers, storing to global NHWC at a
//               channel offset (so a concat sink costs nothing).
// All offsets are tile-independent "local" coordinates; see device_plan.cpp.
#pragma once

#include <cstdint>

namespace xlf {

enum : int { OP_CONV = 0, OP_MAXPOOL = 1, OP_AVGPOOL = 2, OP_ADD = 3 };

constexpr int kMaxOps = 8;
constexpr int kMaxBufs = 4;

struct FOp {
    int kind;
    int stage;        // 1: reads block input `xin`, 2: reads buffer `src` (and `src2` for add)
    int xin;
    int src, src2;    // buffer indices (stage 2)
    int buf;          // buffer written (stage 1), -1 = none
    int emit;         // 1 = store to global
    int own_only;     // stage-1 staged+emitted: store only the tile's ownership slab
    int cin, cout, cout_pad, group, kh, kw, stride, pad, relu;
    int d;            // local source offset: src row = r*stride + kh + d (same for columns)
    int ext_h, ext_w; // cells computed per tile (full tile; edges are masked)
    int org_mul;      // global cell row = tile_origin*org_mul - org_sub + r
    int org_sub;
    int H, W;         // extent of the op's output tensor
    const float* w;   // conv: [cin/group][kh][kw][cout_pad]
    const float* b;   // conv: [cout_pad] (zeros when the layer has no bias)
    float* out;       // NHWC destination base (image 0, channel 0 of the destination tensor)
    int out_cstride;  // channels per pixel of the destination allocation
    int out_coff;     // channel offset inside it
    // Register-blocked conv (kernels_fp32.cu conv_rb): a thread computes cx
    // consecutive cells of one row x ocv output channels.  0 = the generic
    // cell-quad path (grouped convs, kernel widths / strides without an
    // instantiation).  Chosen by the planner (device_plan.cpp rb_variant).
    int cx, ocv;
};

struct FBuf {
    int channels, cpitch, ext_h, ext_w;
    int smem_off;  // in floats
};

// One block input staged into shared memory as [ext_h][ext_w][cpitch] floats.
struct FIn {
    const float* x;  // NHWC, image 0
    int c, cstride, coff, h, w;
    int org_mul, org_sub;  // global row of region row 0 = tile_origin*org_mul - org_sub
    int ext_h, ext_w, cpitch;
    int smem_off;          // in floats
};

constexpr int kMaxIns = 2;

struct FusedParams {
    int nins;
    FIn in[kMaxIns];
    int tile_h, tile_w, grid_h, grid_w, out_h, out_w;
    // Channel tiling (pool-only steps, where input channel c feeds output
    // channel c): CTA z handles channels [z*ctile, (z+1)*ctile); 0 = all.
    int ctile, cgroups;
    int nops, nbufs;
    int smem_floats;
    int threads;  // 256 (two CTAs per SM when shared memory allows) or 512 (one CTA, 16 warps)
    FOp ops[kMaxOps];
    FBuf bufs[kMaxBufs];
};

}  // namespace xlf
