// Launch descriptor of the tensor-core fused-block kernel (kernels_tc.cu;
// "B" = Blackwell).  Same execution model as FusedParams (fused_params.hpp):
// stage the block inputs, stage-1 ops, stage-2 ops; but conv ops with stride
// 1 / group 1 / 32-byte K steps run as implicit GEMMs on tcgen05 with the fp32
// accumulator in TMEM.  Two element types (es = bytes per activation):
//   es = 2  bf16 activations and weights, tcgen05.mma kind::f16 (K = 16 per step),
//   es = 4  fp32 storage rounded to TF32, tcgen05.mma kind::tf32 (K = 8 per step).
// Every layout below is in 16-byte "chunks" (8 bf16 / 4 fp32 channels), so one
// K step is 32 bytes of every row for both types and the descriptors,
// swizzles and weight packing are byte-identical.
//
// Shared-memory activation layout ("planes"): a region of ext_h x ext_w cells
// with C channels is C/cpc planes (cpc = channels per chunk); plane p holds
// chunk p of every cell, cells row-major.  This is the UMMA K-major SWIZZLE_NONE
// canonical layout with the cell index as M: 8 consecutive cells of a row are
// one 8x16-byte core matrix, so
//   * a 1x1 conv over the whole region is an M = cells GEMM (SBO = 128 B),
//   * a kh x kw conv producing an 8-wide strip of rows reads, for tap (dy, dx),
//     the same planes from start address + ((row+dy+d)*ext_w + col+dx+d)*16 with
//     SBO = ext_w*16 B -- the shifted-window implicit GEMM, no im2col copy,
//   * LBO = plane bytes steps K by one chunk.
// Block inputs are loaded by one 4-D TMA per K-block (box {kb_ch, ext_w,
// ext_h, 1 image}, zero fill outside the image = conv padding).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "fused_params.hpp"

namespace xlf {

enum : int { BOP_MMA = 0, BOP_SIMT_CONV = 1, BOP_MAXPOOL = 2, BOP_AVGPOOL = 3, BOP_ADD = 4 };

constexpr int kBMaxOps = 8;
constexpr int kBMaxBufs = 4;
constexpr int kBMaxUnits = 24;  // (op, N block) pairs
constexpr int kRingSlots = 3;
// CTA shapes: 4 or 8 epilogue/SIMT warps + 3 role warps (input producer,
// MMA issuer, weight producer); the kernel is instantiated for both and the
// step's descriptor (epi_warps) selects one.  Resident CTAs per SM: <= 3 / 2.
constexpr int max_ctas_per_sm(int epi_warps) { return epi_warps <= 4 ? 4 : 2; }
constexpr int kChunkBytes = 16 * 1024;  // weight ring slot (smallest; the tuner picks 16 / 32 / 64 KB)
// Dynamic shared memory per CTA: 227 KB minus the static part (barriers, the
// descriptor copy: 4 KB) minus 4 KB headroom (ncu's replay needs some).
constexpr int kSmemBudgetTc = 227 * 1024 - 8192;
constexpr int kRingMax = 8;             // ring slots (P.ring_slots <= this)

struct BOp {
    int kind, stage, xin, src, src2, buf, emit, own_only;
    int cin, kpt, cout, npad, group, kh, kw, stride, pad, relu;  // kpt: MMA K steps (32 B) per tap
    int d;
    int ext_h, ext_w;       // computed region (cells), rows x cols
    int org_mul, org_sub;   // global cell row = tile_origin*org_mul - org_sub + r
    int H, W;               // output tensor extent
    // MMA tiling
    int contig;             // 1: M = consecutive cells of the whole region (1x1 over its source)
    int strips, mtiles;     // windowed: strips of 8 columns x blocks of 16 rows
    int nblocks, nb;        // N split into nblocks of nb (<= 256) accumulator columns
    int ksteps, chunk_steps;
    const uint8_t* wmma;        // [nblock][kh*kw][cin/cpc][nb][cpc] elements (UMMA B image of each K step)
    const float* wsimt;         // [cin/group][kh][kw][cout_pad4] (SIMT convs)
    const float* bias;          // [npad] fp32 (zeros when the layer has no bias)
    void* out;                  // NHWC, element type of the step
    int out_cstride, out_coff;
    int tcol;       // MMA: first TMEM column of this op inside its group
    int wofs;       // MMA, resident weights: byte offset of the op's packed weights in the weight region
    int gap;        // MMA: global-average-pool epilogue (column sums per tile, no output store)
    int bias_smem;  // byte offset of the op's bias copy in shared memory (-1: none)
    // N split over the grid's y dimension (BParams::nsplit): this op computes
    // channels [g*gch, (g+1)*gch) in CTA row g (npad = gch; its packed weights
    // for group g start at wmma + g*gwb bytes).  gch = 0: not split.
    int gch;
    long long gwb;
};

// A group is what one commit / one epilogue pass covers: consecutive MMA ops
// of the same stage (disjoint TMEM columns, issued back to back), or one N
// block of a wide MMA op, or one SIMT op.
struct BGroup {
    int op0, op1;  // ops [op0, op1)
    int nbi;       // N block (multi-block MMA ops), else 0
    int mma;       // 1: tensor-core group
    int tbase;     // first TMEM column of the group (ops add their tcol)
    int wback;     // the issuer waits for the epilogue of group gi - wback (1: in order;
                   // 2: N blocks alternating between two column sets)
    int pwait;     // one accumulator set, gi < wback: the previous tile's last group whose
                   // TMEM columns overlap this one (its epilogue frees them); -1: none
};

// Layout of a shared region: K-blocks of kb_ch channels; inside a K-block
// cell r occupies row_bytes at r*row_bytes (kb_ch = row_bytes / es).
//   kPlanes : row 16 B, no swizzle (epilogue-written buffers)
//   kSw32   : row 32 B, 32-byte swizzle  (TMA box of one 32-byte K step)
//   kSw128  : row 128 B, 128-byte swizzle (TMA box of four K steps)
// Swizzles are functions of the absolute shared address (chunk ^= (addr>>7)
// & mask), identical for TMA writes, UMMA reads and SIMT reads.
enum : int { kPlanes = 0, kSw32 = 1, kSw128 = 3 };

struct BRegion {
    int chunks;         // 16-byte chunks per cell (channels / cpc)
    int ext_h, ext_w;   // cells
    int plane_bytes;    // bytes per K-block (multiple of 1024 for swizzled modes)
    int smem_off;       // bytes from the dynamic smem base
    int mode;           // kPlanes / kSw32 / kSw128
    int kb_ch;          // channels per K-block (row_bytes / es)
    int row_bytes;      // 16 / 32 / 128
};

struct BIn {
    BRegion r;
    int h, w, cstride, coff;  // NHWC tensor (elements)
    int org_mul, org_sub;
    const void* x;
};

struct alignas(64) BParams {
    CUtensorMap xmap[kMaxIns];   // block inputs: 4-D {cstride, W, H, N}, box = one K-block of the region
    int nins;
    BIn in[kMaxIns];
    int tile_h, tile_w, grid_h, grid_w, out_h, out_w;
    int nops, nbufs;
    BOp ops[kBMaxOps];
    BRegion bufs[kBMaxBufs];
    int ngroups;
    BGroup groups[kBMaxUnits];
    int bias_off, bias_bytes;  // shared copy of every MMA op's bias
    int ring_off, chunk_bytes, ring_slots;
    // Resident weights (wres = 1): every MMA op's packed weights are loaded
    // into shared memory ONCE per (persistent) CTA at wres_off (wres_bytes)
    // instead of being streamed through the ring for every tile.
    int wres, wres_off, wres_bytes;
    // gap steps: per-tile column sums (fp32, npad per tile) accumulate in
    // shared memory at gap_off and are written to gap_part[image][tile][c].
    int gap_off;
    float* gap_part;
    int smem_bytes, tmem_cols;
    int ctile, cgroups;  // channel tiling of pool-only steps (0 = all channels)
    // Persistent execution: each CTA walks tiles blockIdx.x, +gridDim.x, ...
    // (tile = (image, channel group, tile row, tile column)).  The block
    // inputs are staged in nxb buffers, xstride bytes apart, so the producer
    // loads tile k+1's regions while tile k computes (nxb = 2).
    int nxb, xstride;
    int ctas_per_sm;  // resident CTAs per SM at smem_bytes (grid = 148 x this, capped by the tiles)
    int grid_all;     // 1: grid = tiles (each CTA one tile), else the persistent grid
    int epi_warps;    // 4 or 8 epilogue/SIMT warps (kernel instantiation)
    int kind;         // step class (kernel instantiation): 0 MMA ops only, 1 with SIMT ops, 2 conv + global average pool
    int tsets;        // accumulator sets in TMEM (2: tile k+1's MMAs run during tile k's epilogue; needs nxb = 2)
    int es;           // bytes per activation element: 2 (bf16, kind::f16) or 4 (fp32/TF32, kind::tf32)
    // N split: the grid is (persistent CTAs, nsplit); CTA row g computes the
    // g-th channel group of every split op (BOp::gch) with only that group's
    // weights resident; unsplit (stage-1 producer) ops are computed by every row.
    int nsplit;
    int gap_np_total;  // gap steps: channels per tile row of gap_part (all groups)
    int pdl;          // programmatic dependent launch (prologue overlaps the previous kernel's drain)
    int xrel_epi;     // 1: the epilogue warps release the staging buffer after the tile even when
                      // only MMAs read it (the earlier synchronisation structure; tested, not tuned)
    // Optional phase trace (engine option trace=1): globaltimer stamps of CTAs with
    // blockIdx.y == 0 and blockIdx.x < kTraceCtas, kTraceEvents each.
    unsigned long long* trace;
    int trace_tiles;  // trace=2: instead, the end stamp of each of the first kTraceEvents tiles
    // Device-memory copy of this descriptor: the kernel pulls it into shared
    // memory with one bulk copy instead of per-thread parameter-bank loads.
    const void* dev_copy;
};

constexpr int kTraceCtas = 8;
constexpr int kTraceEvents = 32;
enum : int {  // trace slots
    kTrStart = 0, kTrXIssued = 1, kTrXLanded = 2, kTrEnd = 3,
    kTrUnit = 4  // + 2u: accumulator ready seen by the epilogue, + 2u + 1: unit done
};

}  // namespace xlf
