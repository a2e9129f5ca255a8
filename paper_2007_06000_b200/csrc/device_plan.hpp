// Device program: how a prepared graph is executed by the sm_100a kernels.
//
// The planner turns a partition (reference FusionBlocks, the B200
// extension, or one-kernel-per-layer) into an ordered list of kernel steps
// whose ops are the graph's layers, plus a tensor table saying where every
// materialised tensor lives in HBM (NHWC, channel pitch padded to 4 floats;
// tensors consumed only by a concat are views into the concat's allocation
// in the B200 partition).  Fused intermediates have no HBM slot at all.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "fused_params.hpp"
#include "fusion.hpp"
#include "graph.hpp"

namespace xlf {

enum class Partition { reference = 0, b200 = 1, unfused = 2 };
const char* to_string(Partition p);

// Engine / planner options: the "key=value,..." string of xlf_engine_create_ex
// (nothing is read from the environment).  The defaults are the product
// configuration; the rest pin one synchronisation / staging mode (tests run
// every mode the tuner may pick) or steer an experiment.
struct Knobs {
    bool always_fuse = false;    // always_fuse=1: no cost-based split of fused blocks
    std::string unfuse;          // unfuse=b3;b4: split these blocks
    double unfuse_ratio = 0.85;  // model margin a split must win by
    double mb_max_weight = -1;   // cap (bytes) on a multi-branch kernel's conv weights (<0: none)
    int mb_pw = 0;               // tensor-core plans: let steps the pointwise kernel would run join multi-branch kernels
    bool no_nalt = false;        // no N-block TMEM column alternation
    bool no_tsep = false;        // groups share TMEM columns
    bool no_pwait = false;       // a tile's first group waits for the previous tile's last unit
    bool xrel_epi = false;       // staging buffer released by the epilogue warps
    int xbuf = 0;                // force 1 / 2 input staging buffers
    int wres = -1;               // force resident (1) / ring-streamed (0) weights
    int tsets = 0;               // force 1 / 2 accumulator sets
    int ctas = 0;                // cap on resident CTAs per SM
    int nsplit = 0;              // force output-channel groups (tensor-core steps that can split)
    bool pdl = true;             // programmatic dependent launch between steps
    bool no_pw = false;          // 1x1 convs through the generic fused-block kernel, not the pointwise GEMM kernel
    bool no_stem = false;        // the first conv + max-pool through the generic fused-block kernel, not the stem kernel
    bool no_s2d = false;         // keep a stride-2 first conv on its own input (no space-to-depth rewrite)
    bool pw_mc = false;          // pointwise channel groups as one cluster with the input multicast (TMA .multicast::cluster)
    bool no_dw = false;          // depthwise (+ pointwise) steps through the generic kernels, not the depthwise kernel
    bool no_fire = false;        // split-mode squeeze -> expand blocks through the generic fused-block kernel, not the fire kernel
    int fire_g = 0, fire_r = 0, fire_nsplit = 0;  // force the fire kernel's unit (G images / R-row bands) and channel groups
    int fire_cps = 0;            // fire kernel CTAs per SM: 0 planner's choice, 1 or 2
    int fire_cb = 0;             // fire kernel squeeze-input chunk: 0 planner's choice, 128 or 64 bytes per pixel per stage
    int fire_sqs = 0;            // fire kernel squeeze weights: 0 planner's choice, 1 streamed through the ring, 2 resident
    int fire_stage = 0;          // fire kernel stores: 0 direct (16-byte fragments), 1 staged through shared memory (whole segments)
    int trace = 0;               // 1: phase stamps of a steady tile, 2: tile end stamps
    bool tune_verbose = false;   // autotune prints every timing to stderr
    int e2e_chunks = 4;          // run_host pipeline depth
    bool e2e_ramp = true;        // run_host: half-size first / last chunk (measured +0.8 % end to end)
    // tile=<layer>:<h>x<w>;...: the step executing <layer> runs at this output
    // tile (a reference TilingPlan's geometry, xlf_block_prepare) or, when the
    // B200 kernel cannot hold it, at its largest feasible exact sub-tile (h' | h,
    // w' | w: every plan tile is a union of kernel tiles; results do not depend
    // on the tiling)
    std::map<std::string, std::pair<int, int>> tiles;
    // The forced tile of step `s` (true), from any of its layers.
    bool forced_tile(const struct StepSpec& s, int* th, int* tw) const;
    // Throws ErrorKind::validation on an unknown key or malformed value.
    static Knobs parse(const std::string& text);
};

struct TensorSlot {
    bool materialized = false;
    int alloc = -1;               // allocation index
    int cstride = 0, coff = 0;    // channel pitch of the allocation, offset of this tensor
    int C = 0, H = 0, W = 0;
};

struct OpSpec {
    std::string layer;
    int stage = 1;
    bool staged = false;     // result kept in a shared buffer
    bool emit = false;       // result stored to HBM
    bool own_only = false;   // staged + emitted escaping intermediate
    int xin = 0;             // stage 1: which block input it reads
    std::vector<int> srcs;   // stage 2: indices (into ops) of the stage-1 ops it reads
};

struct StepSpec {
    enum Kind { FUSED, CONCAT_COPY, ADD, RELU } kind = FUSED;
    std::string id;                    // block id (partition's naming)
    FusionMode mode = FusionMode::unfused;
    std::string tag;                   // "split", "straight+pool", "multi-branch", "conv", ...
    std::vector<std::string> inputs;   // block inputs (tensor names)
    std::vector<OpSpec> ops;
    std::vector<std::string> layers;   // every layer executed by this step
    int out_h = 0, out_w = 0;
    int tile_h = 0, tile_w = 0;
    // tensor-core steps (bf16 / TF32):
    int nxb = 1;        // input staging buffers (2 = next tile's inputs prefetched)
    int wres = 0;       // weights resident in shared memory (else streamed through the ring)
    int ring_slots = 3; // ring depth when streamed
    int grid_all = 0;   // one tile per CTA (grid = tiles) instead of a persistent grid
    int epi_warps = 8;  // epilogue/SIMT warps per CTA (4 or 8)
    int tsets = 1;      // TMEM accumulator sets (2 = cross-tile MMA/epilogue overlap)
    int ring_chunk = 16384;  // bytes per weight-ring slot
    int nsplit = 1;     // output-channel groups over the grid's y dimension (weights of a group resident per CTA)
    int rb = 1;         // fp32: register-blocked conv variants allowed (0 = the generic cell-quad path)
    int threads = 256;  // fp32: threads per CTA (256 or 512)
    // tensor-core conv + global average pool (SqueezeNet conv10 -> pool10): the
    // step's single conv op never stores its output; its epilogue reduces
    // every tile over its cells and the pooled layer `gap_out` (1x1) is
    // finished by a small reduction kernel.  Tiles are over the conv output.
    std::string gap_out;
    int ctile = 0;                     // channel tile of pool-only steps (0 = all)
    int smem_bytes = 0;
    // statistics (per image)
    double macs = 0;            // algorithmic MACs (no halo recompute)
    double macs_executed = 0;   // including halo recompute and edge waste
    double bytes_algorithmic = 0;  // block inputs once + stored outputs once, per image (HBM element size)
    double weight_bytes = 0;       // weights + biases once per launch (HBM element size)
};

struct DevicePlan {
    Partition partition = Partition::b200;
    int tc_es = 0;                       // 0: fp32 SIMT kernels; 2: bf16 / 4: TF32 tensor-core kernels (HBM element bytes)
    std::vector<FusionBlock> blocks;     // the partition, reference vocabulary
    std::vector<StepSpec> steps;
    std::map<std::string, TensorSlot> tensors;
    std::vector<long long> alloc_floats;  // per image
    // weights: offsets (floats) into one packed device buffer, per conv layer
    std::map<std::string, long long> w_off, b_off;
    long long weight_floats = 0;
};

// Blocks of the B200 partition (reference vocabulary: producer/consumer stages).
std::vector<FusionBlock> detect_fusion_blocks_b200(const Graph& g);

// batch_hint steers the tile choice (enough CTAs to fill 148 SMs).
// tc_es = 2 / 4: plan for the tensor-core kernel (kernels_tc.cu): bf16 / fp32
// (TF32) NHWC tensors with channels padded to 16 bytes, tiles from its
// geometry (device_plan_tc.cpp); tc_es = 0: the fp32 SIMT kernel.
DevicePlan plan_device(const Graph& g, Partition part, int batch_hint = 1, int smem_budget_bytes = 227 * 1024, int tc_es = 0,
                       const Knobs& knobs = Knobs{});

// fire_plan.cpp: steps the fire kernel (kernels_fire.cu) runs -- a 1x1 squeeze
// staged on chip feeding stride-1 "same" expand convs (k <= 3) of one width.
bool fire_step_ok(const Graph& g, const StepSpec& s, int es);
// ... and the kernel has a unit / channel split that fits at `batch` images.
bool fire_feasible(const Graph& g, const StepSpec& s, int es, int batch, const Knobs& k);

// device_plan_tc.cpp
bool tc_mma_ok(const Layer& l, int es);
void tc_nblocks(int cout, int* nblocks, int* nb);
long long layout_tc(const Graph& g, const StepSpec& s, int th, int tw, struct BParams* P, int nxb, int wres, int ring_slots, int tsets,
                    int chunk, int es, const Knobs& k);
bool choose_tile_tc(const Graph& g, StepSpec& s, int batch_hint, int smem_budget, int es, const Knobs& k);
// One configuration of a tensor-core step: tile, staging buffers, weight residency /
// ring depth, shared bytes, and the model's score (SM cycles, lower better).
struct BCandidate {
    int th, tw, nxb, wres, slots, smem, epi_warps, tsets, chunk;
    double model;
    int nsplit;
};
// fp32 SIMT steps: every feasible (tile, register-blocked on/off) ranked by
// the SM-cycle model (fp32_tile_cycles), best first; the measured-time tuner
// times the best of each mode.
struct F32Candidate {
    int th, tw, rb, threads, smem;
    double model;
};
std::vector<F32Candidate> candidates_fp32(const Graph& g, const StepSpec& s, int batch_hint, int smem_budget);
// Shared bytes of an fp32 step at a tile (-1 = infeasible); the step's `rb` applies.
long long fp32_layout_bytes(const Graph& g, const StepSpec& s, int th, int tw);
std::vector<BCandidate> candidates_tc(const Graph& g, const StepSpec& s, int batch_hint, int smem_budget, int es, const Knobs& k);
void apply_candidate(StepSpec& s, const BCandidate& c);
std::vector<uint8_t> pack_weights_tc(const Graph& g, const float* flat, size_t count, std::map<std::string, long long>& off, int es);
// One MMA conv's packed weights with an explicit N blocking (nblocks x nb
// columns, zero past cout): the packing of an N-split op (BOp::gch).
std::vector<uint8_t> pack_layer_tc(const Graph& g, const std::string& layer, const float* flat, size_t count, int es, int nb, int nblocks);

// Packs reference-layout weights (save_weights stream order, tensor.cpp:64-95)
// into the device layout of `plan`: per conv [cin/group][kh][kw][cout_pad4]
// followed by bias[cout_pad4].
std::vector<float> pack_weights(const Graph& g, const DevicePlan& plan, const float* flat, size_t count);

// Builds the launch descriptor of a FUSED step; `base(t)` returns the device
// address of image 0 of tensor slot allocation, `wbase` the packed weights.
FusedParams make_params(const Graph& g, const DevicePlan& plan, const StepSpec& s,
                        const std::vector<float*>& alloc_base, const float* wbase);

std::string describe_plan_json(const Graph& g, const DevicePlan& plan);

// Recomputes a step's statistics (macs, bytes_algorithmic, weight_bytes)
// against graph `g` (e.g. the user's graph when the engine rewrote a layer).
void fill_stats(const Graph& g, const DevicePlan& plan, StepSpec& s);

}  // namespace xlf
