/*
 * xlfuse_b200.h -- C ABI of the B200-native cross-layer fused CNN inference
 * path (arXiv 2007.06000).  Plain pointers and sizes only; no torch or C++
 * types cross this boundary.  Library: paper_2007_06000_b200/libxlfuse_b200.so
 *
 * Each entry point names the reference interface it replaces
 * (reference repository proj/, file:line).  All functions return XLF_OK or an
 * error code; the message is available from xlf_last_error() (thread-local).
 * Device entry points are asynchronous on the given cudaStream_t (passed as
 * void*; NULL = the legacy default stream) unless documented otherwise.
 */
#ifndef XLFUSE_B200_H
#define XLFUSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors xlfuse::ErrorKind (include/xlfuse/error.hpp:12-19) plus CUDA / argument errors. */
typedef enum {
    XLF_OK = 0,
    XLF_E_IO = 1,
    XLF_E_PARSE = 2,
    XLF_E_VALIDATION = 3,
    XLF_E_INFEASIBLE = 4,
    XLF_E_VERIFICATION = 5,
    XLF_E_INTERNAL = 6,
    XLF_E_CUDA = 7,
    XLF_E_ARG = 8
} xlf_status;

/* Which partition the device executes. */
typedef enum {
    XLF_PART_REFERENCE = 0, /* detect_fusion_blocks (fusion.cpp:147-226): straight/split/merge, concat unfused */
    XLF_PART_B200 = 1,      /* + pool epilogues, concat sinks, shared-input multi-branch kernels */
    XLF_PART_UNFUSED = 2    /* one kernel per layer (the unfused sm_100a baseline) */
} xlf_partition;

typedef enum {
    XLF_FP32_EXACT = 0, /* bit-exact with run_reference (reference.cpp:16-57) */
    XLF_FP32 = 1,       /* FFMA, <= 1e-5 norm-wise */
    XLF_BF16 = 2,       /* bf16 operands (tcgen05 kind::f16), fp32 accumulate, <= 1e-2 norm-wise */
    XLF_TF32 = 3        /* fp32 storage rounded to TF32 (tcgen05 kind::tf32), fp32 accumulate, <= 1e-3 norm-wise */
} xlf_precision;

typedef struct xlf_graph xlf_graph;
typedef struct xlf_engine xlf_engine;

const char* xlf_last_error(void);
const char* xlf_version(void);

/* ---- graph and planner (host only) ------------------------------------ */

/* parse_graph + infer_shapes + fold_elementwise (graph.cpp:221-256, :405-417,
 * fusion.cpp:24-51) on the reference's structured-text graph format. */
xlf_status xlf_graph_parse(const char* text, xlf_graph** out);
void xlf_graph_destroy(xlf_graph* g);
/* JSON: name, inputs, outputs, layers (kind, inputs, shape, conv/pool params). */
xlf_status xlf_graph_json(const xlf_graph* g, char* buf, size_t cap, size_t* need);
/* serialize_graph (graph.cpp:266-301) of the prepared graph. */
xlf_status xlf_graph_serialize(const xlf_graph* g, char* buf, size_t cap, size_t* need);

/* detect_fusion_blocks (fusion.cpp:147-226) / B200 partition, as
 * block_assignment_report text (fusion.cpp:228-256) or JSON. */
xlf_status xlf_block_report(const xlf_graph* g, int partition, char* buf, size_t cap, size_t* need);
xlf_status xlf_blocks_json(const xlf_graph* g, int partition, char* buf, size_t cap, size_t* need);
/* classify_mode (fusion.cpp:53-128): names separated by ','; JSON result. */
xlf_status xlf_classify_mode(const xlf_graph* g, const char* names_csv, char* buf, size_t cap, size_t* need);
/* plan_tiling (tiling.cpp:240-419) for a block of the reference partition at
 * an explicit geometry on `device` ("titan_xp" | "tesla_p4" | "b200" or a
 * device document, device.cpp:38-62); serialize_plan text (tiling.cpp:493). */
xlf_status xlf_plan_tiling(const xlf_graph* g, const char* block_id, int tile_h, int tile_w, int grid_h, int grid_w,
                           const char* device, char* buf, size_t cap, size_t* need);
/* serialize_device (device.cpp:64-90) of a device ("titan_xp" | "tesla_p4" |
 * "b200" or a device document, parsed and checked by parse_device,
 * device.cpp:38-62): the DeviceSpec documents the planner and
 * xlf_block_prepare accept.  paper_2007_06000_b200/devices/b200.device is
 * this function's output for "b200". */
xlf_status xlf_device_document(const char* device, char* buf, size_t cap, size_t* need);
/* Modelled 16-B store transactions fused / unfused (cost_model.cpp:43-55, titan_xp). */
xlf_status xlf_store_tx(const xlf_graph* g, const char* block_id, long long* fused, long long* unfused);
/* Device program of a partition (host-only planning: kernel steps, tiles,
 * shared bytes, tensor placement) as JSON; batch_hint steers the tile choice. */
xlf_status xlf_device_plan_json(const xlf_graph* g, int partition, int precision, int batch_hint, char* buf, size_t cap,
                                size_t* need);
/* Same, with engine options (see xlf_engine_create_ex). */
xlf_status xlf_device_plan_json_ex(const xlf_graph* g, int partition, int precision, int batch_hint, const char* options, char* buf,
                                   size_t cap, size_t* need);
/* seeded_weights (tensor.cpp:42-62) in save_weights stream order (tensor.cpp:64-95).
 * out may be NULL to query *count. */
xlf_status xlf_seeded_weights(const xlf_graph* g, uint64_t seed, float* out, size_t cap, size_t* count);

/* ---- device executor (replaces simulate_graph fused_exec.cpp:313-349 and
 *      run_fused_block fused_exec.cpp:30-311) ----------------------------- */

/* weights: save_weights stream order, reference layout [oc][ic/g][kh][kw] + bias. */
xlf_status xlf_engine_create(const xlf_graph* g, int device, int partition, int precision, const float* weights,
                             size_t n_weights, int max_batch, xlf_engine** out);
/* Same, with planner / executor options "key=value,..." (NULL or "" = the
 * product defaults; nothing is read from the environment).  Keys:
 * always_fuse, unfuse (block ids separated by ';'), unfuse_ratio, mb_max_weight,
 * xbuf, wres, tsets, ctas, no_nalt, no_tsep, no_pwait, xrel_epi, pdl, trace,
 * tune_verbose, e2e_chunks, e2e_ramp.  XLF_E_VALIDATION for an unknown key. */
xlf_status xlf_engine_create_ex(const xlf_graph* g, int device, int partition, int precision, const float* weights,
                                size_t n_weights, int max_batch, const char* options, xlf_engine** out);
void xlf_engine_destroy(xlf_engine* e);
/* JSON description: steps (kernels, tiles, shared bytes, MACs, algorithmic bytes), tensors. */
xlf_status xlf_engine_json(const xlf_engine* e, char* buf, size_t cap, size_t* need);
int xlf_engine_num_steps(const xlf_engine* e);
int xlf_engine_launches_per_forward(const xlf_engine* e);
/* Device input, NCHW fp32 (reference layout, images stacked): the graph's
 * first input, or the input called `name` (graphs with several inputs). */
xlf_status xlf_engine_set_input(xlf_engine* e, const float* d_nchw, int batch, void* stream);
xlf_status xlf_engine_set_input_named(xlf_engine* e, const char* name, const float* d_nchw, int batch, void* stream);
/* Input generated on device from SeededStream(seed) (tensor.cpp:19-40):
 * image n = stream elements [(first_image+n)*CHW, ...). */
xlf_status xlf_engine_set_input_seeded(xlf_engine* e, uint64_t seed, uint64_t first_image, int batch, void* stream);
/* All blocks of the partition (one CUDA-graph launch when use_graph != 0). */
xlf_status xlf_engine_forward(xlf_engine* e, int batch, int use_graph, void* stream);
/* One step (fused block or singleton) of the partition. */
xlf_status xlf_engine_run_step(xlf_engine* e, int step, int batch, void* stream);
/* Tensor `name` (any materialised layer output) as NCHW fp32 into d_nchw. */
xlf_status xlf_engine_read(xlf_engine* e, const char* name, float* d_nchw, int batch, void* stream);
/* End to end from host memory: H2D of the NCHW input, forward, D2H of tensor
 * `name` into h_out (NCHW). Synchronous. */
xlf_status xlf_engine_run_host(xlf_engine* e, const float* h_in_nchw, int batch, const char* name, float* h_out_nchw,
                               void* stream);
/* Measured-time tuner (no reference counterpart: replaces the reference's
 * model-only tune(), cost_model.cpp:236-294): times the `topk` best
 * configurations of every fused step on the device (`reps` launches each,
 * `batch` images) and keeps the fastest -- tensor-core (bf16 / TF32) steps:
 * tile, staging, weight residency, epilogue warps, accumulator sets, channel
 * groups; fp32 SIMT steps: tile, register-blocked convs on / off, 256 / 512
 * threads per CTA (results do not depend on the choice: fp32_exact stays
 * bit-identical to the reference). The
 * choices are reported by xlf_engine_tune_report (JSON) and by
 * xlf_engine_json's plan. Synchronous; not thread-safe with other calls on
 * the same engine. */
xlf_status xlf_engine_autotune(xlf_engine* e, int batch, int reps, int topk);
xlf_status xlf_engine_tune_report(const xlf_engine* e, char* buf, size_t cap, size_t* need);
/* Applies a tuning report (the JSON xlf_engine_tune_report returns, e.g. saved
 * from an earlier run on the same model / batch / GPU) without measuring:
 * XLF_E_VALIDATION for an unknown step, XLF_E_INFEASIBLE for a configuration
 * this plan cannot run, XLF_E_PARSE for malformed input. */
xlf_status xlf_engine_apply_tuning(xlf_engine* e, const char* json);
/* Profiling aid (engine created with option trace=1, tensor-core precisions):
 * globaltimer stamps of the first CTAs of a step's last launch. */
xlf_status xlf_engine_trace(const xlf_engine* e, int step, unsigned long long* out, size_t cap, size_t* count);

/* ---- one fused block: replaces run_fused_block (fused_exec.hpp:35-37,
 *      fused_exec.cpp:30-311) ------------------------------------------- */

typedef struct xlf_block xlf_block;

typedef enum {
    XLF_LAYOUT_NCHW_F32 = 0, /* reference layout: CHW fp32 per image, images stacked */
    XLF_LAYOUT_NHWC = 1      /* the engine's HBM layout: bf16 (XLF_BF16) or fp32 (other precisions),
                                `cstride` elements per pixel, the tensor at channel `coff` (e.g. its
                                concat slice); both multiples of 16 bytes, address 16-byte aligned.
                                Inputs: channels past C up to the next 16-byte multiple must be zero;
                                outputs: those pad channels are written (as zero). */
} xlf_layout;

/* A caller-owned device tensor (image 0's address; `batch` images follow). */
typedef struct {
    void* data;
    int layout;  /* xlf_layout */
    int cstride; /* NHWC only */
    int coff;    /* NHWC only */
} xlf_tensor_ref;

/* Prepares block `block_id` of `partition` (XLF_PART_REFERENCE: exactly
 * detect_fusion_blocks, fusion.cpp:147-226; or XLF_PART_B200) for `max_batch`
 * images on GPU `gpu`.  weights: the WHOLE graph's weights in save_weights order
 * (the reference's WeightSet).  plan_text: a serialize_plan document
 * (tiling.cpp:493-527; e.g. from xlf_plan_tiling or the reference planner) whose
 * tile geometry the kernel runs at, or NULL for the B200 planner's tile; a plan
 * for another block -> XLF_E_VALIDATION (fused_exec.cpp:33-38), a geometry the
 * B200 kernel cannot hold -> XLF_E_INFEASIBLE.  device: "b200" (default, NULL),
 * "titan_xp", "tesla_p4" or a device document (parse_device, device.cpp:38-62):
 * the transaction size of the counters in xlf_block_json.  An unfused block ->
 * XLF_E_INTERNAL (as the reference).  The handle is immutable for the caller;
 * xlf_block_run may be called from several threads (runs on different streams
 * are ordered by the library: they share the block's staging tensors). */
xlf_status xlf_block_prepare(const xlf_graph* g, const char* block_id, int partition, const char* plan_text, const char* device, int gpu,
                             int precision, const float* weights, size_t n_weights, int max_batch, const char* options, xlf_block** out);
/* JSON: inputs / outputs in the order xlf_block_run takes them (the block's
 * external inputs in layer order; stored_tensors order, cost_model.cpp:21-41),
 * tile, element bytes, per-image counters (stored elements, global store
 * transactions, MACs), the engine's plan. */
xlf_status xlf_block_json(const xlf_block* b, char* buf, size_t cap, size_t* need);
/* Runs the block on `batch` images: reads ins[i], writes outs[i] (caller-owned,
 * any mix of layouts).  Asynchronous and stream-ordered, no host sync.  The
 * first run with a new set of NHWC addresses builds their descriptors (cached). */
xlf_status xlf_block_run(xlf_block* b, const xlf_tensor_ref* ins, int n_ins, const xlf_tensor_ref* outs, int n_outs, int batch,
                         void* stream);
void xlf_block_destroy(xlf_block* b);

/* ---- several GPUs of one node (batch-sharded simulate_graph,
 *      fused_exec.cpp:313-349) ------------------------------ */

typedef struct xlf_multi xlf_multi;

/* Images [*first, *first + *count) of device slot `slot` when `batch` images
 * are split over n devices: contiguous, sizes differ by at most one (the first
 * batch % n slots take one more); n*B images give slot k exactly [k*B, (k+1)*B). */
xlf_status xlf_shard(int batch, int n_devices, int slot, int* first, int* count);
/* One engine per listed device (weights replicated), each driven by its own
 * host worker thread and stream; no collective on the data path. */
xlf_status xlf_multi_create(const xlf_graph* g, const int* devices, int n_devices, int partition, int precision, const float* weights,
                            size_t n_weights, int max_batch_per_device, const char* options, xlf_multi** out);
void xlf_multi_destroy(xlf_multi* m);
/* Every device tunes its engine (concurrently); see xlf_engine_autotune. */
xlf_status xlf_multi_autotune(xlf_multi* m, int batch_per_device, int reps, int topk);
/* End to end from host memory over all devices (xlf_shard ranges of `batch`):
 * each device copies in its images, runs them and writes its slice of tensor
 * `name` into h_out (NCHW).  Synchronous.  ms_per_device (n values, may be
 * NULL): each device's wall time. */
xlf_status xlf_multi_run_host(xlf_multi* m, const float* h_in, int batch, const char* name, float* h_out, double* ms_per_device);
/* Device-resident throughput: device k generates images [k*B, (k+1)*B) of
 * SeededStream(seed) (B = batch_per_device) and times `steps` forwards after
 * `warmup` (CUDA events on its stream); ms_per_device[k] = ms per forward. */
xlf_status xlf_multi_time_seeded(xlf_multi* m, uint64_t seed, int batch_per_device, int steps, int warmup, double* ms_per_device);

#ifdef __cplusplus
}
#endif
#endif /* XLFUSE_B200_H */
