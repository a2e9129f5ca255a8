// Device executor: the B200 successor of simulate_graph (reference
// fused_exec.cpp:313-349).  One Engine = one graph on one GPU at one
// precision and partition, with weights resident in HBM, activations in a
// per-tensor arena sized for max_batch images, and one CUDA graph per batch
// size so a forward pass is a single graph launch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "device_plan.hpp"
#include "graph.hpp"

namespace xlf {

enum class Precision { fp32_exact = 0, fp32 = 1, bf16 = 2, tf32 = 3 };
const char* to_string(Precision p);

class Engine {
public:
    Engine(const Graph& g, int device, Partition part, Precision prec, const float* weights, size_t nweights, int max_batch,
           const Knobs& knobs = Knobs{});
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // Inputs: device NCHW fp32 (reference layout, images stacked), or the
    // seeded stream generated in place (image n = stream elements [n*CHW, ...)).
    void set_input_nchw(const std::string& name, const float* d_nchw, int batch, cudaStream_t st);
    void set_input_seeded(const std::string& name, uint64_t seed, uint64_t first_image, int batch, cudaStream_t st);
    // All steps for `batch` images (replays a captured CUDA graph when use_graph).
    void forward(int batch, cudaStream_t st, bool use_graph = true);
    // Images [n0, n0 + count) of every step (tensor-core plans of fused kernels only).
    void forward_range(int n0, int count, cudaStream_t st);
    bool range_capable() const;
    // One step only (per-block timing / run_fused_block).
    void run_step(int index, int batch, cudaStream_t st);
    // Caller-owned NHWC tensors (xlf_block_run): every step reads / writes the
    // named graph inputs and materialised tensors at external device addresses
    // (element type of the engine's HBM layout, `cstride` elements per pixel,
    // the tensor at channel `coff`).  Descriptors for a set of addresses are
    // built once and cached; no CUDA graph.
    struct External {
        std::string name;
        void* ptr;
        int cstride, coff;
    };
    void forward_external(const std::vector<External>& ext, int batch, cudaStream_t st);
    int element_bytes() const { return esz_; }
    size_t user_input_elements() const { return size_t(in_shape_.elements()); }  // C*H*W of input 0 as the user passes it
    // NHWC arena -> NCHW fp32.
    void read_output_nchw(const std::string& name, float* d_nchw, int batch, cudaStream_t st);
    // C*H*W of a readable tensor (throws for fused intermediates / rewritten inputs).
    size_t tensor_elements(const std::string& name) const;
    // End to end with host buffers: H2D, forward, D2H of `out_name`, sync.
    void run_host(const float* h_in_nchw, int batch, const std::string& out_name, float* h_out_nchw, cudaStream_t st);

    const Graph& graph() const { return g_; }
    const DevicePlan& plan() const { return plan_; }
    int num_steps() const { return int(plan_.steps.size()); }
    int launches_per_forward() const;
    // option trace=1 only: per-CTA phase stamps of step `index` (tensor-core kernels).
    std::vector<unsigned long long> trace(int index) const;
    std::string describe_json() const;
    // Measured-time tuning of the fused steps (tensor-core and fp32 SIMT, see engine.cpp); returns
    // the chosen configurations as JSON.
    std::string autotune(int batch, int reps, int topk);
    std::string autotune_fp32(int batch, int reps, int topk, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1);
    // Applies a report autotune returned (no measurement).
    void apply_tuning(const std::string& json);
    int max_batch() const { return max_batch_; }
    int device() const { return device_; }
    Precision precision() const { return prec_; }

private:
    void launch_step(size_t i, int batch, cudaStream_t st);
    void drop_derived();  // CUDA graphs + external-address descriptors of the current configurations
    std::unique_ptr<struct BParams> build_bparams(const StepSpec& s);
    std::unique_ptr<struct StemParams> build_stem(const StepSpec& s);
    const uint8_t* packed_for(const std::string& layer, int nb, int nblocks);
    std::unique_ptr<struct PwParams> build_pw(const StepSpec& s);
    // nsplit / G / R > 0 force the fire kernel's channel split / unit (else the knobs, else its model)
    std::unique_ptr<struct DwParams> build_dw(const StepSpec& s);
    std::unique_ptr<struct FireParams> build_fire(const StepSpec& s, int nsplit = 0, int G = 0, int R = 0, int sqs = -1, int cb = 0, int cps = 0);
    void launch_tc_step(size_t i, int n0, int count, cudaStream_t st);
    const TensorSlot& slot(const std::string& n) const;
    const TensorSlot& readable(const std::string& n) const;

    Graph g_;
    DevicePlan plan_;
    int device_;
    Precision prec_;
    int max_batch_;
    Knobs knobs_;
    std::vector<float*> allocs_;
    float* weights_ = nullptr;
    float* staging_ = nullptr;  // NCHW input staging for run_host
    cudaStream_t capture_ = nullptr;  // private stream used only to capture CUDA graphs
    size_t staging_floats_ = 0;
    std::vector<struct FusedParams> params_;
    std::vector<std::unique_ptr<struct BParams>> bparams_;  // tensor-core steps
    std::vector<std::unique_ptr<struct StemParams>> stems_;  // steps run by the stem kernel (conv + max-pool)
    std::vector<std::unique_ptr<struct PwParams>> pws_;      // steps run by the pointwise-conv GEMM kernel
    std::vector<std::unique_ptr<struct FireParams>> fires_;  // split blocks run by the fire kernel (squeeze plane on chip)
    std::vector<std::unique_ptr<struct DwParams>> dws_;      // depthwise (+ pointwise) steps (every precision)
    std::vector<unsigned long long*> traces_;                // trace buffers (option trace)
    std::map<std::string, long long> wofftc_;                // packed MMA weights: byte offset per layer
    void* weights_tc_ = nullptr;  // packed MMA weights (bf16 / TF32)
    std::vector<float> host_w_;   // the weights as given (after a space-to-depth rewrite): split packings
    std::map<std::string, void*> packed_;  // layer/nb x nblocks -> packed weights of N-split ops
    int tc_es_ = 0;               // tensor-core element bytes (2 bf16, 4 TF32), 0 = fp32 SIMT kernels
    int esz_ = 4;                 // bytes per activation element in HBM
    bool s2d_ = false;            // tensor cores: first conv rewritten on a space-to-depth input
    int s2d_planar_ = 0;          // ... stored row-planar (the stem kernel reads it)
    TensorShape in_shape_;        // user-facing (NCHW) shape of input 0
    std::map<std::string, TensorShape> user_inputs_;  // graph inputs as the user passes them
    std::map<long long, cudaGraphExec_t> graphs_;  // key > 0: whole batch; < 0: image range (forward_range)
    static constexpr int kMaxChunks = 16;     // run_host pipelining
    cudaStream_t copy_in_ = nullptr, copy_out_ = nullptr;
    cudaEvent_t chunk_ev_[2 * kMaxChunks] = {};
    float* out_staging_ = nullptr;
    std::map<std::string, std::pair<float*, size_t>> gap_parts_;  // conv+gap steps: per-tile partial sums
    std::vector<void*> retired_;                                  // outgrown buffers, freed with the engine
    struct ExtSet {  // descriptors of one set of caller-owned addresses
        std::vector<float*> allocs;
        std::map<std::string, TensorSlot> tensors;
        std::vector<std::unique_ptr<struct BParams>> bp;
        std::vector<struct FusedParams> fp;
        std::vector<std::unique_ptr<struct FireParams>> fr;
        std::vector<std::unique_ptr<struct DwParams>> dw;
    };
    std::map<std::string, std::unique_ptr<ExtSet>> ext_sets_;
};

std::vector<float> seeded_weights(const Graph& g, uint64_t seed);  // tensor.cpp:42-62 semantics
float seeded_value(uint64_t seed, uint64_t index);                    // SeededStream element

void cuda_check(cudaError_t e, const char* what);

}  // namespace xlf
