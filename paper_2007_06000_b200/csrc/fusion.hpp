// Fusion planner of the drop-in API: same types, names and partition as the
// reference (include/xlfuse/fusion.hpp:13-59, src/fusion.cpp:24-256).  The
// reference partition is what `planner = reference` runs on the GPU; the
// B200 partition (device_plan.hpp) extends it with pool epilogues, concat
// sinks and shared-input multi-branch blocks.
#pragma once

#include <string>
#include <vector>

#include "graph.hpp"

namespace xlf {

enum class FusionMode { straight, split, merge, unfused };
const char* to_string(FusionMode m);

struct FusionBlock {
    std::string id;
    FusionMode mode = FusionMode::unfused;
    std::vector<std::string> members;         // producers first, then consumers
    std::vector<std::string> producer_stage;  // kept on chip
    std::vector<std::string> consumer_stage;  // read the on-chip intermediate
    bool stores_intermediate = false;         // a producer escapes the block
    bool fused() const { return mode != FusionMode::unfused; }
};

struct ModeResult {
    bool accepted = false;
    FusionMode mode = FusionMode::unfused;
    bool escaping_intermediate = false;
    std::string reject_reason;
};

Graph fold_elementwise(const Graph& g);
ModeResult classify_mode(const Graph& g, const std::vector<std::string>& candidate);
std::vector<FusionBlock> detect_fusion_blocks(const Graph& g);
std::string block_assignment_report(const Graph& g, const std::vector<FusionBlock>& blocks);

// Tensors a fused block writes to global memory: consumer outputs plus
// producers visible outside the block (cost_model.cpp:21-41 semantics).
std::vector<std::pair<std::string, std::int64_t>> stored_tensors(const Graph& g, const FusionBlock& b);

}  // namespace xlf
