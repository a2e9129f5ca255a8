// Tiling parameters of the drop-in API (reference include/xlfuse/tiling.hpp,
// device.hpp, cost_model.hpp:38-55).  plan_tiling reproduces the reference's
// plan for a given geometry and device (pinned against the reference's plans
// in tests/golden/golden.json); b200_spec() retargets the resource checks to
// B200 (227 KB shared per block, 228 KB per SM, TMEM 512 columns x 128 lanes).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "fusion.hpp"
#include "graph.hpp"

namespace xlf {

struct DeviceSpec {
    std::string name;
    int sm_count = 0;
    double peak_flops = 0, global_bw = 0, shared_bw = 0;
    std::int64_t shared_per_sm = 96 * 1024;
    std::int64_t shared_per_block_max = 48 * 1024;
    std::int64_t constant_capacity = 64 * 1024;
    std::int64_t readonly_cache = 48 * 1024;
    int banks = 32, bank_word = 4, warp_size = 32, transaction_bytes = 16;
    int max_blocks_per_sm = 32, max_threads_per_block = 1024;
    // B200 additions (0 on pre-Blackwell parts).
    int tmem_columns = 0, tmem_lanes = 0;
    void check() const;
};

DeviceSpec titan_xp_spec();
DeviceSpec tesla_p4_spec();
DeviceSpec b200_spec();
DeviceSpec parse_device(const std::string& text);
std::string serialize_device(const DeviceSpec& d);

struct TileGeometry {
    int tile_h = 1, tile_w = 1, grid_h = 1, grid_w = 1, loop_h = 1, loop_w = 1;
    bool operator==(const TileGeometry&) const = default;
};

struct HaloStage {
    std::string layer;
    int kernel_h = 1, kernel_w = 1, stride = 1, pad = 0, channels_out = 0;
    std::int64_t macs_per_cell = 0;
    int extent_h = 0, extent_w = 0, scale_h = 1, scale_w = 1, offset_h = 0, offset_w = 0;
};
struct HaloExtent {
    std::vector<HaloStage> stages;
};

HaloExtent halo_extent(int tile_h, int tile_w, const std::vector<ConvParams>& chain);

struct RedundancyReport {
    std::int64_t staged_input_elements = 0, unique_input_elements = 0, replicated_elements = 0;
    std::int64_t intermediate_staged_cells = 0, intermediate_unique_cells = 0, recomputed_cells = 0, redundant_macs = 0;
};
RedundancyReport redundancy_count(const TileGeometry& geo, const HaloExtent& halo, const TensorShape& input);

std::vector<TileGeometry> enumerate_tilings(int out_h, int out_w);
TileGeometry full_tile_geometry(int out_h, int out_w);

enum class WeightPlacement { constant_memory, readonly_cached_global };

struct SharedLayout {
    std::string name, stage;
    int channels = 0, logical_h = 0, logical_w = 0, border = 0, pad_rows = 0, pad_cols = 1, stride = 1;
    int data_h() const { return logical_h + 2 * border; }
    int data_w() const { return logical_w + 2 * border; }
    int pitch() const { return data_w() + pad_cols; }
    int rows() const { return data_h() + pad_rows; }
    std::int64_t physical_elements() const { return std::int64_t(channels) * rows() * pitch(); }
};

struct TilingPlan {
    std::string graph_name, block_id;
    FusionMode mode = FusionMode::straight;
    std::vector<std::string> producers, consumers;
    bool stores_intermediate = false, shared_input_staging = false;
    TileGeometry geometry;
    int block_dim_x = 1, block_dim_y = 1;
    HaloExtent halo;
    std::vector<SharedLayout> buffers;
    WeightPlacement weights = WeightPlacement::constant_memory;
    std::int64_t replicated_elements = 0, redundant_macs = 0, shared_bytes = 0;
    std::string device_name;
};

struct PlanOptions {
    bool row_bank_padding = false;
};

TilingPlan plan_tiling(const Graph& g, const FusionBlock& b, const TileGeometry& geo, const DeviceSpec& dev,
                       const PlanOptions& opts = {});

struct OccupancyReport {
    int blocks_per_sm = 0;
    double shared_fraction = 0;
    std::vector<std::string> warnings;
};
OccupancyReport check_resources(const TilingPlan& plan, const DeviceSpec& dev);

std::string serialize_plan(const TilingPlan& p);
TilingPlan parse_plan(const std::string& text);

// Modelled 16-byte store transactions (cost_model.cpp:15-55).
std::int64_t transactions_for(std::int64_t elements, const DeviceSpec& d);
std::int64_t global_store_tx_fused(const Graph& g, const FusionBlock& b, const DeviceSpec& d);
std::int64_t global_store_tx_unfused(const Graph& g, const std::vector<std::string>& layers, const DeviceSpec& d);

}  // namespace xlf
