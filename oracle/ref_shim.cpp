// ref_shim.cpp -- extern "C" wrapper over the UNMODIFIED xlfuse reference
// library, compiled from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libxlfuse_ref.so.
//
// TEST INFRASTRUCTURE ONLY: used to pin oracle/xlf_oracle.c, to generate the
// golden vectors under tests/golden/, and as the reference arm / cpu_baseline
// of bench.py.  The product never loads it.
//
// Every entry point returns 0 on success, a negative value on error (message
// via xref_last_error()).
#include <cstdint>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "xlfuse/cost_model.hpp"
#include "xlfuse/device.hpp"
#include "xlfuse/fused_exec.hpp"
#include "xlfuse/fusion.hpp"
#include "xlfuse/graph.hpp"
#include "xlfuse/reference.hpp"
#include "xlfuse/tensor.hpp"
#include "xlfuse/tiling.hpp"

using namespace xlfuse;

namespace {
thread_local std::string g_err;

Graph prepared(const char* text) { return fold_elementwise(infer_shapes(parse_graph(text))); }

int copy_out(const std::string& s, char* buf, size_t cap, size_t* need) {
    if (need) *need = s.size() + 1;
    if (!buf || cap < s.size() + 1) return buf ? -2 : 0;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

// Input for image n of a batch = elements [n*CHW, (n+1)*CHW) of one
// SeededStream(seed) (so image 0 equals seeded_inputs(g, seed)).
std::map<std::string, Tensor> image_inputs(const Graph& g, const float* batch, int n) {
    std::map<std::string, Tensor> in;
    size_t off = 0;
    for (const auto& gi : g.inputs) {
        Tensor t(gi.shape);
        const size_t chw = t.data.size();
        std::memcpy(t.data.data(), batch + (size_t)n * chw + off, chw * 4);
        in.emplace(gi.name, std::move(t));
        off += 0;  // single-input graphs only (all fixtures)
    }
    return in;
}
}  // namespace

extern "C" {

const char* xref_last_error() { return g_err.c_str(); }

// Weights of the prepared graph in file order (filter then bias per conv),
// exactly save_weights' stream (tensor.cpp:64-95).
int xref_seeded_weights(const char* graph_text, uint64_t seed, float* out, size_t cap, size_t* count) {
    try {
        Graph g = prepared(graph_text);
        WeightSet w = seeded_weights(g, seed);
        size_t n = 0;
        for (const auto& l : g.layers) {
            if (l.kind != LayerKind::conv) continue;
            const auto& lw = w.by_layer.at(l.name);
            for (float v : lw.filter) { if (out && n < cap) out[n] = v; ++n; }
            for (float v : lw.bias) { if (out && n < cap) out[n] = v; ++n; }
        }
        if (count) *count = n;
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return -1; }
}

int xref_seeded_inputs(const char* graph_text, uint64_t seed, float* out, size_t n) {
    try {
        Graph g = prepared(graph_text);
        SeededStream rng(seed);
        for (size_t i = 0; i < n; ++i) out[i] = rng.next();
        (void)g;
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return -1; }
}

// run_reference (reference.cpp:126-142) per image on a batch.  `weights`
// in save_weights order (may be null: seeded_weights(g, wseed)).  Writes
// tensor `name` for every image, CHW, contiguous per image.
// mode 0: run_reference (oracle), mode 1: simulate_graph through the
// reference planner + titan_xp tuned plans (the reference fused interpreter).
int xref_run(const char* graph_text, const float* weights, uint64_t wseed, const float* inputs,
             int batch, const char* name, float* out, int mode, int threads) {
    try {
        Graph g = prepared(graph_text);
        WeightSet w;
        if (weights) {
            size_t off = 0;
            for (const auto& l : g.layers) {
                if (l.kind != LayerKind::conv) continue;
                LayerWeights lw;
                lw.filter.assign(weights + off, weights + off + l.conv->weight_count());
                off += (size_t)l.conv->weight_count();
                lw.bias.assign(weights + off, weights + off + l.conv->bias_count());
                off += (size_t)l.conv->bias_count();
                w.by_layer.emplace(l.name, std::move(lw));
            }
        } else {
            w = seeded_weights(g, wseed);
        }
        std::vector<FusionBlock> blocks;
        std::map<std::string, TilingPlan> plans;
        DeviceSpec dev = titan_xp_spec();
        if (mode == 1) {
            blocks = detect_fusion_blocks(g);
            for (const auto& b : blocks)
                if (b.fused()) plans[b.id] = tune(g, b, dev).best;
        }
        const TensorShape os = g.shape_of(name);
        const size_t oelems = (size_t)os.elements();
        std::string err;
        (void)threads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads > 0 ? threads : 1) if (mode == 0)
        for (int n = 0; n < batch; ++n) {
            try {
                auto in = image_inputs(g, inputs, n);
                std::map<std::string, Tensor> vals;
                if (mode == 0) vals = run_reference(g, in, w);
                else vals = simulate_graph(g, blocks, plans, in, w, dev).values;
                const Tensor& t = vals.at(name);
                std::memcpy(out + (size_t)n * oelems, t.data.data(), oelems * 4);
            } catch (const std::exception& e) {
#pragma omp critical
                err = e.what();
            }
        }
        if (!err.empty()) { g_err = err; return -1; }
        return 0;
    } catch (const std::exception& e) { g_err = e.what(); return -1; }
}

// Reference planner output: block_assignment_report (fusion.cpp:228-256).
int xref_block_report(const char* graph_text, char* buf, size_t cap, size_t* need) {
    try {
        Graph g = prepared(graph_text);
        return copy_out(block_assignment_report(g, detect_fusion_blocks(g)), buf, cap, need);
    } catch (const std::exception& e) { g_err = e.what(); return -1; }
}

// Reference plan for one fused block at an explicit geometry (tiling.cpp:240-419),
// serialized by serialize_plan (tiling.cpp:493-527).  device: "titan_xp" | "tesla_p4".
int xref_plan(const char* graph_text, const char* block_id, int tile_h, int tile_w, int grid_h,
              int grid_w, const char* device, char* buf, size_t cap, size_t* need) {
    try {
        Graph g = prepared(graph_text);
        auto blocks = detect_fusion_blocks(g);
        DeviceSpec dev = std::string(device) == "tesla_p4" ? tesla_p4_spec() : titan_xp_spec();
        for (const auto& b : blocks) {
            if (b.id != block_id) continue;
            TilingPlan p;
            if (tile_h <= 0) {
                p = tune(g, b, dev).best;
            } else {
                TileGeometry geo;
                geo.tile_h = tile_h; geo.tile_w = tile_w; geo.grid_h = grid_h; geo.grid_w = grid_w;
                p = plan_tiling(g, b, geo, dev);
            }
            return copy_out(serialize_plan(p), buf, cap, need);
        }
        g_err = "no block " + std::string(block_id);
        return -1;
    } catch (const std::exception& e) { g_err = e.what(); return -1; }
}

// Modelled store transactions of a block (cost_model.cpp:43-55).
int xref_store_tx(const char* graph_text, const char* block_id, long long* fused, long long* unfused) {
    try {
        Graph g = prepared(graph_text);
        DeviceSpec dev = titan_xp_spec();
        for (const auto& b : detect_fusion_blocks(g)) {
            if (b.id != block_id) continue;
            *fused = global_store_tx_fused(g, b, dev);
            *unfused = global_store_tx_unfused(g, b.members, dev);
            return 0;
        }
        g_err = "no block";
        return -1;
    } catch (const std::exception& e) { g_err = e.what(); return -1; }
}

}  // extern "C"
