// extern "C" boundary (include/xlfuse_b200.h).  Every entry point catches
// xlf::Error / std::exception and maps it to an xlf_status with the message
// in a thread-local buffer (the reference throws xlfuse::Error instead,
// error.hpp:21-35).
#include "../../include/xlfuse_b200.h"

#include <algorithm>
#include <cstring>
#include <mutex>
#include <memory>
#include <sstream>
#include <string>

#include "common.hpp"
#include "device_plan.hpp"
#include "engine.hpp"
#include "fusion.hpp"
#include "graph.hpp"
#include "multi.hpp"
#include "tiling.hpp"

struct xlf_graph {
    xlf::Graph g;
};
struct xlf_engine {
    std::unique_ptr<xlf::Engine> e;
    std::string tune_report;  // last xlf_engine_autotune result (JSON)
};

namespace {

thread_local std::string g_error;

// A NULL / malformed argument at the boundary (XLF_E_ARG), as opposed to a
// graph / plan validation failure (XLF_E_VALIDATION).
struct ArgError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

xlf_status code_of(xlf::ErrorKind k) {
    switch (k) {
    case xlf::ErrorKind::io: return XLF_E_IO;
    case xlf::ErrorKind::parse: return XLF_E_PARSE;
    case xlf::ErrorKind::validation: return XLF_E_VALIDATION;
    case xlf::ErrorKind::infeasible: return XLF_E_INFEASIBLE;
    case xlf::ErrorKind::verification: return XLF_E_VERIFICATION;
    case xlf::ErrorKind::internal: return XLF_E_INTERNAL;
    case xlf::ErrorKind::cuda: return XLF_E_CUDA;
    }
    return XLF_E_INTERNAL;
}

template <class F>
xlf_status guard(F&& f) {
    try {
        f();
        g_error.clear();
        return XLF_OK;
    } catch (const xlf::Error& e) {
        g_error = e.what();
        return code_of(e.kind());
    } catch (const ArgError& e) {
        g_error = e.what();
        return XLF_E_ARG;
    } catch (const std::exception& e) {
        g_error = e.what();
        return XLF_E_INTERNAL;
    }
}

void put(const std::string& s, char* buf, size_t cap, size_t* need) {
    if (need) *need = s.size() + 1;
    if (!buf) return;
    if (cap < s.size() + 1) xlf::fail(xlf::ErrorKind::validation, "output buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
}

void need_ptr(const void* p, const char* what) {
    if (!p) throw ArgError(std::string(what) + " is NULL");
}

std::string jstr(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        if (c == '\n') { o += "\\n"; continue; }
        o += c;
    }
    return o + "\"";
}

std::string blocks_json(const std::vector<xlf::FusionBlock>& blocks) {
    std::ostringstream os;
    os << "[";
    for (size_t i = 0; i < blocks.size(); ++i) {
        const auto& b = blocks[i];
        auto list = [&](const std::vector<std::string>& v) {
            std::string s = "[";
            for (size_t k = 0; k < v.size(); ++k) s += (k ? "," : "") + jstr(v[k]);
            return s + "]";
        };
        os << (i ? "," : "") << "{\"id\":" << jstr(b.id) << ",\"mode\":" << jstr(xlf::to_string(b.mode))
           << ",\"members\":" << list(b.members) << ",\"producer_stage\":" << list(b.producer_stage)
           << ",\"consumer_stage\":" << list(b.consumer_stage)
           << ",\"stores_intermediate\":" << (b.stores_intermediate ? "true" : "false") << "}";
    }
    os << "]";
    return os.str();
}

std::vector<xlf::FusionBlock> partition_blocks(const xlf::Graph& g, int part) {
    if (part == XLF_PART_REFERENCE) return xlf::detect_fusion_blocks(g);
    if (part == XLF_PART_B200) return xlf::detect_fusion_blocks_b200(g);
    if (part == XLF_PART_UNFUSED) return xlf::plan_device(g, xlf::Partition::unfused).blocks;
    throw xlf::Error(xlf::ErrorKind::validation, "unknown partition");
}

xlf::DeviceSpec device_named(const char* d) {
    const std::string s = d ? d : "titan_xp";
    if (s == "titan_xp") return xlf::titan_xp_spec();
    if (s == "tesla_p4") return xlf::tesla_p4_spec();
    if (s == "b200") return xlf::b200_spec();
    return xlf::parse_device(s);
}

const xlf::FusionBlock& find_block(const std::vector<xlf::FusionBlock>& blocks, const char* id) {
    for (const auto& b : blocks)
        if (b.id == id) return b;
    throw xlf::Error(xlf::ErrorKind::validation, std::string("no block '") + id + "'");
}

}  // namespace

extern "C" {

const char* xlf_last_error(void) { return g_error.c_str(); }
const char* xlf_version(void) { return "xlfuse-b200 0.1.0 (sm_100a)"; }

xlf_status xlf_graph_parse(const char* text, xlf_graph** out) {
    return guard([&] {
        need_ptr(text, "text"), need_ptr(out, "out");
        auto h = std::make_unique<xlf_graph>();
        h->g = xlf::prepare_graph(text);
        *out = h.release();
    });
}

void xlf_graph_destroy(xlf_graph* g) { delete g; }

xlf_status xlf_graph_json(const xlf_graph* h, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(h, "graph");
        const xlf::Graph& g = h->g;
        std::ostringstream os;
        os << "{\"name\":" << jstr(g.name) << ",\"inputs\":[";
        for (size_t i = 0; i < g.inputs.size(); ++i)
            os << (i ? "," : "") << "{\"name\":" << jstr(g.inputs[i].name) << ",\"shape\":[" << g.inputs[i].shape.channels << ","
               << g.inputs[i].shape.height << "," << g.inputs[i].shape.width << "]}";
        os << "],\"outputs\":[";
        for (size_t i = 0; i < g.outputs.size(); ++i) os << (i ? "," : "") << jstr(g.outputs[i]);
        os << "],\"layers\":[";
        for (size_t i = 0; i < g.layers.size(); ++i) {
            const xlf::Layer& l = g.layers[i];
            os << (i ? "," : "") << "{\"name\":" << jstr(l.name) << ",\"kind\":" << jstr(xlf::to_string(l.kind)) << ",\"inputs\":[";
            for (size_t k = 0; k < l.inputs.size(); ++k) os << (k ? "," : "") << jstr(l.inputs[k]);
            os << "],\"shape\":[" << l.out_shape->channels << "," << l.out_shape->height << "," << l.out_shape->width << "]";
            if (l.conv) {
                const auto& c = *l.conv;
                os << ",\"conv\":{\"out_channels\":" << c.out_channels << ",\"in_channels\":" << c.in_channels
                   << ",\"kernel\":[" << c.kernel_h << "," << c.kernel_w << "],\"pad\":" << c.pad << ",\"stride\":" << c.stride
                   << ",\"group\":" << c.group << ",\"bias\":" << (c.has_bias ? "true" : "false")
                   << ",\"relu\":" << (c.activation == xlf::Activation::relu ? "true" : "false") << "}";
            }
            if (l.pool)
                os << ",\"pool\":{\"kind\":" << jstr(l.pool->kind == xlf::PoolKind::max ? "max" : "avg")
                   << ",\"kernel\":" << l.pool->kernel << ",\"stride\":" << l.pool->stride << ",\"pad\":" << l.pool->pad << "}";
            os << "}";
        }
        os << "]}";
        put(os.str(), buf, cap, need);
    });
}

xlf_status xlf_graph_serialize(const xlf_graph* h, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(h, "graph");
        put(xlf::serialize_graph(h->g), buf, cap, need);
    });
}

xlf_status xlf_block_report(const xlf_graph* h, int part, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(h, "graph");
        put(xlf::block_assignment_report(h->g, partition_blocks(h->g, part)), buf, cap, need);
    });
}

xlf_status xlf_blocks_json(const xlf_graph* h, int part, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(h, "graph");
        put(blocks_json(partition_blocks(h->g, part)), buf, cap, need);
    });
}

xlf_status xlf_classify_mode(const xlf_graph* h, const char* names_csv, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(h, "graph"), need_ptr(names_csv, "names");
        std::vector<std::string> names;
        std::stringstream ss(names_csv);
        std::string tok;
        while (std::getline(ss, tok, ','))
            if (!tok.empty()) names.push_back(tok);
        const xlf::ModeResult r = xlf::classify_mode(h->g, names);
        std::ostringstream os;
        os << "{\"accepted\":" << (r.accepted ? "true" : "false") << ",\"mode\":" << jstr(xlf::to_string(r.mode))
           << ",\"escaping_intermediate\":" << (r.escaping_intermediate ? "true" : "false")
           << ",\"reject_reason\":" << jstr(r.reject_reason) << "}";
        put(os.str(), buf, cap, need);
    });
}

xlf_status xlf_plan_tiling(const xlf_graph* h, const char* block_id, int th, int tw, int gh, int gw, const char* device, char* buf,
                           size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(h, "graph"), need_ptr(block_id, "block_id");
        const auto blocks = xlf::detect_fusion_blocks(h->g);
        xlf::TileGeometry geo;
        geo.tile_h = th, geo.tile_w = tw, geo.grid_h = gh, geo.grid_w = gw;
        put(xlf::serialize_plan(xlf::plan_tiling(h->g, find_block(blocks, block_id), geo, device_named(device))), buf, cap, need);
    });
}

xlf_status xlf_device_document(const char* device, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(device, "device");
        put(xlf::serialize_device(device_named(device)), buf, cap, need);
    });
}

xlf_status xlf_store_tx(const xlf_graph* h, const char* block_id, long long* fused, long long* unfused) {
    return guard([&] {
        need_ptr(h, "graph"), need_ptr(fused, "fused"), need_ptr(unfused, "unfused");
        const auto blocks = xlf::detect_fusion_blocks(h->g);
        const xlf::FusionBlock& b = find_block(blocks, block_id);
        const xlf::DeviceSpec d = xlf::titan_xp_spec();
        *fused = xlf::global_store_tx_fused(h->g, b, d);
        *unfused = xlf::global_store_tx_unfused(h->g, b.members, d);
    });
}

xlf_status xlf_device_plan_json_ex(const xlf_graph* h, int part, int prec, int batch_hint, const char* options, char* buf, size_t cap,
                                   size_t* need) {
    return guard([&] {
        need_ptr(h, "graph");
        if (part < 0 || part > 2) throw ArgError("unknown partition");
        if (prec < 0 || prec > 3) throw ArgError("unknown precision");
        const int es = prec == XLF_BF16 ? 2 : prec == XLF_TF32 ? 4 : 0;
        const xlf::Knobs k = xlf::Knobs::parse(options ? options : "");
        put(xlf::describe_plan_json(h->g, xlf::plan_device(h->g, xlf::Partition(part), batch_hint, 227 * 1024, es, k)), buf, cap, need);
    });
}

xlf_status xlf_device_plan_json(const xlf_graph* h, int part, int prec, int batch_hint, char* buf, size_t cap, size_t* need) {
    return xlf_device_plan_json_ex(h, part, prec, batch_hint, nullptr, buf, cap, need);
}

xlf_status xlf_seeded_weights(const xlf_graph* h, uint64_t seed, float* out, size_t cap, size_t* count) {
    return guard([&] {
        need_ptr(h, "graph");
        const std::vector<float> w = xlf::seeded_weights(h->g, seed);
        if (count) *count = w.size();
        if (out) {
            if (cap < w.size()) xlf::fail(xlf::ErrorKind::validation, "output buffer too small");
            std::memcpy(out, w.data(), w.size() * 4);
        }
    });
}

xlf_status xlf_engine_create_ex(const xlf_graph* h, int device, int part, int prec, const float* weights, size_t n, int max_batch,
                                const char* options, xlf_engine** out) {
    return guard([&] {
        need_ptr(h, "graph"), need_ptr(weights, "weights"), need_ptr(out, "out");
        if (part < 0 || part > 2) throw ArgError("unknown partition");
        if (prec < 0 || prec > 3) throw ArgError("unknown precision");
        const xlf::Knobs k = xlf::Knobs::parse(options ? options : "");
        auto e = std::make_unique<xlf_engine>();
        e->e = std::make_unique<xlf::Engine>(h->g, device, xlf::Partition(part), xlf::Precision(prec), weights, n, max_batch, k);
        *out = e.release();
    });
}

xlf_status xlf_engine_create(const xlf_graph* h, int device, int part, int prec, const float* weights, size_t n, int max_batch,
                             xlf_engine** out) {
    return xlf_engine_create_ex(h, device, part, prec, weights, n, max_batch, nullptr, out);
}

void xlf_engine_destroy(xlf_engine* e) { delete e; }

xlf_status xlf_engine_json(const xlf_engine* e, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(e, "engine");
        put(e->e->describe_json(), buf, cap, need);
    });
}

int xlf_engine_num_steps(const xlf_engine* e) { return e ? e->e->num_steps() : -1; }
int xlf_engine_launches_per_forward(const xlf_engine* e) { return e ? e->e->launches_per_forward() : -1; }

xlf_status xlf_engine_set_input(xlf_engine* e, const float* d, int batch, void* st) {
    return guard([&] {
        need_ptr(e, "engine"), need_ptr(d, "input");
        e->e->set_input_nchw(e->e->graph().inputs[0].name, d, batch, static_cast<cudaStream_t>(st));
    });
}

xlf_status xlf_engine_set_input_named(xlf_engine* e, const char* name, const float* d, int batch, void* st) {
    return guard([&] {
        need_ptr(e, "engine"), need_ptr(name, "name"), need_ptr(d, "input");
        e->e->set_input_nchw(name, d, batch, static_cast<cudaStream_t>(st));
    });
}

xlf_status xlf_engine_set_input_seeded(xlf_engine* e, uint64_t seed, uint64_t first, int batch, void* st) {
    return guard([&] {
        need_ptr(e, "engine");
        e->e->set_input_seeded(e->e->graph().inputs[0].name, seed, first, batch, static_cast<cudaStream_t>(st));
    });
}

xlf_status xlf_engine_forward(xlf_engine* e, int batch, int use_graph, void* st) {
    return guard([&] {
        need_ptr(e, "engine");
        e->e->forward(batch, static_cast<cudaStream_t>(st), use_graph != 0);
    });
}

xlf_status xlf_engine_run_step(xlf_engine* e, int step, int batch, void* st) {
    return guard([&] {
        need_ptr(e, "engine");
        e->e->run_step(step, batch, static_cast<cudaStream_t>(st));
    });
}

xlf_status xlf_engine_read(xlf_engine* e, const char* name, float* d, int batch, void* st) {
    return guard([&] {
        need_ptr(e, "engine"), need_ptr(name, "name"), need_ptr(d, "output");
        e->e->read_output_nchw(name, d, batch, static_cast<cudaStream_t>(st));
    });
}

xlf_status xlf_engine_run_host(xlf_engine* e, const float* h_in, int batch, const char* name, float* h_out, void* st) {
    return guard([&] {
        need_ptr(e, "engine"), need_ptr(h_in, "input"), need_ptr(name, "name"), need_ptr(h_out, "output");
        e->e->run_host(h_in, batch, name, h_out, static_cast<cudaStream_t>(st));
    });
}

}  // extern "C"

extern "C" xlf_status xlf_engine_autotune(xlf_engine* e, int batch, int reps, int topk) {
    return guard([&] {
        need_ptr(e, "engine");
        e->tune_report = e->e->autotune(batch, reps, topk);
    });
}

extern "C" xlf_status xlf_engine_tune_report(const xlf_engine* e, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(e, "engine");
        put(e->tune_report.empty() ? std::string("[]") : e->tune_report, buf, cap, need);
    });
}

extern "C" xlf_status xlf_engine_apply_tuning(xlf_engine* e, const char* json) {
    return guard([&] {
        need_ptr(e, "engine"), need_ptr(json, "json");
        e->e->apply_tuning(json);
        e->tune_report = json;
    });
}

extern "C" xlf_status xlf_engine_trace(const xlf_engine* e, int step, unsigned long long* out, size_t cap, size_t* count) {
    return guard([&] {
        need_ptr(e, "engine");
        const std::vector<unsigned long long> t = e->e->trace(step);
        if (count) *count = t.size();
        if (out) {
            if (cap < t.size()) xlf::fail(xlf::ErrorKind::validation, "output buffer too small");
            std::memcpy(out, t.data(), t.size() * sizeof(unsigned long long));
        }
    });
}

// ---------------------------------------------------------------- one fused block
// run_fused_block (reference fused_exec.hpp:35-37, fused_exec.cpp:30-311) on the
// device: the block's layers become a graph of their own (its external inputs
// = graph inputs, its stored tensors (cost_model.cpp:21-41) = graph outputs),
// executed by an Engine whose single fused step runs at the reference plan's
// tile geometry when one is given.
struct xlf_block {
    std::unique_ptr<xlf::Engine> e;
    xlf::FusionBlock block;
    std::vector<std::string> ins, outs;
    std::string desc;
    std::mutex mu;  // xlf_block_run may be called from several threads
    // runs share the engine's staging tensors (NCHW conversions, partial sums):
    // a run on another stream waits for the previous run's end
    cudaEvent_t done = nullptr;
    cudaStream_t last = nullptr;
    bool ran = false;
    ~xlf_block() {
        if (done) cudaEventDestroy(done);
    }
};

namespace {

xlf::Graph block_graph(const xlf::Graph& g, const xlf::FusionBlock& b, std::vector<std::string>& ins, std::vector<std::string>& outs) {
    xlf::Graph sub;
    sub.name = g.name + "_" + b.id;
    auto member = [&](const std::string& n) { return std::find(b.members.begin(), b.members.end(), n) != b.members.end(); };
    for (const xlf::Layer& l : g.layers) {
        if (!member(l.name)) continue;
        for (const std::string& i : l.inputs)
            if (!member(i) && std::find(ins.begin(), ins.end(), i) == ins.end()) {
                ins.push_back(i);
                sub.inputs.push_back({i, g.shape_of(i)});
            }
        sub.layers.push_back(l);
    }
    for (const auto& [name, elems] : xlf::stored_tensors(g, b)) outs.push_back(name);
    sub.outputs = outs;
    return xlf::infer_shapes(sub);
}

// The block's weights out of the whole graph's (save_weights order, tensor.cpp:64-95).
std::vector<float> block_weights(const xlf::Graph& g, const xlf::FusionBlock& b, const float* w, size_t n) {
    std::vector<float> out;
    size_t pos = 0;
    for (const xlf::Layer& l : g.layers) {
        if (l.kind != xlf::LayerKind::conv) continue;
        const size_t k = size_t(l.conv->weight_count() + l.conv->bias_count());
        if (pos + k > n) xlf::fail(xlf::ErrorKind::validation, "weights: " + std::to_string(n) + " values, the graph needs more");
        if (std::find(b.members.begin(), b.members.end(), l.name) != b.members.end()) out.insert(out.end(), w + pos, w + pos + k);
        pos += k;
    }
    if (pos != n) xlf::fail(xlf::ErrorKind::validation, "weights: " + std::to_string(n) + " values, the graph has " + std::to_string(pos));
    return out;
}

}  // namespace

extern "C" xlf_status xlf_block_prepare(const xlf_graph* h, const char* block_id, int part, const char* plan_text, const char* device,
                                        int gpu, int prec, const float* weights, size_t n_weights, int max_batch, const char* options,
                                        xlf_block** out) {
    return guard([&] {
        need_ptr(h, "graph"), need_ptr(block_id, "block_id"), need_ptr(weights, "weights"), need_ptr(out, "out");
        if (part != XLF_PART_REFERENCE && part != XLF_PART_B200) throw ArgError("blocks come from the reference or b200 partition");
        if (prec < 0 || prec > 3) throw ArgError("unknown precision");
        const xlf::Graph& g = h->g;
        const auto blocks = partition_blocks(g, part);
        auto b = std::make_unique<xlf_block>();
        b->block = find_block(blocks, block_id);
        if (!b->block.fused()) xlf::fail(xlf::ErrorKind::internal, "run_fused_block: block is not fused");
        const xlf::DeviceSpec dev = device_named(device ? device : "b200");
        xlf::Knobs k = xlf::Knobs::parse(options ? options : "");
        k.always_fuse = true;  // the caller asked for this block fused
        k.no_s2d = true;       // inputs keep their own layout (caller-owned NHWC buffers)
        std::string tile_src = "b200 planner";
        int plan_th = 0, plan_tw = 0;
        if (plan_text && *plan_text) {
            const xlf::TilingPlan p = xlf::parse_plan(plan_text);
            if (p.block_id != b->block.id || p.producers != b->block.producer_stage || p.consumers != b->block.consumer_stage)
                xlf::fail(xlf::ErrorKind::validation, "plan/" + p.block_id + " does not match block " + b->block.id);
            const xlf::TensorShape o = g.shape_of(b->block.consumer_stage.at(0));
            const xlf::TileGeometry& geo = p.geometry;
            if (geo.tile_h < 1 || geo.tile_w < 1 || geo.grid_h != (o.height + geo.tile_h - 1) / geo.tile_h ||
                geo.grid_w != (o.width + geo.tile_w - 1) / geo.tile_w)
                xlf::fail(xlf::ErrorKind::validation, "plan/" + p.block_id + ": geometry does not cover the " + std::to_string(o.height) + "x" +
                                                          std::to_string(o.width) + " output");
            for (const std::string& m : b->block.members) k.tiles[m] = {geo.tile_h, geo.tile_w};
            plan_th = geo.tile_h, plan_tw = geo.tile_w;
            tile_src = "plan (" + p.device_name + ")";
        }
        const xlf::Graph sub = block_graph(g, b->block, b->ins, b->outs);
        const std::vector<float> w = block_weights(g, b->block, weights, n_weights);
        b->e = std::make_unique<xlf::Engine>(sub, gpu, xlf::Partition(part), xlf::Precision(prec), w.data(), w.size(), max_batch, k);
        const xlf::DevicePlan& dp = b->e->plan();
        const bool one = dp.steps.size() == 1 && dp.steps[0].kind == xlf::StepSpec::FUSED &&
                         dp.steps[0].layers.size() == b->block.members.size();
        if (!one)
            xlf::fail(xlf::ErrorKind::infeasible, "block " + b->block.id + " does not fit one B200 kernel at this precision" +
                                                      (plan_text && *plan_text ? " and the plan's tile geometry" : "") +
                                                      " (shared memory / TMEM); an engine runs its layers unfused");
        // description + the reference's counter semantics that do not depend on
        // the schedule: stored elements and 16-byte store transactions
        // (cost_model.cpp:15-48, at `device`'s transaction size), ideal MACs
        std::int64_t stored = 0, tx = 0;
        for (const auto& [name, elems] : xlf::stored_tensors(g, b->block)) stored += elems, tx += xlf::transactions_for(elems, dev);
        std::ostringstream os;
        auto shapes = [&](const std::vector<std::string>& v) {
            std::string s = "[";
            for (size_t i = 0; i < v.size(); ++i) {
                const xlf::TensorShape t = g.shape_of(v[i]);
                s += (i ? "," : "") + std::string("{\"name\":") + jstr(v[i]) + ",\"shape\":[" + std::to_string(t.channels) + "," +
                     std::to_string(t.height) + "," + std::to_string(t.width) + "]}";
            }
            return s + "]";
        };
        const xlf::StepSpec& s = dp.steps[0];
        os << "{\"block\":" << jstr(b->block.id) << ",\"mode\":" << jstr(xlf::to_string(b->block.mode)) << ",\"inputs\":" << shapes(b->ins)
           << ",\"outputs\":" << shapes(b->outs) << ",\"element_bytes\":" << b->e->element_bytes() << ",\"tile\":[" << s.tile_h << ","
           << s.tile_w << "],\"plan_tile\":[" << plan_th << "," << plan_tw << "],\"tile_source\":" << jstr(tile_src) << ",\"device\":" << jstr(dev.name)
           << ",\"per_image\":{\"stored_elements\":" << stored << ",\"global_store_tx\":" << tx << ",\"macs\":" << std::int64_t(s.macs)
           << "},\"engine\":" << b->e->describe_json() << "}";
        b->desc = os.str();
        *out = b.release();
    });
}

extern "C" xlf_status xlf_block_json(const xlf_block* b, char* buf, size_t cap, size_t* need) {
    return guard([&] {
        need_ptr(b, "block");
        put(b->desc, buf, cap, need);
    });
}

extern "C" xlf_status xlf_block_run(xlf_block* b, const xlf_tensor_ref* ins, int n_ins, const xlf_tensor_ref* outs, int n_outs, int batch,
                                    void* stream) {
    return guard([&] {
        need_ptr(b, "block"), need_ptr(ins, "ins"), need_ptr(outs, "outs");
        if (n_ins != int(b->ins.size()) || n_outs != int(b->outs.size()))
            throw ArgError("block " + b->block.id + " takes " + std::to_string(b->ins.size()) + " input(s) and " + std::to_string(b->outs.size()) +
                           " output(s)");
        const cudaStream_t st = static_cast<cudaStream_t>(stream);
        std::lock_guard<std::mutex> lock(b->mu);
        xlf::cuda_check(cudaSetDevice(b->e->device()), "cudaSetDevice");
        if (!b->done) xlf::cuda_check(cudaEventCreateWithFlags(&b->done, cudaEventDisableTiming), "cudaEventCreate");
        if (b->ran && b->last != st) xlf::cuda_check(cudaStreamWaitEvent(st, b->done, 0), "cudaStreamWaitEvent");
        std::vector<xlf::Engine::External> ext;
        for (int i = 0; i < n_ins + n_outs; ++i) {
            const xlf_tensor_ref& r = i < n_ins ? ins[i] : outs[i - n_ins];
            const std::string& name = i < n_ins ? b->ins[size_t(i)] : b->outs[size_t(i - n_ins)];
            need_ptr(r.data, "tensor data");
            if (r.layout == XLF_LAYOUT_NHWC) ext.push_back({name, r.data, r.cstride, r.coff});
            else if (r.layout != XLF_LAYOUT_NCHW_F32) throw ArgError("unknown layout for '" + name + "'");
        }
        for (int i = 0; i < n_ins; ++i)
            if (ins[i].layout == XLF_LAYOUT_NCHW_F32) b->e->set_input_nchw(b->ins[size_t(i)], static_cast<const float*>(ins[i].data), batch, st);
        b->e->forward_external(ext, batch, st);
        for (int i = 0; i < n_outs; ++i)
            if (outs[i].layout == XLF_LAYOUT_NCHW_F32) b->e->read_output_nchw(b->outs[size_t(i)], static_cast<float*>(outs[i].data), batch, st);
        xlf::cuda_check(cudaEventRecord(b->done, st), "cudaEventRecord");
        b->last = st, b->ran = true;
    });
}

extern "C" void xlf_block_destroy(xlf_block* b) { delete b; }

// ---------------------------------------------------------------- several GPUs
struct xlf_multi {
    std::unique_ptr<xlf::MultiEngine> m;
};

extern "C" xlf_status xlf_shard(int batch, int n, int slot, int* first, int* count) {
    return guard([&] {
        need_ptr(first, "first"), need_ptr(count, "count");
        xlf::shard_range(batch, n, slot, first, count);
    });
}

extern "C" xlf_status xlf_multi_create(const xlf_graph* h, const int* devices, int n, int part, int prec, const float* weights, size_t nw,
                                       int max_batch_per_device, const char* options, xlf_multi** out) {
    return guard([&] {
        need_ptr(h, "graph"), need_ptr(devices, "devices"), need_ptr(weights, "weights"), need_ptr(out, "out");
        if (part < 0 || part > 2) throw ArgError("unknown partition");
        if (prec < 0 || prec > 3) throw ArgError("unknown precision");
        if (n < 1 || n > 64) throw ArgError("n_devices must be 1..64");
        const xlf::Knobs k = xlf::Knobs::parse(options ? options : "");
        auto m = std::make_unique<xlf_multi>();
        m->m = std::make_unique<xlf::MultiEngine>(h->g, std::vector<int>(devices, devices + n), xlf::Partition(part), xlf::Precision(prec),
                                                  weights, nw, max_batch_per_device, k);
        *out = m.release();
    });
}

extern "C" void xlf_multi_destroy(xlf_multi* m) { delete m; }

extern "C" xlf_status xlf_multi_autotune(xlf_multi* m, int batch_per_device, int reps, int topk) {
    return guard([&] {
        need_ptr(m, "multi");
        m->m->autotune(batch_per_device, reps, topk);
    });
}

extern "C" xlf_status xlf_multi_run_host(xlf_multi* m, const float* h_in, int batch, const char* name, float* h_out, double* ms) {
    return guard([&] {
        need_ptr(m, "multi"), need_ptr(h_in, "input"), need_ptr(name, "name"), need_ptr(h_out, "output");
        const std::vector<double> t = m->m->run_host(h_in, batch, name, h_out);
        if (ms) std::copy(t.begin(), t.end(), ms);
    });
}

extern "C" xlf_status xlf_multi_time_seeded(xlf_multi* m, uint64_t seed, int batch_per_device, int steps, int warmup, double* ms) {
    return guard([&] {
        need_ptr(m, "multi"), need_ptr(ms, "ms");
        const std::vector<double> t = m->m->time_seeded(seed, batch_per_device, steps, warmup);
        std::copy(t.begin(), t.end(), ms);
    });
}
