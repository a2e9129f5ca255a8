// extern "C" boundary (include/xlfuse_b200.h).  Every entry point catches
// xlf::Error / std::exception and maps it to an xlf_status with the message
// in a thread-local buffer (the reference throws xlfuse::Error instead,
// error.hpp:21-35).
#include "../../include/xlfuse_b200.h"

#include <cstring>
#include <memory>
#include <sstream>
#include <string>

#include "common.hpp"
#include "device_plan.hpp"
#include "engine.hpp"
#include "fusion.hpp"
#include "graph.hpp"
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
