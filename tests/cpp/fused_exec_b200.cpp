// proj/src/fused_exec_b200.cpp -- what a maintainer adds to the reference so
// that run_fused_block / simulate_graph (fused_exec.hpp:35-45) execute on a
// B200 through libxlfuse_b200.so.  Reference types in, reference types out:
// the plan's tile geometry drives the GPU kernel, tensors are the reference's
// CHW fp32 Tensors.  (INTEGRATION.md shows this file; tests/test_binding.py
// compiles it against the reference headers and runs it against the reference.)
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <string>
#include <vector>

#include "xlfuse/cost_model.hpp"
#include "xlfuse/error.hpp"
#include "xlfuse/fused_exec.hpp"
#include "xlfuse_b200.h"  // -I<repo>/include, link -lxlfuse_b200

namespace xlfuse {

namespace {

void ok(xlf_status s) {
    if (s == XLF_OK) return;
    const ErrorKind k = s == XLF_E_VALIDATION ? ErrorKind::validation
                        : s == XLF_E_INFEASIBLE ? ErrorKind::infeasible
                        : s == XLF_E_PARSE ? ErrorKind::parse
                                           : ErrorKind::internal;
    throw Error(k, std::string("libxlfuse_b200: ") + xlf_last_error());
}

void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw Error(ErrorKind::internal, std::string("cuda: ") + cudaGetErrorString(e));
}

// WeightSet -> save_weights order (tensor.cpp:64-95): per conv, filter then bias.
std::vector<float> flat_weights(const Graph& g, const WeightSet& w) {
    std::vector<float> flat;
    for (const auto& l : g.layers)
        if (l.kind == LayerKind::conv) {
            const LayerWeights& lw = w.by_layer.at(l.name);
            flat.insert(flat.end(), lw.filter.begin(), lw.filter.end());
            flat.insert(flat.end(), lw.bias.begin(), lw.bias.end());
        }
    return flat;
}

}  // namespace

// run_fused_block on the GPU: same arguments and effect on `values` as the
// reference (producer inputs read by name, stored tensors inserted); the
// returned counters are the schedule-independent ones (stores, ideal MACs).
CounterReport run_fused_block_b200(const Graph& g, const FusionBlock& block, const TilingPlan& plan, const DeviceSpec& device,
                                   std::map<std::string, Tensor>& values, const WeightSet& w, xlf_precision precision = XLF_FP32_EXACT) {
    if (!block.fused()) throw Error(ErrorKind::internal, "run_fused_block: block is not fused");
    xlf_graph* xg = nullptr;
    ok(xlf_graph_parse(serialize_graph(g).c_str(), &xg));
    const std::vector<float> flat = flat_weights(g, w);
    xlf_block* b = nullptr;
    const xlf_status st = xlf_block_prepare(xg, block.id.c_str(), XLF_PART_REFERENCE, serialize_plan(plan).c_str(),
                                            serialize_device(device).c_str(), /*gpu*/ 0, precision, flat.data(), flat.size(),
                                            /*max_batch*/ 1, nullptr, &b);
    xlf_graph_destroy(xg);
    ok(st);
    // inputs / outputs in xlf_block_prepare's order: external inputs in layer
    // order, then stored_tensors order (cost_model.cpp:21-41)
    std::vector<std::string> in_names;
    for (const auto& l : g.layers) {
        if (std::find(block.members.begin(), block.members.end(), l.name) == block.members.end()) continue;
        for (const auto& i : l.inputs)
            if (std::find(block.members.begin(), block.members.end(), i) == block.members.end() &&
                std::find(in_names.begin(), in_names.end(), i) == in_names.end())
                in_names.push_back(i);
    }
    const auto stored = stored_tensors(g, block);
    std::vector<void*> dev;
    std::vector<xlf_tensor_ref> ins, outs;
    try {
        for (const auto& n : in_names) {
            auto it = values.find(n);
            if (it == values.end()) throw Error(ErrorKind::internal, "missing input tensor '" + n + "'");
            void* p = nullptr;
            cuda(cudaMalloc(&p, it->second.data.size() * 4));
            dev.push_back(p);
            cuda(cudaMemcpy(p, it->second.data.data(), it->second.data.size() * 4, cudaMemcpyHostToDevice));
            ins.push_back({p, XLF_LAYOUT_NCHW_F32, 0, 0});
        }
        for (const auto& [n, elems] : stored) {
            void* p = nullptr;
            cuda(cudaMalloc(&p, size_t(elems) * 4));
            dev.push_back(p);
            outs.push_back({p, XLF_LAYOUT_NCHW_F32, 0, 0});
        }
        ok(xlf_block_run(b, ins.data(), int(ins.size()), outs.data(), int(outs.size()), 1, nullptr));
        for (size_t k = 0; k < stored.size(); ++k) {
            Tensor t(g.shape_of(stored[k].first));
            cuda(cudaMemcpy(t.data.data(), outs[k].data, t.data.size() * 4, cudaMemcpyDeviceToHost));
            values.insert_or_assign(stored[k].first, std::move(t));
        }
    } catch (...) {
        for (void* p : dev) cudaFree(p);
        xlf_block_destroy(b);
        throw;
    }
    for (void* p : dev) cudaFree(p);
    xlf_block_destroy(b);
    CounterReport r;
    r.global_store_tx = global_store_tx_fused(g, block, device);
    for (const auto& n : block.members) {
        const Layer* l = g.find_layer(n);
        if (l->kind == LayerKind::conv) r.macs_total += g.shape_of(n).elements() * l->conv->macs_per_output();
    }
    return r;
}

}  // namespace xlfuse
