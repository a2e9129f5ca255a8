// Driver of the reference-side binding (fused_exec_b200.cpp): every fused
// block of a reference graph, planned by the reference's own tune() on its
// own device model, runs through the reference's CPU run_fused_block and
// through run_fused_block_b200 (B200, via the C ABI) with the same plan,
// inputs and weights; the stored tensors must be bit-identical (fp32_exact).
// A plan for another block must be refused with ErrorKind::validation, as the
// reference does (fused_exec.cpp:33-38).  Test infrastructure: links the
// unmodified reference (oracle/_ref/libxlfuse_ref.so).
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>

#include "xlfuse/cost_model.hpp"
#include "xlfuse/error.hpp"
#include "xlfuse/fused_exec.hpp"
#include "xlfuse/fusion.hpp"
#include "xlfuse/reference.hpp"
#include "xlfuse_b200.h"

namespace xlfuse {
CounterReport run_fused_block_b200(const Graph&, const FusionBlock&, const TilingPlan&, const DeviceSpec&, std::map<std::string, Tensor>&,
                                   const WeightSet&, xlf_precision);
}

int main(int argc, char** argv) {
    using namespace xlfuse;
    if (argc < 2) return std::fprintf(stderr, "usage: %s [--device file] graph-file...\n", argv[0]), 2;
    int bad = 0, blocks = 0;
    std::vector<DeviceSpec> devices{titan_xp_spec()};
    int a0 = 1;
    if (std::strcmp(argv[1], "--device") == 0 && argc > 3) devices.push_back(load_device(argv[2])), a0 = 3;  // the reference's parse_device
    for (int a = a0; a < argc; ++a) {
        std::ifstream f(argv[a]);
        std::stringstream ss;
        ss << f.rdbuf();
        const Graph g = fold_elementwise(infer_shapes(parse_graph(ss.str())));
        const WeightSet w = seeded_weights(g, 42);
        const auto all = run_reference(g, seeded_inputs(g, 42), w);
        std::vector<FusionBlock> fused;
        for (const FusionBlock& b : detect_fusion_blocks(g))
            if (b.fused()) fused.push_back(b);
        for (const DeviceSpec& dev : devices)
        for (const FusionBlock& b : fused) {
            const TilingPlan plan = tune(g, b, dev).best;
            std::map<std::string, Tensor> cpu = all, gpu = all;
            for (const auto& [n, e] : stored_tensors(g, b)) cpu.erase(n), gpu.erase(n);
            run_fused_block(g, b, plan, dev, cpu, w);
            const CounterReport r = run_fused_block_b200(g, b, plan, dev, gpu, w, XLF_FP32_EXACT);
            bool same = r.global_store_tx == global_store_tx_fused(g, b, dev);
            for (const auto& [n, e] : stored_tensors(g, b))
                same &= gpu.count(n) && gpu.at(n).data.size() == cpu.at(n).data.size() &&
                        std::memcmp(gpu.at(n).data.data(), cpu.at(n).data.data(), cpu.at(n).data.size() * 4) == 0;
            std::printf("%s %s: tile %dx%d (reference tune on %s): %s\n", g.name.c_str(), b.id.c_str(), plan.geometry.tile_h,
                        plan.geometry.tile_w, dev.name.c_str(), same ? "bit-identical to run_fused_block" : "MISMATCH");
            bad += !same, ++blocks;
            if (fused.size() > 1) {  // another block's plan: refused like the reference
                const FusionBlock& other = fused[&b == &fused[0] ? 1 : 0];
                try {
                    run_fused_block_b200(g, b, tune(g, other, dev).best, dev, gpu, w, XLF_FP32_EXACT);
                    std::printf("  foreign plan accepted: MISMATCH\n"), ++bad;
                } catch (const Error& e) {
                    const bool v = e.kind() == ErrorKind::validation;
                    std::printf("  foreign plan refused (%s)\n", v ? "validation" : "wrong kind"), bad += !v;
                }
            }
        }
    }
    std::printf("%d block(s), %d failure(s)\n", blocks, bad);
    return bad ? 1 : 0;
}
