#include "tiling.hpp"

#include <algorithm>
#include <set>

#include "common.hpp"
#include "textdoc.hpp"

namespace xlf {

// ------------------------------------------------------------------ devices

void DeviceSpec::check() const {
    auto pos = [](double v, const char* what) {
        if (!(v > 0)) fail(ErrorKind::validation, std::string("device spec: ") + what + " must be positive");
    };
    pos(sm_count, "sm_count"), pos(peak_flops, "peak_flops"), pos(global_bw, "global_bw"), pos(shared_bw, "shared_bw");
    pos(double(shared_per_sm), "shared_per_sm"), pos(double(shared_per_block_max), "shared_per_block_max");
    pos(double(constant_capacity), "constant_capacity"), pos(double(readonly_cache), "readonly_cache");
    pos(banks, "banks"), pos(bank_word, "bank_word"), pos(warp_size, "warp_size");
    pos(max_blocks_per_sm, "max_blocks_per_sm"), pos(max_threads_per_block, "max_threads_per_block");
    if (transaction_bytes < 4 || transaction_bytes % 4)
        fail(ErrorKind::validation, "device spec: transaction_bytes must be a positive multiple of 4");
}

DeviceSpec titan_xp_spec() {  // device.cpp:92-100 figures (paper's TITAN Xp)
    DeviceSpec d;
    d.name = "titan_xp", d.sm_count = 30, d.peak_flops = 12.15e12, d.global_bw = 547.7e9, d.shared_bw = 6074e9;
    return d;
}

DeviceSpec tesla_p4_spec() {
    DeviceSpec d;
    d.name = "tesla_p4", d.sm_count = 20, d.peak_flops = 5.5e12, d.global_bw = 192e9, d.shared_bw = 2721e9;
    return d;
}

// B200: 148 SMs, 228 KB shared per SM (227 KB per block), fp32 SIMT peak
// 148 SM x 128 FMA x 2 x 1.965 GHz, HBM from MEASURED_PEAKS.json, TMEM
// 512 x 128 x 32-bit per SM.  Constant-memory placement is not used by the
// B200 kernels (weights live in global memory behind L1/L2 or TMA), but the
// 64 KB figure keeps the reference's placement rule meaningful.
DeviceSpec b200_spec() {
    DeviceSpec d;
    d.name = "b200";
    d.sm_count = 148;
    d.peak_flops = 148.0 * 128 * 2 * 1.965e9;
    d.global_bw = 6536.4e9;
    d.shared_bw = 148.0 * 128 * 1.965e9;
    d.shared_per_sm = 228 * 1024;
    d.shared_per_block_max = 227 * 1024;
    d.constant_capacity = 64 * 1024;
    d.readonly_cache = 128 * 1024;
    d.max_blocks_per_sm = 32;
    d.max_threads_per_block = 1024;
    d.tmem_columns = 512;
    d.tmem_lanes = 128;
    return d;
}

DeviceSpec parse_device(const std::string& text) {
    td::Node doc = td::parse(text);
    DeviceSpec d;
    d.name = doc.need("name").str();
    d.sm_count = int(doc.need("sm_count").integer());
    d.peak_flops = doc.need("peak_flops").real();
    d.global_bw = doc.need("global_bw").real();
    d.shared_bw = doc.need("shared_bw").real();
    d.shared_per_sm = doc.int_or("shared_per_sm", d.shared_per_sm);
    d.shared_per_block_max = doc.int_or("shared_per_block_max", d.shared_per_block_max);
    d.constant_capacity = doc.int_or("constant_capacity", d.constant_capacity);
    d.readonly_cache = doc.int_or("readonly_cache", d.readonly_cache);
    d.banks = int(doc.int_or("banks", d.banks));
    d.bank_word = int(doc.int_or("bank_word", d.bank_word));
    d.warp_size = int(doc.int_or("warp_size", d.warp_size));
    d.transaction_bytes = int(doc.int_or("transaction_bytes", d.transaction_bytes));
    d.max_blocks_per_sm = int(doc.int_or("max_blocks_per_sm", d.max_blocks_per_sm));
    d.max_threads_per_block = int(doc.int_or("max_threads_per_block", d.max_threads_per_block));
    d.tmem_columns = int(doc.int_or("tmem_columns", 0));
    d.tmem_lanes = int(doc.int_or("tmem_lanes", 0));
    d.check();
    return d;
}

std::string serialize_device(const DeviceSpec& d) {
    td::Node doc;
    auto I = [&](const char* k, long long v) { doc.children.push_back(td::leaf(k, v)); };
    doc.children.push_back(td::leaf("name", d.name));
    I("sm_count", d.sm_count);
    doc.children.push_back(td::leaf("peak_flops", d.peak_flops));
    doc.children.push_back(td::leaf("global_bw", d.global_bw));
    doc.children.push_back(td::leaf("shared_bw", d.shared_bw));
    I("shared_per_sm", d.shared_per_sm), I("shared_per_block_max", d.shared_per_block_max);
    I("constant_capacity", d.constant_capacity), I("readonly_cache", d.readonly_cache);
    I("banks", d.banks), I("bank_word", d.bank_word), I("warp_size", d.warp_size);
    I("transaction_bytes", d.transaction_bytes), I("max_blocks_per_sm", d.max_blocks_per_sm);
    I("max_threads_per_block", d.max_threads_per_block);
    if (d.tmem_columns) I("tmem_columns", d.tmem_columns), I("tmem_lanes", d.tmem_lanes);
    return td::serialize(doc);
}

// ------------------------------------------------------------------ halo

// Receptive-field recursion from the output tile back to the chain input
// (tiling.cpp:24-56 semantics): extent_k = (extent_{k+1} - 1) * stride_k + kernel_k.
HaloExtent halo_extent(int tile_h, int tile_w, const std::vector<ConvParams>& chain) {
    if (chain.empty()) fail(ErrorKind::internal, "halo_extent: empty chain");
    if (tile_h < 1 || tile_w < 1) fail(ErrorKind::internal, "halo_extent: tile must be >= 1x1");
    HaloExtent h;
    h.stages.resize(chain.size());
    int eh = tile_h, ew = tile_w, sh = 1, sw = 1, oh = 0, ow = 0;
    for (size_t r = chain.size(); r-- > 0;) {
        const ConvParams& c = chain[r];
        HaloStage& s = h.stages[r];
        s.kernel_h = c.kernel_h, s.kernel_w = c.kernel_w, s.stride = c.stride, s.pad = c.pad;
        s.channels_out = c.out_channels;
        s.macs_per_cell = c.in_channels > 0 ? c.macs_per_output() : 0;
        eh = (eh - 1) * c.stride + c.kernel_h;
        ew = (ew - 1) * c.stride + c.kernel_w;
        oh = oh * c.stride - c.pad;
        ow = ow * c.stride - c.pad;
        sh *= c.stride, sw *= c.stride;
        s.extent_h = eh, s.extent_w = ew, s.scale_h = sh, s.scale_w = sw, s.offset_h = oh, s.offset_w = ow;
    }
    return h;
}

// Marks every cell each tile stages, per chain stage, and compares against
// the unique cell count (tiling.cpp:83-151 semantics).
RedundancyReport redundancy_count(const TileGeometry& geo, const HaloExtent& halo, const TensorShape& input) {
    RedundancyReport rep;
    const size_t n = halo.stages.size();
    if (!n) return rep;
    std::vector<std::pair<int, int>> plane(n + 1);  // plane[i] = input dims of stage i; plane[n] = output
    plane[0] = {input.height, input.width};
    for (size_t i = 0; i < n; ++i) {
        const HaloStage& s = halo.stages[i];
        plane[i + 1] = {conv_out_dim(plane[i].first, s.kernel_h, s.pad, s.stride),
                        conv_out_dim(plane[i].second, s.kernel_w, s.pad, s.stride)};
    }
    const int oh = plane[n].first, ow = plane[n].second;
    if (geo.tile_h * geo.grid_h < oh || geo.tile_w * geo.grid_w < ow)
        fail(ErrorKind::internal, "redundancy_count: geometry does not cover the output");
    std::vector<std::vector<unsigned char>> mark(n);
    std::vector<std::int64_t> staged(n, 0);
    for (size_t i = 0; i < n; ++i) mark[i].assign(size_t(plane[i].first) * plane[i].second, 0);
    for (int ty = 0; ty < geo.grid_h; ++ty)
        for (int tx = 0; tx < geo.grid_w; ++tx) {
            int y = ty * geo.tile_h, x = tx * geo.tile_w;
            int h = std::min(geo.tile_h, oh - y), w = std::min(geo.tile_w, ow - x);
            if (h <= 0 || w <= 0) continue;
            for (size_t r = n; r-- > 0;) {
                const HaloStage& s = halo.stages[r];
                y = y * s.stride - s.pad, x = x * s.stride - s.pad;
                h = (h - 1) * s.stride + s.kernel_h, w = (w - 1) * s.stride + s.kernel_w;
                const int y0 = std::max(0, y), y1 = std::min(plane[r].first, y + h);
                const int x0 = std::max(0, x), x1 = std::min(plane[r].second, x + w);
                if (y1 <= y0 || x1 <= x0) continue;
                staged[r] += std::int64_t(y1 - y0) * (x1 - x0);
                for (int yy = y0; yy < y1; ++yy)
                    std::fill_n(mark[r].begin() + size_t(yy) * plane[r].second + x0, x1 - x0, 1);
            }
        }
    auto uniq = [&](size_t i) { return std::int64_t(std::count(mark[i].begin(), mark[i].end(), 1)); };
    rep.staged_input_elements = staged[0] * input.channels;
    rep.unique_input_elements = uniq(0) * input.channels;
    rep.replicated_elements = rep.staged_input_elements - rep.unique_input_elements;
    for (size_t i = 1; i < n; ++i) {
        const HaloStage& p = halo.stages[i - 1];
        const std::int64_t u = uniq(i), extra = staged[i] - u;
        rep.intermediate_staged_cells += staged[i] * p.channels_out;
        rep.intermediate_unique_cells += u * p.channels_out;
        rep.recomputed_cells += extra * p.channels_out;
        rep.redundant_macs += extra * p.channels_out * p.macs_per_cell;
    }
    return rep;
}

// ------------------------------------------------------------------ search space

namespace {
bool composite(int n) {
    if (n < 4) return false;
    for (int d = 2; d * d <= n; ++d)
        if (n % d == 0) return true;
    return false;
}
// (tile, grid) pairs from the factors of n (or of the next composite above a
// prime n, leaving a partial last tile); tile 1 and tile == n excluded.
std::vector<std::pair<int, int>> factor_pairs(int n) {
    std::vector<std::pair<int, int>> r;
    if (n <= 1) return r;
    int basis = n;
    while (!composite(basis)) ++basis;
    for (int t = 2; t < basis; ++t) {
        if (basis % t || t == n) continue;
        const int g = basis / t;
        if (g >= 2 && t * (g - 1) < n) r.emplace_back(t, g);
    }
    return r;
}
}  // namespace

std::vector<TileGeometry> enumerate_tilings(int out_h, int out_w) {
    std::vector<TileGeometry> out;
    auto make = [](int th, int gh, int tw, int gw) {
        TileGeometry g;
        g.tile_h = th, g.grid_h = gh, g.tile_w = tw, g.grid_w = gw;
        return g;
    };
    if (out_h == out_w) {
        for (auto [t, g] : factor_pairs(out_h)) out.push_back(make(t, g, t, g));
        return out;
    }
    auto hs = factor_pairs(out_h), ws = factor_pairs(out_w);
    if (hs.empty()) hs.emplace_back(out_h, 1);
    if (ws.empty()) ws.emplace_back(out_w, 1);
    for (auto [th, gh] : hs)
        for (auto [tw, gw] : ws)
            if (gh != 1 || gw != 1) out.push_back(make(th, gh, tw, gw));
    return out;
}

TileGeometry full_tile_geometry(int out_h, int out_w) {
    TileGeometry g;
    g.tile_h = out_h, g.tile_w = out_w;
    return g;
}

// ------------------------------------------------------------------ plan

namespace {
std::string staging_key(const Layer& p) {
    const ConvParams& c = *p.conv;
    return p.inputs[0] + "/" + std::to_string(c.kernel_h) + "x" + std::to_string(c.kernel_w) + "/" +
           std::to_string(c.stride) + "/" + std::to_string(c.pad);
}
}  // namespace

TilingPlan plan_tiling(const Graph& g, const FusionBlock& b, const TileGeometry& geo, const DeviceSpec& dev,
                       const PlanOptions& opts) {
    if (!b.fused()) fail(ErrorKind::internal, "plan_tiling: unfused blocks have no tiling plan");
    std::vector<const Layer*> prod, cons;
    for (const std::string& n : b.producer_stage) {
        const Layer* l = g.find_layer(n);
        if (!l) fail(ErrorKind::internal, "plan_tiling: unknown layer '" + n + "'");
        prod.push_back(l);
    }
    for (const std::string& n : b.consumer_stage) {
        const Layer* l = g.find_layer(n);
        if (!l) fail(ErrorKind::internal, "plan_tiling: unknown layer '" + n + "'");
        cons.push_back(l);
    }
    const TensorShape out = *cons[0]->out_shape;
    for (const Layer* c : cons)
        if (c->out_shape->height != out.height || c->out_shape->width != out.width)
            fail(ErrorKind::infeasible, "block " + b.id + ": consumer output extents differ");

    // Staged region relative to the tile: lead rows before, trail rows after
    // (in consumer input coordinates), consumer stride S.
    int S = 1, lead_h = 0, lead_w = 0, trail_h = 1, trail_w = 1;
    if (b.mode != FusionMode::merge) {
        S = cons[0]->conv->stride;
        for (const Layer* c : cons) {
            const ConvParams& cc = *c->conv;
            if (cc.stride != S) fail(ErrorKind::infeasible, "block " + b.id + ": consumer strides differ");
            lead_h = std::max(lead_h, cc.pad), lead_w = std::max(lead_w, cc.pad);
            trail_h = std::max(trail_h, cc.kernel_h - cc.pad), trail_w = std::max(trail_w, cc.kernel_w - cc.pad);
        }
    }
    if (b.stores_intermediate) trail_h = std::max(trail_h, S), trail_w = std::max(trail_w, S);
    if (trail_h <= lead_h - geo.tile_h || trail_w <= lead_w - geo.tile_w)
        fail(ErrorKind::infeasible, "block " + b.id + ": padding exceeds kernel extent");
    if (geo.tile_h < 1 || geo.tile_w < 1 || geo.grid_h < 1 || geo.grid_w < 1)
        fail(ErrorKind::validation, "tile geometry fields must be >= 1");
    if (geo.tile_h * geo.grid_h < out.height || geo.tile_w * geo.grid_w < out.width)
        fail(ErrorKind::validation, "tile geometry does not cover the output");
    if (geo.tile_h * (geo.grid_h - 1) >= out.height || geo.tile_w * (geo.grid_w - 1) >= out.width)
        fail(ErrorKind::validation, "tile geometry has an empty trailing tile");

    TilingPlan p;
    p.graph_name = g.name, p.block_id = b.id, p.mode = b.mode;
    p.producers = b.producer_stage, p.consumers = b.consumer_stage;
    p.stores_intermediate = b.stores_intermediate;
    p.geometry = geo;
    p.device_name = dev.name;
    const int ext_h = (geo.tile_h - 1) * S + lead_h + trail_h;
    const int ext_w = (geo.tile_w - 1) * S + lead_w + trail_w;
    const int border = std::max(lead_h, lead_w);
    for (size_t i = 0; i < prod.size(); ++i) {
        const ConvParams& c = *prod[i]->conv;
        SharedLayout buf;
        buf.name = "s" + std::to_string(i);
        buf.stage = prod[i]->name;
        buf.channels = prod[i]->out_shape->channels;
        buf.border = border;
        buf.logical_h = ext_h - 2 * border, buf.logical_w = ext_w - 2 * border;
        buf.pad_cols = 1, buf.pad_rows = opts.row_bank_padding ? 1 : 0;
        buf.stride = S;
        p.buffers.push_back(buf);
        HaloStage hs;
        hs.layer = prod[i]->name;
        hs.kernel_h = c.kernel_h, hs.kernel_w = c.kernel_w, hs.stride = c.stride, hs.pad = c.pad;
        hs.channels_out = c.out_channels, hs.macs_per_cell = c.macs_per_output();
        hs.extent_h = (ext_h - 1) * c.stride + c.kernel_h, hs.extent_w = (ext_w - 1) * c.stride + c.kernel_w;
        hs.scale_h = hs.scale_w = S * c.stride;
        hs.offset_h = hs.offset_w = -border * c.stride - c.pad;
        p.halo.stages.push_back(hs);
    }
    for (const Layer* c : cons) {
        HaloStage hs;
        hs.layer = c->name;
        if (b.mode == FusionMode::merge) {
            hs.channels_out = c->out_shape->channels;
            hs.extent_h = geo.tile_h, hs.extent_w = geo.tile_w;
        } else {
            const ConvParams& cc = *c->conv;
            hs.kernel_h = cc.kernel_h, hs.kernel_w = cc.kernel_w, hs.stride = cc.stride, hs.pad = cc.pad;
            hs.channels_out = cc.out_channels, hs.macs_per_cell = cc.macs_per_output();
            hs.extent_h = (geo.tile_h - 1) * cc.stride + cc.kernel_h;
            hs.extent_w = (geo.tile_w - 1) * cc.stride + cc.kernel_w;
        }
        hs.scale_h = hs.scale_w = hs.stride;
        hs.offset_h = hs.offset_w = -hs.pad;
        p.halo.stages.push_back(hs);
    }
    p.block_dim_x = std::min(geo.tile_w, dev.max_threads_per_block);
    p.block_dim_y = std::min(geo.tile_h, std::max(1, dev.max_threads_per_block / p.block_dim_x));
    p.geometry.loop_w = (geo.tile_w + p.block_dim_x - 1) / p.block_dim_x;
    p.geometry.loop_h = (geo.tile_h + p.block_dim_y - 1) / p.block_dim_y;

    std::int64_t wbytes = 0;
    for (const Layer* l : prod) wbytes += (l->conv->weight_count() + l->conv->bias_count()) * 4;
    for (const Layer* l : cons)
        if (l->kind == LayerKind::conv) wbytes += (l->conv->weight_count() + l->conv->bias_count()) * 4;
    p.weights = wbytes <= dev.constant_capacity ? WeightPlacement::constant_memory : WeightPlacement::readonly_cached_global;

    // Redundancy: each producer chained with a pseudo-consumer that reads the
    // staged region (kernel lead+trail, pad lead, stride S).
    std::set<std::string> keys;
    for (const Layer* l : prod) {
        ConvParams pseudo;
        pseudo.kernel_h = lead_h + trail_h, pseudo.kernel_w = lead_w + trail_w;
        pseudo.pad = lead_h, pseudo.stride = S, pseudo.out_channels = l->out_shape->channels;
        HaloExtent h = halo_extent(geo.tile_h, geo.tile_w, {*l->conv, pseudo});
        h.stages[0].channels_out = l->conv->out_channels;
        h.stages[0].macs_per_cell = l->conv->macs_per_output();
        const RedundancyReport rr = redundancy_count(geo, h, g.shape_of(l->inputs[0]));
        if (!keys.insert(staging_key(*l)).second) p.shared_input_staging = true;
        else p.replicated_elements += rr.replicated_elements;
        p.redundant_macs += rr.redundant_macs;
    }
    for (const SharedLayout& s : p.buffers) p.shared_bytes += s.physical_elements() * 4;
    if (p.shared_bytes > dev.shared_per_block_max)
        fail(ErrorKind::infeasible, "block " + b.id + ": staging buffers need " + std::to_string(p.shared_bytes) +
                                        " B of shared memory, per-block limit is " +
                                        std::to_string(dev.shared_per_block_max) + " B");
    return p;
}

OccupancyReport check_resources(const TilingPlan& plan, const DeviceSpec& dev) {
    OccupancyReport r;
    const std::int64_t bytes = std::max<std::int64_t>(plan.shared_bytes, 1);
    r.blocks_per_sm = int(std::min<std::int64_t>(dev.shared_per_sm / bytes, dev.max_blocks_per_sm));
    r.shared_fraction = double(plan.shared_bytes) / double(dev.shared_per_sm);
    if (r.blocks_per_sm < 1) r.warnings.push_back("staging buffers exceed per-SM shared capacity");
    if (plan.shared_bytes * 3 > dev.shared_per_sm) r.warnings.push_back("plan uses more than 1/3 of per-SM shared memory");
    if (r.blocks_per_sm == 1) r.warnings.push_back("occupancy is 1 block/SM; memory latency cannot be hidden");
    return r;
}

// ------------------------------------------------------------------ plan files

std::string serialize_plan(const TilingPlan& p) {
    td::Node doc, sec = td::branch("plan");
    auto add = [&](td::Node n) { sec.children.push_back(std::move(n)); };
    add(td::leaf("graph", p.graph_name));
    add(td::leaf("block", p.block_id));
    add(td::leaf("mode", std::string(to_string(p.mode))));
    add(td::leaf_list("producers", p.producers));
    add(td::leaf_list("consumers", p.consumers));
    add(td::leaf("stores_intermediate", std::string(p.stores_intermediate ? "true" : "false")));
    add(td::leaf("shared_input_staging", std::string(p.shared_input_staging ? "true" : "false")));
    td::Node geo = td::branch("geometry");
    geo.children.push_back(td::leaf_ints("tile", {p.geometry.tile_h, p.geometry.tile_w}));
    geo.children.push_back(td::leaf_ints("grid", {p.geometry.grid_h, p.geometry.grid_w}));
    geo.children.push_back(td::leaf_ints("loops", {p.geometry.loop_h, p.geometry.loop_w}));
    add(geo);
    add(td::leaf_ints("threads", {p.block_dim_x, p.block_dim_y}));
    td::Node halo = td::branch("halo");
    for (const HaloStage& s : p.halo.stages) {
        td::Node n = td::branch("stage");
        n.children.push_back(td::leaf("layer", s.layer));
        n.children.push_back(td::leaf_ints("kernel", {s.kernel_h, s.kernel_w}));
        n.children.push_back(td::leaf("stride", (long long)s.stride));
        n.children.push_back(td::leaf("pad", (long long)s.pad));
        n.children.push_back(td::leaf("channels_out", (long long)s.channels_out));
        n.children.push_back(td::leaf("macs_per_cell", (long long)s.macs_per_cell));
        n.children.push_back(td::leaf_ints("extent", {s.extent_h, s.extent_w}));
        n.children.push_back(td::leaf_ints("scale", {s.scale_h, s.scale_w}));
        n.children.push_back(td::leaf_ints("offset", {s.offset_h, s.offset_w}));
        halo.children.push_back(std::move(n));
    }
    add(halo);
    for (const SharedLayout& b : p.buffers) {
        td::Node n = td::branch("buffer");
        n.children.push_back(td::leaf("name", b.name));
        n.children.push_back(td::leaf("stage", b.stage));
        n.children.push_back(td::leaf("channels", (long long)b.channels));
        n.children.push_back(td::leaf_ints("logical", {b.logical_h, b.logical_w}));
        n.children.push_back(td::leaf("border", (long long)b.border));
        n.children.push_back(td::leaf_ints("bank_pad", {b.pad_rows, b.pad_cols}));
        n.children.push_back(td::leaf("stride", (long long)b.stride));
        n.children.push_back(td::leaf("physical_elements", (long long)b.physical_elements()));
        add(n);
    }
    add(td::leaf("weights", std::string(p.weights == WeightPlacement::constant_memory ? "constant_memory"
                                                                                      : "readonly_cached_global")));
    add(td::leaf("replicated_elements", (long long)p.replicated_elements));
    add(td::leaf("redundant_macs", (long long)p.redundant_macs));
    add(td::leaf("shared_bytes", (long long)p.shared_bytes));
    add(td::leaf("device", p.device_name));
    doc.children.push_back(std::move(sec));
    return td::serialize(doc);
}

TilingPlan parse_plan(const std::string& text) {
    const td::Node doc = td::parse(text);
    const td::Node& s = doc.need("plan");
    TilingPlan p;
    p.graph_name = s.need("graph").str();
    p.block_id = s.need("block").str();
    const std::string mode = s.need("mode").str();
    if (mode == "straight") p.mode = FusionMode::straight;
    else if (mode == "split") p.mode = FusionMode::split;
    else if (mode == "merge") p.mode = FusionMode::merge;
    else if (mode == "unfused") p.mode = FusionMode::unfused;
    else fail(ErrorKind::parse, "unknown fusion mode '" + mode + "'", s.need("mode").line);
    p.producers = s.need("producers").values;
    p.consumers = s.need("consumers").values;
    p.stores_intermediate = s.bool_or("stores_intermediate", false);
    p.shared_input_staging = s.bool_or("shared_input_staging", false);
    const td::Node& geo = s.need("geometry");
    auto two = [](const td::Node& n) {
        auto v = n.ints();
        if (v.size() != 2) fail(ErrorKind::parse, "'" + n.key + "' needs two values", n.line);
        return std::pair<int, int>{int(v[0]), int(v[1])};
    };
    std::tie(p.geometry.tile_h, p.geometry.tile_w) = two(geo.need("tile"));
    std::tie(p.geometry.grid_h, p.geometry.grid_w) = two(geo.need("grid"));
    std::tie(p.geometry.loop_h, p.geometry.loop_w) = two(geo.need("loops"));
    std::tie(p.block_dim_x, p.block_dim_y) = two(s.need("threads"));
    for (const td::Node* st : s.need("halo").all("stage")) {
        HaloStage h;
        h.layer = st->str_or("layer", "");
        std::tie(h.kernel_h, h.kernel_w) = two(st->need("kernel"));
        h.stride = int(st->need("stride").integer());
        h.pad = int(st->need("pad").integer());
        h.channels_out = int(st->int_or("channels_out", 0));
        h.macs_per_cell = st->int_or("macs_per_cell", 0);
        std::tie(h.extent_h, h.extent_w) = two(st->need("extent"));
        std::tie(h.scale_h, h.scale_w) = two(st->need("scale"));
        std::tie(h.offset_h, h.offset_w) = two(st->need("offset"));
        p.halo.stages.push_back(h);
    }
    for (const td::Node* bn : s.all("buffer")) {
        SharedLayout b;
        b.name = bn->need("name").str();
        b.stage = bn->need("stage").str();
        b.channels = int(bn->need("channels").integer());
        std::tie(b.logical_h, b.logical_w) = two(bn->need("logical"));
        b.border = int(bn->need("border").integer());
        std::tie(b.pad_rows, b.pad_cols) = two(bn->need("bank_pad"));
        b.stride = int(bn->need("stride").integer());
        if (bn->need("physical_elements").integer() != b.physical_elements())
            fail(ErrorKind::parse, "buffer '" + b.name + "': physical_elements mismatch", bn->line);
        p.buffers.push_back(b);
    }
    const std::string w = s.need("weights").str();
    if (w == "constant_memory") p.weights = WeightPlacement::constant_memory;
    else if (w == "readonly_cached_global") p.weights = WeightPlacement::readonly_cached_global;
    else fail(ErrorKind::parse, "unknown weight placement '" + w + "'");
    p.replicated_elements = s.need("replicated_elements").integer();
    p.redundant_macs = s.need("redundant_macs").integer();
    p.shared_bytes = s.need("shared_bytes").integer();
    p.device_name = s.str_or("device", "");
    return p;
}

std::int64_t transactions_for(std::int64_t elements, const DeviceSpec& d) {
    return elements <= 0 ? 0 : (elements * 4 + d.transaction_bytes - 1) / d.transaction_bytes;
}
std::int64_t global_store_tx_fused(const Graph& g, const FusionBlock& b, const DeviceSpec& d) {
    std::int64_t tx = 0;
    for (const auto& [n, e] : stored_tensors(g, b)) tx += transactions_for(e, d);
    return tx;
}
std::int64_t global_store_tx_unfused(const Graph& g, const std::vector<std::string>& layers, const DeviceSpec& d) {
    std::int64_t tx = 0;
    for (const std::string& n : layers) tx += transactions_for(g.shape_of(n).elements(), d);
    return tx;
}

}  // namespace xlf
