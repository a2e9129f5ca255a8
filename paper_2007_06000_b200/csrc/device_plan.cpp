#include "device_plan.hpp"
#include "tc_params.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <set>
#include <sstream>

#include "common.hpp"

namespace xlf {

const char* to_string(Partition p) {
    switch (p) {
    case Partition::reference: return "reference";
    case Partition::b200: return "b200";
    case Partition::unfused: return "unfused";
    }
    return "?";
}

namespace {

int round4(int c) { return (c + 3) & ~3; }
int smem_pitch(int c) {
    int p = round4(c) + 4;  // +4 floats: consecutive cells land on different banks
    if (p % 32 == 0) p += 4;
    return p;
}

std::map<std::string, int> topo_index(const Graph& g) {
    std::map<std::string, int> idx;
    int i = 0;
    for (const Layer* l : topo_order(g)) idx[l->name] = i++;
    return idx;
}

// Window of a layer as a reader of its input: kernel, stride, pad.
struct Window {
    int kh = 1, kw = 1, stride = 1, pad = 0;
};
Window window_of(const Layer& l) {
    Window w;
    if (l.kind == LayerKind::conv) w = {l.conv->kernel_h, l.conv->kernel_w, l.conv->stride, l.conv->pad};
    else if (l.kind == LayerKind::pool) w = {l.pool->kernel, l.pool->kernel, l.pool->stride, l.pool->pad};
    return w;
}

bool escapes(const Graph& g, const std::string& p, const std::vector<std::string>& members) {
    if (g.is_output(p)) return true;
    for (const std::string& c : g.consumers_of(p))
        if (std::find(members.begin(), members.end(), c) == members.end()) return true;
    return false;
}

FusionBlock make_block(int& next, FusionMode m, std::vector<std::string> prod, std::vector<std::string> cons, bool esc) {
    FusionBlock b;
    b.id = "b" + std::to_string(next++);
    b.mode = m;
    b.producer_stage = prod;
    b.consumer_stage = cons;
    b.members = prod;
    b.members.insert(b.members.end(), cons.begin(), cons.end());
    b.stores_intermediate = esc;
    return b;
}

}  // namespace

// B200 partition.  Pass 1 is the reference's greedy conv pass (merge > split >
// straight) except that a split keeps EVERY compatible conv reader (an
// inception-style reduce feeding three branches stays one block).  Pass 2
// adds what the reference always rejects (fusion.cpp:66-69): a pool as the
// consumer of a conv (conv -> bias -> ReLU -> pool, the paper's straight mode)
// and a pool as the producer of a conv (inception's pool-projection branch).
std::vector<FusionBlock> detect_fusion_blocks_b200(const Graph& g) {
    if (!g.shapes_inferred()) fail(ErrorKind::internal, "detect_fusion_blocks requires inferred shapes");
    std::vector<FusionBlock> blocks;
    std::set<std::string> taken;
    int next = 0;
    auto is_free = [&](const std::string& n, LayerKind k) {
        const Layer* l = g.find_layer(n);
        return l && l->kind == k && !taken.count(n);
    };
    auto push = [&](FusionBlock b) {
        for (const std::string& m : b.members) taken.insert(m);
        blocks.push_back(std::move(b));
    };
    const auto order = topo_order(g);
    for (const Layer* l : order) {
        if (taken.count(l->name) || l->kind != LayerKind::conv) continue;
        const auto readers = g.consumers_of(l->name);
        bool merged = false;
        for (const std::string& rn : readers) {
            const Layer* r = g.find_layer(rn);
            if (r->kind != LayerKind::add || taken.count(rn)) continue;
            const std::string &a = r->inputs[0], &b = r->inputs[1];
            if (a == b || !is_free(a, LayerKind::conv) || !is_free(b, LayerKind::conv)) continue;
            std::vector<std::string> mem{a, b, rn};
            push(make_block(next, FusionMode::merge, {a, b}, {rn}, escapes(g, a, mem) || escapes(g, b, mem)));
            merged = true;
            break;
        }
        if (merged) continue;
        std::vector<std::string> convs;
        for (const std::string& rn : readers)
            if (is_free(rn, LayerKind::conv)) convs.push_back(rn);
        if (convs.empty()) continue;
        // Largest set of readers sharing stride and output extent (first wins ties).
        std::vector<std::string> best;
        for (const std::string& c0 : convs) {
            const Layer* a = g.find_layer(c0);
            std::vector<std::string> grp;
            for (const std::string& c : convs) {
                const Layer* b = g.find_layer(c);
                if (b->conv->stride == a->conv->stride && b->out_shape->height == a->out_shape->height &&
                    b->out_shape->width == a->out_shape->width)
                    grp.push_back(c);
            }
            if (grp.size() > best.size()) best = grp;
        }
        std::vector<std::string> mem{l->name};
        mem.insert(mem.end(), best.begin(), best.end());
        push(make_block(next, best.size() >= 2 ? FusionMode::split : FusionMode::straight, {l->name}, best,
                        escapes(g, l->name, mem)));
    }
    for (const Layer* l : order) {
        if (taken.count(l->name) || g.is_output(l->name)) continue;
        const auto readers = g.consumers_of(l->name);
        if (readers.size() != 1) continue;
        const std::string& c = readers[0];
        if (l->kind == LayerKind::conv && is_free(c, LayerKind::pool))
            push(make_block(next, FusionMode::straight, {l->name}, {c}, false));
        else if (l->kind == LayerKind::pool && is_free(c, LayerKind::conv))
            push(make_block(next, FusionMode::straight, {l->name}, {c}, false));
    }
    for (const Layer* l : order) {
        if (taken.count(l->name)) continue;
        FusionBlock b;
        b.id = "b" + std::to_string(next++);
        b.members = {l->name};
        taken.insert(l->name);
        blocks.push_back(std::move(b));
    }
    return blocks;
}

namespace {

// Step for one block of any partition.
StepSpec step_for_block(const Graph& g, const FusionBlock& b) {
    StepSpec s;
    s.id = b.id;
    s.mode = b.mode;
    s.layers = b.members;
    if (!b.fused()) {
        const Layer& l = *g.find_layer(b.members[0]);
        switch (l.kind) {
        case LayerKind::concat: s.kind = StepSpec::CONCAT_COPY, s.tag = "concat"; break;
        case LayerKind::add: s.kind = StepSpec::ADD, s.tag = "add"; break;
        case LayerKind::relu: s.kind = StepSpec::RELU, s.tag = "relu"; break;
        default: {
            s.kind = StepSpec::FUSED;
            s.tag = to_string(l.kind);
            OpSpec op;
            op.layer = l.name, op.stage = 1, op.emit = true;
            s.ops.push_back(op);
        }
        }
        s.inputs = l.inputs;
        s.out_h = l.out_shape->height, s.out_w = l.out_shape->width;
        return s;
    }
    s.kind = StepSpec::FUSED;
    s.tag = to_string(b.mode);
    for (const std::string& p : b.producer_stage) {
        const Layer& l = *g.find_layer(p);
        OpSpec op;
        op.layer = p, op.stage = 1, op.staged = true;
        op.emit = op.own_only = escapes(g, p, b.members);
        auto it = std::find(s.inputs.begin(), s.inputs.end(), l.inputs[0]);
        if (it == s.inputs.end()) s.inputs.push_back(l.inputs[0]), op.xin = int(s.inputs.size()) - 1;
        else op.xin = int(it - s.inputs.begin());
        s.ops.push_back(op);
    }
    for (const std::string& c : b.consumer_stage) {
        const Layer& l = *g.find_layer(c);
        OpSpec op;
        op.layer = c, op.stage = 2, op.emit = true;
        for (const std::string& in : l.inputs)
            for (size_t i = 0; i < b.producer_stage.size(); ++i)
                if (b.producer_stage[i] == in) op.srcs.push_back(int(i));
        s.ops.push_back(op);
        if (g.find_layer(c)->kind == LayerKind::pool && s.tag == "straight") s.tag = "straight+pool";
    }
    const Layer& last = *g.find_layer(b.consumer_stage[0]);
    s.out_h = last.out_shape->height, s.out_w = last.out_shape->width;
    return s;
}

// Cells of slack after a staged region / buffer that a kxk (k > 1) conv
// reads: the register-blocked conv computes whole CX-cell row windows, so the
// last row's window reads up to (CX-1)*S + kw-1 <= 9 cells past the region
// (values discarded, never stored).  1x1 convs clamp instead (conv_rb).
constexpr int kSlackCells = 10;

// Per-thread instructions of one register-blocked conv unit (kernels_fp32.cu
// conv_rb): per (ic, kh) the row window loads, OCV/4 weight loads per tap and
// CX*OCV FMAs per tap; 1x1: per 4 channels CX 16-byte loads, OCV weight loads
// and 4*CX*OCV FMAs.
double rb_unit_instr(const FOp& o, int cx, int ocv) {
    if (o.kw == 1) return (o.cin / 4.0) * (cx + ocv + 4.0 * cx * ocv);
    const int win = (cx - 1) * o.stride + o.kw;
    return double(o.cin) * o.kh * (win + o.kw * ocv / 4.0 + double(o.kw) * cx * ocv);
}

// Threads of one register-blocked conv op per tile (conv_rb's lane mapping:
// channel groups padded to a multiple of min(8, groups)).
double rb_units(const FOp& o, int cx, int ocv) {
    const int QV = o.cout_pad / ocv, B = std::min(8, QV);
    return double(o.ext_h) * ((o.ext_w + cx - 1) / cx) * double((QV + B - 1) / B * B);
}

// Register-blocked variant of a conv op: the (cx, ocv) instantiation that
// minimises one CTA's serial work for the op (rounds of 256 threads x
// per-thread instructions), the larger block on ties; cx = 0 keeps the
// generic cell-quad path (grouped convs, widths / strides not instantiated).
void rb_variant(FOp& o, int threads) {
    o.cx = o.ocv = 0;
    if (o.kind != OP_CONV || o.group != 1) return;
    // instantiated shapes (conv_rb_v): 1x1 stride 1, 3x3 stride 1 / 2, k x 5 stride 1
    const bool inst = (o.kw == 1 && o.kh == 1 && o.stride == 1) || (o.kw == 3 && o.kh == 3 && o.stride <= 2) || (o.kw == 5 && o.stride == 1);
    if (!inst) return;
    static const int kVariants[4][2] = {{8, 8}, {4, 8}, {4, 4}, {2, 4}};
    // Variants that give every thread of the CTA a unit: fewest warp
    // instructions (the largest block that fits); otherwise (small tiles) the
    // one with the shortest serial chain.
    double best_full = 1e300, best_lat = 1e300;
    int full[2] = {0, 0}, lat[2] = {0, 0};
    for (const auto& v : kVariants) {
        if (o.cout_pad % v[1] || (v[0] == 8 && (o.stride != 1 || o.kw > 3))) continue;  // instantiated set (conv_rb_v)
        const double units = rb_units(o, v[0], v[1]);
        const double per = rb_unit_instr(o, v[0], v[1]);
        const double wi = std::ceil(units / 32.0) * per, l = std::ceil(units / threads) * per;
        if (units >= threads && wi < best_full * 0.999) best_full = wi, full[0] = v[0], full[1] = v[1];
        if (l < best_lat * 0.999) best_lat = l, lat[0] = v[0], lat[1] = v[1];
    }
    const int* pick = full[0] ? full : lat;
    o.cx = pick[0], o.ocv = pick[1];
}

struct OpGeom {
    int ext_h, ext_w, org_mul, org_sub, d;
};

// Lays out one fused step at tile (th, tw).  Returns shared bytes, or -1 when
// the ops cannot share one tiling (differing strides / scales).
long long layout_step(const Graph& g, const StepSpec& s, int th, int tw, FusedParams* fp) {
    const int nops = int(s.ops.size());
    if (nops > kMaxOps || s.inputs.size() > size_t(kMaxIns)) return -1;
    std::vector<OpGeom> geo(size_t(nops), OpGeom{th, tw, 1, 0, 0});
    // staged buffers: lead L, stride S, trails per producer op
    std::vector<int> bufidx(size_t(nops), -1);
    int nbufs = 0;
    for (int i = 0; i < nops; ++i) {
        const OpSpec& op = s.ops[size_t(i)];
        if (op.stage != 1 || !op.staged) continue;
        int S = -1, L = 0, Th = 1, Tw = 1;
        bool add_reader = false;
        for (const OpSpec& c : s.ops) {
            if (c.stage != 2 || std::find(c.srcs.begin(), c.srcs.end(), i) == c.srcs.end()) continue;
            const Layer& cl = *g.find_layer(c.layer);
            if (cl.kind == LayerKind::add) {
                add_reader = true;
                continue;
            }
            const Window w = window_of(cl);
            if (S >= 0 && S != w.stride) return -1;
            S = w.stride;
            L = std::max(L, w.pad);
            Th = std::max(Th, w.kh - w.pad), Tw = std::max(Tw, w.kw - w.pad);
        }
        if (add_reader) {
            if (S > 1 || L > 0) return -1;
            S = 1;
        }
        if (S < 0) S = 1;
        if (op.own_only) Th = std::max(Th, S), Tw = std::max(Tw, S);
        geo[size_t(i)] = {(th - 1) * S + L + Th, (tw - 1) * S + L + Tw, S, L, 0};
        bufidx[size_t(i)] = nbufs++;
    }
    if (nbufs > kMaxBufs) return -1;
    // stage-2 offsets into their buffers
    for (int i = 0; i < nops; ++i) {
        const OpSpec& op = s.ops[size_t(i)];
        if (op.stage != 2) continue;
        const Layer& l = *g.find_layer(op.layer);
        const int L = geo[size_t(op.srcs[0])].org_sub;
        geo[size_t(i)].d = l.kind == LayerKind::add ? 0 : L - window_of(l).pad;
    }
    // block input regions
    long long floats = 0;
    std::vector<FIn> ins(s.inputs.size());
    for (size_t xi = 0; xi < s.inputs.size(); ++xi) {
        int scale = -1, XL = 0;
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            if (op.stage != 1 || op.xin != int(xi)) continue;
            const Window w = window_of(*g.find_layer(op.layer));
            const int sc = geo[size_t(i)].org_mul * w.stride;
            if (scale >= 0 && sc != scale) return -1;
            scale = sc;
            XL = std::max(XL, geo[size_t(i)].org_sub * w.stride + w.pad);
        }
        int eh = 0, ew = 0;
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            if (op.stage != 1 || op.xin != int(xi)) continue;
            const Window w = window_of(*g.find_layer(op.layer));
            OpGeom& og = geo[size_t(i)];
            og.d = XL - (og.org_sub * w.stride + w.pad);
            eh = std::max(eh, og.d + (og.ext_h - 1) * w.stride + w.kh);
            ew = std::max(ew, og.d + (og.ext_w - 1) * w.stride + w.kw);
        }
        const TensorShape xs = g.shape_of(s.inputs[xi]);
        FIn& in = ins[xi];
        in = FIn{};
        in.c = s.ctile ? s.ctile : round4(xs.channels), in.h = xs.height, in.w = xs.width;
        in.org_mul = scale < 0 ? 1 : scale, in.org_sub = XL;
        in.ext_h = eh, in.ext_w = ew, in.cpitch = smem_pitch(in.c);
        in.smem_off = int(floats);
        bool window_reader = false;
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            const Layer& l = *g.find_layer(op.layer);
            window_reader |= op.stage == 1 && op.xin == int(xi) && l.kind == LayerKind::conv && l.conv->kernel_w > 1;
        }
        floats += (long long)(eh * ew + (window_reader ? kSlackCells : 0)) * in.cpitch;
    }
    std::vector<FBuf> bufs(static_cast<size_t>(nbufs));
    for (int i = 0; i < nops; ++i) {
        if (bufidx[size_t(i)] < 0) continue;
        const TensorShape os = *g.find_layer(s.ops[size_t(i)].layer)->out_shape;
        FBuf& b = bufs[size_t(bufidx[size_t(i)])];
        b.channels = os.channels, b.cpitch = smem_pitch(os.channels);
        b.ext_h = geo[size_t(i)].ext_h, b.ext_w = geo[size_t(i)].ext_w;
        b.smem_off = int(floats);
        bool window_reader = false;
        for (const OpSpec& c : s.ops) {
            const Layer& l = *g.find_layer(c.layer);
            window_reader |= c.stage == 2 && std::find(c.srcs.begin(), c.srcs.end(), i) != c.srcs.end() && l.kind == LayerKind::conv &&
                             l.conv->kernel_w > 1;
        }
        floats += (long long)(b.ext_h * b.ext_w + (window_reader ? kSlackCells : 0)) * b.cpitch;
    }
    if (fp) {
        *fp = FusedParams{};
        fp->nins = int(ins.size());
        for (size_t i = 0; i < ins.size(); ++i) fp->in[i] = ins[i];
        fp->tile_h = th, fp->tile_w = tw;
        fp->out_h = s.out_h, fp->out_w = s.out_w;
        fp->grid_h = (s.out_h + th - 1) / th, fp->grid_w = (s.out_w + tw - 1) / tw;
        fp->nops = nops, fp->nbufs = nbufs, fp->smem_floats = int(floats);
        fp->ctile = s.ctile;
        fp->threads = s.threads == 512 ? 512 : 256;
        fp->cgroups = s.ctile ? round4(g.shape_of(s.inputs[0]).channels) / s.ctile : 1;
        for (int i = 0; i < nbufs; ++i) fp->bufs[i] = bufs[size_t(i)];
        for (int i = 0; i < nops; ++i) {
            const OpSpec& os = s.ops[size_t(i)];
            const Layer& l = *g.find_layer(os.layer);
            FOp& o = fp->ops[i];
            o = FOp{};
            o.stage = os.stage, o.xin = os.xin;
            o.src = os.srcs.empty() ? -1 : bufidx[size_t(os.srcs[0])];
            o.src2 = os.srcs.size() > 1 ? bufidx[size_t(os.srcs[1])] : -1;
            o.buf = bufidx[size_t(i)];
            o.emit = os.emit, o.own_only = os.own_only;
            const TensorShape out = *l.out_shape;
            o.H = out.height, o.W = out.width;
            o.cout = out.channels, o.cout_pad = round4(out.channels);
            const Window w = window_of(l);
            o.kh = w.kh, o.kw = w.kw, o.stride = w.stride, o.pad = w.pad;
            o.group = 1;
            if (l.kind == LayerKind::conv) {
                o.kind = OP_CONV;
                o.cin = l.conv->in_channels, o.group = l.conv->group, o.relu = l.conv->activation == Activation::relu;
            } else if (l.kind == LayerKind::pool) {
                o.kind = l.pool->kind == PoolKind::max ? OP_MAXPOOL : OP_AVGPOOL;
                o.cin = out.channels;
                if (s.ctile) o.cout_pad = s.ctile;
            } else {
                o.kind = OP_ADD;
                o.cin = out.channels;
            }
            o.d = geo[size_t(i)].d;
            o.ext_h = geo[size_t(i)].ext_h, o.ext_w = geo[size_t(i)].ext_w;
            o.org_mul = geo[size_t(i)].org_mul, o.org_sub = geo[size_t(i)].org_sub;
            if (s.rb) rb_variant(o, fp->threads);
        }
    }
    return floats * 4;
}

// Modelled SM cycles of one fp32 step at a tile: per CTA, the serial
// per-thread instruction count (rounds of 256 threads over each op's units,
// input staging) and the warp instructions it issues; the busiest SM runs
// ceil(CTAs / 148) CTAs, `occ` at a time, issuing <= 4 warp instructions per
// cycle.  Halo recompute and partial tiles / row windows show up as units.
double fp32_tile_cycles(const FusedParams& fp, int batch, long long smem) {
    double lat = 0, wi = 0;
    const double nt = fp.threads;
    auto add = [&](double units, double per) {
        lat += std::ceil(units / nt) * per;
        wi += std::ceil(units / 32.0) * per;
    };
    for (int i = 0; i < fp.nins; ++i) add(double(fp.in[i].ext_h) * fp.in[i].ext_w * fp.in[i].c / 4.0, 6.0);
    for (int i = 0; i < fp.nops; ++i) {
        const FOp& o = fp.ops[i];
        const double cells = double(o.ext_h) * o.ext_w, Q = o.cout_pad / 4;
        if (o.kind == OP_CONV && o.cx)
            add(rb_units(o, o.cx, o.ocv), rb_unit_instr(o, o.cx, o.ocv) * 1.3);
        else if (o.kind == OP_CONV) {
            const int PX = cells * Q >= 8 * nt && o.group == 1 ? 8 : 4;
            add(std::ceil(cells / PX) * Q, double(o.cin / o.group) * o.kh * o.kw * (1 + PX + 4 * PX) * 1.3);
        } else
            add(cells * Q, 3.0 * o.kh * o.kw + 8);
    }
    // Weights stream from L2 through L1 (~64 B/cycle per SM); past what L1
    // keeps beside the CTAs' shared memory, every round of units re-reads them.
    const int occ = std::max(1, std::min(fp.threads == 512 ? 1 : 2, int((228 * 1024) / (smem + 1024))));  // registers: 128 x 512 per SM
    const double l1_keep = std::max(16.0 * 1024, (256.0 * 1024 - double(occ) * smem) / occ / 2);
    double l2 = 0;
    for (int i = 0; i < fp.nops; ++i) {
        const FOp& o = fp.ops[i];
        if (o.kind != OP_CONV) continue;
        const double wb = double(o.cin / o.group) * o.kh * o.kw * o.cout_pad * 4;
        const double units = o.cx ? rb_units(o, o.cx, o.ocv)
                                  : double(o.ext_h) * o.ext_w * o.cout_pad / 16;
        l2 += wb > l1_keep ? wb * std::ceil(units / nt) : wb;
    }
    const double ctas = double(fp.grid_h) * fp.grid_w * fp.cgroups * std::max(batch, 1);
    const double per_sm = std::ceil(ctas / 148.0);
    const double conc = std::min(double(occ), per_sm);
    return std::max({per_sm * wi / 3.0, per_sm * l2 / 64.0, std::ceil(per_sm / conc) * (lat + 1500.0)}) + 300.0 * per_sm;
}

// Tile choice: minimise the modelled SM cycles (fp32_tile_cycles).
bool choose_tile_at(const Graph& g, StepSpec& s, int batch_hint, int smem_budget, const Knobs& k);

// Pool-only steps whose full-channel region never fits shared memory (a
// global average pool over 13x13x1000) are tiled over channels as well.
bool choose_tile(const Graph& g, StepSpec& s, int batch_hint, int smem_budget, const Knobs& k) {
    s.ctile = 0;
    if (choose_tile_at(g, s, batch_hint, smem_budget, k)) return true;
    bool pools = s.inputs.size() == 1;
    for (const OpSpec& op : s.ops) pools &= op.stage == 1 && g.find_layer(op.layer)->kind == LayerKind::pool;
    if (!pools) return false;
    const int C = round4(g.shape_of(s.inputs[0]).channels);
    for (int ct = C - 4; ct >= 4; ct -= 4) {
        if (C % ct) continue;
        s.ctile = ct;
        if (choose_tile_at(g, s, batch_hint, smem_budget, k)) return true;
    }
    s.ctile = 0;
    return false;
}

bool choose_tile_at(const Graph& g, StepSpec& s, int batch_hint, int smem_budget, const Knobs& k) {
    double best = 1e300;
    int bh = 0, bw = 0, bsm = 0;
    int fh = 0, fw = 0;
    const bool forced = k.forced_tile(s, &fh, &fw);
    const int lim_h = forced ? fh : std::min(s.out_h, 32), lim_w = forced ? fw : std::min(s.out_w, 32);
    for (int th = 1; th <= lim_h; ++th)
        for (int tw = 1; tw <= lim_w; ++tw) {
            if (forced && (fh % th || fw % tw)) continue;  // sub-tiles of the plan's tile (see Knobs::tiles)
            FusedParams fp;
            const long long sm = layout_step(g, s, th, tw, &fp);
            if (sm < 0 || sm > smem_budget) continue;
            const double t = fp32_tile_cycles(fp, batch_hint, sm);
            const double key = forced ? -double(th) * tw : t;  // the plan's tile, else its largest feasible sub-tile
            if (key < best * 0.999 || (key <= best * 1.001 && long(th) * tw > long(bh) * bw)) best = key, bh = th, bw = tw, bsm = int(sm);
        }
    if (!bh) return false;
    s.tile_h = bh, s.tile_w = bw, s.smem_bytes = bsm;
    return true;
}

}  // namespace

std::vector<F32Candidate> candidates_fp32(const Graph& g, const StepSpec& s, int batch_hint, int smem_budget) {
    std::vector<F32Candidate> out;
    StepSpec t = s;
    for (int mode = 0; mode < 4; ++mode) {
        t.rb = mode & 1, t.threads = mode & 2 ? 512 : 256;
        for (int th = 1; th <= std::min(s.out_h, 32); ++th)
            for (int tw = 1; tw <= std::min(s.out_w, 32); ++tw) {
                FusedParams fp;
                const long long sm = layout_step(g, t, th, tw, &fp);
                if (sm < 0 || sm > smem_budget) continue;
                out.push_back({th, tw, t.rb, t.threads, int(sm), fp32_tile_cycles(fp, batch_hint, sm)});
            }
    }
    std::stable_sort(out.begin(), out.end(), [](const F32Candidate& a, const F32Candidate& b) { return a.model < b.model; });
    return out;
}

long long fp32_layout_bytes(const Graph& g, const StepSpec& s, int th, int tw) { return layout_step(g, s, th, tw, nullptr); }

// Algorithmic traffic / work of a step: block inputs once +
// stored outputs once per image (bytes_algorithmic), weights + biases once
// per launch (weight_bytes), MACs without halo recompute.
void fill_stats(const Graph& g, const DevicePlan& plan, StepSpec& s) {
    const double es = plan.tc_es ? double(plan.tc_es) : 4.0;  // bytes per activation / weight element
    s.macs = 0, s.bytes_algorithmic = 0, s.macs_executed = 0, s.weight_bytes = 0;
    for (const std::string& in : s.inputs) s.bytes_algorithmic += double(g.shape_of(in).elements()) * es;
    if (s.kind == StepSpec::CONCAT_COPY) {
        s.bytes_algorithmic *= 2;
        return;
    }
    for (const OpSpec& op : s.ops) {
        const Layer& l = *g.find_layer(op.layer);
        if (l.kind == LayerKind::conv) {
            s.macs += double(l.out_shape->elements()) * double(l.conv->macs_per_output());
            s.weight_bytes += double(l.conv->weight_count() + l.conv->bias_count()) * es;
        }
        if (op.emit) s.bytes_algorithmic += double(g.shape_of(s.gap_out.empty() ? op.layer : s.gap_out).elements()) * es;
    }
    if (s.kind != StepSpec::FUSED) {
        s.bytes_algorithmic += double(g.shape_of(s.layers[0]).elements()) * es;
        return;
    }
    if (plan.tc_es) {
        s.macs_executed = s.macs;
        return;
    }
    FusedParams fp;
    layout_step(g, s, s.tile_h, s.tile_w, &fp);
    const double tiles = double(fp.grid_h) * fp.grid_w;
    for (int i = 0; i < fp.nops; ++i) {
        const Layer& l = *g.find_layer(s.ops[size_t(i)].layer);
        if (l.kind == LayerKind::conv)
            s.macs_executed += tiles * fp.ops[i].ext_h * fp.ops[i].ext_w * l.out_shape->channels * double(l.conv->macs_per_output());
    }
}

bool Knobs::forced_tile(const StepSpec& s, int* th, int* tw) const {
    if (tiles.empty()) return false;
    for (const std::string& l : s.layers) {
        auto it = tiles.find(l);
        if (it != tiles.end()) {
            *th = it->second.first, *tw = it->second.second;
            return true;
        }
    }
    return false;
}

Knobs Knobs::parse(const std::string& text) {
    Knobs k;
    size_t pos = 0;
    while (pos < text.size()) {
        size_t end = text.find(',', pos);
        if (end == std::string::npos) end = text.size();
        const std::string item = text.substr(pos, end - pos);
        pos = end + 1;
        if (item.find_first_not_of(" \t") == std::string::npos) continue;
        const size_t eq = item.find('=');
        if (eq == std::string::npos) fail(ErrorKind::validation, "options: '" + item + "' is not key=value");
        const std::string key = item.substr(0, eq), val = item.substr(eq + 1);
        char* rest = nullptr;
        const double num = std::strtod(val.c_str(), &rest);
        const bool is_num = !val.empty() && rest && *rest == 0;
        auto need_num = [&]() {
            if (!is_num) fail(ErrorKind::validation, "options: '" + key + "' needs a number, got '" + val + "'");
            return num;
        };
        if (key == "always_fuse") k.always_fuse = need_num() != 0;
        else if (key == "unfuse") k.unfuse = ";" + val + ";";
        else if (key == "unfuse_ratio") k.unfuse_ratio = need_num();
        else if (key == "mb_max_weight") k.mb_max_weight = need_num();
        else if (key == "mb_pw") k.mb_pw = int(need_num());
        else if (key == "no_nalt") k.no_nalt = need_num() != 0;
        else if (key == "no_tsep") k.no_tsep = need_num() != 0;
        else if (key == "no_pwait") k.no_pwait = need_num() != 0;
        else if (key == "xrel_epi") k.xrel_epi = need_num() != 0;
        else if (key == "xbuf") k.xbuf = int(need_num());
        else if (key == "wres") k.wres = int(need_num());
        else if (key == "tsets") k.tsets = int(need_num());
        else if (key == "ctas") k.ctas = int(need_num());
        else if (key == "nsplit") k.nsplit = int(need_num());
        else if (key == "pdl") k.pdl = need_num() != 0;
        else if (key == "no_s2d") k.no_s2d = need_num() != 0;
        else if (key == "no_stem") k.no_stem = need_num() != 0;
        else if (key == "no_pw") k.no_pw = need_num() != 0;
        else if (key == "no_fire") k.no_fire = need_num() != 0;
        else if (key == "no_dw") k.no_dw = need_num() != 0;
        else if (key == "pw_mc") k.pw_mc = need_num() != 0;
        else if (key == "fire_g") k.fire_g = int(need_num());
        else if (key == "fire_r") k.fire_r = int(need_num());
        else if (key == "fire_nsplit") k.fire_nsplit = int(need_num());
        else if (key == "fire_stage") k.fire_stage = int(need_num());
        else if (key == "fire_sqs") k.fire_sqs = int(need_num());
        else if (key == "fire_cb") k.fire_cb = int(need_num());
        else if (key == "fire_cps") k.fire_cps = int(need_num());
        else if (key == "trace") k.trace = int(need_num());
        else if (key == "tune_verbose") k.tune_verbose = need_num() != 0;
        else if (key == "e2e_chunks") k.e2e_chunks = std::max(1, int(need_num()));
        else if (key == "e2e_ramp") k.e2e_ramp = need_num() != 0;
        else if (key == "tile") {
            std::stringstream ss(val);
            std::string it;
            while (std::getline(ss, it, ';')) {
                const size_t c = it.rfind(':'), x = it.rfind('x');
                int h = 0, w = 0;
                if (c == std::string::npos || x == std::string::npos || x < c ||
                    std::sscanf(it.c_str() + c + 1, "%dx%d", &h, &w) != 2 || h < 1 || w < 1)
                    fail(ErrorKind::validation, "options: tile entries are <layer>:<h>x<w>, got '" + it + "'");
                k.tiles[it.substr(0, c)] = {h, w};
            }
        }
        else fail(ErrorKind::validation, "options: unknown key '" + key + "'");
    }
    return k;
}

DevicePlan plan_device(const Graph& g, Partition part, int batch_hint, int smem_budget, int tc_es, const Knobs& knobs) {
    if (!g.shapes_inferred()) fail(ErrorKind::internal, "plan_device requires inferred shapes");
    if (tc_es != 0 && tc_es != 2 && tc_es != 4) fail(ErrorKind::validation, "plan_device: element size must be 0, 2 or 4");
    DevicePlan plan;
    plan.partition = part;
    plan.tc_es = tc_es;
    const bool tc = tc_es != 0;
    const int cpad = tc_es == 2 ? 8 : 4;  // channel padding of HBM tensors (16 bytes)
    auto tile = [&](StepSpec& st) {
        return tc ? choose_tile_tc(g, st, batch_hint, std::min(smem_budget, kSmemBudgetTc), tc_es, knobs) : choose_tile(g, st, batch_hint, smem_budget, knobs);
    };
    if (part == Partition::reference) plan.blocks = detect_fusion_blocks(g);
    else if (part == Partition::b200) plan.blocks = detect_fusion_blocks_b200(g);
    else {
        int next = 0;
        for (const Layer* l : topo_order(g)) {
            FusionBlock b;
            b.id = "b" + std::to_string(next++);
            b.members = {l->name};
            plan.blocks.push_back(b);
        }
    }
    // Execute in topological order of each block's first member (fused_exec.cpp:322-332).
    const auto tix = topo_index(g);
    auto first = [&](const FusionBlock& b) {
        int m = 1 << 30;
        for (const std::string& n : b.members) m = std::min(m, tix.at(n));
        return m;
    };
    std::vector<FusionBlock> ordered = plan.blocks;
    std::stable_sort(ordered.begin(), ordered.end(), [&](const FusionBlock& a, const FusionBlock& b) { return first(a) < first(b); });

    std::vector<StepSpec> steps;
    for (const FusionBlock& b : ordered) {
        StepSpec s = step_for_block(g, b);
        // Split blocks the fire kernel takes stay fused: its squeeze plane never
        // leaves shared memory and its units are whole images or row bands, so
        // neither the generic kernel's tile limits nor the tile-size penalty the
        // cost model below prices apply.
        if (tc && b.fused() && fire_feasible(g, s, tc_es, batch_hint, knobs)) {
            tile(s);  // generic geometry for the statistics only (the engine replaces it)
            steps.push_back(s);
            continue;
        }
        if (s.kind == StepSpec::FUSED && !tile(s)) {
            if (!b.fused()) fail(ErrorKind::infeasible, "layer " + b.members[0] + " does not fit shared memory at any tile");
            // tensor cores: conv -> global average pool runs as one kernel
            // whose epilogue reduces (the conv output never reaches HBM).
            if (tc && part == Partition::b200 && s.ops.size() == 2 && s.ops[0].stage == 1 && s.ops[1].stage == 2) {
                const Layer& c = *g.find_layer(s.ops[0].layer);
                const Layer& p = *g.find_layer(s.ops[1].layer);
                if (c.kind == LayerKind::conv && p.kind == LayerKind::pool && p.pool->kind == PoolKind::avg && p.pool->pad == 0 &&
                    p.pool->kernel == c.out_shape->height && p.pool->kernel == c.out_shape->width && tc_mma_ok(c, tc_es) &&
                    !g.is_output(c.name) && g.consumers_of(c.name).size() == 1) {
                    StepSpec t = s;
                    t.tag = "conv+gap";
                    t.ops.resize(1);
                    t.ops[0].staged = false, t.ops[0].emit = true, t.ops[0].own_only = false;
                    t.gap_out = p.name;
                    t.out_h = c.out_shape->height, t.out_w = c.out_shape->width;
                    if (tile(t)) {
                        steps.push_back(t);
                        continue;
                    }
                }
            }
            // Fused block infeasible on chip: run its members as singletons.
            for (const std::string& m : b.members) {
                FusionBlock one;
                one.id = b.id + "." + m;
                one.members = {m};
                StepSpec t = step_for_block(g, one);
                if (t.kind == StepSpec::FUSED && !tile(t))
                    fail(ErrorKind::infeasible, "layer " + m + " does not fit shared memory at any tile");
                steps.push_back(t);
            }
            continue;
        }
        // tensor-core B200: fusion is not free -- a fused block stages its producers'
        // (wider) inputs, so its tiles are smaller and a weight-heavy consumer
        // re-streams its weights for more tiles.  Keep the block fused only if
        // the planner's model says it beats its layers run as single kernels
        // plus the HBM round trip of the intermediates (SURVEY §8f rank 1's
        // model, the same scores the measured tuner starts from).
        // Weightless consumers (conv -> pool) re-stream nothing: the split's
        // premise does not hold, and the model mis-ranks them (TF32 C1 at
        // batch 1: 29.7 us split vs 23.1 us fused), so they stay fused.
        bool pool_consumers = false;
        for (const OpSpec& op : s.ops)
            if (op.stage == 2) pool_consumers = true;
        for (const OpSpec& op : s.ops)
            if (op.stage == 2 && g.find_layer(op.layer)->kind != LayerKind::pool) pool_consumers = false;
        if (tc && part == Partition::b200 && s.kind == StepSpec::FUSED && b.fused() && s.gap_out.empty() && !knobs.always_fuse && !pool_consumers) {
            const int budget = std::min(smem_budget, kSmemBudgetTc);
            const std::vector<BCandidate> fc = candidates_tc(g, s, batch_hint, budget, tc_es, knobs);
            double fused = fc.empty() ? 1e300 : fc.front().model, single = 0;
            std::vector<StepSpec> singles;
            for (const std::string& m : b.members) {
                FusionBlock one;
                one.id = b.id + "." + m;
                one.members = {m};
                StepSpec t = step_for_block(g, one);
                if (t.kind != StepSpec::FUSED) {
                    single = 1e300;
                    break;
                }
                const std::vector<BCandidate> sc = candidates_tc(g, t, batch_hint, budget, tc_es, knobs);
                if (sc.empty()) {
                    single = 1e300;
                    break;
                }
                apply_candidate(t, sc.front());
                single += sc.front().model;
                singles.push_back(t);
            }
            // experiment knob: unfuse=<block id>[;<block id>...]
            const bool force_split = knobs.unfuse.find(";" + b.id + ";") != std::string::npos;
            if (force_split || single < knobs.unfuse_ratio * fused) {
                for (StepSpec& t : singles) steps.push_back(t);
                continue;
            }
        }
        steps.push_back(s);
    }

    // B200: shared-input multi-branch kernels.  Steps whose stage-1 ops all
    // read the same single tensor and whose outputs share one extent run as
    // one kernel (one staged input region), if the union still fits.
    if (part == Partition::b200) {
        const double mb_max_weight = knobs.mb_max_weight;
        std::vector<char> gone(steps.size(), 0), fire(steps.size(), 0);
        // steps the fire kernel runs keep their own kernel
        for (size_t i = 0; i < steps.size(); ++i) fire[i] = tc && fire_feasible(g, steps[i], tc_es, batch_hint, knobs);
        // Steps the pointwise kernel runs (one 1x1 conv: all pixels of the
        // launch as one M dimension, resident channel-group weights) beat the
        // generic kernel's tiles; merging them only saves a re-read of the
        // shared input, which L2 serves.  Measured (bf16): inception-3a at
        // batch 64 117 us with its four branches merged, 113 us with the 1x1
        // branch merged into the pool projection, 97 us with every 1x1 conv on
        // the pointwise kernel; C2 merge at batch 8 23.7 vs 24.4 us.  So
        // pointwise steps stay out of multi-branch kernels (option mb_pw=1
        // merges them).
        std::vector<int> npw(steps.size(), 0);
        for (size_t i = 0; i < steps.size(); ++i) {
            const StepSpec& t = steps[i];
            if (!tc || t.kind != StepSpec::FUSED || t.ops.size() != 1 || !t.gap_out.empty()) continue;
            const Layer& l = *g.find_layer(t.ops[0].layer);
            npw[i] = l.kind == LayerKind::conv && l.conv->kernel_h == 1 && l.conv->kernel_w == 1 && l.conv->stride == 1 &&
                     l.conv->pad == 0 && l.conv->group == 1;
        }
        for (size_t i = 0; i < steps.size(); ++i) {
            if (gone[i] || fire[i] || steps[i].kind != StepSpec::FUSED || steps[i].inputs.size() != 1) continue;
            for (size_t j = i + 1; j < steps.size(); ++j) {
                if (gone[j] || fire[j] || steps[j].kind != StepSpec::FUSED || steps[j].inputs != steps[i].inputs) continue;
                if (steps[j].out_h != steps[i].out_h || steps[j].out_w != steps[i].out_w) continue;
                if (!knobs.mb_pw && (npw[i] || npw[j])) continue;
                StepSpec m = steps[i];
                const int base = int(m.ops.size());
                for (OpSpec op : steps[j].ops) {
                    for (int& si : op.srcs) si += base;
                    m.ops.push_back(op);
                }
                std::stable_sort(m.ops.begin(), m.ops.end(), [](const OpSpec& a, const OpSpec& b) { return a.stage < b.stage; });
                // re-map srcs after the stage sort
                std::vector<std::string> names;
                for (const OpSpec& op : m.ops) names.push_back(op.layer);
                for (OpSpec& op : m.ops) {
                    if (op.stage != 2) continue;
                    const Layer& l = *g.find_layer(op.layer);
                    op.srcs.clear();
                    for (const std::string& in : l.inputs)
                        for (size_t k = 0; k < names.size(); ++k)
                            if (names[k] == in) op.srcs.push_back(int(k));
                }
                m.layers.insert(m.layers.end(), steps[j].layers.begin(), steps[j].layers.end());
                m.id += "+" + steps[j].id;
                m.tag = "multi-branch";
                m.mode = FusionMode::merge;
                if (mb_max_weight >= 0) {  // experiment knob: cap on the merged kernel's conv weights (bytes)
                    double wb = 0;
                    for (const OpSpec& op : m.ops) {
                        const Layer& l = *g.find_layer(op.layer);
                        if (l.kind == LayerKind::conv) wb += double(l.conv->weight_count()) * (tc_es == 2 ? 2 : 4);
                    }
                    if (wb > mb_max_weight) continue;
                }
                if (!tile(m)) continue;
                steps[i] = m;
                npw[i] += npw[j];
                gone[j] = 1;
            }
        }
        std::vector<StepSpec> kept;
        for (size_t i = 0; i < steps.size(); ++i)
            if (!gone[i]) kept.push_back(steps[i]);
        steps.swap(kept);
    }

    // Which tensors exist in HBM: graph inputs, every emitted op output, every
    // non-fused singleton output.
    std::set<std::string> materialized;
    for (const GraphInput& in : g.inputs) materialized.insert(in.name);
    for (const StepSpec& s : steps) {
        if (s.kind != StepSpec::FUSED) materialized.insert(s.layers[0]);
        for (const OpSpec& op : s.ops)
            if (op.emit) materialized.insert(s.gap_out.empty() ? op.layer : s.gap_out);
    }
    // Concat elision (B200): every input of a concat that is consumed by the
    // concat alone becomes a channel-offset view of the concat's allocation.
    std::map<std::string, std::pair<std::string, int>> view_of;  // tensor -> (concat, channel offset)
    std::set<std::string> elided;
    if (part == Partition::b200) {
        for (const Layer& l : g.layers) {
            if (l.kind != LayerKind::concat || !materialized.count(l.name)) continue;
            bool ok = true;
            int off = 0;
            for (const std::string& in : l.inputs) {
                const Layer* p = g.find_layer(in);
                const TensorShape s = g.shape_of(in);
                ok &= p != nullptr && !g.is_output(in) && g.consumers_of(in).size() == 1 && materialized.count(in) &&
                      s.channels % cpad == 0 && !view_of.count(in);
                off += s.channels;
            }
            if (!ok) continue;
            off = 0;
            for (const std::string& in : l.inputs) {
                view_of[in] = {l.name, off};
                off += g.shape_of(in).channels;
            }
            elided.insert(l.name);
        }
        std::vector<StepSpec> kept;
        for (StepSpec& s : steps)
            if (!(s.kind == StepSpec::CONCAT_COPY && elided.count(s.layers[0]))) kept.push_back(s);
        steps.swap(kept);
    }
    std::function<TensorSlot(const std::string&)> resolve = [&](const std::string& n) -> TensorSlot {
        auto it = plan.tensors.find(n);
        if (it != plan.tensors.end()) return it->second;
        const TensorShape s = g.shape_of(n);
        TensorSlot t;
        t.materialized = true, t.C = s.channels, t.H = s.height, t.W = s.width;
        auto v = view_of.find(n);
        if (v != view_of.end()) {
            const TensorSlot host = resolve(v->second.first);
            t.alloc = host.alloc, t.cstride = host.cstride, t.coff = host.coff + v->second.second;
        } else {
            t.alloc = int(plan.alloc_floats.size()), t.cstride = (s.channels + cpad - 1) / cpad * cpad, t.coff = 0;
            plan.alloc_floats.push_back((long long)s.height * s.width * t.cstride);
        }
        plan.tensors[n] = t;
        return t;
    };
    for (const GraphInput& in : g.inputs) resolve(in.name);
    for (const Layer* l : topo_order(g))
        if (materialized.count(l->name)) resolve(l->name);
    for (const Layer& l : g.layers)
        if (!plan.tensors.count(l.name)) plan.tensors[l.name] = TensorSlot{};

    long long woff = 0;
    for (const Layer& l : g.layers) {
        if (l.kind != LayerKind::conv) continue;
        const ConvParams& c = *l.conv;
        plan.w_off[l.name] = woff;
        woff += (long long)(c.in_channels / c.group) * c.kernel_h * c.kernel_w * round4(c.out_channels);
        plan.b_off[l.name] = woff;
        woff += round4(c.out_channels);
    }
    plan.weight_floats = woff;
    for (StepSpec& s : steps) fill_stats(g, plan, s);
    plan.steps = steps;
    return plan;
}

std::vector<float> pack_weights(const Graph& g, const DevicePlan& plan, const float* flat, size_t count) {
    std::vector<float> out(size_t(plan.weight_floats), 0.0f);
    size_t pos = 0;
    for (const Layer& l : g.layers) {
        if (l.kind != LayerKind::conv) continue;
        const ConvParams& c = *l.conv;
        const int cin_g = c.in_channels / c.group, cp = round4(c.out_channels);
        const size_t nf = size_t(c.weight_count()), nb = size_t(c.bias_count());
        if (pos + nf + nb > count) fail(ErrorKind::validation, "weights: stream too short for layer '" + l.name + "'");
        float* w = out.data() + plan.w_off.at(l.name);
        for (int oc = 0; oc < c.out_channels; ++oc)
            for (int ic = 0; ic < cin_g; ++ic)
                for (int y = 0; y < c.kernel_h; ++y)
                    for (int x = 0; x < c.kernel_w; ++x)
                        w[((size_t(ic) * c.kernel_h + y) * c.kernel_w + x) * cp + oc] =
                            flat[pos + ((size_t(oc) * cin_g + ic) * c.kernel_h + y) * c.kernel_w + x];
        pos += nf;
        float* b = out.data() + plan.b_off.at(l.name);
        for (size_t i = 0; i < nb; ++i) b[i] = flat[pos + i];
        pos += nb;
    }
    if (pos != count)
        fail(ErrorKind::validation, "weights: stream holds " + std::to_string(count) + " floats, graph needs " + std::to_string(pos));
    return out;
}

FusedParams make_params(const Graph& g, const DevicePlan& plan, const StepSpec& s,
                        const std::vector<float*>& alloc_base, const float* wbase) {
    FusedParams fp;
    if (layout_step(g, s, s.tile_h, s.tile_w, &fp) < 0) fail(ErrorKind::internal, "step " + s.id + ": layout failed");
    for (int i = 0; i < fp.nins; ++i) {
        const TensorSlot& t = plan.tensors.at(s.inputs[size_t(i)]);
        fp.in[i].x = alloc_base[size_t(t.alloc)];
        fp.in[i].cstride = t.cstride, fp.in[i].coff = t.coff;
    }
    for (int i = 0; i < fp.nops; ++i) {
        const OpSpec& os = s.ops[size_t(i)];
        FOp& o = fp.ops[i];
        if (o.kind == OP_CONV) {
            o.w = wbase + plan.w_off.at(os.layer);
            o.b = wbase + plan.b_off.at(os.layer);
        }
        if (o.emit) {
            const TensorSlot& t = plan.tensors.at(os.layer);
            o.out = alloc_base[size_t(t.alloc)];
            o.out_cstride = t.cstride, o.out_coff = t.coff;
        }
    }
    return fp;
}

std::string describe_plan_json(const Graph& g, const DevicePlan& plan) {
    std::ostringstream os;
    auto q = [](const std::string& s) { return "\"" + s + "\""; };
    os << "{\"partition\":" << q(to_string(plan.partition)) << ",\"steps\":[";
    for (size_t i = 0; i < plan.steps.size(); ++i) {
        const StepSpec& s = plan.steps[i];
        static const char* kinds[] = {"fused", "concat_copy", "add", "relu"};
        os << (i ? "," : "") << "{\"id\":" << q(s.id) << ",\"kind\":" << q(kinds[s.kind]) << ",\"tag\":" << q(s.tag)
           << ",\"mode\":" << q(to_string(s.mode)) << ",\"tile\":[" << s.tile_h << "," << s.tile_w
           << "],\"out\":[" << s.out_h << "," << s.out_w << "],\"smem_bytes\":" << s.smem_bytes << ",\"nxb\":" << s.nxb << ",\"wres\":" << s.wres << ",\"ring_slots\":" << s.ring_slots << ",\"grid_all\":" << s.grid_all << ",\"epi_warps\":" << s.epi_warps << ",\"tsets\":" << s.tsets << ",\"nsplit\":" << s.nsplit << ",\"rb\":" << s.rb << ",\"threads\":" << s.threads << ",\"macs\":" << s.macs
           << ",\"macs_executed\":" << s.macs_executed << ",\"bytes_algorithmic\":" << s.bytes_algorithmic
           << ",\"weight_bytes\":" << s.weight_bytes << ",\"ring_chunk\":" << s.ring_chunk << ",\"inputs\":[";
        for (size_t k = 0; k < s.inputs.size(); ++k) os << (k ? "," : "") << q(s.inputs[k]);
        os << "],\"layers\":[";
        for (size_t k = 0; k < s.layers.size(); ++k) os << (k ? "," : "") << q(s.layers[k]);
        os << "],\"ops\":[";
        for (size_t k = 0; k < s.ops.size(); ++k) {
            const OpSpec& o = s.ops[k];
            os << (k ? "," : "") << "{\"layer\":" << q(o.layer) << ",\"stage\":" << o.stage << ",\"staged\":"
               << (o.staged ? "true" : "false") << ",\"emit\":" << (o.emit ? "true" : "false") << "}";
        }
        os << "]}";
    }
    os << "],\"tensors\":{";
    bool firstt = true;
    for (const auto& [n, t] : plan.tensors) {
        os << (firstt ? "" : ",") << q(n) << ":{\"materialized\":" << (t.materialized ? "true" : "false")
           << ",\"alloc\":" << t.alloc << ",\"cstride\":" << t.cstride << ",\"coff\":" << t.coff << ",\"shape\":[" << t.C
           << "," << t.H << "," << t.W << "]}";
        firstt = false;
    }
    os << "},\"alloc_floats\":[";
    for (size_t i = 0; i < plan.alloc_floats.size(); ++i) os << (i ? "," : "") << plan.alloc_floats[i];
    os << "],\"weight_floats\":" << plan.weight_floats << "}";
    (void)g;
    return os.str();
}

}  // namespace xlf
