// Host geometry of the fire kernel (kernels_fire.cu, fire_params.hpp): which
// steps it takes, the unit shape (G whole images or a band of R rows), the
// output-channel split, ring depth and plane count, and the shared-memory /
// TMEM layout.  The unit is chosen by a small model of one SM's time per unit
// (squeeze + expand MMA cycles, HBM bytes at the SM's share of bandwidth,
// epilogue columns) times the rounds the persistent grid needs.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.hpp"
#include "device_plan.hpp"
#include "fire_params.hpp"

namespace xlf {

namespace {
int cdiv(int a, int b) { return (a + b - 1) / b; }
int up(int v, int a) { return (v + a - 1) / a * a; }
}  // namespace

bool fire_step_ok(const Graph& g, const StepSpec& s, int es) {
    if (es != 2 && es != 4) return false;
    if (s.kind != StepSpec::FUSED || !s.gap_out.empty() || s.inputs.size() != 1 || s.ops.size() < 2 || s.ops.size() > 1 + kFireMaxOps)
        return false;
    const OpSpec& o0 = s.ops[0];
    const Layer* sq = g.find_layer(o0.layer);
    if (!sq || !tc_mma_ok(*sq, es) || o0.stage != 1 || o0.emit || o0.xin != 0) return false;
    const ConvParams& c = *sq->conv;
    if (c.kernel_h != 1 || c.kernel_w != 1 || c.pad != 0 || c.out_channels % 16 || c.out_channels > 128) return false;
    if (sq->inputs.size() != 1 || sq->inputs[0] != s.inputs[0]) return false;
    const TensorShape so = *sq->out_shape;
    int cout = -1;
    for (size_t k = 1; k < s.ops.size(); ++k) {
        const OpSpec& o = s.ops[k];
        const Layer* l = g.find_layer(o.layer);
        if (!l || o.stage != 2 || !o.emit || o.srcs.size() != 1 || o.srcs[0] != 0 || !tc_mma_ok(*l, es)) return false;
        const ConvParams& e = *l->conv;
        if (e.in_channels != c.out_channels || e.kernel_h != e.kernel_w || e.kernel_h % 2 == 0 || e.pad != (e.kernel_h - 1) / 2 || e.pad > 1)
            return false;
        if (!(*l->out_shape == TensorShape{e.out_channels, so.height, so.width})) return false;
        if (e.out_channels % 16 || (cout >= 0 && e.out_channels != cout)) return false;
        cout = e.out_channels;
    }
    return true;
}

// Unit geometry for (G, R) on an H x W map: squeeze / expand M tiles and the
// plane's cells (see fire_params.hpp).
static void fire_geometry(int H, int W, int G, int R, int pmax, int* Ts, int* Te, int* cells) {
    const int Wp = W + 1, prows = G * (R + 1) + 1;
    const int px = G > 1 ? G * H * W : std::min(R + 2, H) * W;
    *Ts = cdiv(px, 128);
    *Te = cdiv((G * (R + 1) - 1) * Wp, 128);
    const int read_end = 1 + Wp + *Te * 128 + pmax * Wp + pmax;
    const int write_end = 1 + prows * Wp + 1;  // + the zero column of the row after the last
    *cells = up(std::max(read_end, write_end), 8);
}

// Lays out shared memory for a choice; returns the bytes (or -1: does not fit).
int fire_layout(FireParams& P, int nst, int nplane, bool staged) {
    const int cpc = 16 / P.es;
    int off = 0;
    P.nst = nst, P.nplane = nplane;
    P.ring_off = 0;
    P.stage_bytes = 128 * P.cb + (P.sq_stream ? up((P.cb / 32) * P.S * 32, 1024) : 0);  // stages stay 1024-aligned (swizzle atoms)
    off = nst * P.stage_bytes;
    P.wsq_off = off;
    if (!P.sq_stream) off = up(off + P.ksteps * P.S * 32, 128);
    for (int o = 0; o < P.nops; ++o) {
        P.op[o].w_off = off;
        off = up(off + int(P.op[o].gwb), 128);
    }
    P.plane_off = off;
    P.plane_bytes = P.plane_cells * 16 * (P.S / cpc);
    off = up(off + nplane * P.plane_bytes, 128);
    P.stage_off = staged ? off : -1;
    if (staged) off += (P.cps == 2 ? 4 : 8) * 4096;  // epilogue warps x 32 cells x (64 or 128 bytes)
    P.sqbias_off = off;
    off += P.S * 4;
    for (int o = 0; o < P.nops; ++o) {
        P.op[o].bias_off = off;
        off += P.gch * 4;
    }
    P.smem_bytes = up(off, 128);
    return P.smem_bytes <= (P.cps == 2 ? kFireSmemMax2 : kFireSmemMax) ? P.smem_bytes : -1;
}

// Every feasible (nsplit, G, R) for P (H, W, S, ksteps, nops, op[].kh / pad /
// cout, es filled in), laid out (deepest ring with two planes, else one
// plane), sorted by the model (SM cycles for `batch` images on `sms` SMs).
// Forced values (> 0) restrict the search.
std::vector<std::pair<double, FireParams>> fire_candidates(const FireParams& P, int batch, int sms, int force_nsplit, int force_g, int force_r) {
    const int cpc = 16 / P.es;
    const int cout = P.op[0].cout;
    int pmax = 0, taps = 0;
    for (int o = 0; o < P.nops; ++o) pmax = std::max(pmax, P.op[o].pad), taps += P.op[o].kh * P.op[o].kw;
    const int sq_cols = P.S <= 32 ? 32 : P.S <= 64 ? 64 : 128;
    const double bw_chip = 3300.0;  // HBM bytes per SM cycle, whole chip (~6.5 TB/s at 1.965 GHz)
    std::vector<std::pair<double, FireParams>> out;
    for (int cps : {1, 2})
    for (int cb : {128, 64})
    for (int sqs : {0, 1})
    for (int ns : {1, 2, 3, 4}) {  // 3: 192- and 384-channel expands at 64-channel groups (TF32 fire6/7 weights fit)
        if (force_nsplit > 0 && ns != force_nsplit) continue;
        // 64-byte chunks only on request: they let wider expand weights stay
        // resident (fire8/9 at two channel groups) but measured slower on
        // every SqueezeNet fire step and on inception's r3 -> b3
        if (cb != (P.cb_mode ? P.cb_mode : 128)) continue;
        if (P.cps_mode && cps != P.cps_mode) continue;
        const int tcols = 512 / cps;  // TMEM columns of one CTA
        if (P.sq_stream_mode == 1 && sqs == 0) continue;
        if (P.sq_stream_mode == 2 && sqs == 1) continue;
        if (cout % (32 * ns)) continue;  // whole 32-column store segments per op and group
        const int gch = cout / ns;
        // N < 64 expand MMAs cost as much as N = 64 ones (measured: inception-3a's
        // reduce -> 3x3 at 4 groups of 32 took 61 us against 42 us unfused)
        if (gch < std::min(64, cout)) continue;
        if (gch > 256 || 2 * sq_cols + 2 * gch > tcols) continue;  // two expand accumulators, at least one op each
        // every op of an M tile in one job when two such accumulators fit TMEM, else one job per op
        const int per_op = 2 * sq_cols + 2 * P.nops * gch > tcols ? 1 : 0;
        std::vector<std::pair<int, int>> shapes;  // (G, R)
        for (int G = 1; G <= 8; ++G) shapes.push_back({G, P.H});
        for (int R = 1; R < P.H; ++R) shapes.push_back({1, R});
        for (auto [G, R] : shapes) {
            if (force_g > 0 && G != force_g) continue;
            if (force_r > 0 && R != force_r) continue;
            if (G > 1 && G > batch) continue;
            FireParams Q = P;
            Q.cb = cb;
            Q.cps = cps;
            Q.kchunks = (Q.ksteps * 32 + cb - 1) / cb;
            Q.sq_stream = sqs;
            Q.nsplit = ns, Q.gch = gch, Q.G = G, Q.R = R, Q.bands = cdiv(P.H, R);
            Q.seg = P.es == 2 && gch % 64 == 0 ? 64 : 32;  // 128-byte store segments when the op's channels allow
            fire_geometry(P.H, P.W, G, R, pmax, &Q.Ts, &Q.Te, &Q.plane_cells);
            for (int o = 0; o < Q.nops; ++o) Q.op[o].gwb = (long long)Q.op[o].kh * Q.op[o].kw * (Q.S / cpc) * gch * 16;
            // the deepest ring with two planes, else one plane; stores direct
            // (staged through shared memory only on request: measured 7 %
            // slower on fire2/3, the staging adds shared-memory traffic and a
            // shuffle per store to a kernel bound by per-warp latency)
            int nst = 0, npl = 0;
            bool stg = true;
            for (int st = 0; st <= 1 && !nst; ++st) {
                if (st != (P.stage_mode == 1 ? 1 : 0)) continue;
                for (int pl = 2; pl >= 1 && !nst; --pl)
                    for (int s = kFireStages; s >= (cb == 64 ? 2 : 3); --s)
                        if (fire_layout(Q, s, pl, st != 0) > 0) {
                            nst = s, npl = pl, stg = st != 0;
                            break;
                        }
            }
            if (!nst) continue;
            fire_layout(Q, nst, npl, stg);
            Q.sq_cols = sq_cols;
            Q.per_op = per_op;
            Q.nexslots = std::min(kFireMaxExSlots, (tcols - 2 * sq_cols) / ((per_op ? 1 : Q.nops) * gch));
            // model (SM cycles)
            const int units = G > 1 ? cdiv(batch, G) : batch * Q.bands;
            const long long items = (long long)units * ns;
            const int active = int(std::min<long long>(items, (long long)sms * cps));
            const double rounds = std::ceil(double(items) / (sms * cps));
            const double share = cps == 2 && items > sms ? 2.0 : 1.0;  // two CTAs share an SM's tensor pipe and TMEM read ports
            const double mma_n = std::max(16.0, 0.53 * gch);
            const double sq_mma = double(Q.Ts) * Q.ksteps * std::max(16.0, 0.53 * Q.S);
            const double ex_mma = double(Q.Te) * taps * (Q.S / cpc / 2) * mma_n;
            const double px_in = G > 1 ? double(G) * P.H * P.W : double(std::min(R + 2, P.H)) * P.W;
            const double px_out = G > 1 ? double(G) * P.H * P.W : double(std::min(R, P.H)) * P.W;
            const double bytes = px_in * Q.ksteps * 32 / std::max(1, ns) + px_out * Q.nops * gch * P.es;
            const double mem = bytes / (bw_chip / active);
            // every CTA of a unit's channel groups reads the whole input through L2 (~6 KB / cycle chip-wide)
            const double l2 = (px_in * Q.ksteps * 32 + px_out * Q.nops * gch * P.es) / (6000.0 / active);
            // TMEM reads (64 B / cycle per SM) of every squeeze and expand accumulator
            const double tmem = (double(Q.Ts) * P.S + double(Q.Te) * Q.nops * gch) * 128 * 4 / 64.0;
            // streamed squeeze weights: re-read from L2 per squeeze tile
            const double l2w = sqs ? double(Q.Ts) * Q.ksteps * P.S * 32 / (6000.0 / active) : 0.0;
            const double unit = std::max({(sq_mma + ex_mma) * share, mem, l2 + l2w, tmem * 2.0 * share}) + (npl == 2 ? 600.0 : 1500.0);
            out.push_back({rounds * unit, Q});
        }
    }
    std::stable_sort(out.begin(), out.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    return out;
}

bool fire_choose(FireParams& P, int batch, int sms, int force_nsplit, int force_g, int force_r, double* model_out) {
    const auto c = fire_candidates(P, batch, sms, force_nsplit, force_g, force_r);
    if (c.empty()) return false;
    P = c.front().second;
    if (model_out) *model_out = c.front().first;
    return true;
}

// Shape fields of the fire descriptor from the graph (no device addresses).
void fire_shape(const Graph& g, const StepSpec& s, int es, FireParams& P) {
    const Layer& sq = *g.find_layer(s.ops[0].layer);
    const TensorShape in = g.shape_of(s.inputs[0]);
    P.es = es, P.H = in.height, P.W = in.width, P.HW = in.height * in.width, P.Wp = in.width + 1;
    P.ksteps = sq.conv->in_channels * es / 32;
    P.cb = 128, P.cps = 1;
    P.kchunks = (P.ksteps + 3) / 4;
    P.S = sq.conv->out_channels;
    P.schunks = P.S * es / 16;
    P.sq_relu = sq.conv->activation == Activation::relu;
    P.nops = int(s.ops.size()) - 1;
    for (int o = 0; o < P.nops; ++o) {
        const Layer& l = *g.find_layer(s.ops[size_t(o) + 1].layer);
        FireOp& op = P.op[o];
        op.kh = l.conv->kernel_h, op.kw = l.conv->kernel_w, op.pad = l.conv->pad;
        op.cout = l.conv->out_channels;
        op.relu = l.conv->activation == Activation::relu;
    }
}

bool fire_feasible(const Graph& g, const StepSpec& s, int es, int batch, const Knobs& k) {
    if (k.no_fire || !fire_step_ok(g, s, es)) return false;
    int th, tw;
    if (k.forced_tile(s, &th, &tw)) return false;  // a reference plan's tile drives the generic kernel (xlf_block_prepare)
    FireParams P{};
    fire_shape(g, s, es, P);
    P.stage_mode = k.fire_stage;
    P.sq_stream_mode = k.fire_sqs;
    P.cb_mode = k.fire_cb;
    P.cps_mode = k.fire_cps;
    return fire_choose(P, std::max(1, batch), 148, k.fire_nsplit, k.fire_g, k.fire_r, nullptr);
}

}  // namespace xlf
