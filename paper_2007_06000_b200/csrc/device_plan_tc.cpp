// Geometry of the tensor-core kernel (kernels_tc.cu) for a step of the device
// program: per-op MMA/SIMT choice, regions, TMEM columns, shared bytes, and
// the weight packing the MMA B operand reads.  `es` is the element size of
// the step (2: bf16, 4: fp32 storage of TF32 values); every shared layout is
// in 16-byte chunks (cpc = 16 / es channels) and 32-byte K steps.
#include <algorithm>
#include <vector>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "tc_params.hpp"
#include "common.hpp"
#include "device_plan.hpp"

namespace xlf {

namespace {

int r16(int c) { return (c + 15) & ~15; }
int rc(int c, int es) { const int cpc = 16 / es; return (c + cpc - 1) / cpc * cpc; }  // channels rounded up to a chunk
int r128(int c) { return (c + 127) & ~127; }
int cdiv(int a, int b) { return (a + b - 1) / b; }
int pow2_cols(int c) {
    if (c <= 0) return 0;
    int p = 32;
    while (p < c) p <<= 1;
    return p;
}

struct Win {
    int kh = 1, kw = 1, stride = 1, pad = 0;
};
Win win(const Layer& l) {
    if (l.kind == LayerKind::conv) return {l.conv->kernel_h, l.conv->kernel_w, l.conv->stride, l.conv->pad};
    if (l.kind == LayerKind::pool) return {l.pool->kernel, l.pool->kernel, l.pool->stride, l.pool->pad};
    return {};
}

constexpr int kSlack = 2048;  // contiguous-M tiles may read up to 127 cells past a plane

}  // namespace

bool tc_mma_ok(const Layer& l, int es) {  // whole 32-byte K steps: Cin % 16 (bf16) / % 8 (TF32)
    return l.kind == LayerKind::conv && l.conv->stride == 1 && l.conv->group == 1 && (l.conv->in_channels * es) % 32 == 0;
}

// N blocking of an MMA conv: nblocks x nb accumulator columns, nb % 16 == 0, nb <= 256.
void tc_nblocks(int cout, int* nblocks, int* nb) {
    const int n16 = r16(cout);
    *nblocks = cdiv(n16, 256);
    *nb = r16(cdiv(n16, *nblocks));
}

long long layout_tc(const Graph& g, const StepSpec& s, int th, int tw, BParams* P, int nxb, int wres, int ring_slots, int tsets,
                    int chunk, int es, const Knobs& k) {
    const int nops = int(s.ops.size());
    if (es != 2 && es != 4) return -1;
    const int cpc = 16 / es;
    // tuning-report values come from outside: reject what the kernel cannot run
    if (nxb < 1 || nxb > 2 || tsets < 1 || tsets > 2 || th < 1 || tw < 1) return -1;
    if (!wres && (ring_slots < 1 || ring_slots > kRingMax || chunk < 1024 || chunk % 1024)) return -1;
    if (nops > kBMaxOps || s.inputs.size() > size_t(kMaxIns)) return -1;
    struct G {
        int ext_h, ext_w, mul, sub, d;
        bool mma, contig;
    };
    std::vector<G> geo(static_cast<size_t>(nops));
    std::vector<int> bufidx(static_cast<size_t>(nops), -1);
    const int rows_m = cdiv(th, 16) * 16;  // windowed MMA ops over the tile compute whole 16-row blocks
    const int cols_m = cdiv(tw, 8) * 8;
    int nbufs = 0;
    for (int i = 0; i < nops; ++i) {
        const Layer& l = *g.find_layer(s.ops[size_t(i)].layer);
        geo[size_t(i)] = {th, tw, 1, 0, 0, tc_mma_ok(l, es), false};
    }
    // staged buffers: lead L, stride S, trail T from the readers (+ the rows /
    // columns windowed MMA readers over-read)
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
            const Win w = win(cl);
            if (S >= 0 && S != w.stride) return -1;
            S = w.stride, L = std::max(L, w.pad);
            Th = std::max(Th, w.kh - w.pad), Tw = std::max(Tw, w.kw - w.pad);
        }
        if (add_reader) {
            if (S > 1 || L > 0) return -1;
            S = 1;
        }
        if (S < 0) S = 1;
        if (op.own_only) Th = std::max(Th, S), Tw = std::max(Tw, S);
        int eh = (th - 1) * S + L + Th, ew = (tw - 1) * S + L + Tw;
        for (const OpSpec& c : s.ops) {
            if (c.stage != 2 || std::find(c.srcs.begin(), c.srcs.end(), i) == c.srcs.end()) continue;
            const Layer& cl = *g.find_layer(c.layer);
            if (!tc_mma_ok(cl, es)) continue;
            const Win w = win(cl);
            eh = std::max(eh, rows_m - 1 + w.kh - 1 + (L - w.pad) + 1);
            ew = std::max(ew, cols_m - 1 + w.kw - 1 + (L - w.pad) + 1);
        }
        G& gi = geo[size_t(i)];
        gi.ext_h = eh, gi.ext_w = ew, gi.mul = S, gi.sub = L;
        bufidx[size_t(i)] = nbufs++;
    }
    if (nbufs > kBMaxBufs) return -1;

    // block inputs
    std::vector<BIn> ins(s.inputs.size());
    std::vector<int> XLs(s.inputs.size()), scales(s.inputs.size());
    for (size_t xi = 0; xi < s.inputs.size(); ++xi) {
        int scale = -1, XL = 0;
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            if (op.stage != 1 || op.xin != int(xi)) continue;
            const Win w = win(*g.find_layer(op.layer));
            const int sc = geo[size_t(i)].mul * w.stride;
            if (scale >= 0 && sc != scale) return -1;
            scale = sc;
            XL = std::max(XL, geo[size_t(i)].sub * w.stride + w.pad);
        }
        XLs[xi] = XL, scales[xi] = scale < 0 ? 1 : scale;
    }
    // 1x1 stride-1 MMA producers whose buffer readers all have stride 1 run in
    // contiguous-M mode: their region IS the input region (d = 0), so every
    // 128 consecutive cells form one GEMM tile.
    for (int i = 0; i < nops; ++i) {
        const OpSpec& op = s.ops[size_t(i)];
        G& gi = geo[size_t(i)];
        const Layer& l = *g.find_layer(op.layer);
        if (op.stage != 1 || !gi.mma || l.conv->kernel_h != 1 || l.conv->kernel_w != 1 || l.conv->pad != 0) continue;
        if (scales[size_t(op.xin)] != 1) continue;
        gi.contig = true;
    }
    for (size_t xi = 0; xi < s.inputs.size(); ++xi) {
        const int XL = XLs[xi];
        int eh = 0, ew = 0;
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            if (op.stage != 1 || op.xin != int(xi)) continue;
            const Win w = win(*g.find_layer(op.layer));
            G& gi = geo[size_t(i)];
            if (gi.contig) continue;
            gi.d = XL - (gi.sub * w.stride + w.pad);
            const int rh = gi.mma ? cdiv(gi.ext_h, 16) * 16 : gi.ext_h;
            const int rw = gi.mma ? cdiv(gi.ext_w, 8) * 8 : gi.ext_w;
            eh = std::max(eh, gi.d + (rh - 1) * w.stride + w.kh);
            ew = std::max(ew, gi.d + (rw - 1) * w.stride + w.kw);
        }
        // contiguous producers: their buffer = this region; readers' reach
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            if (op.stage != 1 || op.xin != int(xi) || !geo[size_t(i)].contig) continue;
            eh = std::max(eh, geo[size_t(i)].ext_h + (XL - geo[size_t(i)].sub));
            ew = std::max(ew, geo[size_t(i)].ext_w + (XL - geo[size_t(i)].sub));
            for (const OpSpec& c : s.ops) {
                if (c.stage != 2 || std::find(c.srcs.begin(), c.srcs.end(), i) == c.srcs.end()) continue;
                const Layer& cl = *g.find_layer(c.layer);
                const Win w = win(cl);
                const bool cm = tc_mma_ok(cl, es);
                const int rh = cm ? rows_m : th, rw = cm ? cols_m : tw;
                const int d = cl.kind == LayerKind::add ? 0 : XL - w.pad;
                eh = std::max(eh, d + (rh - 1) * w.stride + w.kh);
                ew = std::max(ew, d + (rw - 1) * w.stride + w.kw);
            }
        }
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            if (op.stage != 1 || op.xin != int(xi) || !geo[size_t(i)].contig) continue;
            G& gi = geo[size_t(i)];
            gi.ext_h = eh, gi.ext_w = ew, gi.sub = XL, gi.d = 0;
        }
        const TensorShape xs = g.shape_of(s.inputs[xi]);
        BIn& in = ins[xi];
        in = BIn{};
        in.r.chunks = (s.ctile ? s.ctile : rc(xs.channels, es)) / cpc;
        in.r.ext_h = eh, in.r.ext_w = ew;
        in.h = xs.height, in.w = xs.width;
        in.org_mul = scales[xi], in.org_sub = XL;
        if (eh > 256 || ew > 256) return -1;  // TMA box limit
    }
    // readers' offsets into buffers
    for (int i = 0; i < nops; ++i) {
        const OpSpec& op = s.ops[size_t(i)];
        if (op.stage != 2) continue;
        const Layer& l = *g.find_layer(op.layer);
        const int L = geo[size_t(op.srcs[0])].sub;
        geo[size_t(i)].d = l.kind == LayerKind::add ? 0 : L - win(l).pad;
    }
    // shared memory
    long long bytes = 0;
    // Epilogue-written plane buffers get a plane stride of 16 (mod 128) bytes:
    // SIMT readers fetch the 8 planes of one cell from 8 different bank groups.
    auto region = [&](BRegion& r, bool skew = false) {
        const int kbs = r.row_bytes / 16;  // chunks per K-block
        if (r.mode == kPlanes) r.plane_bytes = r128(r.ext_h * r.ext_w * r.row_bytes) + (skew ? 16 : 0);
        else r.plane_bytes = (r.ext_h * r.ext_w * r.row_bytes + 1023) & ~1023;
        bytes = (bytes + 1023) & ~1023LL;  // swizzle atoms / TMA destinations
        r.smem_off = int(bytes);
        bytes += (long long)(r.chunks / kbs) * r.plane_bytes + kSlack;
    };
    // Block inputs arrive by TMA: 128-byte (SWIZZLE_128B) or 32-byte
    // (SWIZZLE_32B) boxes per cell when the channel count allows -- few, wide
    // requests -- else 16-byte planes.
    for (BIn& in : ins) {
        const int bytes_per_cell = in.r.chunks * 16;
        if (bytes_per_cell % 128 == 0) in.r.mode = kSw128, in.r.row_bytes = 128;
        else if (bytes_per_cell % 32 == 0) in.r.mode = kSw32, in.r.row_bytes = 32;
        else in.r.mode = kPlanes, in.r.row_bytes = 16;
        in.r.kb_ch = in.r.row_bytes / es;
        region(in.r);
    }
    std::vector<BRegion> bufs(static_cast<size_t>(nbufs));
    for (int i = 0; i < nops; ++i) {
        if (bufidx[size_t(i)] < 0) continue;
        BRegion& b = bufs[size_t(bufidx[size_t(i)])];
        b.chunks = rc(g.find_layer(s.ops[size_t(i)].layer)->out_shape->channels, es) / cpc;
        b.ext_h = geo[size_t(i)].ext_h, b.ext_w = geo[size_t(i)].ext_w;
        b.mode = kPlanes, b.kb_ch = cpc, b.row_bytes = 16;  // written by the epilogue threads
        region(b, true);
    }
    // N split (s.nsplit > 1): MMA-only steps whose terminal ops (stage 2 of a
    // two-stage block, else every op) split their output channels over the
    // grid's y dimension; stage-1 producers of a two-stage block are
    // recomputed by every channel group, and must not escape to HBM.
    const int nsplit = std::max(1, s.nsplit);
    bool two_stage = false;
    for (const OpSpec& op : s.ops) two_stage |= op.stage == 2;
    if (nsplit > 1) {
        for (int i = 0; i < nops; ++i) {
            const OpSpec& op = s.ops[size_t(i)];
            if (!geo[size_t(i)].mma) return -1;
            if (two_stage ? (op.stage == 1 ? op.emit : !op.emit) : !op.emit) return -1;
        }
    }
    auto split_op = [&](int i) { return nsplit > 1 && (!two_stage || s.ops[size_t(i)].stage == 2); };
    bool any_mma = false;
    int tmem = 0;
    std::vector<BOp> ops(static_cast<size_t>(nops));
    for (int i = 0; i < nops; ++i) {
        const OpSpec& os = s.ops[size_t(i)];
        const Layer& l = *g.find_layer(os.layer);
        const G& gi = geo[size_t(i)];
        BOp& o = ops[size_t(i)];
        o = BOp{};
        o.stage = os.stage, o.xin = os.xin;
        o.src = os.srcs.empty() ? -1 : bufidx[size_t(os.srcs[0])];
        o.src2 = os.srcs.size() > 1 ? bufidx[size_t(os.srcs[1])] : -1;
        o.buf = bufidx[size_t(i)];
        o.emit = os.emit, o.own_only = os.own_only;
        const TensorShape out = *l.out_shape;
        o.H = out.height, o.W = out.width, o.cout = out.channels;
        const Win w = win(l);
        o.kh = w.kh, o.kw = w.kw, o.stride = w.stride, o.pad = w.pad, o.group = 1;
        o.d = gi.d, o.ext_h = gi.ext_h, o.ext_w = gi.ext_w, o.org_mul = gi.mul, o.org_sub = gi.sub;
        o.npad = rc(out.channels, es);
        if (l.kind == LayerKind::conv) {
            o.cin = l.conv->in_channels, o.group = l.conv->group, o.relu = l.conv->activation == Activation::relu;
            if (gi.mma) {
                o.kind = BOP_MMA;
                o.contig = gi.contig;
                o.kpt = o.cin * es / 32;
                tc_nblocks(out.channels, &o.nblocks, &o.nb);
                if (split_op(i)) {  // one N block of gch channels per group
                    const int gch = r16(cdiv(r16(out.channels), nsplit));
                    if (gch > 256 || gch * (nsplit - 1) >= out.channels) return -1;  // one block per group, no empty group
                    o.nblocks = 1, o.nb = gch, o.gch = gch;
                    o.gwb = (long long)o.kh * o.kw * o.kpt * gch * 32;
                }
                o.npad = o.nblocks * o.nb;
                if (o.contig) o.strips = 1, o.mtiles = cdiv(o.ext_h * o.ext_w, 128);
                else o.strips = cdiv(o.ext_w, 8), o.mtiles = o.strips * cdiv(o.ext_h, 16);
                o.ksteps = o.kh * o.kw * o.kpt;
                o.chunk_steps = std::max(1, chunk / (o.nb * 32));
                if (!wres && chunk < o.nb * 32) return -1;  // a ring slot holds at least one K step
                if (o.mtiles * o.nb > 512) return -1;  // TMEM: 512 columns
                tmem = std::max(tmem, o.mtiles * o.nb);
                any_mma = true;
            } else {
                o.kind = BOP_SIMT_CONV;
            }
        } else if (l.kind == LayerKind::pool) {
            o.kind = l.pool->kind == PoolKind::max ? BOP_MAXPOOL : BOP_AVGPOOL;
            o.cin = out.channels;
            if (s.ctile) o.npad = s.ctile;
        } else {
            o.kind = BOP_ADD;
            o.cin = out.channels;
        }
    }
    // Groups: consecutive same-stage single-block MMA ops share one commit and
    // one epilogue pass (disjoint TMEM columns); wide ops get a group per N
    // block; SIMT ops are their own group.
    std::vector<BGroup> groups;
    int gcols = 0;
    tmem = 0;
    for (int i = 0; i < nops; ++i) {
        BOp& o = ops[size_t(i)];
        if (o.kind != BOP_MMA) {
            groups.push_back({i, i + 1, 0, 0, 0, 1, -1});
            continue;
        }
        const int cols = o.mtiles * o.nb;
        if (o.nblocks > 1) {
            // N blocks alternate between two column sets when both fit: block
            // k+1's MMAs run while the epilogue drains block k
            const bool alt = 2 * cols <= 512 && !k.no_nalt;
            for (int k = 0; k < o.nblocks; ++k) groups.push_back({i, i + 1, k, 1, alt ? (k & 1) * cols : 0, alt && k > 0 ? 2 : 1, -1});
            o.tcol = 0;
            tmem = std::max(tmem, alt ? 2 * cols : cols);
            continue;
        }
        const bool join = !groups.empty() && groups.back().mma && groups.back().op1 == i &&
                          ops[size_t(groups.back().op0)].stage == o.stage && ops[size_t(groups.back().op0)].nblocks == 1 &&
                          gcols + cols <= 512;
        if (join) {
            o.tcol = gcols;
            gcols += cols;
            groups.back().op1 = i + 1;
        } else {
            o.tcol = 0;
            gcols = cols;
            groups.push_back({i, i + 1, 0, 1, 0, 1, -1});
        }
        tmem = std::max(tmem, gcols);
    }
    if (groups.size() > size_t(kBMaxUnits)) return -1;
    // Single-block MMA groups get disjoint TMEM columns when that fits the
    // allocation they need anyway, so a group of the next tile can start
    // while a later group of this tile still drains.
    auto single = [&](const BGroup& G) { return G.mma && ops[size_t(G.op0)].nblocks == 1; };
    {
        int sum = 0;
        for (const BGroup& G : groups)
            if (single(G)) sum += ops[size_t(G.op1 - 1)].tcol + ops[size_t(G.op1 - 1)].mtiles * ops[size_t(G.op1 - 1)].nb;
        bool all_single = true;
        for (const BGroup& G : groups) all_single &= !G.mma || single(G);
        if (all_single && sum <= pow2_cols(tmem) && !k.no_tsep) {
            int base = 0;
            for (BGroup& G : groups)
                if (single(G)) G.tbase = base, base += ops[size_t(G.op1 - 1)].tcol + ops[size_t(G.op1 - 1)].mtiles * ops[size_t(G.op1 - 1)].nb;
        }
    }
    // what the issuer waits for before a tile's first groups (one accumulator set)
    auto span = [&](const BGroup& G, int& lo, int& hi) {
        lo = 1 << 30, hi = 0;
        for (int i = G.op0; i < G.op1; ++i) {
            const BOp& o = ops[size_t(i)];
            lo = std::min(lo, G.tbase + o.tcol), hi = std::max(hi, G.tbase + o.tcol + o.mtiles * o.nb);
        }
    };
    for (size_t gi = 0; gi < groups.size(); ++gi) {
        BGroup& G = groups[gi];
        G.pwait = -1;
        if (!G.mma) continue;
        int lo, hi;
        span(G, lo, hi);
        for (int j = int(groups.size()) - 1; j >= 0; --j) {
            if (!groups[size_t(j)].mma) continue;
            int l2, h2;
            span(groups[size_t(j)], l2, h2);
            if (l2 < hi && lo < h2) {
                G.pwait = k.no_pwait ? int(groups.size()) - 1 : j;
                break;
            }
        }
    }
    long long gap_off = 0;
    if (!s.gap_out.empty()) {
        if (nops != 1 || ops[0].kind != BOP_MMA) return -1;
        ops[0].gap = 1;
        gap_off = (bytes + 15) & ~15LL;
        bytes = gap_off + 4LL * ops[0].nblocks * ops[0].nb * 4;  // column sums, one slot per TMEM lane quadrant
    }
    // shared copy of the biases the epilogues read
    const long long bias_off = bytes;
    for (BOp& o : ops) {
        o.bias_smem = -1;
        if (o.kind == BOP_MMA) o.bias_smem = int(bytes), bytes += (long long)o.npad * 4;
    }
    const long long bias_bytes = bytes - bias_off;
    bytes = (bytes + 1023) & ~1023LL;
    const long long ring_off = bytes;
    long long wres_off = 0, wres_bytes = 0;
    if (any_mma && wres) {
        wres_off = bytes;
        for (BOp& o : ops)
            if (o.kind == BOP_MMA) {
                o.wofs = int(wres_bytes);
                wres_bytes += ((long long)o.nblocks * o.ksteps * o.nb * 32 + 127) & ~127LL;
            }
        bytes += wres_bytes;
    } else if (any_mma) {
        bytes += (long long)ring_slots * chunk;
    }
    // MMA A-operand reads run past their region: contiguous-M ops read whole
    // 128-row tiles, windowed ops whole 16-row x 8-column blocks shifted by
    // the taps.  The allocation must cover the furthest read of every region
    // (into whatever follows it is harmless: those rows are masked).
    auto read_end = [&](const BOp& o, const BRegion& r) -> long long {
        const long long nkb = r.chunks * 16 / r.row_bytes;
        long long last_cell;  // one past the last cell any M tile reads
        if (o.contig) last_cell = (long long)o.mtiles * 128;
        else last_cell = (long long)(o.mtiles / o.strips * 16 - 1 + o.kh - 1 + o.d) * r.ext_w + (o.strips * 8 - 1 + o.kw - 1 + o.d) + 1;
        return r.smem_off + std::max(nkb * r.plane_bytes, (nkb - 1) * r.plane_bytes + last_cell * r.row_bytes);
    };
    long long in_read = 0;  // furthest read into the input staging region
    for (const BOp& o : ops) {
        if (o.kind != BOP_MMA) continue;
        const BRegion& r = o.stage == 1 ? ins[size_t(o.xin)].r : bufs[size_t(o.src)];
        const long long e = read_end(o, r);
        bytes = std::max(bytes, e);
        if (o.stage == 1) in_read = std::max(in_read, e);
    }
    bytes = (bytes + 127) & ~127LL;
    // second staging buffer of the block inputs (they sit first, from offset 0)
    long long in_end = 0;
    for (const BIn& in : ins) in_end = std::max(in_end, (long long)in.r.smem_off + (long long)(in.r.chunks * 16 / in.r.row_bytes) * in.r.plane_bytes + kSlack);
    long long xstride = 0;
    if (nxb == 2) {
        xstride = (bytes + 1023) & ~1023LL;
        bytes = xstride + std::max(in_end, in_read);
    }
    if (tsets == 2 && (nxb != 2 || !any_mma || 2 * pow2_cols(tmem) > 512)) return -1;
    if (P) {
        std::memset(static_cast<void*>(P), 0, sizeof(BParams));
        P->nins = int(ins.size());
        for (size_t i = 0; i < ins.size(); ++i) P->in[i] = ins[i];
        P->tile_h = th, P->tile_w = tw;
        P->out_h = s.out_h, P->out_w = s.out_w;
        P->grid_h = cdiv(s.out_h, th), P->grid_w = cdiv(s.out_w, tw);
        P->nops = nops, P->nbufs = nbufs;
        for (int i = 0; i < nops; ++i) P->ops[i] = ops[size_t(i)];
        for (int i = 0; i < nbufs; ++i) P->bufs[i] = bufs[size_t(i)];
        P->ngroups = int(groups.size());
        for (size_t i = 0; i < groups.size(); ++i) P->groups[i] = groups[i];
        P->bias_off = int(bias_off), P->bias_bytes = int(bias_bytes);
        P->ring_off = int(ring_off), P->chunk_bytes = chunk, P->ring_slots = ring_slots;
        P->wres = any_mma && wres, P->wres_off = int(wres_off), P->wres_bytes = int(wres_bytes);
        P->smem_bytes = int(bytes);
        P->ctile = s.ctile;
        P->cgroups = s.ctile ? rc(g.shape_of(s.inputs[0]).channels, es) / s.ctile : 1;
        P->tmem_cols = pow2_cols(tmem);
        P->nxb = nxb, P->xstride = int(xstride);
        P->tsets = tsets;
        P->gap_off = int(gap_off);
        P->es = es;
        P->nsplit = nsplit;
        P->gap_np_total = ops[0].gap ? nsplit * ops[0].npad : ops[0].npad;
        P->pdl = k.pdl ? 1 : 0;
        P->xrel_epi = k.xrel_epi ? 1 : 0;
    }
    return bytes;
}

// Tile choice for the tensor-core kernel: memory-bound blocks, so the model is
// the bytes a CTA moves (input region incl. halo re-reads, outputs) plus a
// small MMA term, over waves of CTAs resident per SM (shared memory and TMEM).
static bool choose_tile_tc_at(const Graph& g, StepSpec& s, int batch_hint, int smem_budget, int es, const Knobs& k);

// Pool-only steps too wide for shared memory (13x13x1000 global average pool)
// are also tiled over channels (channel c in -> channel c out).
bool choose_tile_tc(const Graph& g, StepSpec& s, int batch_hint, int smem_budget, int es, const Knobs& k) {
    s.ctile = 0;
    if (choose_tile_tc_at(g, s, batch_hint, smem_budget, es, k)) return true;
    bool pools = s.inputs.size() == 1;
    for (const OpSpec& op : s.ops) pools &= op.stage == 1 && g.find_layer(op.layer)->kind == LayerKind::pool;
    if (!pools) return false;
    const int cpc = 16 / es, C = rc(g.shape_of(s.inputs[0]).channels, es);
    for (int ct = C - cpc; ct >= cpc; ct -= cpc) {
        if (C % ct) continue;
        s.ctile = ct;
        if (choose_tile_tc_at(g, s, batch_hint, smem_budget, es, k)) return true;
    }
    s.ctile = 0;
    return false;
}

// Every feasible configuration of a step, scored by the model below (SM
// cycles, lower is better), best first.
//
// Persistent CTAs (kernels_tc.cu): each walks tiles; with two staging
// buffers (nxb = 2) the next tile's inputs load while this one computes.
// Model: a tile costs load (its input region incl. halo at the per-SM HBM
// share, ~24 B/cycle) + compute (MMA, SIMT, weights streamed through the ring
// at ring-bytes per ~2000-cycle L2 round trip, fixed per-unit sync/epilogue
// latency); nxb = 2 hides the load behind the compute.  `occ` CTAs per SM
// overlap; HBM bounds the total.  The model only ranks candidates: the engine
// autotuner (Engine::autotune) measures the top ones on the device.
std::vector<BCandidate> candidates_tc(const Graph& g, const StepSpec& s, int batch_hint, int smem_budget, int es, const Knobs& k) {
    const int force = k.xbuf, force_w = k.wres;
    struct WMode {
        int wres, slots, chunk;
    };
    // weights resident, or a ring of `slots` x `chunk` bytes (bytes in flight
    // per L2 round trip; larger chunks amortise the per-copy latency)
    const WMode wmodes[] = {{1, 3, kChunkBytes}, {0, 3, kChunkBytes}, {0, 6, kChunkBytes}, {0, 8, kChunkBytes},
                            {0, 3, 2 * kChunkBytes}, {0, 4, 2 * kChunkBytes}, {0, 2, 4 * kChunkBytes}, {0, 3, 4 * kChunkBytes}};
    std::vector<BCandidate> out;
    int fh = 0, fw = 0;
    const bool forced = k.forced_tile(s, &fh, &fw);  // a reference plan's geometry
    BParams* P = new BParams;
    // channel-group counts this step can split into (1 = no split)
    std::vector<int> splits{1};
    for (int ns : {2, 4, 8}) {
        StepSpec t = s;
        t.nsplit = ns;
        if (layout_tc(g, t, 1, 1, nullptr, 1, 1, 3, 1, kChunkBytes, es, k) >= 0 ||
            layout_tc(g, t, std::min(s.out_h, 8), std::min(s.out_w, 8), nullptr, 1, 0, 3, 1, 4 * kChunkBytes, es, k) >= 0)
            splits.push_back(ns);
    }
    StepSpec sv = s;
    for (int ns : splits)
    for (int ew : {8, 4})
    for (int ts = 1; ts <= 2; ++ts)
    for (int nxb = ts; nxb <= 2; ++nxb)
        for (const WMode& wm : wmodes) {
            // channel groups exist to keep a group's weights resident: with a
            // split, only resident weights and the shallowest ring are tried
            if (ns > 1 && !wm.wres && (wm.slots != 3 || wm.chunk != kChunkBytes)) continue;
            sv.nsplit = ns;
            for (int th = 1; th <= (forced ? fh : std::min(s.out_h, 32)); ++th)
                for (int tw = 1; tw <= (forced ? fw : std::min(s.out_w, 32)); ++tw) {
                    if (forced && (fh % th || fw % tw)) continue;  // the plan's tile or an exact sub-tile
                    const long long sm = layout_tc(g, sv, th, tw, P, nxb, wm.wres, wm.slots, ts, wm.chunk, es, k);
                    if (sm < 0 || sm > smem_budget) continue;
                    if (wm.wres && !P->wres) continue;  // no MMA op: the ring/resident choice is moot
                    double in_bytes = 0, mma = 0, simt = 0;
                    for (int i = 0; i < P->nins; ++i) in_bytes += double(P->in[i].r.chunks) * P->in[i].r.ext_h * P->in[i].r.ext_w * 16;
                    for (int i = 0; i < P->nops; ++i) {
                        const BOp& o = P->ops[i];
                        if (o.kind == BOP_MMA) mma += double(o.mtiles) * 128 * o.nblocks * o.nb * o.ksteps * 16;
                        else simt += double(o.ext_h) * o.ext_w * o.npad * o.kh * o.kw * (o.kind == BOP_SIMT_CONV ? o.cin : 1);
                    }
                    double out_bytes = 0;
                    for (int i = 0; i < P->nops; ++i)
                        if (P->ops[i].emit) out_bytes += double(th) * tw * P->ops[i].npad * es;
                    const double tiles = double(P->grid_h) * P->grid_w * P->cgroups * std::max(batch_hint, 1) * ns;
                    // 228 KB per SM; per CTA: dynamic + static (~4 KB) + 1 KB driver reserve
                    int occ = std::max(1, std::min(max_ctas_per_sm(ew), int((228 * 1024) / (sm + 5120))));
                    if (P->tmem_cols) occ = std::min(occ, 512 / (P->tmem_cols * ts));
                    double wbytes = 0;  // weights each tile streams from L2 through the ring
                    for (int i = 0; i < P->nops; ++i)
                        if (P->ops[i].kind == BOP_MMA) wbytes += double(P->ops[i].nblocks) * P->ops[i].ksteps * P->ops[i].nb * 32;
                    const double wcost = P->wres ? 0.0 : wbytes * 2000.0 / (double(wm.slots) * wm.chunk);
                    const double load = in_bytes / 24.0 + 1000.0;
                    // epilogue / SIMT work spreads over the epilogue warps
                    const double compute = out_bytes / 48.0 + wcost + mma / 8192.0 + simt / 128.0 * (8.0 / ew) + 800.0 * P->ngroups;
                    // two accumulator sets hide the MMA time behind the previous tile's epilogue
                    const double per_tile = (nxb == 2 ? std::max(load, compute) : load + compute) - (ts == 2 ? mma / 8192.0 : 0.0);
                    const double t = std::max(std::ceil(tiles / (148.0 * occ)) * per_tile,
                                              tiles * (in_bytes + out_bytes) / (148.0 * 24.0));
                    out.push_back({th, tw, nxb, P->wres, wm.slots, int(sm), ew, ts, wm.chunk, t, ns});
                }
        }
    delete P;
    // testing aids (options xbuf / wres / tsets): keep only the matching
    // configurations when any exists for this step
    auto prefer = [&](auto pred) {
        std::vector<BCandidate> keep;
        for (const BCandidate& c : out)
            if (pred(c)) keep.push_back(c);
        if (!keep.empty()) out.swap(keep);
    };
    if (force) prefer([&](const BCandidate& c) { return c.nxb == force; });
    if (force_w >= 0) prefer([&](const BCandidate& c) { return c.wres == force_w; });
    if (k.tsets) prefer([&](const BCandidate& c) { return c.tsets == k.tsets; });
    if (k.nsplit) prefer([&](const BCandidate& c) { return c.nsplit == k.nsplit; });
    std::stable_sort(out.begin(), out.end(), [](const BCandidate& a, const BCandidate& b) {
        if (a.model < b.model * 0.999) return true;
        if (b.model < a.model * 0.999) return false;
        return long(a.th) * a.tw > long(b.th) * b.tw;  // ties: the larger tile
    });
    if (forced && !out.empty()) {  // the plan's tile, else its largest feasible sub-tile (any staging / weight mode)
        long best = 0;
        for (const BCandidate& c : out) best = std::max(best, long(c.th) * c.tw);
        std::vector<BCandidate> keep;
        for (const BCandidate& c : out)
            if (long(c.th) * c.tw == best) keep.push_back(c);
        out.swap(keep);
    }
    return out;
}

static bool choose_tile_tc_at(const Graph& g, StepSpec& s, int batch_hint, int smem_budget, int es, const Knobs& k) {
    const std::vector<BCandidate> c = candidates_tc(g, s, batch_hint, smem_budget, es, k);
    if (c.empty()) return false;
    apply_candidate(s, c.front());
    return true;
}

void apply_candidate(StepSpec& s, const BCandidate& c) {
    s.tile_h = c.th, s.tile_w = c.tw, s.smem_bytes = c.smem, s.nxb = c.nxb, s.wres = c.wres, s.ring_slots = c.slots;
    s.epi_warps = c.epi_warps, s.tsets = c.tsets, s.ring_chunk = c.chunk, s.nsplit = c.nsplit;
}

// Weights of every MMA-eligible conv as the UMMA K-major B operand of each
// 32-byte K step: [nblock][tap][cin/cpc][nb][cpc] elements, bf16 (RN even) or
// fp32 rounded to TF32 (RN, ties away -- the rounding the TF32 epilogue
// applies to activations).  `off`: byte offset per layer.
namespace {
void put_tc(std::vector<uint8_t>& out, size_t byte, float f, int es) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if (es == 2) {
        u += 0x7FFF + ((u >> 16) & 1);  // round to nearest even
        const uint16_t h = uint16_t(u >> 16);
        std::memcpy(&out[byte], &h, 2);
    } else {
        if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & ~0x1FFFu;  // TF32: 10 mantissa bits, ties away
        std::memcpy(&out[byte], &u, 4);
    }
}

// Appends layer l's packed weights (nblocks x nb columns) read from w (its
// filter [oc][ic][kh][kw]) to out.
void pack_conv_tc(std::vector<uint8_t>& out, const ConvParams& c, const float* w, int es, int nblocks, int nb) {
    const int cpc = 16 / es;
    const int kpt = c.in_channels * es / 32, taps = c.kernel_h * c.kernel_w, ksteps = taps * kpt;
    const size_t base = out.size();
    out.resize(base + size_t(nblocks) * ksteps * nb * 32, 0);
    for (int oc = 0; oc < c.out_channels; ++oc)
        for (int ic = 0; ic < c.in_channels; ++ic)
            for (int y = 0; y < c.kernel_h; ++y)
                for (int x = 0; x < c.kernel_w; ++x) {
                    const int nbi = oc / nb, n = oc - nbi * nb, tap = y * c.kernel_w + x;
                    const int step = tap * kpt + ic / (2 * cpc), half = (ic % (2 * cpc)) / cpc;
                    const size_t el = ((size_t(nbi) * ksteps + step) * 2 + half) * nb * cpc + size_t(n) * cpc + ic % cpc;
                    put_tc(out, base + el * es, w[((size_t(oc) * c.in_channels + ic) * c.kernel_h + y) * c.kernel_w + x], es);
                }
}
}  // namespace

std::vector<uint8_t> pack_weights_tc(const Graph& g, const float* flat, size_t count, std::map<std::string, long long>& off, int es) {
    std::vector<uint8_t> out;
    size_t pos = 0;
    for (const Layer& l : g.layers) {
        if (l.kind != LayerKind::conv) continue;
        const ConvParams& c = *l.conv;
        const size_t nf = size_t(c.weight_count()), nb_ = size_t(c.bias_count());
        if (pos + nf + nb_ > count) fail(ErrorKind::validation, "weights: stream too short for layer '" + l.name + "'");
        if (tc_mma_ok(l, es)) {
            int nblocks, nb;
            tc_nblocks(c.out_channels, &nblocks, &nb);
            off[l.name] = (long long)out.size();
            pack_conv_tc(out, c, flat + pos, es, nblocks, nb);
        }
        pos += nf + nb_;
    }
    return out;
}

std::vector<uint8_t> pack_layer_tc(const Graph& g, const std::string& layer, const float* flat, size_t count, int es, int nb, int nblocks) {
    size_t pos = 0;
    for (const Layer& l : g.layers) {
        if (l.kind != LayerKind::conv) continue;
        const size_t n = size_t(l.conv->weight_count() + l.conv->bias_count());
        if (l.name == layer) {
            if (pos + n > count || !tc_mma_ok(l, es) || nblocks * nb < l.conv->out_channels)
                fail(ErrorKind::internal, "pack_layer_tc: cannot pack '" + layer + "'");
            std::vector<uint8_t> out;
            pack_conv_tc(out, *l.conv, flat + pos, es, nblocks, nb);
            return out;
        }
        pos += n;
    }
    fail(ErrorKind::internal, "pack_layer_tc: no conv '" + layer + "'");
}

}  // namespace xlf
