// Tensor-core fused-block kernel for sm_100a (tcgen05 + TMEM + TMA), for two
// element types (template parameter T): bf16 (tcgen05.mma kind::f16) and
// fp32 storage carrying TF32 values (kind::tf32).  All shared-memory layouts
// and UMMA descriptors are in 16-byte chunks / 32-byte K steps, identical for
// both types; T changes the MMA kind, the chunk's channel count (8 / 4) and
// the epilogue's conversion (bf16 RN / TF32 RNA).
//
// Persistent: grid = 148 x (resident CTAs per SM), capped by the tile count;
// CTA b walks tiles b, b + gridDim.x, ... (tile = image x channel group x
// output tile).  352 threads in four roles:
//   warp E      input producer: TMA of the block inputs (one 4-D box per
//               K-block, zero fill outside the image = conv padding) into
//               staging buffer k % nxb; with nxb = 2 tile k+1's inputs load
//               while tile k computes;
//   warp 10     weight producer: cp.async.bulk of the packed weights through a
//               3-slot ring (full/empty mbarriers), running ahead across tiles;
//   warp 9      MMA issuer: one thread issues tcgen05.mma (M=128, N<=256,
//               one 32-byte K step, bf16 or TF32 -> fp32 in TMEM) for every conv "unit"
//               (op x N block), commits to the ring and to the unit's
//               accumulator barrier; the warp owns TMEM alloc/dealloc (once);
//   warps 0-7   epilogue + SIMT ops: tcgen05.ld the accumulator (lane = GEMM
//               row = output cell), bias + ReLU + halo mask, bf16 / TF32, and either
//               keep it on chip (shared "planes" buffer that the next stage's
//               MMAs read with shifted descriptors) or store NHWC to HBM at
//               the concat channel offset.  Pools / stride-2 convs / adds run
//               here as SIMT code on the same shared planes.
// Units execute in order; the issuer starts unit u only after every earlier
// unit's epilogue signalled (its TMEM columns are free and any buffer it
// reads is written); every per-tile barrier flips phase once per tile.
// Barrier init, TMEM allocation, the descriptor and bias copies happen once
// per CTA, not per tile.  See tc_params.hpp for the shared-memory layout.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "tc_params.hpp"
#include "umma.cuh"

namespace xlf {

namespace {

using namespace umma;

// Element traits: channels per 16-byte chunk, conversions, the MMA kind.
template <class T>
struct Elem;

template <>
struct Elem<__nv_bfloat16> {
    static constexpr int cpc = 8;
    static constexpr uint32_t idesc(int M, int N) { return idesc_bf16(M, N); }
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_bf16(t, a, b, id, acc); }
    __device__ static float rnd(float x) { return x; }  // rounding happens in pack()
    __device__ static __nv_bfloat16 from(float x) { return __float2bfloat16(x); }
    __device__ static float to(__nv_bfloat16 x) { return __bfloat162float(x); }
    // v[0..7] -> one chunk
    __device__ static uint4 pack(const float* v) {
        uint4 u;
        __nv_bfloat162 h;
        h = __floats2bfloat162_rn(v[0], v[1]), u.x = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[2], v[3]), u.y = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[4], v[5]), u.z = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[6], v[7]), u.w = *reinterpret_cast<uint32_t*>(&h);
        return u;
    }
    __device__ static void unpack(uint4 u, float* f) {
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[q]));
            f[2 * q] = p.x, f[2 * q + 1] = p.y;
        }
    }
    __device__ static uint32_t max2(uint32_t a, uint32_t b) {
        __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a), y = *reinterpret_cast<__nv_bfloat162*>(&b);
        __nv_bfloat162 m = __hmax2(x, y);
        return *reinterpret_cast<uint32_t*>(&m);
    }
    __device__ static uint4 vmax(uint4 a, uint4 b) { return make_uint4(max2(a.x, b.x), max2(a.y, b.y), max2(a.z, b.z), max2(a.w, b.w)); }
};

template <>
struct Elem<float> {
    static constexpr int cpc = 4;
    static constexpr uint32_t idesc(int M, int N) { return idesc_tf32(M, N); }
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_tf32(t, a, b, id, acc); }
    __device__ static float rnd(float x) { return round_tf32(x); }
    __device__ static float from(float x) { return round_tf32(x); }
    __device__ static float to(float x) { return x; }
    // v[0..3] -> one chunk (TF32-rounded)
    __device__ static uint4 pack(const float* v) {
        return make_uint4(__float_as_uint(round_tf32(v[0])), __float_as_uint(round_tf32(v[1])), __float_as_uint(round_tf32(v[2])),
                          __float_as_uint(round_tf32(v[3])));
    }
    __device__ static void unpack(uint4 u, float* f) {
        f[0] = __uint_as_float(u.x), f[1] = __uint_as_float(u.y), f[2] = __uint_as_float(u.z), f[3] = __uint_as_float(u.w);
    }
    __device__ static uint32_t max1(uint32_t a, uint32_t b) { return __float_as_uint(fmaxf(__uint_as_float(a), __uint_as_float(b))); }
    __device__ static uint4 vmax(uint4 a, uint4 b) { return make_uint4(max1(a.x, b.x), max1(a.y, b.y), max1(a.z, b.z), max1(a.w, b.w)); }
};

// CTA shape, a template parameter of the kernel (the tuner picks per step):
// EW epilogue/SIMT warps (4 or 8), then the input producer, MMA issuer and
// weight producer warps.  Fewer epilogue warps -> fewer registers per CTA ->
// more CTAs (more independent tile chains) per SM.
constexpr int kSubs = 4;  // accumulator-ready barriers per group (per op, the last shared by the rest)

template <int EW>
struct Cta {
    static constexpr int compute = EW * 32;        // warps 0..EW-1: epilogue + SIMT ops
    static constexpr int threads = compute + 96;
    static constexpr int wx = EW, wmma = EW + 1, ww = EW + 2;
    static constexpr int halves = compute / 128;   // epilogue warp groups splitting the accumulator columns
    static constexpr int min_blocks = EW <= 4 ? 4 : 2;
};

struct BTile {
    int n, ty, tx, oy0, ox0, c0;
};

// Trace stamps of the first tile of CTAs 0..kTraceCtas-1 (k = tile ordinal of the CTA).
__device__ __forceinline__ void stamp(const BParams& P, int ev, int k = 0) {
    if (blockIdx.y != 0) return;
    if (P.trace && P.trace_tiles && ev == kTrEnd && k < kTraceEvents && blockIdx.x < kTraceCtas) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.trace[blockIdx.x * kTraceEvents + k] = t;
        return;
    }
    if (P.trace && !P.trace_tiles && k == 2 && blockIdx.x < kTraceCtas && ev < kTraceEvents) {  // a steady-state tile
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.trace[blockIdx.x * kTraceEvents + ev] = t;
    }
}

// Programmatic dependent launch: a step's CTAs start (barriers, TMEM, the
// descriptor and resident weights) while the previous step drains; reads of
// the previous step's outputs wait here.
__device__ __forceinline__ void grid_dependency_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <int EW>
__device__ __forceinline__ void named_sync_compute() { asm volatile("bar.sync 1, %0;\n" ::"n"(Cta<EW>::compute) : "memory"); }

// Epilogue-side wait: ONE thread polls the mbarrier, the other compute warps
// block in a hardware named barrier (no issue slots).  Eight warps polling a
// try_wait loop issued a third of all instructions of the kernel and starved
// the co-resident CTA's epilogue (ncu, profiles/r1_ncu_summary.md).
template <int EW>
__device__ __forceinline__ void compute_wait(uint64_t* bar, uint32_t parity) {
#ifdef XLF_WAIT_CTA
    if (threadIdx.x == 0) mbar_sleep_wait(bar, parity);
    named_sync_compute<EW>();
#else
    // every epilogue thread observes the phase itself: warps start on an
    // accumulator as soon as it is ready, without a CTA-wide barrier
    mbar_sleep_wait(bar, parity);
#endif
}

__device__ __forceinline__ const BRegion& src_region(const BParams& P, const BOp& op, int which) {
    return op.stage == 1 ? P.in[op.xin].r : P.bufs[which];
}

// The region an op reads, with a stage-1 (block input) region moved to the
// staging buffer of the current tile.
__device__ __forceinline__ BRegion src_region_at(const BParams& P, const BOp& op, int which, int xdelta) {
    BRegion R = src_region(P, op, which);
    if (op.stage == 1) R.smem_off += xdelta;
    return R;
}

// Tile tau of the persistent walk: image-major, then channel group, rows, columns.
__device__ __forceinline__ BTile tile_at(const BParams& P, int tau, int n0) {
    const int per_img = P.grid_h * P.grid_w * P.cgroups, per_cg = P.grid_h * P.grid_w;
    BTile t;
    const int ni = tau / per_img;
    int r = tau - ni * per_img;
    t.n = n0 + ni;  // absolute image (a launch may cover images [n0, n0 + batch))
    const int cg = r / per_cg;
    r -= cg * per_cg;
    t.ty = r / P.grid_w;
    t.tx = r - t.ty * P.grid_w;
    t.oy0 = t.ty * P.tile_h;
    t.ox0 = t.tx * P.tile_w;
    t.c0 = cg * P.ctile;
    return t;
}

// The persistent walk tau = blockIdx.x, +gridDim.x, ... decoded incrementally:
// tau and the stride are split once into mixed-radix digits (image, channel
// group, tile row, tile column) and each step adds the stride's digits with
// carries -- no integer division per tile.
struct TileWalk {
    int n, cg, ty, tx;      // current tile (n relative to n0)
    int dn, dcg, dty, dtx;  // digits of gridDim.x
    __device__ __forceinline__ void split(const BParams& P, int v, int& a, int& b, int& c, int& d) const {
        const int per_cg = P.grid_h * P.grid_w, per_img = per_cg * P.cgroups;
        a = v / per_img, v -= a * per_img;
        b = v / per_cg, v -= b * per_cg;
        c = v / P.grid_w, d = v - c * P.grid_w;
    }
    __device__ __forceinline__ void init(const BParams& P) {
        split(P, int(blockIdx.x), n, cg, ty, tx);
        split(P, int(gridDim.x), dn, dcg, dty, dtx);
    }
    __device__ __forceinline__ void next(const BParams& P) {
        tx += dtx, ty += dty, cg += dcg, n += dn;
        if (tx >= P.grid_w) tx -= P.grid_w, ++ty;
        if (ty >= P.grid_h) ty -= P.grid_h, ++cg;
        if (cg >= P.cgroups) cg -= P.cgroups, ++n;
    }
    __device__ __forceinline__ BTile tile(const BParams& P, int n0) const {
        BTile t;
        t.n = n0 + n, t.ty = ty, t.tx = tx;
        t.oy0 = ty * P.tile_h, t.ox0 = tx * P.tile_w, t.c0 = cg * P.ctile;
        return t;
    }
};

// Last group whose MMAs read the staging buffer, when only MMAs read it (no
// SIMT group): the issuer then releases the buffer with a tcgen05.commit
// right after that group, so the next tile's input load overlaps the rest of
// this tile (expand MMAs, epilogues).  -1: the epilogue warps release it after
// the tile (SIMT ops read the staged input).
__device__ __forceinline__ int x_release_group(const BParams& P) {
    if (P.xrel_epi) return -1;
    int last = -1;
    for (int gi = 0; gi < P.ngroups; ++gi) {
        const BGroup& G = P.groups[gi];
        if (!G.mma) return -1;
        for (int i = G.op0; i < G.op1; ++i)
            if (P.ops[i].stage == 1) last = gi;
    }
    return last;
}

// ------------------------------------------------------------------ producers

// Block inputs of every tile of this CTA into staging buffer k % nxb; a buffer
// is refilled once it is released (x_free: the MMAs that read it completed, or
// the epilogue finished the tile; see x_release_group).
__device__ void x_producer(const BParams& P, const CUtensorMap* xmaps, uint8_t* smem, int total, int n0, uint64_t* bar_x,
                           uint64_t* x_free) {
    uint32_t bytes = 0;
    for (int k = 0; k < P.nins; ++k) bytes += uint32_t(P.in[k].r.chunks) * uint32_t(P.in[k].r.ext_h * P.in[k].r.ext_w * 16);
    const int nxb = P.nxb;
    int k = 0;
    grid_dependency_wait();  // the previous step's outputs are this step's inputs
    TileWalk tw;
    tw.init(P);
    for (int tau = blockIdx.x; tau < total; tau += gridDim.x, ++k, tw.next(P)) {
        const BTile t = tw.tile(P, n0);
        const int b = nxb == 2 ? (k & 1) : 0, use = nxb == 2 ? (k >> 1) : k;
        if (use > 0) mbar_sleep_wait(&x_free[b], (use - 1) & 1);
        stamp(P, kTrStart, k);
        mbar_expect_tx(&bar_x[b], bytes);
        uint8_t* xb = smem + b * P.xstride;
        for (int i = 0; i < P.nins; ++i) {
            const BIn& in = P.in[i];
            const int x0 = t.ox0 * in.org_mul - in.org_sub, y0 = t.oy0 * in.org_mul - in.org_sub;
            const int nkb = in.r.chunks * 16 / in.r.row_bytes;
            for (int kb = 0; kb < nkb; ++kb)
                tma_load_4d(xb + in.r.smem_off + kb * in.r.plane_bytes, &xmaps[i], in.coff + t.c0 + kb * in.r.kb_ch, x0, y0, t.n,
                            &bar_x[b]);
        }
        stamp(P, kTrXIssued, k);
    }
}

// Weights, in exactly the order the issuer consumes them, tile after tile
// (the ring runs ahead into the next tile while this one's epilogue runs).
__device__ void w_producer(const BParams& P, uint8_t* smem, int total, uint64_t* ring_full, uint64_t* ring_empty, uint64_t* bar_w) {
    if (P.wres) {  // resident: every op's packed weights once, then done
        uint32_t total_b = 0;
        for (int i = 0; i < P.nops; ++i)
            if (P.ops[i].kind == BOP_MMA) total_b += uint32_t(P.ops[i].nblocks * P.ops[i].ksteps * P.ops[i].nb * 32);
        mbar_expect_tx(bar_w, total_b);
        for (int i = 0; i < P.nops; ++i) {
            const BOp& op = P.ops[i];
            if (op.kind != BOP_MMA) continue;
            const uint32_t b = uint32_t(op.nblocks * op.ksteps * op.nb * 32);
            const uint8_t* src = op.wmma + (op.gch ? op.gwb * blockIdx.y : 0);  // this CTA row's channel group
            for (uint32_t o = 0; o < b; o += 65536)  // pieces of <= 64 KB
                bulk_g2s(smem + P.wres_off + op.wofs + o, src + o, min(65536u, b - o), bar_w);
        }
        return;
    }
    const int slots = P.ring_slots;
    int c = 0;
    for (int tau = blockIdx.x; tau < total; tau += gridDim.x) {
        for (int gi = 0; gi < P.ngroups; ++gi) {
            const BGroup& G = P.groups[gi];
            if (!G.mma) continue;
            for (int i = G.op0; i < G.op1; ++i) {
                const BOp& op = P.ops[i];
                const uint8_t* wb = op.wmma + (op.gch ? op.gwb * blockIdx.y : 0) + size_t(G.nbi) * op.ksteps * op.nb * 32;
                for (int s0 = 0; s0 < op.ksteps; s0 += op.chunk_steps, ++c) {
                    const int steps = min(op.chunk_steps, op.ksteps - s0);
                    const int slot = c % slots;
                    if (c >= slots) mbar_sleep_wait(&ring_empty[slot], ((c / slots) - 1) & 1);
                    const uint32_t b = uint32_t(steps) * op.nb * 32;
                    mbar_expect_tx(&ring_full[slot], b);
                    bulk_g2s(smem + P.ring_off + slot * P.chunk_bytes, wb + size_t(s0) * op.nb * 32, b, &ring_full[slot]);
                }
            }
        }
    }
}

// ------------------------------------------------------------------ MMA issuer

// All MMAs of one op (one N block): K steps in tap-major order (s = tap*c16
// + kc, the packing order of the weights), every M tile per step.  Every op
// field is hoisted into locals first and the descriptors are advanced by
// precomputed deltas (in 16-byte units of the start-address field), so one MMA
// costs a handful of uniform-datapath instructions.
template <class T>
__device__ __forceinline__ void issue_op(const BParams& P, const BOp& op, int nbi, uint32_t sbase, uint32_t tmem, int& c,
                                         uint64_t* ring_full, uint64_t* ring_empty, int xdelta) {
    const BRegion R = src_region_at(P, op, op.src, xdelta);
    const int mode = R.mode, plane = R.plane_bytes, rowb = R.row_bytes, ew = R.ext_w;
    const int ksteps = op.ksteps, csteps = op.chunk_steps, nb = op.nb, mtiles = op.mtiles, strips = op.strips;
    const int kw = op.kw, d = op.d, contig = op.contig, c16 = op.kpt;
    const uint32_t idesc = Elem<T>::idesc(128, nb);
    uint32_t lbo, layout;
    if (mode == kPlanes) lbo = plane, layout = kNoSwizzle;
    else lbo = 16, layout = mode == kSw32 ? kSW32 : kSW128;
    const uint32_t sbo = contig ? 8 * rowb : ew * rowb;
    const uint64_t bdesc0 = sdesc(0, nb * 16, 128, kNoSwizzle);
    const uint32_t ring0 = sbase + P.ring_off, chunkb = P.chunk_bytes;
    const int slots = P.ring_slots, wres = P.wres;
    const uint32_t wbase = sbase + P.wres_off + op.wofs + uint32_t(nbi * ksteps * nb * 32);
    // start-field deltas (16-byte units)
    const uint32_t d_mt = contig ? (128 * rowb) >> 4 : (8 * rowb) >> 4;       // next M tile / next strip
    const uint32_t d_rb = ((16 * ew - 8 * (strips - 1)) * rowb) >> 4;          // last strip -> next 16-row block
    const uint32_t d_dx = rowb >> 4, d_row = ((ew - kw) * rowb) >> 4;          // next tap column / next tap row
    uint64_t a_tap = sdesc(sbase + R.smem_off + (contig ? 0 : (d * ew + d) * rowb), lbo, sbo, layout);
    const uint32_t tm0 = tmem + op.tcol;
    int kc = 0, dx = 0;
    uint32_t acc = 0;
    for (int s0 = 0; s0 < ksteps; s0 += csteps) {
        const int steps = min(csteps, ksteps - s0);
        const int slot = wres ? 0 : c % slots;
        uint64_t bd;
        if (wres) {
            bd = bdesc0 + ((wbase + uint32_t(s0 * nb * 32)) >> 4);
        } else {
            mbar_wait(&ring_full[slot], (c / slots) & 1);
            fence_after();
            bd = bdesc0 + ((ring0 + slot * chunkb) >> 4);
        }
        for (int sl = 0; sl < steps; ++sl) {
            uint32_t kofs;  // 32-byte K step kc inside the region's K-blocks, 16-byte units
            if (mode == kPlanes) kofs = (kc * 2 * plane) >> 4;
            else if (mode == kSw32) kofs = (kc * plane) >> 4;
            else kofs = (((kc >> 2) * plane) >> 4) + (kc & 3) * 2;
            uint64_t a = a_tap + kofs;
            uint32_t tcur = tm0;
            int st = 0;
            for (int mt = 0; mt < mtiles; ++mt) {
                Elem<T>::mma(tcur, a, bd, idesc, acc);
                tcur += nb;
                if (contig || ++st < strips) a += d_mt;
                else st = 0, a += d_rb;
            }
            acc = 1;
            bd += (nb * 32) >> 4;
            if (++kc == c16) {
                kc = 0;
                a_tap += d_dx;
                if (++dx == kw) dx = 0, a_tap += d_row;
            }
        }
        if (!wres) commit(&ring_empty[slot]), ++c;
    }
}

template <class T>
__device__ void issuer(const BParams& P, uint8_t* smem, uint32_t tmem, int total, uint64_t* bar_x, uint64_t* x_free, uint64_t* ring_full,
                       uint64_t* ring_empty, uint64_t* acc_full, uint64_t* unit_done, uint64_t* acc_free, uint64_t* bar_w) {
    int c = 0, k = 0;
    const uint32_t sbase = smem_u32(smem);
    const int G = P.ngroups, nxb = P.nxb;
    // SIMT-only steps: nothing to issue, and the epilogue (not gated by any
    // accumulator) may run tiles ahead, so the issuer must not track phases.
    bool any = false;
    for (int gi = 0; gi < G; ++gi) any |= P.groups[gi].mma != 0;
    if (!any) return;
    if (P.wres) mbar_sleep_wait(bar_w, 0);
    const int ts = P.tsets;
    const int xrel = x_release_group(P);
    for (int tau = blockIdx.x; tau < total; tau += gridDim.x, ++k) {
        const int b = nxb == 2 ? (k & 1) : 0, use = nxb == 2 ? (k >> 1) : k;
        const int xdelta = b * P.xstride;
        // accumulator set: with two sets the issuer runs one tile ahead --
        // tile k+1's MMAs overlap tile k's epilogue
        const int s = ts == 2 ? (k & 1) : 0, j = ts == 2 ? (k >> 1) : k;
        uint64_t* ud = unit_done + s * kBMaxUnits;
        mbar_sleep_wait(&bar_x[b], use & 1);
        stamp(P, kTrXLanded, k);
        if (ts == 2) {
            if (j > 0) mbar_sleep_wait(&acc_free[s], (j - 1) & 1);  // tile k-2 (same set) fully done
        }
        for (int gi = 0; gi < G; ++gi) {
            // earlier units' epilogues done, in order; with one set, a tile's
            // first units wait for the previous tile's last unit on their TMEM
            // columns (pwait: with disjoint group columns the next tile's
            // first group starts while this tile's later groups drain)
            if (gi >= P.groups[gi].wback) mbar_sleep_wait(&ud[gi - P.groups[gi].wback], j & 1);
            else if (ts == 1 && k > 0 && P.groups[gi].pwait >= 0) mbar_sleep_wait(&ud[P.groups[gi].pwait], (k - 1) & 1);
            const BGroup& Gr = P.groups[gi];
            if (!Gr.mma) continue;
            fence_after();
            if (gi < 2) stamp(P, 29 + 2 * gi, k);  // group's inputs ready, issue starts
            // one commit per op of the group (the first kSubs-1 ops, then one
            // for the rest): the epilogue starts on an op while the group's
            // later ops are still on the tensor cores
            uint64_t* fb = acc_full + (s * kBMaxUnits + gi) * kSubs;
            for (int i = Gr.op0; i < Gr.op1; ++i) {
                issue_op<T>(P, P.ops[i], Gr.nbi, sbase, tmem + uint32_t(s * P.tmem_cols + Gr.tbase), c, ring_full, ring_empty, xdelta);
                const int sub = i - Gr.op0;
                if (sub < kSubs - 1 || i == Gr.op1 - 1) commit(&fb[sub < kSubs - 1 ? sub : kSubs - 1]);
            }
            if (gi == xrel) commit(&x_free[b]);      // staging buffer read by every MMA that needs it
            if (gi < 2) stamp(P, 30 + 2 * gi, k);  // group issued
        }
    }
}

// ------------------------------------------------------------------ epilogue / SIMT

// Register copy of everything an epilogue / SIMT op needs from the (shared)
// descriptor.  Epilogues store to shared memory, so the compiler cannot cache
// descriptor fields read from shared memory across those stores; hoisting
// them once per op avoids a dependent shared load per field per channel.
template <class T>
struct EpiOp {
    int relu, cend, emit, own_only, gap, gap_np;  // cend: output channels rounded up to a chunk
    int org_mul, org_sub, H, W, out_cstride, out_coff;
    int tile_h, tile_w, grid_h, grid_w;
    int buf_ew, buf_plane;
    uint8_t* buf;           // shared buffer base (planes), or null
    T* out;
    uint32_t bias_s;        // shared address of the op's fp32 bias (MMA ops)
    const float* bias_p;    // the same, as a generic pointer
};

template <class T>
__device__ __forceinline__ EpiOp<T> epi_op(const BParams& P, const BOp& op, uint8_t* smem) {
    constexpr int cpc = Elem<T>::cpc;
    EpiOp<T> e;
    e.relu = op.relu, e.cend = (op.cout + cpc - 1) / cpc * cpc, e.emit = op.emit, e.own_only = op.own_only, e.gap = op.gap;
    e.gap_np = op.gap ? op.nblocks * op.nb : 0;
    e.org_mul = op.org_mul, e.org_sub = op.org_sub, e.H = op.H, e.W = op.W;
    e.out_cstride = op.out_cstride, e.out_coff = op.out_coff;
    if (op.gch) {  // channel group blockIdx.y: channels [g*gch, g*gch + gch) stored at their offset
        const int g0 = int(blockIdx.y) * op.gch;
        e.out_coff += g0;
        e.cend = max(0, min(op.gch, e.cend - g0));
    }
    e.tile_h = P.tile_h, e.tile_w = P.tile_w, e.grid_h = P.grid_h, e.grid_w = P.grid_w;
    e.buf = nullptr, e.buf_ew = 0, e.buf_plane = 0;
    if (op.buf >= 0) {
        const BRegion& B = P.bufs[op.buf];
        e.buf = smem + B.smem_off, e.buf_ew = B.ext_w, e.buf_plane = B.plane_bytes;
    }
    e.out = static_cast<T*>(op.out);
    e.bias_s = op.bias_smem >= 0 ? smem_u32(smem + op.bias_smem) : 0u;
    e.bias_p = op.bias_smem >= 0 ? reinterpret_cast<const float*>(smem + op.bias_smem) : nullptr;
    return e;
}

template <class T>
__device__ __forceinline__ bool owns(const EpiOp<T>& e, const BTile& t, int gy, int gx) {
    if (!e.own_only)  // emitted cells: exactly this tile (contiguous-M ops compute a halo'd region)
        return gy >= t.oy0 && gy < t.oy0 + e.tile_h && gx >= t.ox0 && gx < t.ox0 + e.tile_w;
    const int S = e.org_mul;
    const int y1 = t.ty == e.grid_h - 1 ? e.H : min(e.H, (t.oy0 + e.tile_h) * S);
    const int x1 = t.tx == e.grid_w - 1 ? e.W : min(e.W, (t.ox0 + e.tile_w) * S);
    return gy >= t.oy0 * S && gy < y1 && gx >= t.ox0 * S && gx < x1;
}

// Destination of one computed cell: the on-chip buffer (planes layout) and/or
// its NHWC pixel in HBM.  Computed once per cell, reused for every channel.
template <class T>
struct CellDst {
    bool valid, inside;
    uint8_t* sbuf;  // plane-0 address of the cell in the shared buffer, or null
    T* gdst;        // channel-0 address of the pixel (concat offset applied), or null
};

template <class T>
__device__ __forceinline__ CellDst<T> cell_dst(const EpiOp<T>& e, const BTile& t, int r, int c, bool valid) {
    CellDst<T> d;
    const int gy = t.oy0 * e.org_mul - e.org_sub + r, gx = t.ox0 * e.org_mul - e.org_sub + c;
    d.valid = valid;
    d.inside = gy >= 0 && gy < e.H && gx >= 0 && gx < e.W;
    d.sbuf = e.buf ? e.buf + (r * e.buf_ew + c) * 16 : nullptr;
    d.gdst = nullptr;
    if (e.emit && !e.gap && e.out && valid && d.inside && owns(e, t, gy, gx))
        d.gdst = e.out + ((size_t(t.n) * e.H + gy) * e.W + gx) * e.out_cstride + e.out_coff + t.c0;
    return d;
}

__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

__device__ __forceinline__ uint4 lds_u4(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}

// Stores chunk k (channels [k*cpc, (k+1)*cpc)) of one cell, already packed.
template <class T>
__device__ __forceinline__ void put_chunk(const CellDst<T>& d, int k, uint4 u, const EpiOp<T>& e) {
    if (d.sbuf) *reinterpret_cast<uint4*>(d.sbuf + k * e.buf_plane) = d.inside ? u : make_uint4(0, 0, 0, 0);
    if (d.gdst) *reinterpret_cast<uint4*>(d.gdst + k * Elem<T>::cpc) = u;
}

// Stores 8 channels [ch, ch+8) of one cell (values already final; ch < cend):
// one bf16 chunk, or two fp32 chunks (the second only below cend -- fp32
// tensors are padded to 4 channels, not 8).
template <class T>
__device__ __forceinline__ void put8(const CellDst<T>& d, int ch, const float* v8, const EpiOp<T>& e) {
    constexpr int cpc = Elem<T>::cpc;
    put_chunk(d, ch / cpc, Elem<T>::pack(v8), e);
    if constexpr (cpc == 4) {
        if (ch + 4 < e.cend) put_chunk(d, ch / cpc + 1, Elem<T>::pack(v8 + 4), e);
    }
}

// Bias + ReLU + store of 16 accumulator columns (channels ch0 ...), unrolled.
template <class T>
__device__ __forceinline__ void finish16(const EpiOp<T>& e, const CellDst<T>& d, int ch0, float* v) {
#pragma unroll
    for (int j = 0; j < 16; j += 8) {
        if (ch0 + j >= e.cend) break;
        const float4 b0 = lds_f4(e.bias_s + uint32_t(ch0 + j) * 4u);
        const float4 b1 = lds_f4(e.bias_s + uint32_t(ch0 + j + 4) * 4u);
        float* x = v + j;
        x[0] += b0.x, x[1] += b0.y, x[2] += b0.z, x[3] += b0.w, x[4] += b1.x, x[5] += b1.y, x[6] += b1.z, x[7] += b1.w;
        if (e.relu)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaxf(x[k], 0.0f);
        put8(d, ch0 + j, x, e);
    }
}

// 32 accumulator columns: the TMEM load is issued first and the 32 bias
// values are fetched from shared memory while it is in flight (the bias
// fetch after the wait was the epilogue's main stall, ncu short_sb).
template <class T>
__device__ __forceinline__ void finish32(const EpiOp<T>& e, const CellDst<T>& d, bool valid, int ch0, uint32_t ta) {
    uint32_t r[32];
    tmem_ld32_issue(ta, r);
    const uint32_t bp = e.bias_s + uint32_t(ch0) * 4u;
    float4 b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = lds_f4(bp + 16u * j);  // volatile: stays between the TMEM load issue and its wait
    tmem_ld_wait32(r);
    if (!valid) return;
#pragma unroll
    for (int j = 0; j < 32; j += 8) {
        if (ch0 + j >= e.cend) break;
        if (j == 16) {
#pragma unroll
            for (int q = 0; q < 4; ++q) b[q] = lds_f4(bp + 64u + 16u * q);
        }
        float x[8];
        const float4 b0 = b[(j & 15) / 4], b1 = b[(j & 15) / 4 + 1];
        x[0] = __uint_as_float(r[j]) + b0.x, x[1] = __uint_as_float(r[j + 1]) + b0.y;
        x[2] = __uint_as_float(r[j + 2]) + b0.z, x[3] = __uint_as_float(r[j + 3]) + b0.w;
        x[4] = __uint_as_float(r[j + 4]) + b1.x, x[5] = __uint_as_float(r[j + 5]) + b1.y;
        x[6] = __uint_as_float(r[j + 6]) + b1.z, x[7] = __uint_as_float(r[j + 7]) + b1.w;
        if (e.relu)
#pragma unroll
            for (int k = 0; k < 8; ++k) x[k] = fmaxf(x[k], 0.0f);
        put8(d, ch0 + j, x, e);
    }
}

// Warp transpose-reduction: on entry lane l holds v[0..31] (row l, columns
// 0..31); on exit lane l returns the sum of column l over the warp's 32 rows
// (31 shuffles: at each step a lane keeps the half of its columns selected by
// its own lane bit and adds the partner's copy of that half).
__device__ __forceinline__ float warp_colsum32(float* v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int j = 0; j < off; ++j) {
            const float send = upper ? v[j] : v[j + off];
            const float keep = upper ? v[j + off] : v[j];
            v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

// Global-average-pool epilogue: relu(acc + bias) of the cells this tile owns
// (others contribute 0), summed over the warp's rows and added to the tile's
// per-column sums in shared memory.  Warp-uniform (all lanes shuffle).
template <class T>
__device__ __forceinline__ void finish_gap(const EpiOp<T>& e, bool take, int ch0, int ncols, uint32_t ta, float* gsum) {
    float v[32];
    if (ncols == 32) {
        tmem_ld32(ta, v);
    } else {
        tmem_ld16(ta, v);
#pragma unroll
        for (int j = 16; j < 32; ++j) v[j] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        if (j >= ncols) {
            v[j] = v[j + 1] = v[j + 2] = v[j + 3] = 0.0f;
            continue;
        }
        const float4 b = lds_f4(e.bias_s + uint32_t(ch0 + j) * 4u);
        float x0 = v[j] + b.x, x1 = v[j + 1] + b.y, x2 = v[j + 2] + b.z, x3 = v[j + 3] + b.w;
        if (e.relu) x0 = fmaxf(x0, 0.0f), x1 = fmaxf(x1, 0.0f), x2 = fmaxf(x2, 0.0f), x3 = fmaxf(x3, 0.0f);
        // select, not multiply: rows outside the tile hold whatever the
        // over-read shared memory produced (possibly Inf/NaN)
        v[j] = take ? x0 : 0.0f, v[j + 1] = take ? x1 : 0.0f, v[j + 2] = take ? x2 : 0.0f, v[j + 3] = take ? x3 : 0.0f;
    }
    const float colsum = warp_colsum32(v);
    const int lane = threadIdx.x & 31;
    // per-warp slot (no shared float atomics: sm_100 lowers them to a CAS loop)
    float* slot = gsum + ((threadIdx.x >> 5) & 3) * e.gap_np;  // warps w, w+4 own disjoint columns
    if (lane < ncols && ch0 + lane < e.cend) slot[ch0 + lane] += colsum;
}

// Accumulator -> bias/ReLU/mask -> bf16 / TF32 -> shared buffer and/or HBM.  Thread
// (row = tid % 128) owns TMEM lane `row` = GEMM row = one cell.  With two
// warp groups, narrow ops (<= 32 columns) split the M tiles between them,
// wider ones split the columns in 32-column slices.
template <class T, int EW, bool GAP>
__device__ void epilogue_mma(const BParams& P, const BOp& op, int nbi, uint8_t* smem, uint32_t tmem, const BTile& t) {
    constexpr int kHalves = Cta<EW>::halves;
    const EpiOp<T> e = epi_op<T>(P, op, smem);
    const int mtiles = op.mtiles, contig = op.contig, ext_w = op.ext_w, ext_h = op.ext_h, strips = op.strips, nb = op.nb;
    const int row = threadIdx.x & 127, half = kHalves > 1 ? int(threadIdx.x >> 7) : 0;
    const uint32_t tbase = tmem + op.tcol + (uint32_t(row & ~31) << 16);
    const int chbase = nbi * nb;
    const bool split_m = kHalves > 1 && nb <= 32;
    const int mt0 = split_m ? half : 0, mstep = split_m ? kHalves : 1;
    const int col0 = split_m ? 0 : half * 32, cstep = split_m ? 32 : 32 * kHalves;
    // windowed M tiles: (16-row block, 8-column strip) stepped, not divided
    int wst = mt0 % strips, wrb = mt0 / strips;
    for (int mt = mt0; mt < mtiles; mt += mstep) {
        int r, c;
        bool valid;
        if (contig) {
            const int idx = mt * 128 + row;
            r = idx / ext_w, c = idx - r * ext_w;
            valid = idx < ext_h * ext_w;
        } else {
            r = wrb * 16 + (row >> 3), c = wst * 8 + (row & 7);
            valid = r < ext_h && c < ext_w;
            wst += mstep;
            while (wst >= strips) wst -= strips, ++wrb;
        }
        const CellDst<T> d = cell_dst(e, t, r, c, valid);
        if (GAP) {
            float* gsum = reinterpret_cast<float*>(smem + P.gap_off);
            const bool take = valid && d.inside;
            for (int col = col0; col < nb; col += cstep) finish_gap(e, take, chbase + col, min(32, nb - col), tbase + mt * nb + col, gsum);
            continue;
        }
        for (int col = col0; col < nb; col += cstep) {
            const uint32_t ta = tbase + mt * nb + col;
            if (nb - col >= 32) {
                finish32(e, d, valid, chbase + col, ta);
            } else {
                float v[16];
                tmem_ld16(ta, v);
                if (valid) finish16(e, d, chbase + col, v);
            }
        }
    }
}

// Register copy of a shared region's addressing.  Swizzled regions start on
// 1024-byte boundaries with 1024-multiple K-block strides, so the swizzle of
// cell r is (r & 7) for SW128 and ((r >> 2) & 1) for SW32.
struct RegionView {
    uint8_t* base;
    int mode, per, plane, rowb, ew;  // per = 16-byte chunks per row
};

__device__ __forceinline__ RegionView region_view(const BRegion& R, uint8_t* smem) {
    return {smem + R.smem_off, R.mode, R.row_bytes >> 4, R.plane_bytes, R.row_bytes, R.ext_w};
}

__device__ __forceinline__ const uint8_t* chunk_ptr(const RegionView& v, int cell, int oct) {
    const int kb = oct / v.per, j = oct - kb * v.per;
    const int sw = v.mode == kSw128 ? (cell & 7) : v.mode == kSw32 ? ((cell >> 2) & 1) : 0;
    return v.base + kb * v.plane + cell * v.rowb + ((j ^ sw) << 4);
}

// Byte offset of 16-byte chunk j (within K-block kb) of cell `cell`, for a
// region whose K-blocks start on 1024-byte boundaries (MODE = region mode).
template <int MODE>
__device__ __forceinline__ uint32_t chunk_off(uint32_t kb_base, int cell, int j) {
    if (MODE == kSw128) return kb_base + uint32_t(cell) * 128u + uint32_t((j ^ (cell & 7)) << 4);
    if (MODE == kSw32) return kb_base + uint32_t(cell) * 32u + uint32_t((j ^ ((cell >> 2) & 1)) << 4);
    return kb_base + uint32_t(cell) * 16u;
}

// Pools over a shared region (zero padding is already in the region: TMA
// zero fill / masked epilogue cells), max in bf16 (exact), average in fp32
// over the full window (reference.cpp:59-88).  Thread u handles one chunk
// (oct: 8 bf16 / 4 fp32 channels) of one output cell, chunks fastest: the 8
// chunks of a cell sit in 8 different bank groups in every region mode, and 8
// neighbouring threads store one 128-byte run of the NHWC output.
template <class T, int EW, int MODE, int K, bool MX>
__device__ void pool_fast(const EpiOp<T>& e, const BRegion& Rg, uint8_t* smem, const BOp& op, const BTile& t) {
    const uint32_t base = smem_u32(smem + Rg.smem_off);
    const int plane = Rg.plane_bytes, rew = Rg.ext_w;
    const int ext_w = op.ext_w, stride = op.stride, dd = op.d;
    const int kh_ = K ? K : op.kh, kw_ = K ? K : op.kw;
    const int ncell = op.ext_h * ext_w, c8 = op.npad / Elem<T>::cpc;  // chunks per cell
    const float inv = 1.0f / float(kh_ * kw_);
    constexpr int kPer = MODE == kSw128 ? 8 : MODE == kSw32 ? 2 : 1;
    // u = cell * c8 + oct, u = tid, tid + NT, ...: when c8 divides NT the
    // thread's oct is fixed and its cell advances by NT / c8 -- (r, c) are
    // stepped instead of divided (two integer divisions per unit otherwise).
    constexpr int NT = Cta<EW>::compute;
    const bool step = (NT % c8) == 0;
    const int oct0 = threadIdx.x % c8, cs = NT / c8;
    const int dr = cs / ext_w, dc = cs - dr * ext_w;
    int rr = (threadIdx.x / c8) / ext_w, cc = (threadIdx.x / c8) - rr * ext_w;
    for (int u = threadIdx.x; u < ncell * c8; u += NT) {
        int r, c, oct;
        if (step) {
            r = rr, c = cc, oct = oct0;
            rr += dr, cc += dc;
            if (cc >= ext_w) cc -= ext_w, ++rr;
        } else {
            const int cell = u / c8;
            oct = u - cell * c8, r = cell / ext_w, c = cell - r * ext_w;
        }
        const int kb = oct / kPer, j = oct - kb * kPer;
        const uint32_t kbb = base + uint32_t(kb * plane);
        const int c0 = (r * stride + dd) * rew + c * stride + dd;
        uint4 out;
        if (MX) {
            uint4 m = lds_u4(chunk_off<MODE>(kbb, c0, j));
#pragma unroll
            for (int ky = 0; ky < (K ? K : 1); ++ky)
                for (int ky2 = 0; ky2 < (K ? 1 : kh_); ++ky2)
#pragma unroll
                    for (int kx = 0; kx < (K ? K : 1); ++kx)
                        for (int kx2 = 0; kx2 < (K ? 1 : kw_); ++kx2) {
                            const int dy = K ? ky : ky2, dx = K ? kx : kx2;
                            if (dy == 0 && dx == 0) continue;
                            m = Elem<T>::vmax(m, lds_u4(chunk_off<MODE>(kbb, c0 + dy * rew + dx, j)));
                        }
            out = m;
        } else {
            constexpr int cpc = Elem<T>::cpc;
            float acc[cpc];
#pragma unroll
            for (int q = 0; q < cpc; ++q) acc[q] = 0.0f;
            for (int dy = 0; dy < kh_; ++dy)
                for (int dx = 0; dx < kw_; ++dx) {
                    float f[cpc];
                    Elem<T>::unpack(lds_u4(chunk_off<MODE>(kbb, c0 + dy * rew + dx, j)), f);
#pragma unroll
                    for (int q = 0; q < cpc; ++q) acc[q] += f[q];
                }
#pragma unroll
            for (int q = 0; q < cpc; ++q) acc[q] *= inv;
            out = Elem<T>::pack(acc);
        }
        put_chunk(cell_dst(e, t, r, c, true), oct, out, e);
    }
}

template <class T, int EW, int MODE>
__device__ __forceinline__ void pool_mode(const EpiOp<T>& e, const BRegion& R, uint8_t* smem, const BOp& op, const BTile& t) {
    if (op.kind == BOP_MAXPOOL) {
        if (op.kh == 3 && op.kw == 3) pool_fast<T, EW, MODE, 3, true>(e, R, smem, op, t);
        else pool_fast<T, EW, MODE, 0, true>(e, R, smem, op, t);
    } else {
        pool_fast<T, EW, MODE, 0, false>(e, R, smem, op, t);
    }
}

// Residual add of two shared plane buffers.
template <class T, int EW>
__device__ void simt_add(const EpiOp<T>& e, const BRegion& A, const BRegion& B, uint8_t* smem, const BOp& op, const BTile& t) {
    constexpr int cpc = Elem<T>::cpc;
    const int ext_w = op.ext_w, ncell = op.ext_h * ext_w, c8 = op.npad / cpc;
    for (int u = threadIdx.x; u < ncell * c8; u += Cta<EW>::compute) {
        const int cell = u / c8, oct = u - cell * c8;
        const int r = cell / ext_w, c = cell - r * ext_w;
        float fa[cpc], fb[cpc];
        Elem<T>::unpack(lds_u4(smem_u32(smem + A.smem_off + oct * A.plane_bytes + (r * A.ext_w + c) * 16)), fa);
        Elem<T>::unpack(lds_u4(smem_u32(smem + B.smem_off + oct * B.plane_bytes + (r * B.ext_w + c) * 16)), fb);
#pragma unroll
        for (int q = 0; q < cpc; ++q) fa[q] += fb[q];
        put_chunk(cell_dst(e, t, r, c, true), oct, Elem<T>::pack(fa), e);
    }
}

template <class T, int EW>
__device__ void simt_pool_add(const BParams& P, const BOp& op, uint8_t* smem, const BTile& t, int xdelta) {
    const EpiOp<T> e = epi_op<T>(P, op, smem);
    const BRegion R = src_region_at(P, op, op.src, xdelta);
    if (op.kind == BOP_ADD) {
        simt_add<T, EW>(e, R, P.bufs[op.src2], smem, op, t);
        return;
    }
    if (R.mode == kSw128) pool_mode<T, EW, kSw128>(e, R, smem, op, t);
    else if (R.mode == kSw32) pool_mode<T, EW, kSw32>(e, R, smem, op, t);
    else pool_mode<T, EW, kPlanes>(e, R, smem, op, t);
}

// Direct conv for what the tensor-core path does not take (stride != 1,
// groups, Cin not a multiple of 16).  fp32 accumulate.
template <class T, int EW>
__device__ void simt_conv(const BParams& P, const BOp& op, uint8_t* smem, const BTile& t, int xdelta) {
    constexpr int cpc = Elem<T>::cpc;
    const EpiOp<T> e = epi_op<T>(P, op, smem);
    const RegionView R = region_view(src_region_at(P, op, op.src, xdelta), smem);
    const int ext_w = op.ext_w, kh_ = op.kh, kw_ = op.kw, stride = op.stride, dd = op.d, cout = op.cout;
    const int ncell = op.ext_h * ext_w, c8 = (op.npad + 7) / 8;  // groups of 8 output channels per cell
    const int cin_g = op.cin / op.group, cout_g = cout / op.group, cp4 = (cout + 3) & ~3;
    const float* wsimt = op.wsimt;
    const float* gbias = op.bias;
    for (int u = threadIdx.x; u < ncell * c8; u += Cta<EW>::compute) {
        const int cell = u / c8, oct = u - cell * c8;
        const int r = cell / ext_w, c = cell - r * ext_w;
        float acc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
        const int base = (r * stride + dd) * R.ew + c * stride + dd;
        for (int ic = 0; ic < cin_g; ++ic)
            for (int kh = 0; kh < kh_; ++kh)
                for (int kw = 0; kw < kw_; ++kw) {
                    const int cell_in = base + kh * R.ew + kw;
                    const float* wrow = wsimt + ((ic * kh_ + kh) * kw_ + kw) * cp4;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int oc = oct * 8 + j;
                        if (oc >= cout) break;
                        const int in_c = (oc / cout_g) * cin_g + ic;
                        const T xv = *reinterpret_cast<const T*>(chunk_ptr(R, cell_in, in_c / cpc) + (in_c % cpc) * int(sizeof(T)));
                        acc[j] = fmaf(Elem<T>::to(xv), __ldg(wrow + oc), acc[j]);
                    }
                }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int oc = oct * 8 + j;
            const float x = oc < cout ? acc[j] + __ldg(gbias + oc) : 0.0f;
            acc[j] = e.relu ? fmaxf(x, 0.0f) : x;
        }
        put8(cell_dst(e, t, r, c, true), oct * 8, acc, e);
    }
}

// KIND (compile-time step class): kMmaOnly steps (fire modules, plain convs)
// carry no SIMT / pool / global-average-pool code, so their register
// allocation is not set by those paths; kSimt adds pools / stride-2 convs /
// adds; kGap is the conv + global-average-pool epilogue.
enum : int { kMmaOnly = 0, kSimt = 1, kGap = 2 };

template <class T, int EW, int KIND>
__global__ void __launch_bounds__(Cta<EW>::threads, Cta<EW>::min_blocks) fused_tc_kernel(const __grid_constant__ BParams Pg, int batch,
                                                                                      int n0) {
    constexpr int kCompute = Cta<EW>::compute, kWarpX = Cta<EW>::wx, kWarpMma = Cta<EW>::wmma, kWarpW = Cta<EW>::ww;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t bar_x[2], x_free[2], ring_full[kRingMax], ring_empty[kRingMax], acc_full[2 * kBMaxUnits * kSubs],
        unit_done[2 * kBMaxUnits], acc_free[2];
    __shared__ uint32_t tmem_slot;
    // The descriptor lives in the kernel-parameter constant bank; the op loops
    // index it with run-time op numbers, and indexed constant loads that miss
    // the small constant cache stall for hundreds of cycles.  The epilogue
    // warps work from a shared-memory copy, pulled from the device copy with
    // one bulk copy; the producers (few loads, latency-critical X issue) and
    // the MMA issuer (uniform indices) read the bank, which also holds the
    // tensor maps TMA reads.
    __shared__ __align__(64) BParams Ps;
    __shared__ __align__(8) uint64_t bar_p, bar_w;
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;  // provably warp-uniform
    const int total = Pg.grid_h * Pg.grid_w * Pg.cgroups * batch;
    grid_launch_dependents();  // every CTA is resident: the next step may be scheduled as SMs free up
    if (threadIdx.x == 0) {
        mbar_init(&bar_p, 1);
        const int xrel = x_release_group(Pg);
        for (int i = 0; i < 2; ++i) mbar_init(&bar_x[i], 1), mbar_init(&x_free[i], xrel >= 0 ? 1 : EW);  // MMA commit, or one arrival per epilogue warp
        for (int i = 0; i < kRingMax; ++i) mbar_init(&ring_full[i], 1), mbar_init(&ring_empty[i], 1);
        mbar_init(&bar_w, 1);
        for (int t = 0; t < Pg.tsets; ++t)
            for (int i = 0; i < Pg.ngroups; ++i) {
                mbar_init(&unit_done[t * kBMaxUnits + i], EW);
                for (int q = 0; q < kSubs; ++q) mbar_init(&acc_full[(t * kBMaxUnits + i) * kSubs + q], 1);
            }
        mbar_init(&acc_free[0], EW), mbar_init(&acc_free[1], EW);
        mbar_fence_init();
        mbar_expect_tx(&bar_p, uint32_t(sizeof(BParams)));
        bulk_g2s(&Ps, Pg.dev_copy, uint32_t(sizeof(BParams)), &bar_p);
    }
    if (warp == kWarpMma && Pg.tmem_cols) tmem_alloc(&tmem_slot, Pg.tmem_cols * Pg.tsets);
    fence_before();
    __syncthreads();
    fence_after();
    const BParams& P = Ps;
    const uint32_t tmem = Pg.tmem_cols ? tmem_slot : 0;

    if (warp == kWarpX) {
        if (lane == 0) x_producer(Pg, Pg.xmap, smem, total, n0, bar_x, x_free);  // starts before Ps lands
    } else if (warp == kWarpW) {
        if (lane == 0) w_producer(Pg, smem, total, ring_full, ring_empty, &bar_w);
    } else if (warp == kWarpMma) {
        // One thread issues everything: a per-MMA elect.sync + __syncwarp in a
        // warp-wide loop costs ~175 cycles per tcgen05.mma against ~50 for a
        // single-thread loop (tests/probes/tcgen05_rate.cu) -- and these
        // convolutions are many small MMAs (N 16..256, K 16).
        // (elect.sync, not lane == 0: the compiler then knows one thread is
        // active and moves descriptors to uniform registers without the
        // per-MMA ELECT waterfall it emits for a lane-predicated branch)
        if (elect_one()) issuer<T>(Pg, smem, tmem, total, bar_x, x_free, ring_full, ring_empty, acc_full, unit_done, acc_free, &bar_w);
        __syncwarp();
    } else {
        compute_wait<EW>(&bar_p, 0);
        // biases of the MMA ops -> shared memory (read by every epilogue)
        for (int i = 0; i < P.nops; ++i) {
            const BOp& op = P.ops[i];
            if (op.bias_smem < 0) continue;
            float* dst = reinterpret_cast<float*>(smem + op.bias_smem);
            const int g0 = op.gch ? int(blockIdx.y) * op.gch : 0;  // channel group of this CTA row
            for (int k = threadIdx.x; k < op.npad; k += kCompute) dst[k] = g0 + k < op.cout ? __ldg(op.bias + g0 + k) : 0.0f;
            if (op.gap)
                for (int k = threadIdx.x; k < 4 * op.npad; k += kCompute) reinterpret_cast<float*>(smem + P.gap_off)[k] = 0.0f;
        }
        named_sync_compute<EW>();
        const int gap_np = KIND == kGap ? P.ops[0].npad : 0;  // gap steps have one op
        const int nxb = P.nxb;
        const int xrel = x_release_group(P);
        int k = 0;
        const int ts = P.tsets;
        grid_dependency_wait();  // global stores after the previous step completed (no write/read overlap)
        TileWalk tw;
        tw.init(P);
        for (int tau = blockIdx.x; tau < total; tau += gridDim.x, ++k, tw.next(P)) {
            const BTile t = tw.tile(P, n0);
            const int b = nxb == 2 ? (k & 1) : 0, use = nxb == 2 ? (k >> 1) : k;
            const int xdelta = b * P.xstride;
            const int s = ts == 2 ? (k & 1) : 0, j = ts == 2 ? (k >> 1) : k;
            const uint32_t tm = tmem + uint32_t(s * P.tmem_cols);
            bool have_x = false;
            for (int gi = 0; gi < P.ngroups; ++gi) {
                const BGroup& G = P.groups[gi];
                if (G.mma) {
                    uint64_t* fb = acc_full + (s * kBMaxUnits + gi) * kSubs;
                    for (int i = G.op0; i < G.op1; ++i) {
                        const int sub = i - G.op0;
                        if (sub < kSubs) {  // op `sub`'s accumulators (the last slot covers the rest of the group)
                            compute_wait<EW>(&fb[sub], j & 1);
                            if (threadIdx.x == 0 && sub == 0) stamp(P, kTrUnit + 2 * gi, k);
                            fence_after();
                        }
                        epilogue_mma<T, EW, KIND == kGap>(P, P.ops[i], G.nbi, smem, tm + uint32_t(G.tbase), t);
                    }
                } else {
                    if constexpr (KIND == kSimt) {
                        const BOp& op = P.ops[G.op0];
                        if (!have_x) compute_wait<EW>(&bar_x[b], use & 1), have_x = true;
                        if (op.kind == BOP_SIMT_CONV) simt_conv<T, EW>(P, op, smem, t, xdelta);
                        else simt_pool_add<T, EW>(P, op, smem, t, xdelta);
                    }
                }
                fence_async_smem();  // epilogue-written buffers are read by later MMAs (async proxy)
                fence_before();
                // MMA-only steps: no epilogue reads what another warp wrote, so
                // each warp releases the unit on its own (the barrier counts
                // one arrival per warp); SIMT ops and the pooled column sums
                // read across warps and need the whole group first
                if constexpr (KIND != kMmaOnly) named_sync_compute<EW>();
                __syncwarp();
                if (lane == 0) mbar_arrive(&unit_done[s * kBMaxUnits + gi]);
                if (threadIdx.x == 0) stamp(P, kTrUnit + 2 * gi + 1, k);
            }
            // every unit of this tile is done (MMAs complete, SIMT reads
            // finished): its staging buffer and accumulator set are free
            if (lane == 0) {
                if (xrel < 0) mbar_arrive(&x_free[b]);
                if (ts == 2) mbar_arrive(&acc_free[s]);
            }
            if (threadIdx.x == 0) stamp(P, kTrEnd, k);
            if (KIND == kGap) {  // this tile's column sums -> gap_part[image][tile][c], reset
                float* gsum = reinterpret_cast<float*>(smem + P.gap_off);
                const int per_img = P.grid_h * P.grid_w;
                float* dst = P.gap_part + (size_t(t.n) * per_img + t.ty * P.grid_w + t.tx) * P.gap_np_total + blockIdx.y * gap_np;
                for (int c = threadIdx.x; c < gap_np; c += kCompute) {
                    float a = 0.0f;
#pragma unroll
                    for (int w = 0; w < 4; ++w) a += gsum[w * gap_np + c], gsum[w * gap_np + c] = 0.0f;
                    dst[c] = a;
                }
                named_sync_compute<EW>();
            }
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == kWarpMma && Pg.tmem_cols) tmem_free(tmem, Pg.tmem_cols * Pg.tsets);
}

// ----------------------------------------------------------------- layout kernels
// Conversions at the boundary (NCHW fp32 <-> NHWC T, channels padded to the
// pitch with zeros) and the small steps outside fused kernels.  Values a
// tensor-core step reads are rounded once here (bf16 RN / TF32 RNA).

template <class T>
__global__ void nchw_f32_to_nhwc_tc(const float* __restrict__ src, T* __restrict__ dst, int N, int C, int H, int W, int cs) {
    const long long total = (long long)N * H * W * cs;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int c = int(i % cs);
        const long long p = i / cs;
        const int x = int(p % W), y = int((p / W) % H);
        const long long n = p / ((long long)W * H);
        dst[i] = Elem<T>::from(c < C ? src[((n * C + c) * H + y) * W + x] : 0.0f);
    }
}

template <class T>
__global__ void nhwc_tc_to_nchw_f32(const T* __restrict__ src, int cs, int coff, float* __restrict__ dst, int N, int C, int H, int W) {
    const long long total = (long long)N * C * H * W;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int x = int(i % W);
        const int y = int((i / W) % H);
        const int c = int((i / ((long long)W * H)) % C);
        const long long n = i / ((long long)W * H * C);
        dst[i] = Elem<T>::to(src[((n * H + y) * W + x) * cs + coff + c]);
    }
}

__device__ __forceinline__ float seeded_at(unsigned long long seed, unsigned long long idx) {  // SeededStream element idx (tensor.cpp:19-40)
    unsigned long long z = seed + (idx + 1ull) * 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z = z ^ (z >> 31);
    return static_cast<float>(z >> 40) * (1.0f / 16777216.0f) - 0.5f;
}

template <class T>
__global__ void seeded_nhwc_tc(T* __restrict__ dst, unsigned long long seed, unsigned long long first_image, int N, int C, int H, int W,
                               int cs) {
    const long long total = (long long)N * H * W * cs;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int c = int(i % cs);
        const long long p = i / cs;
        const int x = int(p % W), y = int((p / W) % H);
        const long long n = p / ((long long)W * H);
        const float v = c < C ? seeded_at(seed, (((first_image + n) * C + c) * H + y) * (unsigned long long)W + x) : 0.0f;
        dst[i] = Elem<T>::from(v);
    }
}

// Space-to-depth input for a stride-2 first conv (see Engine: the conv is
// rewritten as a stride-1 conv on 2x2 phases so it runs on tensor cores):
// dst[n][Y][X][(py*2+px)*C + c] = src[n][c][2Y+py][2X+px], channels >= 4C zero.
// Source is NCHW fp32 (src != nullptr) or the SeededStream (seed, first_image).
// planar != 0: "row-planar" instead of NHWC -- image n, row Y holds the row's
// 16-byte channel planes one after the other ([n][Y][plane][X][cpc]), so a
// whole input row is one contiguous run (the stem kernel's TMA layout).
template <class T>
__global__ void s2d_tc(const float* __restrict__ src, unsigned long long seed, unsigned long long first_image, T* __restrict__ dst, int N,
                       int C, int H, int W, int cs, int planar) {
    const int H2 = H / 2, W2 = W / 2;
    const long long total = (long long)N * H2 * W2 * cs;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int ci = int(i % cs);
        const long long p = i / cs;
        const int X = int(p % W2), Y = int((p / W2) % H2);
        const long long n = p / ((long long)W2 * H2);
        float v = 0.0f;
        if (ci < 4 * C) {
            const int ph = ci / C, c = ci - ph * C;
            const int y = 2 * Y + (ph >> 1), x = 2 * X + (ph & 1);
            const unsigned long long idx = (((unsigned long long)n * C + c) * H + y) * (unsigned long long)W + x;
            v = src ? src[idx] : seeded_at(seed, first_image * (unsigned long long)C * H * W + idx);
        }
        constexpr int cpc = Elem<T>::cpc;
        const long long o = planar ? (((n * H2 + Y) * (cs / cpc) + ci / cpc) * W2 + X) * cpc + ci % cpc : i;
        dst[o] = Elem<T>::from(v);
    }
}

template <class T>
__global__ void concat_copy_tc(const T* __restrict__ src, int scs, int sco, T* __restrict__ dst, int dcs, int dco, int C, long long pixels) {
    const long long total = pixels * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long p = i / C;
        const int c = int(i - p * C);
        dst[p * dcs + dco + c] = src[p * scs + sco + c];
    }
}

template <class T>
__global__ void eltwise_tc(int op, const T* __restrict__ a, int acs, int aco, const T* __restrict__ b, int bcs, int bco, T* __restrict__ o,
                           int ocs, int oco, int C, long long pixels) {
    const long long total = pixels * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long p = i / C;
        const int c = int(i - p * C);
        const float x = Elem<T>::to(a[p * acs + aco + c]);
        o[p * ocs + oco + c] = Elem<T>::from(op == 0 ? x + Elem<T>::to(b[p * bcs + bco + c]) : fmaxf(x, 0.0f));
    }
}

// gap steps: out[n][coff + c] = scale * sum over the image's tiles of
// part[n][tile][c] for images [n0, n0 + N), in tile order (deterministic).
template <class T>
__global__ void gap_finish_tc(const float* __restrict__ part, int tiles, int np, float scale, T* __restrict__ out, int cs, int coff, int C,
                              int n0, int N) {
    const long long total = (long long)N * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const long long n = n0 + i / C;
        const int c = int(i % C);
        const float* p = part + size_t(n) * tiles * np + c;
        float acc = 0.0f;
        for (int t = 0; t < tiles; ++t) acc += p[size_t(t) * np];
        out[size_t(n) * cs + coff + c] = Elem<T>::from(acc * scale);
    }
}

int grid_b(long long work) {
    long long b = (work + 255) / 256;
    return int(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

// SMs of the calling thread's current device (cached per device).
int sm_count() {
    static int cache[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    if (!cache[dev]) {
        int n = 148;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1) n = 148;
        cache[dev] = n;
    }
    return cache[dev];
}

}  // namespace

namespace {

template <class T, int EW>
cudaError_t init_ew() {
    // 227 KB per block minus the static part (barriers + the BParams copy) and headroom
    for (auto fn : {fused_tc_kernel<T, EW, kMmaOnly>, fused_tc_kernel<T, EW, kSimt>, fused_tc_kernel<T, EW, kGap>}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudgetTc);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

// Resident CTAs per SM from shared memory (228 KB per SM, 1 KB reserved per
// CTA, the static barriers + descriptor copy), registers (64 K per SM in four
// 16 K sub-partition files, warps placed round-robin) and the launch bound
// (the occupancy API under-reports this kernel).  Over-subscribing is
// harmless (tiles are independent), under-subscribing halves the overlap.
template <class T, int EW, int KIND>
int occupancy_ew(int smem_bytes, int tmem_cols) {
    cudaFuncAttributes a{};
    cudaFuncGetAttributes(&a, fused_tc_kernel<T, EW, KIND>);
    const int by_smem = int((228 * 1024) / (size_t(smem_bytes) + a.sharedSizeBytes + 1024));
    const int warps = Cta<EW>::threads / 32, regs = std::max(a.numRegs, 1);
    int by_regs = 1;
    while ((by_regs + 1) * warps <= 64 && ((by_regs + 1) * warps + 3) / 4 * 32 * regs <= 16384) ++by_regs;
    int occ = std::max(1, std::min(std::min(Cta<EW>::min_blocks, by_regs), by_smem));
    // TMEM: 512 columns per SM; a CTA whose tcgen05.alloc cannot be served
    // waits for another CTA to exit, i.e. serialises behind a persistent one
    if (tmem_cols > 0) occ = std::min(occ, std::max(1, 512 / tmem_cols));
    return occ;
}

template <class T>
int occupancy_t(int smem_bytes, int tmem_cols, int epi_warps, int kind) {
    if (epi_warps == 4)
        return kind == kGap ? occupancy_ew<T, 4, kGap>(smem_bytes, tmem_cols)
               : kind == kSimt ? occupancy_ew<T, 4, kSimt>(smem_bytes, tmem_cols) : occupancy_ew<T, 4, kMmaOnly>(smem_bytes, tmem_cols);
    return kind == kGap ? occupancy_ew<T, 8, kGap>(smem_bytes, tmem_cols)
           : kind == kSimt ? occupancy_ew<T, 8, kSimt>(smem_bytes, tmem_cols) : occupancy_ew<T, 8, kMmaOnly>(smem_bytes, tmem_cols);
}

template <class T>
cudaError_t launch_t(const BParams& P, int batch, cudaStream_t st, int n0) {
    const long long tiles = (long long)P.grid_h * P.grid_w * P.cgroups * batch;
    const int ns = std::max(1, P.nsplit);  // channel groups: grid rows
    const long long grid = P.grid_all ? tiles
                                      : std::min<long long>(tiles, std::max<long long>(1, (long long)sm_count() * std::max(1, P.ctas_per_sm) / ns));
    if (grid < 1) return cudaSuccess;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid), unsigned(ns), 1u), cfg.blockDim = dim3(unsigned(P.epi_warps * 32 + 96));
    cfg.dynamicSmemBytes = size_t(P.smem_bytes), cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = P.pdl ? 1 : 0;
    cfg.attrs = attr, cfg.numAttrs = 1;
#define XLF_LAUNCH(EWV, K) cudaLaunchKernelEx(&cfg, fused_tc_kernel<T, EWV, K>, P, batch, n0)
    if (P.epi_warps == 4) {
        if (P.kind == kGap) XLF_LAUNCH(4, kGap);
        else if (P.kind == kSimt) XLF_LAUNCH(4, kSimt);
        else XLF_LAUNCH(4, kMmaOnly);
    } else {
        if (P.kind == kGap) XLF_LAUNCH(8, kGap);
        else if (P.kind == kSimt) XLF_LAUNCH(8, kSimt);
        else XLF_LAUNCH(8, kMmaOnly);
    }
#undef XLF_LAUNCH
    return cudaGetLastError();
}

}  // namespace

cudaError_t init_fused_tc() {
    for (cudaError_t e : {init_ew<__nv_bfloat16, 4>(), init_ew<__nv_bfloat16, 8>(), init_ew<float, 4>(), init_ew<float, 8>()})
        if (e != cudaSuccess) return e;
    return cudaSuccess;
}

int occupancy_fused_tc(int smem_bytes, int tmem_cols, int epi_warps, int kind, int es) {  // tmem_cols: per CTA (all sets)
    return es == 4 ? occupancy_t<float>(smem_bytes, tmem_cols, epi_warps, kind) : occupancy_t<__nv_bfloat16>(smem_bytes, tmem_cols, epi_warps, kind);
}

// Step class of a descriptor (selects the kernel instantiation).
int step_kind_tc(const BParams& P) {
    for (int i = 0; i < P.nops; ++i)
        if (P.ops[i].gap) return kGap;
    for (int i = 0; i < P.nops; ++i)
        if (P.ops[i].kind != BOP_MMA) return kSimt;
    return kMmaOnly;
}

cudaError_t launch_fused_tc(const BParams& P, int batch, cudaStream_t st, int n0) {
    return P.es == 4 ? launch_t<float>(P, batch, st, n0) : launch_t<__nv_bfloat16>(P, batch, st, n0);
}

#define XLF_BY_ES(es, CALL_F32, CALL_BF16)                      \
    do {                                                         \
        if ((es) == 4) CALL_F32; else CALL_BF16;                 \
    } while (0)

cudaError_t launch_nchw_to_nhwc_tc(int es, const float* src, void* dst, int N, int C, int H, int W, int cs, cudaStream_t st) {
    const int g = grid_b((long long)N * H * W * cs);
    XLF_BY_ES(es, (nchw_f32_to_nhwc_tc<float><<<g, 256, 0, st>>>(src, static_cast<float*>(dst), N, C, H, W, cs)),
              (nchw_f32_to_nhwc_tc<__nv_bfloat16><<<g, 256, 0, st>>>(src, static_cast<__nv_bfloat16*>(dst), N, C, H, W, cs)));
    return cudaGetLastError();
}

cudaError_t launch_nhwc_tc_to_nchw(int es, const void* src, int cs, int coff, float* dst, int N, int C, int H, int W, cudaStream_t st) {
    const int g = grid_b((long long)N * C * H * W);
    XLF_BY_ES(es, (nhwc_tc_to_nchw_f32<float><<<g, 256, 0, st>>>(static_cast<const float*>(src), cs, coff, dst, N, C, H, W)),
              (nhwc_tc_to_nchw_f32<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), cs, coff, dst, N, C, H, W)));
    return cudaGetLastError();
}

cudaError_t launch_seeded_nhwc_tc(int es, void* dst, unsigned long long seed, unsigned long long first_image, int N, int C, int H, int W,
                                  int cs, cudaStream_t st) {
    const int g = grid_b((long long)N * H * W * cs);
    seed = seed ? seed : 0x9e3779b97f4a7c15ull;
    XLF_BY_ES(es, (seeded_nhwc_tc<float><<<g, 256, 0, st>>>(static_cast<float*>(dst), seed, first_image, N, C, H, W, cs)),
              (seeded_nhwc_tc<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<__nv_bfloat16*>(dst), seed, first_image, N, C, H, W, cs)));
    return cudaGetLastError();
}

cudaError_t launch_s2d_tc(int es, const float* src, unsigned long long seed, unsigned long long first_image, void* dst, int N, int C, int H,
                          int W, int cs, int planar, cudaStream_t st) {
    const int g = grid_b((long long)N * (H / 2) * (W / 2) * cs);
    seed = seed ? seed : 0x9e3779b97f4a7c15ull;
    XLF_BY_ES(es, (s2d_tc<float><<<g, 256, 0, st>>>(src, seed, first_image, static_cast<float*>(dst), N, C, H, W, cs, planar)),
              (s2d_tc<__nv_bfloat16><<<g, 256, 0, st>>>(src, seed, first_image, static_cast<__nv_bfloat16*>(dst), N, C, H, W, cs, planar)));
    return cudaGetLastError();
}

cudaError_t launch_concat_copy_tc(int es, const void* src, int scs, int sco, void* dst, int dcs, int dco, int C, long long pixels,
                                  cudaStream_t st) {
    const int g = grid_b(pixels * C);
    XLF_BY_ES(es, (concat_copy_tc<float><<<g, 256, 0, st>>>(static_cast<const float*>(src), scs, sco, static_cast<float*>(dst), dcs, dco, C, pixels)),
              (concat_copy_tc<__nv_bfloat16><<<g, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), scs, sco,
                                                                 static_cast<__nv_bfloat16*>(dst), dcs, dco, C, pixels)));
    return cudaGetLastError();
}

cudaError_t launch_gap_finish_tc(int es, const float* part, int tiles, int np, float scale, void* out, int cs, int coff, int C, int n0, int N,
                                 cudaStream_t st) {
    const int g = grid_b((long long)N * C);
    XLF_BY_ES(es, (gap_finish_tc<float><<<g, 256, 0, st>>>(part, tiles, np, scale, static_cast<float*>(out), cs, coff, C, n0, N)),
              (gap_finish_tc<__nv_bfloat16><<<g, 256, 0, st>>>(part, tiles, np, scale, static_cast<__nv_bfloat16*>(out), cs, coff, C, n0, N)));
    return cudaGetLastError();
}

cudaError_t launch_eltwise_tc(int es, int op, const void* a, int acs, int aco, const void* b, int bcs, int bco, void* o, int ocs, int oco, int C,
                              long long pixels, cudaStream_t st) {
    const int g = grid_b(pixels * C);
    XLF_BY_ES(es, (eltwise_tc<float><<<g, 256, 0, st>>>(op, static_cast<const float*>(a), acs, aco, static_cast<const float*>(b), bcs, bco,
                                                       static_cast<float*>(o), ocs, oco, C, pixels)),
              (eltwise_tc<__nv_bfloat16><<<g, 256, 0, st>>>(op, static_cast<const __nv_bfloat16*>(a), acs, aco,
                                                           static_cast<const __nv_bfloat16*>(b), bcs, bco, static_cast<__nv_bfloat16*>(o), ocs,
                                                           oco, C, pixels)));
    return cudaGetLastError();
}
#undef XLF_BY_ES

}  // namespace xlf
