// Fire kernel for sm_100a (see fire_params.hpp): a split-mode fused block --
// 1x1 squeeze -> several stride-1 expand convs -> concat -- in one persistent
// kernel whose squeeze output never leaves shared memory.
//
//   warp 8   producer: this group's packed weights once (resident), then the
//            squeeze input as 128-pixel x 128-byte chunks through a TMA ring
//            (2-D map over all pixels of the launch, SWIZZLE_128B), unit
//            after unit, running ahead of the MMAs;
//   warp 9   MMA issuer (one thread): per unit the squeeze GEMM (M = 128
//            pixels, N = S, K = input channels) into one of two TMEM
//            accumulators, then -- once the squeeze plane is complete -- every
//            expand op of every expand M tile (M = 128 plane cells, one MMA
//            per tap and K step, A = the plane at a shifted start address)
//            into a ring of TMEM accumulators.  With two planes the next
//            unit's squeeze is issued before this unit's expand;
//   warps 0-7 epilogue: squeeze accumulator -> bias + ReLU -> the plane cell
//            of each pixel (zero column / zero rows written per unit); expand
//            accumulator -> bias + ReLU -> NHWC store at the op's concat
//            offset.  Thread t of warp w owns TMEM lane 32 (w % 4) + t; the
//            two warp groups take alternate column segments (32 or 64
//            channels of one op), staged through shared memory so each store
//            instruction writes whole segments (TMEM reads, 64 B/cycle per
//            SM, bound this stage; 16 warps measured slower: register spills).
// The reference computes the same block tile by tile on the CPU
// (fused_exec.cpp:116-210 producer stage into a zero-bordered buffer,
// :214-280 consumer stage, :192-209 stores).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "fire_params.hpp"
#include "umma.cuh"

namespace xlf {

namespace {

using namespace umma;

// CTAs per SM (P.cps): 1 -- 8 epilogue warps (two per TMEM lane quadrant), all
// 512 TMEM columns; 2 -- two independent unit pipelines per SM, each with 4
// epilogue warps, 256 TMEM columns and half the shared memory.
// Squeeze-input stages: 128 pixels x a K chunk of P.cb bytes (128: SWIZZLE_128B,
// 4 K steps; 64: SWIZZLE_64B, 2 K steps -- narrow stages leave room for
// larger resident expand weights).
template <int CPS>
struct Cfg {
    static constexpr int kEpi = CPS == 1 ? 256 : 128;
    static constexpr int kThreads = kEpi + 64;
    static constexpr int kProd = kEpi / 32, kMma = kEpi / 32 + 1;
    static constexpr int kGroups = kEpi / 128;  // epilogue warps per TMEM lane quadrant
    static constexpr int kTmemCols = 512 / CPS;
};

template <class T>
struct FElem;
template <>
struct FElem<__nv_bfloat16> {
    static constexpr int cpc = 8;
    __device__ static uint32_t idesc(int N) { return idesc_bf16(128, N); }
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_bf16(t, a, b, id, acc); }
    __device__ static uint4 pack(const float* v) {
        uint4 u;
        __nv_bfloat162 h;
        h = __floats2bfloat162_rn(v[0], v[1]), u.x = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[2], v[3]), u.y = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[4], v[5]), u.z = *reinterpret_cast<uint32_t*>(&h);
        h = __floats2bfloat162_rn(v[6], v[7]), u.w = *reinterpret_cast<uint32_t*>(&h);
        return u;
    }
};
template <>
struct FElem<float> {
    static constexpr int cpc = 4;
    __device__ static uint32_t idesc(int N) { return idesc_tf32(128, N); }
    __device__ static void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) { mma_tf32(t, a, b, id, acc); }
    __device__ static uint4 pack(const float* v) {
        return make_uint4(__float_as_uint(round_tf32(v[0])), __float_as_uint(round_tf32(v[1])), __float_as_uint(round_tf32(v[2])),
                          __float_as_uint(round_tf32(v[3])));
    }
};

__device__ __forceinline__ void tma_2d(void* smem, const void* desc, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            smem_u32(smem)),
        "l"(desc), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

// 32-byte (256-bit) global store: a whole L2 sector per thread
__device__ __forceinline__ void st_global32(void* p, uint4 a, uint4 b) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y),
                 "r"(b.z), "r"(b.w)
                 : "memory");
}

__device__ __forceinline__ void st_shared16(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// A unit: images [nA, nA + ni) (rows r0 .. r0 + R - 1 of each), its squeeze
// pixels [p0, p1) of the launch's pixel rows.
struct Unit {
    int nA, ni, r0;
    int p0, p1;
};

__device__ __forceinline__ Unit unit_of(const FireParams& P, int u, int n0, int count) {
    Unit U;
    if (P.G > 1) {
        U.nA = n0 + u * P.G, U.r0 = 0;
        U.ni = min(P.G, n0 + count - U.nA);
        U.p0 = U.nA * P.HW, U.p1 = (U.nA + U.ni) * P.HW;
    } else {
        const int b = u % P.bands;
        U.nA = n0 + u / P.bands, U.ni = 1, U.r0 = b * P.R;
        U.p0 = U.nA * P.HW + max(U.r0 - 1, 0) * P.W;
        U.p1 = U.nA * P.HW + min(U.r0 + P.R + 1, P.H) * P.W;
    }
    return U;
}

// Job order.  Round r of a CTA with nu units: with two planes, the squeeze
// tiles of unit r interleaved (evenly, Bresenham) with the expand tiles of
// unit r - 1, so the next unit's squeeze overlaps this unit's expand on the
// tensor pipe, the TMA ring and the epilogue warps alike; with one plane,
// unit r's squeeze tiles then its expand tiles.  The MMA issuer and the
// epilogue warps walk the same sequence.
struct Round {
    int sq, ex;  // unit indices of this CTA (-1: none)
    int ns, ne;  // squeeze / expand jobs
};
__device__ __forceinline__ Round round_of(const FireParams& P, int r, int nu) {
    Round R;
    if (P.nplane == 2) R.sq = r < nu ? r : -1, R.ex = r >= 1 ? r - 1 : -1;
    else R.sq = r, R.ex = r;
    R.ns = R.sq >= 0 ? P.Ts : 0, R.ne = R.ex >= 0 ? P.Te * (P.per_op ? P.nops : 1) : 0;
    return R;
}
// Walks the jobs of a round: squeeze tile (idx, true) or expand tile (idx,
// false).  Two planes: the squeeze tiles spread evenly over the round
// (Bresenham: after job i, floor((i + 1) * ns / tot) of them).
struct Jobs {
    int ns, tot, i = 0, nsq = 0, rem = 0;
    bool two;
    __device__ Jobs(const FireParams& P, const Round& R) : ns(R.ns), tot(R.ns + R.ne), two(P.nplane == 2) {}
    __device__ __forceinline__ bool next(int* idx) {
        bool sq;
        if (two) {
            rem += ns;
            sq = rem >= tot;
            if (sq) rem -= tot;
        } else {
            sq = i < ns;
        }
        nsq += sq;
        *idx = sq ? nsq - 1 : i - nsq;
        ++i;
        return sq;
    }
};

// x / d for 0 <= x < 2^24 through a float reciprocal (inv = 1 / d), corrected
// to the exact quotient.
__device__ __forceinline__ int fdiv(int x, int d, float inv) {
    int q = __float2int_rz(__int2float_rn(x) * inv);
    const int r = x - q * d;
    q += (r >= d) - (r < 0);
    return q;
}

// Profiling aid (option trace=1): globaltimer stamps of CTA (0, 0), one
// region of kFireTraceN (code << 32 | index, time) pairs per role.
__device__ __forceinline__ void stamp(const FireParams& P, int role, int& n, int code, int idx) {
    if (!P.trace || blockIdx.x != 0 || blockIdx.y != 0 || n >= kFireTraceN) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    unsigned long long* e = P.trace + (size_t(role) * kFireTraceN + n++) * 2;
    e[0] = (unsigned long long)code << 32 | unsigned(idx);
    e[1] = t;
}

__device__ __forceinline__ uint4 ld_shared_u4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}

__device__ __forceinline__ float4 ld_shared_f4(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

template <class T, int CPS>
__global__ void __launch_bounds__(Cfg<CPS>::kThreads, CPS) fire_kernel(const __grid_constant__ FireParams P, int n0, int count) {
    constexpr int kEpi = Cfg<CPS>::kEpi, kProd = Cfg<CPS>::kProd, kMma = Cfg<CPS>::kMma, kTmemCols = Cfg<CPS>::kTmemCols;
    constexpr int NGR = Cfg<CPS>::kGroups;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[kFireStages], empty[kFireStages], sqf[2], sqe[2], exf[kFireMaxExSlots], exe[kFireMaxExSlots],
        plf[2], ple[2], wbar;
    __shared__ uint32_t tmem_slot;
    constexpr int cpc = FElem<T>::cpc;
    const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
    const int g = blockIdx.y;
    const int units = P.G > 1 ? (count + P.G - 1) / P.G : count * P.bands;
    const int nu = int(blockIdx.x) < units ? (units - 1 - int(blockIdx.x)) / int(gridDim.x) + 1 : 0;
    const int rounds = nu == 0 ? 0 : P.nplane == 2 ? nu + 1 : nu;
    const int NE = P.nexslots;
    const int JW = (P.per_op ? 1 : P.nops) * P.gch;  // TMEM columns of one expand job (every op of one M tile, or one op)
    const int nj = P.per_op ? P.nops : 1;             // expand jobs per M tile
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int s = 0; s < P.nst; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
        for (int a = 0; a < 2; ++a) mbar_init(&sqf[a], 1), mbar_init(&sqe[a], kEpi / 32), mbar_init(&plf[a], kEpi / 32), mbar_init(&ple[a], 1);
        for (int a = 0; a < NE; ++a) mbar_init(&exf[a], 1), mbar_init(&exe[a], kEpi / 32);
        mbar_init(&wbar, 1);
        mbar_fence_init();
    }
    if (warp == kMma) tmem_alloc(&tmem_slot, uint32_t(kTmemCols));
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t ring = smem_u32(smem + P.ring_off), plane0 = smem_u32(smem + P.plane_off);
    const uint32_t PS = uint32_t(P.plane_cells) * 16u;  // bytes between the 16-byte channel chunks of a plane
    const uint32_t exc0 = 2u * uint32_t(P.sq_cols);      // first expand accumulator column

    if (warp == kProd) {
        if (lane == 0) {
            const uint32_t sqb = P.sq_stream ? 0u : uint32_t(P.ksteps) * uint32_t(P.S) * 32u;  // resident squeeze weights
            uint32_t wb = sqb;
            for (int o = 0; o < P.nops; ++o) wb += uint32_t(P.op[o].gwb);
            mbar_expect_tx(&wbar, wb);
            for (uint32_t o = 0; o < sqb; o += 65536) bulk_g2s(smem + P.wsq_off + o, P.wsq + o, min(65536u, sqb - o), &wbar);
            for (int k = 0; k < P.nops; ++k) {
                const uint32_t b = uint32_t(P.op[k].gwb);
                const uint8_t* src = P.op[k].w + P.op[k].gwb * g;
                for (uint32_t o = 0; o < b; o += 65536) bulk_g2s(smem + P.op[k].w_off + o, src + o, min(65536u, b - o), &wbar);
            }
            asm volatile("griddepcontrol.wait;" ::: "memory");  // the input is the previous step's output
            const int kc_elems = P.cb / P.es;
            const int kpc = P.cb / 32;                  // K steps per chunk
            const uint32_t abytes = 128u * uint32_t(P.cb);  // input bytes per stage
            int it = 0, tn = 0;
            for (int k = 0; k < nu; ++k) {  // squeeze tiles in unit order (every round order keeps them in it)
                const Unit U = unit_of(P, int(blockIdx.x) + k * int(gridDim.x), n0, count);
                for (int ts = 0; ts < P.Ts; ++ts)
                    for (int kc = 0; kc < P.kchunks; ++kc, ++it) {
                        const int s = it % P.nst;
                        if (it >= P.nst) mbar_sleep_wait(&empty[s], uint32_t(it / P.nst - 1) & 1u);
                        stamp(P, 2, tn, 50, it);
                        uint8_t* stage = smem + P.ring_off + s * P.stage_bytes;
                        if (P.sq_stream) {  // this K chunk's squeeze weights ride along with the input chunk
                            const uint32_t b = uint32_t(min(kpc, P.ksteps - kc * kpc)) * uint32_t(P.S) * 32u;
                            mbar_expect_tx(&full[s], abytes + b);
                            bulk_g2s(stage + abytes, P.wsq + size_t(kc) * kpc * P.S * 32, b, &full[s]);
                        } else {
                            mbar_expect_tx(&full[s], abytes);
                        }
                        tma_2d(stage, &P.amap, P.coff_in + kc * kc_elems, U.p0 + ts * 128, &full[s]);
                    }
            }
        }
    } else if (warp == kMma) {
        // One elected thread issues every MMA.  Everything the loops need is
        // hoisted into registers first and descriptors advance by deltas in
        // the 16-byte start-address field, so an MMA costs a few
        // uniform-datapath instructions (recomputing descriptors per MMA made
        // the issue loop, not the tensor pipe, the limit).
        if (elect_one()) {
            mbar_sleep_wait(&wbar, 0);
            const uint32_t idsq = FElem<T>::idesc(P.S), idex = FElem<T>::idesc(P.gch);
            const uint64_t bsq0 = sdesc(smem_u32(smem + P.wsq_off), uint32_t(P.S) * 16u, 128u, kNoSwizzle);
            const uint32_t bsq_step = (uint32_t(P.S) * 32u) >> 4;
            const uint64_t ring0 = P.cb == 128 ? sdesc(ring, 16u, 1024u, kSW128) : sdesc(ring, 16u, 512u, kSW64);
            const uint64_t bsq_ring = sdesc(ring + 128u * uint32_t(P.cb), uint32_t(P.S) * 16u, 128u, kNoSwizzle);
            const int kpc = P.cb / 32;  // K steps per input chunk
            const int nst = P.nst, kchunks = P.kchunks, ksteps = P.ksteps, Ts = P.Ts, nops = P.nops, gch = P.gch, Wp = P.Wp;
            const int nks = P.schunks / 2;                        // expand K steps per tap
            const uint32_t da = (2u * PS) >> 4, db = 2u * uint32_t(gch);  // next K step: A (two plane chunks), B
            // per op: taps, weights descriptor, first tap's cell shift
            int okh[kFireMaxOps], okw[kFireMaxOps], osh[kFireMaxOps];
            uint64_t ob[kFireMaxOps];
#pragma unroll
            for (int o = 0; o < kFireMaxOps; ++o) {
                const bool on = o < nops;
                okh[o] = on ? P.op[o].kh : 0, okw[o] = on ? P.op[o].kw : 0;
                osh[o] = on ? -P.op[o].pad * Wp - P.op[o].pad : 0;
                ob[o] = sdesc(smem_u32(smem + (on ? P.op[o].w_off : 0)), uint32_t(gch) * 16u, 128u, kNoSwizzle);
            }
            // expand A of tile 0 at shift 0: output cell Wp (+1 slack cell)
            const uint64_t aplane0 = sdesc(plane0 + uint32_t(1 + Wp) * 16u, PS, 128u, kNoSwizzle);
            const uint32_t plane_step = uint32_t(P.plane_bytes) >> 4;
            int it = 0, sq_cnt = 0, ex_cnt = 0, tn = 0;
            for (int r = 0; r < rounds; ++r) {
                const Round R = round_of(P, r, nu);
                const int pl = R.ex >= 0 ? R.ex % P.nplane : 0;
                const uint64_t aplane = aplane0 + uint64_t(pl) * plane_step;
                bool waited = false;
                Jobs J(P, R);
                for (int i = 0; i < R.ns + R.ne; ++i) {
                    int idx;
                    if (J.next(&idx)) {  // squeeze tile: M = 128 pixels, N = S, K = input channels
                        const int a = sq_cnt & 1;
                        stamp(P, 0, tn, 11, sq_cnt);
                        if (sq_cnt >= 2) mbar_wait(&sqe[a], uint32_t((sq_cnt >> 1) - 1) & 1u);
                        fence_after();
                        stamp(P, 0, tn, 21, sq_cnt);
                        const uint32_t d = tmem + uint32_t(a * P.sq_cols);
                        uint32_t acc = 0;
                        uint64_t bd = bsq0;
                        for (int kc = 0; kc < kchunks; ++kc, ++it) {
                            const int s = it % nst;
                            mbar_wait(&full[s], uint32_t(it / nst) & 1u);
                            fence_after();
                            const int steps = min(kpc, ksteps - kc * kpc);
                            uint64_t ad = ring0 + uint64_t(s * (P.stage_bytes >> 4));
                            if (P.sq_stream) bd = bsq_ring + uint64_t(s * (P.stage_bytes >> 4));  // this chunk's weights in the stage
                            for (int kk = 0; kk < steps; ++kk) {
                                FElem<T>::mma(d, ad, bd, idsq, acc);
                                acc = 1;
                                ad += 2;  // +32 bytes inside the swizzle row
                                bd += bsq_step;
                            }
                            commit(&empty[s]);
                        }
                        commit(&sqf[a]);
                        stamp(P, 0, tn, 31, sq_cnt);
                        ++sq_cnt;
                        (void)Ts;
                    } else {  // expand tile idx: every op, every tap, A = the plane at a shifted start
                        stamp(P, 0, tn, 12, ex_cnt);
                        if (!waited) {
                            mbar_wait(&plf[pl], uint32_t(R.ex / P.nplane) & 1u);
                            waited = true;
                        }
                        const int a = ex_cnt % NE;
                        if (ex_cnt >= NE) mbar_wait(&exe[a], uint32_t(ex_cnt / NE - 1) & 1u);
                        fence_after();
                        stamp(P, 0, tn, 22, ex_cnt);
                        const int te = idx / nj, o0 = idx - te * nj;  // per-op jobs: op o0 of tile te; else every op
                        const uint64_t ajob = aplane + uint64_t(te * 128);
                        const uint32_t dj = tmem + exc0 + uint32_t(a * JW);
#pragma unroll
                        for (int o = 0; o < kFireMaxOps; ++o) {
                            if (o >= nops) break;
                            if (nj > 1 && o != o0) continue;
                            const uint32_t d = dj + uint32_t((nj > 1 ? 0 : o) * gch);
                            uint64_t arow = ajob + uint64_t(int64_t(osh[o]));  // shift >= -(Wp + 1): no borrow out of the field
                            uint64_t bd = ob[o];
                            uint32_t acc = 0;
                            for (int ky = 0; ky < okh[o]; ++ky, arow += uint64_t(Wp)) {
                                uint64_t atap = arow;
                                for (int kx = 0; kx < okw[o]; ++kx, ++atap) {
                                    uint64_t ad = atap;
                                    for (int kk = 0; kk < nks; ++kk) {
                                        FElem<T>::mma(d, ad, bd, idex, acc);
                                        acc = 1;
                                        ad += da;
                                        bd += db;
                                    }
                                }
                            }
                        }
                        commit(&exf[a]);
                        stamp(P, 0, tn, 32, ex_cnt);
                        ++ex_cnt;
                    }
                }
                if (R.ex >= 0) commit(&ple[pl]);  // every MMA reading this plane has completed
            }
        }
        __syncwarp();
    } else {
        // ---------------------------------------------------------------- epilogue warps
        // TMEM lane (M row); column chunks / segments of this warp: index % NGR == half
        const int t = threadIdx.x & 127, half = threadIdx.x >> 7;
        float* sqbias = reinterpret_cast<float*>(smem + P.sqbias_off);
        for (int c = threadIdx.x; c < P.S; c += kEpi) sqbias[c] = __ldg(P.sq_bias + c);
        for (int o = 0; o < P.nops; ++o) {
            float* b = reinterpret_cast<float*>(smem + P.op[o].bias_off);
            for (int c = threadIdx.x; c < P.gch; c += kEpi) b[c] = g * P.gch + c < P.op[o].cout ? __ldg(P.op[o].bias + g * P.gch + c) : 0.0f;
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("bar.sync 1, %0;\n" ::"n"(kEpi) : "memory");
        const uint32_t tl = uint32_t(t & ~31) << 16;
        const int Rp = P.R + 1;
        const int prows = P.G * Rp + 1;  // plane rows of a unit
        const float iWp = __frcp_rn(float(P.Wp)), iRp = __frcp_rn(float(Rp)), iHW = __frcp_rn(float(P.HW)), iW = __frcp_rn(float(P.W)),
                    iSC = __frcp_rn(float(P.schunks));
        const int SEG = P.seg;                            // store segment: columns of one op per warp pass
        const int spo = P.gch / SEG;                      // segments per op
        const int pieces = SEG * int(sizeof(T)) / 16;     // 16-byte pieces of a cell's segment (4 or 8)
        const int RB = pieces * 16;                       // staging row bytes
        const int rshift = pieces == 8 ? 0 : 1;           // swizzle key = (cell >> rshift) & (pieces - 1): conflict-free both ways
        const int skey = (lane >> rshift) & (pieces - 1);
        const bool staged = P.stage_off >= 0;            // else direct 16-byte stores (shared memory did not fit the staging rows)
        const uint32_t stg = smem_u32(smem + max(P.stage_off, 0)) + uint32_t(warp) * 4096u;  // this warp's staging rows
        const uint32_t sqb_s = smem_u32(sqbias);
        int sq_cnt = 0, ex_cnt = 0, tn = 0;
        const bool tr = threadIdx.x == 0;
        for (int r = 0; r < rounds; ++r) {
            const Round R = round_of(P, r, nu);
            const Unit Us = unit_of(P, int(blockIdx.x) + max(R.sq, 0) * int(gridDim.x), n0, count);
            const Unit Ue = unit_of(P, int(blockIdx.x) + max(R.ex, 0) * int(gridDim.x), n0, count);
            const int pls = max(R.sq, 0) % P.nplane;
            const uint32_t pbs = plane0 + uint32_t(pls * P.plane_bytes);
            Jobs J(P, R);
            for (int i = 0; i < R.ns + R.ne; ++i) {
                int idx;
                if (J.next(&idx)) {  // ------------------------------ squeeze tile idx of unit R.sq
                    if (idx == 0) {
                        if (R.sq >= P.nplane) mbar_sleep_wait(&ple[pls], uint32_t(R.sq / P.nplane - 1) & 1u);  // expand of unit sq - nplane done
                        // The zero cells of this unit's plane: the zero column of every
                        // row (+ the row after the last: the (+1, +1) tap of the last
                        // pixel of the last row reads it), and the rows of image rows -1 / H.
                        const uint4 z = make_uint4(0, 0, 0, 0);
                        for (int id = threadIdx.x; id < (prows + 1) * P.schunks; id += kEpi) {
                            const int pr = fdiv(id, P.schunks, iSC), ch = id - pr * P.schunks;
                            st_shared16(pbs + uint32_t(ch) * PS + uint32_t(pr * P.Wp + 1) * 16u, z);
                        }
                        // zero rows: multi-image units every Rp-th row; bands row 0 (r0 = 0)
                        // and the row of image row H (if inside the plane)
                        int zr0 = -1, zr1 = -1, nzr;
                        if (P.G > 1) nzr = P.G + 1;
                        else {
                            if (Us.r0 == 0) zr0 = 0;
                            if (P.H - Us.r0 + 1 <= Rp) zr1 = P.H - Us.r0 + 1;
                            nzr = 2;
                        }
                        const int rowitems = P.Wp * P.schunks;
                        for (int id = threadIdx.x; id < nzr * rowitems; id += kEpi) {
                            const int k = id >= rowitems ? (P.G > 1 ? fdiv(id, rowitems, __frcp_rn(float(rowitems))) : 1) : 0;
                            const int rem = id - k * rowitems;
                            const int ch = fdiv(rem, P.Wp, iWp), cc = rem - ch * P.Wp;
                            const int pr = P.G > 1 ? k * Rp : (k == 0 ? zr0 : zr1);
                            if (pr >= 0) st_shared16(pbs + uint32_t(ch) * PS + uint32_t(pr * P.Wp + cc + 1) * 16u, z);
                        }
                    }
                    const int a = sq_cnt & 1;
                    if (tr) stamp(P, 1, tn, 41, sq_cnt);
                    mbar_sleep_wait(&sqf[a], uint32_t(sq_cnt >> 1) & 1u);
                    fence_after();
                    if (tr) stamp(P, 1, tn, 51, sq_cnt);
                    const int p = Us.p0 + idx * 128 + t;
                    int cell = -1;  // plane cell of this thread's pixel (-1: outside the unit)
                    if (p < Us.p1) {
                        const int lp = p - Us.nA * P.HW;  // pixel index inside the unit's first image
                        const int n = fdiv(lp, P.HW, iHW), rem = lp - n * P.HW;
                        const int rw = fdiv(rem, P.W, iW), c = rem - rw * P.W;
                        cell = (n * Rp + (rw - Us.r0 + 1)) * P.Wp + c + 1;
                    }
                    for (int c0 = 32 * half; c0 < P.S; c0 += 32 * NGR) {  // 32-column chunks of the squeeze, alternating between warp groups
                        const int nc = min(32, P.S - c0);
                        float v[32];
                        if (nc == 32) tmem_ld32(tmem + tl + uint32_t(a * P.sq_cols + c0), v);
                        else tmem_ld16(tmem + tl + uint32_t(a * P.sq_cols + c0), v);
                        if (cell >= 0) {
                            const uint32_t dst = pbs + uint32_t(c0 / cpc) * PS + uint32_t(cell + 1) * 16u;
#pragma unroll
                            for (int j = 0; j < 32; j += 8) {
                                if (j >= nc) break;
                                const float4 b0 = ld_shared_f4(sqb_s + uint32_t(c0 + j) * 4u), b1 = ld_shared_f4(sqb_s + uint32_t(c0 + j + 4) * 4u);
                                float w[8] = {v[j] + b0.x, v[j + 1] + b0.y, v[j + 2] + b0.z, v[j + 3] + b0.w,
                                              v[j + 4] + b1.x, v[j + 5] + b1.y, v[j + 6] + b1.z, v[j + 7] + b1.w};
                                if (P.sq_relu)
#pragma unroll
                                    for (int e = 0; e < 8; ++e) w[e] = fmaxf(w[e], 0.0f);
#pragma unroll
                                for (int h = 0; h < 8; h += cpc) st_shared16(dst + uint32_t((j + h) / cpc) * PS, FElem<T>::pack(w + h));
                            }
                        }
                    }
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sqe[a]);
                    ++sq_cnt;
                    if (idx == P.Ts - 1) {
                        fence_async_smem();  // plane writes -> visible to the MMAs (async proxy)
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&plf[pls]);
                    }
                } else {  // ---------------------------------------------------- expand job idx of unit R.ex
                    const int te = idx / nj, o0 = idx - te * nj;  // M tile; op of a per-op job
                    const int q = P.Wp + te * 128 + t;
                    const int pr = fdiv(q, P.Wp, iWp), cc = q - pr * P.Wp;
                    const int ii = fdiv(pr, Rp, iRp), rr = pr - ii * Rp, ir = Ue.r0 + rr - 1;
                    const bool valid = cc >= 1 && ii < Ue.ni && rr >= 1 && ir < P.H;
                    const long long pix = (long long)((Ue.nA + ii) * P.H + ir) * P.W + (cc - 1);
                    const int a = ex_cnt % NE;
                    if (tr) stamp(P, 1, tn, 42, ex_cnt);
                    mbar_sleep_wait(&exf[a], uint32_t(ex_cnt / NE) & 1u);
                    fence_after();
                    if (tr) stamp(P, 1, tn, 52, ex_cnt);
                    // Stores go through a per-warp staging row: each thread writes
                    // its cell's segment (SEG channels) to shared memory, then the
                    // warp stores whole segments -- 32 / pieces cells per
                    // instruction, every 16-byte piece of a cell by its own lane --
                    // instead of 32 cells' 16-byte fragments per instruction.
                    if (!staged) {
                        // direct stores: this warp's 32-column chunks of the job (global
                        // chunk index of parity `half`), two TMEM loads in flight per pass
                        // (TMEM reads are latency-bound per warp: one wait for both)
                        T* dst[kFireMaxOps];
#pragma unroll
                        for (int o = 0; o < kFireMaxOps; ++o)
                            dst[o] = valid && o < P.nops ? static_cast<T*>(P.op[o].out) + pix * P.op[o].out_cstride + P.op[o].out_coff + g * P.gch
                                                         : nullptr;
                        const int nch = JW / 32;
                        const uint32_t tj = tmem + tl + exc0 + uint32_t(a * JW);
                        const bool st32 = P.st32 != 0;
                        for (int cb = half; cb < nch; cb += 2 * NGR) {
                            const bool two = cb + NGR < nch;
                            uint32_t r0[32], r1[32];
                            tmem_ld32_issue(tj + uint32_t(cb * 32), r0);
                            if (two) tmem_ld32_issue(tj + uint32_t((cb + NGR) * 32), r1);
                            tmem_ld_wait32(r0);
                            if (two) tmem_ld_wait32(r1);
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                if (u == 1 && !two) break;
                                int o = nj > 1 ? o0 : 0, c0 = (cb + NGR * u) * 32;
                                while (c0 >= P.gch) c0 -= P.gch, ++o;
                                const FireOp& op = P.op[o];
                                const uint32_t bsm = smem_u32(smem + op.bias_off) + uint32_t(c0) * 4u;
                                T* d = dst[0];
#pragma unroll
                                for (int oo = 1; oo < kFireMaxOps; ++oo)
                                    if (o == oo) d = dst[oo];
                                const bool relu = op.relu;
                                // 32-byte stores: 2 x 16-byte packs per 32-byte piece (16 bf16 / 8 fp32 channels)
                                constexpr int JP = 2 * cpc;  // channels per 32-byte piece
#pragma unroll
                                for (int j = 0; j < 32; j += JP) {
                                    const uint32_t* r = u ? r1 : r0;
                                    uint4 pk[2];
#pragma unroll
                                    for (int hh = 0; hh < 2; ++hh) {
                                        const int jj = j + hh * cpc;
                                        float w[cpc];
#pragma unroll
                                        for (int e = 0; e < cpc; e += 4) {
                                            const float4 b4 = ld_shared_f4(bsm + uint32_t(jj + e) * 4u);
                                            w[e] = __uint_as_float(r[jj + e]) + b4.x, w[e + 1] = __uint_as_float(r[jj + e + 1]) + b4.y;
                                            w[e + 2] = __uint_as_float(r[jj + e + 2]) + b4.z, w[e + 3] = __uint_as_float(r[jj + e + 3]) + b4.w;
                                        }
                                        if (relu)
#pragma unroll
                                            for (int e = 0; e < cpc; ++e) w[e] = fmaxf(w[e], 0.0f);
                                        pk[hh] = FElem<T>::pack(w);
                                    }
                                    if (d) {
                                        if (st32) st_global32(d + c0 + j, pk[0], pk[1]);
                                        else *reinterpret_cast<uint4*>(d + c0 + j) = pk[0], *reinterpret_cast<uint4*>(d + c0 + j + cpc) = pk[1];
                                    }
                                }
                            }
                        }
                    } else {
                        const int cpl = 32 / pieces;  // cells per store instruction
                        for (int o = 0; o < P.nops; ++o) {
                            if (nj > 1 && o != o0) continue;
                            const FireOp& op = P.op[o];
                            const uint32_t bsm = smem_u32(smem + op.bias_off);
                            const int ocol = nj > 1 ? 0 : o;  // the op's column block inside the job
                            T* dsto = valid ? static_cast<T*>(op.out) + pix * op.out_cstride + op.out_coff + g * P.gch : nullptr;
                            for (int k = NGR == 1 ? 0 : (half + o * spo) & 1; k < spo; k += NGR) {  // segments of the op whose global index has this parity
                                const int c0 = k * SEG;
                                for (int h = 0; h < SEG; h += 32) {
                                    float v[32];
                                    tmem_ld32(tmem + tl + exc0 + uint32_t(a * JW + ocol * P.gch + c0 + h), v);
    #pragma unroll
                                    for (int j = 0; j < 32; j += 8) {
                                        const float4 b0 = ld_shared_f4(bsm + uint32_t(c0 + h + j) * 4u), b1 = ld_shared_f4(bsm + uint32_t(c0 + h + j + 4) * 4u);
                                        float w[8] = {v[j] + b0.x, v[j + 1] + b0.y, v[j + 2] + b0.z, v[j + 3] + b0.w,
                                                      v[j + 4] + b1.x, v[j + 5] + b1.y, v[j + 6] + b1.z, v[j + 7] + b1.w};
                                        if (op.relu)
    #pragma unroll
                                            for (int e = 0; e < 8; ++e) w[e] = fmaxf(w[e], 0.0f);
    #pragma unroll
                                        for (int e = 0; e < 8; e += cpc) {
                                            if (staged) {
                                                const int pc = (h + j + e) / cpc;  // piece of this cell's segment
                                                st_shared16(stg + uint32_t(lane * RB + ((pc ^ skey) << 4)), FElem<T>::pack(w + e));
                                            } else if (dsto) {
                                                *reinterpret_cast<uint4*>(dsto + c0 + h + j + e) = FElem<T>::pack(w + e);
                                            }
                                        }
                                    }
                                }
                                if (!staged) continue;
                                __syncwarp();
    #pragma unroll 4
                                for (int m = 0; m < 32; m += cpl) {
                                    const int c = m + lane / pieces, q = lane % pieces;
                                    const unsigned long long dp = __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dsto), c);
                                    const int key = (c >> rshift) & (pieces - 1);
                                    const uint4 val = ld_shared_u4(stg + uint32_t(c * RB + ((q ^ key) << 4)));
                                    if (dp) *reinterpret_cast<uint4*>(reinterpret_cast<T*>(dp) + c0 + q * cpc) = val;
                                }
                                __syncwarp();
                            }
                        }
                    }
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&exe[a]);
                    if (tr) stamp(P, 1, tn, 62, ex_cnt);
                    ++ex_cnt;
                }
            }
        }
    }
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == kMma) tmem_free(tmem, uint32_t(kTmemCols));
}

template <class T, int CPS>
cudaError_t launch_t(const FireParams& P, int n0, int count, cudaStream_t st) {
    static bool init = false;
    if (!init) {
        cudaError_t e = cudaFuncSetAttribute(fire_kernel<T, CPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFireSmemMax);
        if (e != cudaSuccess) return e;
        init = true;
    }
    const int units = P.G > 1 ? (count + P.G - 1) / P.G : count * P.bands;
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int gx = std::max(1, std::min(units, CPS * sms / std::max(1, P.nsplit)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(gx), unsigned(std::max(1, P.nsplit)), 1u), cfg.blockDim = dim3(Cfg<CPS>::kThreads);
    cfg.dynamicSmemBytes = size_t(P.smem_bytes), cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = P.pdl ? 1 : 0;
    cfg.attrs = attr, cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, fire_kernel<T, CPS>, P, n0, count);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_fire(const FireParams& P, int n0, int count, cudaStream_t st) {
    if (P.cps == 2) return P.es == 4 ? launch_t<float, 2>(P, n0, count, st) : launch_t<__nv_bfloat16, 2>(P, n0, count, st);
    return P.es == 4 ? launch_t<float, 1>(P, n0, count, st) : launch_t<__nv_bfloat16, 1>(P, n0, count, st);
}

}  // namespace xlf
