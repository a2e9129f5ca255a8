#include "engine.hpp"

#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <set>
#include <tuple>

#include "tc_params.hpp"
#include "stem_params.hpp"
#include "pw_params.hpp"
#include "fire_params.hpp"
#include "dw_params.hpp"
#include "common.hpp"
#include "fused_params.hpp"

namespace xlf {

// kernels_fp32.cu
cudaError_t init_fused_fp32();
cudaError_t launch_fused_fp32(const FusedParams& P, int batch, bool exact, cudaStream_t st);
cudaError_t launch_concat_copy(const float* src, int scs, int sco, float* dst, int dcs, int dco, int C, long long pixels, cudaStream_t st);
cudaError_t launch_eltwise(int op, const float* a, int acs, int aco, const float* b, int bcs, int bco, float* o, int ocs, int oco,
                           int C, long long pixels, cudaStream_t st);
cudaError_t launch_nchw_to_nhwc(const float* src, float* dst, int N, int C, int H, int W, int cs, cudaStream_t st);
cudaError_t launch_nhwc_to_nchw(const float* src, int cs, int coff, float* dst, int N, int C, int H, int W, cudaStream_t st);
cudaError_t launch_seeded_nhwc(float* dst, unsigned long long seed, unsigned long long first_image, int N, int C, int H, int W,
                               int cs, cudaStream_t st);
// kernels_tc.cu (es = element bytes: 2 bf16, 4 fp32/TF32)
cudaError_t init_fused_tc();
cudaError_t launch_fused_tc(const BParams& P, int batch, cudaStream_t st, int n0);
int occupancy_fused_tc(int smem_bytes, int tmem_cols, int epi_warps, int kind, int es);
int step_kind_tc(const BParams& P);
cudaError_t launch_gap_finish_tc(int es, const float* part, int tiles, int np, float scale, void* out, int cs, int coff, int C, int n0, int N,
                                 cudaStream_t st);
cudaError_t launch_nchw_to_nhwc_tc(int es, const float* src, void* dst, int N, int C, int H, int W, int cs, cudaStream_t st);
cudaError_t launch_nhwc_tc_to_nchw(int es, const void* src, int cs, int coff, float* dst, int N, int C, int H, int W, cudaStream_t st);
cudaError_t launch_seeded_nhwc_tc(int es, void* dst, unsigned long long seed, unsigned long long first_image, int N, int C, int H, int W,
                                  int cs, cudaStream_t st);
cudaError_t launch_s2d_tc(int es, const float* src, unsigned long long seed, unsigned long long first_image, void* dst, int N, int C, int H,
                          int W, int cs, int planar, cudaStream_t st);
cudaError_t launch_concat_copy_tc(int es, const void* src, int scs, int sco, void* dst, int dcs, int dco, int C, long long pixels,
                                  cudaStream_t st);
// kernels_stem.cu
cudaError_t launch_stem(const StemParams& P, int batch, cudaStream_t st, int n0);
// kernels_pw.cu
cudaError_t launch_pw(const PwParams& P, int n0, int count, cudaStream_t st);
cudaError_t launch_fire(const FireParams& P, int n0, int count, cudaStream_t st);
cudaError_t launch_dw(const DwParams& P, int n0, int count, cudaStream_t st);
int fire_layout(FireParams& P, int nst, int nplane, bool staged);
void fire_shape(const Graph& g, const StepSpec& s, int es, FireParams& P);
bool fire_choose(FireParams& P, int batch, int sms, int force_nsplit, int force_g, int force_r, double* model_out);
std::vector<std::pair<double, FireParams>> fire_candidates(const FireParams& P, int batch, int sms, int force_nsplit, int force_g, int force_r);
cudaError_t launch_pw_gap_finish(const PwParams& P, int C, float scale, void* out, int cs, int coff, int n0, int count, cudaStream_t st);
cudaError_t launch_eltwise_tc(int es, int op, const void* a, int acs, int aco, const void* b, int bcs, int bco, void* o, int ocs, int oco, int C,
                              long long pixels, cudaStream_t st);

const char* to_string(Precision p) {
    switch (p) {
    case Precision::fp32_exact: return "fp32_exact";
    case Precision::fp32: return "fp32";
    case Precision::bf16: return "bf16";
    case Precision::tf32: return "tf32";
    }
    return "?";
}

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(ErrorKind::cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

float seeded_value(uint64_t seed, uint64_t i) {
    uint64_t z = (seed ? seed : 0x9e3779b97f4a7c15ULL) + (i + 1) * 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    return static_cast<float>(z >> 40) * (1.0f / 16777216.0f) - 0.5f;
}

std::vector<float> seeded_weights(const Graph& g, uint64_t seed) {
    const uint64_t ws = seed ^ 0xabcdef1234567890ULL;
    std::vector<float> out;
    for (const Layer& l : g.layers) {
        if (l.kind != LayerKind::conv) continue;
        if (l.conv->in_channels <= 0) fail(ErrorKind::internal, "seeded_weights: run infer_shapes first (layer '" + l.name + "')");
        const size_t n = size_t(l.conv->weight_count() + l.conv->bias_count());
        const size_t base = out.size();
        out.resize(base + n);
        for (size_t i = 0; i < n; ++i) out[base + i] = seeded_value(ws, base + i);
    }
    return out;
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        cuda_check(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q), "cuTensorMapEncodeTiled lookup");
        if (q != cudaDriverEntryPointSuccess || !p) fail(ErrorKind::cuda, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 4-D map over an NHWC tensor {cstride, W, H, N} of `es`-byte elements; box =
// one K-block (16 bytes per cell unswizzled, 32 with SWIZZLE_32B, 128 with
// SWIZZLE_128B) of an ext_h x ext_w region, zero fill outside the image.
void encode_region_map(CUtensorMap* map, const void* base, int cstride, int W, int H, int N, const BRegion& r, int es) {
    const cuuint64_t dims[4] = {cuuint64_t(cstride), cuuint64_t(W), cuuint64_t(H), cuuint64_t(N)};
    const cuuint64_t strides[3] = {cuuint64_t(cstride) * es, cuuint64_t(W) * cstride * es, cuuint64_t(H) * W * cstride * es};
    const cuuint32_t box[4] = {cuuint32_t(r.kb_ch), cuuint32_t(r.ext_w), cuuint32_t(r.ext_h), 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUtensorMapSwizzle sw = r.mode == kSw128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : r.mode == kSw32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                    : CU_TENSOR_MAP_SWIZZLE_NONE;
    const CUresult res = tensor_map_encoder()(map, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) fail(ErrorKind::cuda, "cuTensorMapEncodeTiled failed (" + std::to_string(int(res)) + ")");
}

// Tensor-core plans: a stride-2, pad-0 conv reading the graph input (SqueezeNet conv1:
// 3x3/2 on 3 channels) cannot use the stride-1 implicit GEMM.  Rewrite it as a
// stride-1 ceil(k/2) x ceil(k/2) conv over the space-to-depth input
// (4 phases x C channels, padded to 16): out(y,x) = sum over phase (py,px),
// tap (ty,tx) of in(2(y+ty)+py, 2(x+tx)+px) * W[2ty+py][2tx+px]; identical
// sums, so the conv runs on tensor cores.  Returns false when not applicable.
bool rewrite_s2d(Graph& g, std::vector<float>& w) {
    if (g.inputs.size() != 1) return false;
    const GraphInput in = g.inputs[0];
    const int C = in.shape.channels;
    if (4 * C > 16 || in.shape.height % 2 || in.shape.width % 2) return false;
    const auto readers = g.consumers_of(in.name);
    if (readers.size() != 1) return false;
    Layer* l = g.find_layer(readers[0]);
    if (l->kind != LayerKind::conv || l->conv->stride != 2 || l->conv->pad != 0 || l->conv->group != 1 || l->conv->kernel_h > 4 ||
        l->conv->kernel_w > 4)
        return false;
    // new weights for this layer (save_weights order: filter then bias, layers in file order)
    size_t off = 0;
    for (const Layer& x : g.layers) {
        if (&x == l) break;
        if (x.kind == LayerKind::conv) off += size_t(x.conv->weight_count() + x.conv->bias_count());
    }
    const ConvParams c = *l->conv;
    const int kh2 = (c.kernel_h + 1) / 2, kw2 = (c.kernel_w + 1) / 2, cin2 = 16;
    std::vector<float> f2(size_t(c.out_channels) * cin2 * kh2 * kw2, 0.0f);
    for (int oc = 0; oc < c.out_channels; ++oc)
        for (int ci = 0; ci < C; ++ci)
            for (int ky = 0; ky < c.kernel_h; ++ky)
                for (int kx = 0; kx < c.kernel_w; ++kx) {
                    const int ph = (ky % 2) * 2 + kx % 2, ty = ky / 2, tx = kx / 2;
                    f2[((size_t(oc) * cin2 + ph * C + ci) * kh2 + ty) * kw2 + tx] =
                        w[off + ((size_t(oc) * C + ci) * c.kernel_h + ky) * c.kernel_w + kx];
                }
    const size_t nf = size_t(c.weight_count());
    w.erase(w.begin() + long(off), w.begin() + long(off + nf));
    w.insert(w.begin() + long(off), f2.begin(), f2.end());
    g.inputs[0].shape = {cin2, in.shape.height / 2, in.shape.width / 2};
    l->conv->kernel_h = kh2, l->conv->kernel_w = kw2, l->conv->stride = 1, l->conv->in_channels = cin2;
    const TensorShape before = *l->out_shape;
    g = infer_shapes(g);
    if (!(*g.find_layer(readers[0])->out_shape == before)) fail(ErrorKind::internal, "s2d rewrite changed the conv output shape");
    return true;
}

}  // namespace

Engine::Engine(const Graph& g, int device, Partition part, Precision prec, const float* weights, size_t nweights, int max_batch,
               const Knobs& knobs)
    : g_(g), device_(device), prec_(prec), max_batch_(max_batch), knobs_(knobs) {
    if (!g_.shapes_inferred()) fail(ErrorKind::internal, "engine: graph shapes not inferred");
    if (max_batch < 1) fail(ErrorKind::validation, "engine: max_batch must be >= 1");
    if (g_.inputs.empty()) fail(ErrorKind::validation, "engine: the graph has no input");
    tc_es_ = prec == Precision::bf16 ? 2 : prec == Precision::tf32 ? 4 : 0;
    const bool tc = tc_es_ != 0;
    esz_ = tc_es_ == 2 ? 2 : 4;
    for (const GraphInput& in : g_.inputs) user_inputs_[in.name] = in.shape;
    in_shape_ = g_.inputs[0].shape;
    const Graph user = g_;
    std::vector<float> wcopy;
    if (tc) {
        wcopy.assign(weights, weights + nweights);
        s2d_ = !knobs_.no_s2d && rewrite_s2d(g_, wcopy);
        if (s2d_) weights = wcopy.data(), nweights = wcopy.size();
    }
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    plan_ = plan_device(g_, part, max_batch, 227 * 1024, tc_es_, knobs_);
    // statistics against the user's graph (the s2d rewrite pads conv1's input
    // to 16 channels; the algorithmic bytes / MACs are the real layer's)
    if (s2d_)
        for (StepSpec& s : plan_.steps) fill_stats(user, plan_, s);
    cuda_check(tc ? init_fused_tc() : init_fused_fp32(), "kernel attributes");
    // fp32 packed weights (+ slack: bf16 epilogues read bias up to the N-block padding)
    std::vector<float> packed = pack_weights(g_, plan_, weights, nweights);
    packed.resize(packed.size() + 1024, 0.0f);
    cuda_check(cudaMalloc(&weights_, packed.size() * 4), "cudaMalloc(weights)");
    cuda_check(cudaMemcpy(weights_, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice), "weights H2D");
    if (tc) {
        host_w_.assign(weights, weights + nweights);  // N-split ops are packed per channel group on demand (packed_for)
        std::vector<uint8_t> wt = pack_weights_tc(g_, weights, nweights, wofftc_, tc_es_);
        wt.resize(wt.size() + 128, 0);
        cuda_check(cudaMalloc(&weights_tc_, wt.size()), "cudaMalloc(tensor-core weights)");
        cuda_check(cudaMemcpy(weights_tc_, wt.data(), wt.size(), cudaMemcpyHostToDevice), "tensor-core weights H2D");
    }
    for (long long f : plan_.alloc_floats) {
        void* p = nullptr;
        const size_t bytes = size_t(f) * size_t(max_batch) * esz_;
        cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(activations)");
        cuda_check(cudaMemset(p, 0, bytes), "cudaMemset");  // channel padding stays zero
        allocs_.push_back(static_cast<float*>(p));
    }
    size_t most = 0;
    for (const auto& [n, t] : plan_.tensors)
        if (t.materialized) most = std::max(most, size_t(t.C) * t.H * t.W);
    staging_floats_ = most * size_t(max_batch);
    cuda_check(cudaMalloc(&staging_, staging_floats_ * 4), "cudaMalloc(staging)");
    params_.resize(plan_.steps.size());
    bparams_.resize(plan_.steps.size());
    stems_.resize(plan_.steps.size());
    pws_.resize(plan_.steps.size());
    fires_.resize(plan_.steps.size());
    dws_.resize(plan_.steps.size());
    for (size_t i = 0; i < plan_.steps.size(); ++i) {
        const StepSpec& s = plan_.steps[i];
        if (s.kind != StepSpec::FUSED) continue;
        if (auto dp = build_dw(s)) {
            dws_[i] = std::move(dp);
            plan_.steps[i].tag = s.ops.size() == 2 ? "depthwise+pointwise" : "depthwise";
            plan_.steps[i].tile_h = dws_[i]->tile_h, plan_.steps[i].tile_w = dws_[i]->tile_w;
            plan_.steps[i].smem_bytes = dws_[i]->smem_bytes;
            continue;
        }
        if (!tc) {
            params_[i] = make_params(g_, plan_, s, allocs_, weights_);
            continue;
        }
        if (auto st = build_stem(s)) {
            stems_[i] = std::move(st);
            plan_.steps[i].tag = "stem";
            s2d_planar_ = 1;  // the stem reads the space-to-depth input row-planar (see s2d_tc)
            continue;
        }
        if (auto fp = build_fire(s)) {
            fires_[i] = std::move(fp);
            StepSpec& t = plan_.steps[i];
            t.tag = "fire";
            t.nsplit = fires_[i]->nsplit;
            t.tile_h = fires_[i]->G > 1 ? fires_[i]->G * fires_[i]->H : fires_[i]->R;  // unit: G images or an R-row band
            t.tile_w = fires_[i]->W;
            t.smem_bytes = fires_[i]->smem_bytes;
            continue;
        }
        if (auto pw = build_pw(s)) {
            pws_[i] = std::move(pw);
            plan_.steps[i].tag = s.gap_out.empty() ? "pointwise" : "pointwise+gap";
            plan_.steps[i].nsplit = pws_[i]->nsplit;
            continue;
        }
        bparams_[i] = build_bparams(s);
    }
}

// The stem kernel (kernels_stem.cu) takes a step that is exactly: the first
// conv of the graph rewritten on the space-to-depth input (stride 1, whole
// 32-byte K steps, one N block of 32 | npad <= 128 columns, output rows <= 128
// wide) -> its 3x3/2 pad-0 max-pool, the conv output not stored.  Returns
// null for any other step (the generic fused-block kernel runs it).
std::unique_ptr<StemParams> Engine::build_stem(const StepSpec& s) {
    if (!s2d_ || !tc_es_ || knobs_.no_stem || s.kind != StepSpec::FUSED || s.ops.size() != 2 || s.inputs.size() != 1 ||
        s.inputs[0] != g_.inputs[0].name)
        return nullptr;
    const OpSpec &oc = s.ops[0], &op = s.ops[1];
    const Layer& c = *g_.find_layer(oc.layer);
    const Layer& p = *g_.find_layer(op.layer);
    if (c.kind != LayerKind::conv || p.kind != LayerKind::pool || oc.stage != 1 || op.stage != 2 || oc.emit || !op.emit ||
        p.pool->kind != PoolKind::max || p.pool->kernel != 3 || p.pool->stride != 2 || p.pool->pad != 0 || !tc_mma_ok(c, tc_es_) ||
        c.conv->activation != Activation::relu)
        return nullptr;
    int nblocks = 0, nb = 0;
    tc_nblocks(c.conv->out_channels, &nblocks, &nb);
    const TensorShape in = g_.shape_of(s.inputs[0]), co = *c.out_shape, po = *p.out_shape;
    if (nblocks != 1 || (nb != 64 && nb != 128) || co.width > 128 || in.width > 256 || c.conv->kernel_h > 4 || c.conv->kernel_w > 4) return nullptr;
    auto P = std::make_unique<StemParams>();
    const TensorSlot& xt = plan_.tensors.at(s.inputs[0]);
    const TensorSlot& ot = plan_.tensors.at(p.name);
    const int cpc = 16 / tc_es_;
    P->es = tc_es_;
    P->Hin = in.height, P->Win = in.width, P->planes = xt.cstride / cpc;
    P->kh = c.conv->kernel_h, P->kw = c.conv->kernel_w;
    P->Hc = co.height, P->Wc = co.width, P->cout = co.channels, P->npad = nb;
    P->Hp = po.height, P->Wp = po.width;
    if (P->planes * cpc != c.conv->in_channels || P->planes % 2) return nullptr;
    P->wmma = static_cast<const uint8_t*>(weights_tc_) + wofftc_.at(c.name);
    P->w_bytes = P->kh * P->kw * P->planes * nb * 16;
    P->bias = weights_ + plan_.b_off.at(c.name);
    P->out = allocs_[size_t(ot.alloc)], P->out_cstride = ot.cstride, P->out_coff = ot.coff;
    // bands of pooled rows: balance units over the persistent grid at max_batch
    P->ctas_per_sm = 2;
    const long long grid = 148LL * P->ctas_per_sm;
    double best = 1e300;
    for (int br = 2; br <= std::min(P->Hp, 16); ++br) {
        const int bands = (P->Hp + br - 1) / br;
        const double t = std::ceil(double(max_batch_) * bands / grid) * (2.0 * br + 1 + 2.0);  // conv rows per band + per-band latency
        if (t < best) best = t, P->band_rows = br, P->bands = bands;
    }
    P->slots = kStemSlots;
    P->acc_slots = nb == 64 ? 4 : 2;  // as the kernel instantiation (kernels_stem.cu)
    P->tmem_cols = 32;
    while (P->tmem_cols < P->acc_slots * nb) P->tmem_cols *= 2;
    auto up = [](int v, int a) { return (v + a - 1) / a * a; };
    P->plane_bytes = in.width * 16;  // planes of a row are contiguous (row-planar input)
    P->slot_bytes = up(P->planes * P->plane_bytes, 128);
    P->ring_off = 0;
    P->w_off = up(P->slots * P->slot_bytes, 1024);
    P->stage_off = up(P->w_off + P->w_bytes, 1024);
    P->stage_bytes = 128 * nb * tc_es_;
    P->bias_off = P->stage_off + 2 * P->stage_bytes;
    P->smem_bytes = P->bias_off + nb * 4;
    if (P->smem_bytes > kStemSmemMax) return nullptr;
    P->pdl = knobs_.pdl ? 1 : 0;
    // input rows, row-planar (s2d_tc planar): one input row = row_elems contiguous
    // elements = `lines` lines of `inner` elements; the map is 2-D {inner, lines
    // of the whole batch}, one box = one input row (lines of >= 256 bytes: TMA
    // moves a box line by line, 16-byte lines would starve it)
    const long long row_elems = (long long)P->planes * in.width * cpc;
    int inner = 0;
    for (int d = 256; d >= cpc; d -= cpc)
        if (row_elems % d == 0) {
            inner = d;
            break;
        }
    if (!inner || row_elems / inner > 256) return nullptr;
    P->row_lines = int(row_elems / inner);
    const cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t((long long)max_batch_ * in.height * P->row_lines)};
    const cuuint64_t strides[1] = {cuuint64_t(inner) * tc_es_};
    const cuuint32_t box[2] = {cuuint32_t(inner), cuuint32_t(P->row_lines)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult res = tensor_map_encoder()(&P->xmap, tc_es_ == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                              allocs_[size_t(xt.alloc)], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) fail(ErrorKind::cuda, "cuTensorMapEncodeTiled (stem) failed (" + std::to_string(int(res)) + ")");
    return P;
}

// The pointwise-conv GEMM kernel (kernels_pw.cu) takes a step that is one
// 1x1 / stride-1 / pad-0 conv (optionally + global average pool): its pixels
// across images form one GEMM M dimension.  Output channels are split into
// groups whose weights stay resident (<= 128 KB per CTA).
std::unique_ptr<PwParams> Engine::build_pw(const StepSpec& s) {
    if (!tc_es_ || knobs_.no_pw || s.kind != StepSpec::FUSED || s.ops.size() != 1 || s.inputs.size() != 1) return nullptr;
    const OpSpec& op = s.ops[0];
    const Layer& l = *g_.find_layer(op.layer);
    if (op.stage != 1 || !op.emit || !tc_mma_ok(l, tc_es_) || l.conv->kernel_h != 1 || l.conv->kernel_w != 1 || l.conv->pad != 0) return nullptr;
    if (s2d_ && s.inputs[0] == g_.inputs[0].name) return nullptr;  // row-planar / rewritten input
    const TensorSlot& xt = plan_.tensors.at(s.inputs[0]);
    const int HW = xt.H * xt.W;
    const bool gap = !s.gap_out.empty();
    if (gap && HW < 32) return nullptr;
    auto P = std::make_unique<PwParams>();
    const int cpc = 16 / tc_es_, N = (l.conv->out_channels + 15) / 16 * 16;
    P->es = tc_es_, P->HW = HW, P->coff_in = xt.coff;
    P->ksteps = l.conv->in_channels * tc_es_ / 32;
    P->kchunks = (P->ksteps + 3) / 4;
    P->cout = l.conv->out_channels, P->relu = l.conv->activation == Activation::relu;
    // channel groups: the fewest whose weights fit 128 KB resident and N <= 256
    int G = 1;
    for (;; ++G) {
        const int gch = (((N + G - 1) / G) + 15) / 16 * 16;
        if (gch <= 256 && (long long)P->ksteps * gch * 32 <= 128 * 1024) {
            P->gch = gch;
            break;
        }
        if (G > 16) return nullptr;
    }
    if (knobs_.nsplit > 0) {  // testing aid: force the group count when it is valid
        const int gch = (((N + knobs_.nsplit - 1) / knobs_.nsplit) + 15) / 16 * 16;
        if (gch <= 256 && (long long)P->ksteps * gch * 32 <= 200 * 1024 && gch * (knobs_.nsplit - 1) < P->cout) G = knobs_.nsplit, P->gch = gch;
    }
    P->nsplit = G;
    // option pw_mc=1: the channel groups of an M tile as one cluster, its A
    // chunks loaded once and multicast (measured slower on conv10: 67 -> 79 us,
    // 8-CTA clusters limit the resident grid and run the groups in lock step)
    P->mc = knobs_.pw_mc && G >= 2 && G <= 8 ? G : 1;
    P->wmma = G == 1 && P->gch == [&] { int nbk, nb; tc_nblocks(l.conv->out_channels, &nbk, &nb); return nbk == 1 ? nb : -1; }()
                  ? static_cast<const uint8_t*>(weights_tc_) + wofftc_.at(l.name)
                  : packed_for(l.name, P->gch, G);
    P->gwb = (long long)P->ksteps * P->gch * 32;
    P->bias = weights_ + plan_.b_off.at(l.name);
    const std::string out_name = gap ? s.gap_out : l.name;
    const TensorSlot& ot = plan_.tensors.at(gap ? l.name : out_name);
    (void)cpc;
    if (!gap) P->out = allocs_[size_t(ot.alloc)], P->out_cstride = ot.cstride, P->out_coff = ot.coff;
    P->gap = gap;
    P->ring_off = 0;
    P->w_off = kPwStages * 128 * 128;
    P->bias_off = P->w_off + int(P->gwb);
    P->smem_bytes = P->bias_off + P->gch * 4;
    P->tmem_cols = 32;
    while (P->tmem_cols < 2 * P->gch) P->tmem_cols *= 2;
    P->ctas_per_sm = 1;  // 10 warps x ~124 registers: one CTA per SM
    P->pdl = knobs_.pdl ? 1 : 0;
    if (gap) {
        const size_t warps = size_t((max_batch_ * (long long)HW + 127) / 128) * 4;
        const size_t need = warps * 2 * size_t(G) * P->gch;
        auto& buf = gap_parts_[s.id];
        if (buf.second < need) {
            if (buf.first) retired_.push_back(buf.first);
            cuda_check(cudaMalloc(&buf.first, need * 4), "cudaMalloc(gap partials)");
            buf.second = need;
        }
        P->gap_part = buf.first;
    }
    // A: 2-D {cstride, max_batch * HW}, box = 128 bytes of channels x 128 pixels, 128-byte swizzle
    const cuuint64_t dims[2] = {cuuint64_t(xt.cstride), cuuint64_t((long long)max_batch_ * HW)};
    const cuuint64_t strides[1] = {cuuint64_t(xt.cstride) * tc_es_};
    const cuuint32_t box[2] = {cuuint32_t(128 / tc_es_), 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult res = tensor_map_encoder()(&P->amap, tc_es_ == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                              allocs_[size_t(xt.alloc)], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) fail(ErrorKind::cuda, "cuTensorMapEncodeTiled (pointwise) failed (" + std::to_string(int(res)) + ")");
    return P;
}

// The depthwise kernel (kernels_dw.cu) takes a step that is one depthwise
// conv (groups == in == out channels <= 32, <= 25 taps, stride 1 / 2) on the
// step's input, alone or followed by a 1x1 conv reading only its output (the
// depthwise output then stays in registers).  Every precision: fp32 SIMT
// arithmetic (reference order in fp32_exact), HBM tensors in the engine's
// element type.
std::unique_ptr<DwParams> Engine::build_dw(const StepSpec& s) {
    if (knobs_.no_dw || s.kind != StepSpec::FUSED || s.inputs.size() != 1 || s.ops.empty() || s.ops.size() > 2 || !s.gap_out.empty()) return nullptr;
    if (s2d_ && s.inputs[0] == g_.inputs[0].name) return nullptr;
    const OpSpec& o0 = s.ops[0];
    const Layer& d = *g_.find_layer(o0.layer);
    if (d.kind != LayerKind::conv || o0.stage != 1 || o0.xin != 0) return nullptr;
    const ConvParams& c = *d.conv;
    if (c.group != c.in_channels || c.out_channels != c.in_channels || c.in_channels > kDwMaxC || c.kernel_h * c.kernel_w > kDwMaxTaps ||
        (c.stride != 1 && c.stride != 2) || d.inputs.size() != 1 || d.inputs[0] != s.inputs[0])
        return nullptr;
    const Layer* p = nullptr;
    if (s.ops.size() == 2) {
        const OpSpec& o1 = s.ops[1];
        p = g_.find_layer(o1.layer);
        if (!p || p->kind != LayerKind::conv || o0.emit || o1.stage != 2 || !o1.emit || o1.srcs.size() != 1 || o1.srcs[0] != 0) return nullptr;
        const ConvParams& q = *p->conv;
        if (q.kernel_h != 1 || q.kernel_w != 1 || q.stride != 1 || q.pad != 0 || q.group != 1 || q.in_channels != c.out_channels) return nullptr;
    } else if (!o0.emit) {
        return nullptr;
    }
    auto P = std::make_unique<DwParams>();
    const TensorSlot& xt = plan_.tensors.at(s.inputs[0]);
    const TensorSlot& ot = plan_.tensors.at(p ? p->name : d.name);
    const TensorShape out = *d.out_shape;
    P->es = esz_;
    P->exact = prec_ == Precision::fp32_exact;
    P->tf32 = prec_ == Precision::tf32;
    P->H = xt.H, P->W = xt.W, P->C = c.in_channels, P->Ho = out.height, P->Wo = out.width;
    P->kh = c.kernel_h, P->kw = c.kernel_w, P->pad = c.pad, P->stride = c.stride;
    P->in = allocs_[size_t(xt.alloc)], P->in_cstride = xt.cstride, P->in_coff = xt.coff;
    P->wdw = weights_ + plan_.w_off.at(d.name);
    P->bdw = c.has_bias ? weights_ + plan_.b_off.at(d.name) : nullptr;
    P->relu_dw = c.activation == Activation::relu;
    P->pw = p != nullptr;
    if (p) {
        P->cout = p->conv->out_channels;
        P->wpw = weights_ + plan_.w_off.at(p->name);
        P->bpw = p->conv->has_bias ? weights_ + plan_.b_off.at(p->name) : nullptr;
        P->relu_pw = p->conv->activation == Activation::relu;
    }
    P->out = allocs_[size_t(ot.alloc)], P->out_cstride = ot.cstride, P->out_coff = ot.coff;
    P->out_c = p ? P->cout : P->C;
    P->px = c.stride == 1 && c.in_channels <= kDwMaxC / 2 ? 2 : 1;
    P->tile_w = c.stride == 1 ? 32 : 16;
    P->tile_h = kDwThreads * P->px / P->tile_w;
    P->cin_h = (P->tile_h - 1) * c.stride + c.kernel_h;
    P->cin_w = (P->tile_w - 1) * c.stride + c.kernel_w;
    const int c4 = (P->C + 3) / 4 * 4;
    P->cp = (c4 / 4) % 2 ? c4 : c4 + 4;  // odd number of float4s per cell: conflict-free float4 reads across a warp
    P->cw = c4;
    P->cpw = p ? (P->cout + 3) / 4 * 4 : 0;
    P->smem_bytes = (P->cin_h * P->cin_w * P->cp + c.kernel_h * c.kernel_w * P->cw + P->cw + (p ? P->C * P->cpw + P->cpw : 0)) * 4;
    if (P->smem_bytes > 227 * 1024) return nullptr;
    P->pdl = knobs_.pdl ? 1 : 0;
    return P;
}

// The fire kernel (kernels_fire.cu) takes a split block whose producer is a
// 1x1 squeeze staged on chip and whose consumers are stride-1 "same" expand
// convs of one width (fire_step_ok); its unit / channel split / ring are
// chosen by fire_choose at max_batch.
std::unique_ptr<FireParams> Engine::build_fire(const StepSpec& s, int fns, int fg, int fr, int sqs, int cb, int cps) {
    int th, tw;
    if (!tc_es_ || knobs_.no_fire || !fire_step_ok(g_, s, tc_es_) || knobs_.forced_tile(s, &th, &tw)) return nullptr;
    if (s2d_ && s.inputs[0] == g_.inputs[0].name) return nullptr;  // row-planar / rewritten input
    const Layer& sq = *g_.find_layer(s.ops[0].layer);
    const TensorSlot& xt = plan_.tensors.at(s.inputs[0]);
    auto P = std::make_unique<FireParams>();
    const int es = tc_es_;
    fire_shape(g_, s, es, *P);
    P->stage_mode = knobs_.fire_stage;
    P->sq_stream_mode = sqs < 0 ? knobs_.fire_sqs : sqs ? 1 : 2;
    P->cb_mode = cb > 0 ? cb : knobs_.fire_cb;
    P->cps_mode = cps > 0 ? cps : knobs_.fire_cps;
    P->coff_in = xt.coff;
    P->sq_bias = weights_ + plan_.b_off.at(sq.name);
    for (int o = 0; o < P->nops; ++o) {
        const Layer& l = *g_.find_layer(s.ops[size_t(o) + 1].layer);
        FireOp& op = P->op[o];
        op.bias = weights_ + plan_.b_off.at(l.name);
        const TensorSlot& ot = plan_.tensors.at(l.name);
        op.out = allocs_[size_t(ot.alloc)], op.out_cstride = ot.cstride, op.out_coff = ot.coff;
    }
    P->st32 = 1;
    for (int o = 0; o < P->nops; ++o)
        if ((P->op[o].out_cstride * es) % 32 || (P->op[o].out_coff * es) % 32 || reinterpret_cast<uintptr_t>(P->op[o].out) % 32) P->st32 = 0;
    int sms = 148;
    cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device_), "SM count");
    double model = 0;
    if (fns <= 0 && fg <= 0 && fr <= 0) fns = knobs_.fire_nsplit, fg = knobs_.fire_g, fr = knobs_.fire_r;
    if (!fire_choose(*P, max_batch_, sms, fns, fg, fr, &model)) return nullptr;
    P->wsq = packed_for(sq.name, P->S, 1);
    for (int o = 0; o < P->nops; ++o) P->op[o].w = packed_for(s.ops[size_t(o) + 1].layer, P->gch, P->nsplit);
    P->pdl = knobs_.pdl ? 1 : 0;
    if (knobs_.trace) {  // globaltimer stamps of CTA (0, 0) (profiling aid)
        unsigned long long* tr = nullptr;
        const size_t n = size_t(3) * kFireTraceN * 2;
        cuda_check(cudaMalloc(&tr, n * 8), "cudaMalloc(trace)");
        cuda_check(cudaMemset(tr, 0, n * 8), "cudaMemset(trace)");
        P->trace = tr;
        traces_.push_back(tr);
    }
    // squeeze A: 2-D {cstride, max_batch * HW}, box = cb bytes of channels x 128 pixels, cb-byte swizzle
    const cuuint64_t dims[2] = {cuuint64_t(xt.cstride), cuuint64_t((long long)max_batch_ * P->HW)};
    const cuuint64_t strides[1] = {cuuint64_t(xt.cstride) * es};
    const cuuint32_t box[2] = {cuuint32_t(P->cb / es), 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult res = tensor_map_encoder()(&P->amap, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                              allocs_[size_t(xt.alloc)], dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                              P->cb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (res != CUDA_SUCCESS) fail(ErrorKind::cuda, "cuTensorMapEncodeTiled (fire) failed (" + std::to_string(int(res)) + ")");
    return P;
}

// Packed weights of `layer` with nblocks x nb columns (N-split ops: one block
// per channel group), built once per shape from the host copy.
const uint8_t* Engine::packed_for(const std::string& layer, int nb, int nblocks) {
    const std::string key = layer + "/" + std::to_string(nb) + "x" + std::to_string(nblocks);
    auto it = packed_.find(key);
    if (it != packed_.end()) return static_cast<const uint8_t*>(it->second);
    const std::vector<uint8_t> w = pack_layer_tc(g_, layer, host_w_.data(), host_w_.size(), tc_es_, nb, nblocks);
    void* d = nullptr;
    cuda_check(cudaMalloc(&d, w.size() + 128), "cudaMalloc(split weights)");
    cuda_check(cudaMemcpy(d, w.data(), w.size(), cudaMemcpyHostToDevice), "split weights H2D");
    packed_[key] = d;
    return static_cast<const uint8_t*>(d);
}

// Launch descriptor of a tensor-core step in its current configuration (tile,
// staging, weight residency), bound to this engine's tensors and weights,
// with its device copy.
std::unique_ptr<BParams> Engine::build_bparams(const StepSpec& s) {
    auto P = std::make_unique<BParams>();
    if (layout_tc(g_, s, s.tile_h, s.tile_w, P.get(), s.nxb, s.wres, s.ring_slots, s.tsets, s.ring_chunk, tc_es_, knobs_) < 0)
        fail(ErrorKind::internal, "step " + s.id + ": tensor-core layout failed");
    P->epi_warps = s.epi_warps;
    P->kind = step_kind_tc(*P);
    P->ctas_per_sm = occupancy_fused_tc(P->smem_bytes, P->tmem_cols * P->tsets, P->epi_warps, P->kind, tc_es_);
    if (knobs_.ctas > 0) P->ctas_per_sm = std::min(P->ctas_per_sm, knobs_.ctas);
    P->grid_all = s.grid_all;
    if (knobs_.trace)
        std::fprintf(stderr, "[xlf] step %s: tile %dx%d, %d B shared, %d staging buffer(s), weights %s, %d CTA(s)/SM%s\n",
                     s.id.c_str(), s.tile_h, s.tile_w, P->smem_bytes, P->nxb,
                     P->wres ? "resident" : (std::to_string(P->ring_slots) + "-slot ring").c_str(), P->ctas_per_sm,
                     s.grid_all ? ", one tile per CTA" : "");
    for (int k = 0; k < P->nins; ++k) {
        const TensorSlot& t = plan_.tensors.at(s.inputs[size_t(k)]);
        BIn& in = P->in[k];
        in.x = allocs_[size_t(t.alloc)];
        in.cstride = t.cstride, in.coff = t.coff;
        encode_region_map(&P->xmap[k], in.x, t.cstride, t.W, t.H, max_batch_, in.r, tc_es_);
    }
    for (int k = 0; k < P->nops; ++k) {
        const OpSpec& os = s.ops[size_t(k)];
        BOp& o = P->ops[k];
        if (o.kind == BOP_MMA || o.kind == BOP_SIMT_CONV) {
            o.wsimt = weights_ + plan_.w_off.at(os.layer);
            o.bias = weights_ + plan_.b_off.at(os.layer);
            if (o.kind == BOP_MMA)
                o.wmma = o.gch ? packed_for(os.layer, o.nb, P->nsplit) : static_cast<const uint8_t*>(weights_tc_) + wofftc_.at(os.layer);
        }
        if (o.emit) {
            const TensorSlot& t = plan_.tensors.at(s.gap_out.empty() ? os.layer : s.gap_out);
            o.out = allocs_[size_t(t.alloc)];
            o.out_cstride = t.cstride, o.out_coff = t.coff;
        }
    }
    if (!s.gap_out.empty()) {  // per-tile column sums, [image][tile][npad of all channel groups] fp32
        const size_t need = size_t(max_batch_) * P->grid_h * P->grid_w * P->gap_np_total;
        auto& buf = gap_parts_[s.id];
        if (buf.second < need) {
            // grow only; the old buffer stays allocated until the engine dies
            // (descriptors built earlier -- the tuner's candidates, the current
            // step -- may still point at it)
            if (buf.first) retired_.push_back(buf.first);
            cuda_check(cudaMalloc(&buf.first, need * 4), "cudaMalloc(gap partials)");
            buf.second = need;
        }
        P->gap_part = buf.first;
    }
    if (knobs_.trace) {  // phase stamps of a few CTAs (profiling aid)
        unsigned long long* tr = nullptr;
        const size_t n = size_t(kTraceCtas) * kTraceEvents;
        cuda_check(cudaMalloc(&tr, n * 8), "cudaMalloc(trace)");
        cuda_check(cudaMemset(tr, 0, n * 8), "cudaMemset(trace)");
        P->trace = tr;
        P->trace_tiles = knobs_.trace == 2;
        traces_.push_back(tr);
    }
    void* dev = nullptr;
    cuda_check(cudaMalloc(&dev, sizeof(BParams)), "cudaMalloc(step descriptor)");
    P->dev_copy = dev;
    cuda_check(cudaMemcpy(dev, P.get(), sizeof(BParams), cudaMemcpyHostToDevice), "step descriptor H2D");
    return P;
}

// Measured-time tuner (successor of the reference's
// model-based tune(), cost_model.cpp:236-294): for every bf16 fused step the
// `topk` best configurations by the planner's model, each launched both as a
// persistent grid and one tile per CTA, are timed on the device with CUDA
// events (`reps` launches after one warm-up, on the engine's own tensors) and
// the fastest is kept.  Arithmetic does not depend on the configuration, so
// results stay within the bf16 tolerance whatever is chosen.
// fp32 SIMT steps: the model's best `topk` tiles with and without the
// register-blocked convs, plus the largest feasible tile of each and the
// planner's choice, timed on the device; the fastest is kept.  Every choice
// computes the same per-element arithmetic (fixed accumulation order), so
// fp32_exact stays bit-identical to the oracle whatever is picked.
std::string Engine::autotune_fp32(int batch, int reps, int topk, cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1) {
    std::ostringstream js;
    bool first = true;
    const bool exact = prec_ == Precision::fp32_exact;
    for (size_t i = 0; i < plan_.steps.size(); ++i) {
        StepSpec& s = plan_.steps[i];
        if (s.kind != StepSpec::FUSED || dws_[i]) continue;
        const std::vector<F32Candidate> all = candidates_fp32(g_, s, batch, 227 * 1024);
        std::vector<F32Candidate> cands = {{s.tile_h, s.tile_w, s.rb, s.threads, s.smem_bytes, 0.0}};
        int per_mode[4] = {0, 0, 0, 0};
        const F32Candidate* biggest[4] = {nullptr, nullptr, nullptr, nullptr};
        for (const F32Candidate& c : all) {  // the SIMT model is coarse: time >= 6 per (rb, threads) mode
            const int m = c.rb + (c.threads == 512 ? 2 : 0);
            if (per_mode[m]++ < std::max(6, 2 * topk)) cands.push_back(c);
            if (!biggest[m] || c.th * c.tw > biggest[m]->th * biggest[m]->tw) biggest[m] = &c;
        }
        for (const F32Candidate* c : biggest)
            if (c) cands.push_back(*c);
        float best_ms = 1e30f;
        StepSpec best = s;
        FusedParams bestP{};
        int tried = 0;
        std::set<std::array<int, 4>> seen;
        for (const F32Candidate& c : cands) {
            if (!seen.insert({c.th, c.tw, c.rb, c.threads}).second) continue;
            StepSpec t = s;
            t.tile_h = c.th, t.tile_w = c.tw, t.rb = c.rb, t.threads = c.threads;
            const long long sm = fp32_layout_bytes(g_, t, c.th, c.tw);
            if (sm < 0 || sm > 227 * 1024) continue;
            t.smem_bytes = int(sm);
            const FusedParams P = make_params(g_, plan_, t, allocs_, weights_);
            cuda_check(launch_fused_fp32(P, batch, exact, st), "autotune warm-up");
            cuda_check(cudaEventRecord(e0, st), "cudaEventRecord");
            for (int r = 0; r < reps; ++r) cuda_check(launch_fused_fp32(P, batch, exact, st), "autotune launch");
            cuda_check(cudaEventRecord(e1, st), "cudaEventRecord");
            cuda_check(cudaEventSynchronize(e1), "cudaEventSynchronize");
            float ms = 0;
            cuda_check(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
            ms /= float(reps);
            ++tried;
            if (knobs_.tune_verbose)
                std::fprintf(stderr, "[xlf] tune %s (fp32): tile %dx%d rb %d threads %d smem %d: %.1f us (model %.0f)\n", s.id.c_str(), c.th, c.tw,
                             c.rb, c.threads, int(sm), ms * 1000.0f, c.model);
            if (ms < best_ms) best_ms = ms, best = t, bestP = P;
        }
        if (!tried) continue;
        s = best;
        params_[i] = bestP;
        js << (first ? "" : ",") << "{\"id\":\"" << s.id << "\",\"kernel\":\"fp32\",\"tried\":" << tried << ",\"us\":" << best_ms * 1000.0f
           << ",\"tile\":[" << s.tile_h << "," << s.tile_w << "],\"rb\":" << s.rb << ",\"threads\":" << s.threads << ",\"smem_bytes\":" << s.smem_bytes << "}";
        first = false;
    }
    return js.str();
}

std::string Engine::autotune(int batch, int reps, int topk) {
    if (batch <= 0 || batch > max_batch_) batch = max_batch_;
    reps = std::max(1, reps), topk = std::max(1, topk);
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    cudaStream_t st;
    cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate(tune)");
    // captured forwards and external-address descriptors hold the current
    // configurations, which are replaced below
    drop_derived();
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "cudaEventCreate"), cuda_check(cudaEventCreate(&e1), "cudaEventCreate");
    std::ostringstream js;
    js << "[";
    bool first = true;
    if (!tc_es_) js << autotune_fp32(batch, std::max(1, reps), std::max(1, topk), st, e0, e1);
    // fire steps: the model's best configurations of every channel split (and
    // the current one) timed on the device; the fastest is kept
    for (size_t i = 0; i < plan_.steps.size(); ++i) {
        if (!fires_[i]) continue;
        const StepSpec& s = plan_.steps[i];
        FireParams shape{};
        fire_shape(g_, s, tc_es_, shape);
        shape.stage_mode = knobs_.fire_stage;
        shape.sq_stream_mode = knobs_.fire_sqs;
        shape.cb_mode = knobs_.fire_cb;
        shape.cps_mode = knobs_.fire_cps;
        std::vector<std::array<int, 6>> cands = {{fires_[i]->nsplit, fires_[i]->G, fires_[i]->R, fires_[i]->sq_stream, fires_[i]->cb, fires_[i]->cps}};
        // the model ranks unit shapes only roughly (it misses per-unit latency
        // chains): time the best 8 * topk by the model and at least topk of
        // every (split, whole images / row bands, squeeze-weight mode) family
        std::map<std::array<int, 4>, int> per_family;
        const auto all = fire_candidates(shape, batch, 148, 0, 0, 0);
        for (size_t k = 0; k < all.size(); ++k) {
            const FireParams& Q = all[k].second;
            const std::array<int, 6> c = {Q.nsplit, Q.G, Q.R, Q.sq_stream, Q.cb, Q.cps};
            int& fam = per_family[{Q.nsplit, Q.G > 1, Q.sq_stream, Q.cps}];
            if ((int(k) < 8 * topk || fam < topk) && std::find(cands.begin(), cands.end(), c) == cands.end())
                cands.push_back(c), ++fam;
        }
        float best_ms = 1e30f;
        std::unique_ptr<FireParams> bestP;
        int tried = 0;
        for (const auto& c : cands) {
            std::unique_ptr<FireParams> P = build_fire(s, c[0], c[1], c[2], c[3], c[4], c[5]);
            if (!P) continue;
            cuda_check(launch_fire(*P, 0, batch, st), "autotune warm-up");
            cuda_check(cudaEventRecord(e0, st), "cudaEventRecord");
            for (int r = 0; r < reps; ++r) cuda_check(launch_fire(*P, 0, batch, st), "autotune launch");
            cuda_check(cudaEventRecord(e1, st), "cudaEventRecord");
            cuda_check(cudaEventSynchronize(e1), "cudaEventSynchronize");
            float ms = 0;
            cuda_check(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
            ms /= float(reps);
            ++tried;
            if (knobs_.tune_verbose)
                std::fprintf(stderr, "[xlf] tune %s (fire): nsplit %d G %d R %d sqs %d cb %d cps %d ring %d planes %d smem %d: %.1f us\n", s.id.c_str(), P->nsplit,
                             P->G, P->R, P->sq_stream, P->cb, P->cps, P->nst, P->nplane, P->smem_bytes, ms * 1000.0f);
            if (ms < best_ms) best_ms = ms, bestP = std::move(P);
        }
        if (!bestP) continue;
        fires_[i] = std::move(bestP);
        StepSpec& t = plan_.steps[i];
        t.nsplit = fires_[i]->nsplit;
        t.tile_h = fires_[i]->G > 1 ? fires_[i]->G * fires_[i]->H : fires_[i]->R;
        t.smem_bytes = fires_[i]->smem_bytes;
        js << (first ? "" : ",") << "{\"id\":\"" << s.id << "\",\"kernel\":\"fire\",\"tried\":" << tried << ",\"us\":" << best_ms * 1000.0f
           << ",\"nsplit\":" << fires_[i]->nsplit << ",\"G\":" << fires_[i]->G << ",\"R\":" << fires_[i]->R << ",\"sqs\":" << fires_[i]->sq_stream << ",\"cb\":" << fires_[i]->cb << ",\"cps\":" << fires_[i]->cps
           << ",\"smem_bytes\":" << fires_[i]->smem_bytes
           << "}";
        first = false;
    }
    for (size_t i = 0; i < plan_.steps.size(); ++i) {
        StepSpec& s = plan_.steps[i];
        if (s.kind != StepSpec::FUSED || !bparams_[i]) continue;
        // the model ranks tiles within one staging / weight mode reasonably
        // but not across modes: keep the best `topk` of every mode
        std::vector<BCandidate> all = candidates_tc(g_, s, batch, kSmemBudgetTc, tc_es_, knobs_), cands;
        std::map<std::tuple<int, int, int, int>, int> per_mode;
        std::map<std::tuple<int, int, int, int>, const BCandidate*> biggest;  // largest tile of each mode
        for (const BCandidate& c : all) {
            const auto key = std::make_tuple(c.nxb, c.wres, c.slots * 1000 + c.chunk / 1024, (c.epi_warps * 4 + c.tsets) * 16 + c.nsplit);
            if (per_mode[key]++ < topk) cands.push_back(c);
            const BCandidate*& bg = biggest[key];
            if (!bg || c.th * c.tw > bg->th * bg->tw) bg = &c;
        }
        // the model under-rates large tiles (weight re-streaming per tile):
        // also time the largest feasible tile of every mode
        for (auto& [key, c] : biggest) {
            bool have = false;
            for (const BCandidate& d : cands) have |= d.th == c->th && d.tw == c->tw && d.nxb == c->nxb && d.wres == c->wres &&
                                                      d.slots == c->slots && d.epi_warps == c->epi_warps && d.tsets == c->tsets &&
                                                      d.chunk == c->chunk && d.nsplit == c->nsplit;
            if (!have) cands.push_back(*c);
        }
        float best_ms = 1e30f;
        StepSpec best = s;
        std::unique_ptr<BParams> bestP;
        int tried = 0;
        for (const BCandidate& c : cands)
            for (int ga = 0; ga < 2; ++ga) {
                StepSpec t = s;
                apply_candidate(t, c);
                t.grid_all = ga;
                std::unique_ptr<BParams> P = build_bparams(t);
                if (ga && P->ctas_per_sm * 148LL >= (long long)P->grid_h * P->grid_w * P->cgroups * batch * std::max(1, P->nsplit)) {
                    cudaFree(const_cast<void*>(P->dev_copy));
                    continue;  // persistent grid already covers every tile
                }
                cuda_check(launch_fused_tc(*P, batch, st, 0), "autotune warm-up");
                cuda_check(cudaEventRecord(e0, st), "cudaEventRecord");
                for (int r = 0; r < reps; ++r) cuda_check(launch_fused_tc(*P, batch, st, 0), "autotune launch");
                cuda_check(cudaEventRecord(e1, st), "cudaEventRecord");
                cuda_check(cudaEventSynchronize(e1), "cudaEventSynchronize");
                float ms = 0;
                cuda_check(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
                ms /= float(reps);
                ++tried;
                if (knobs_.tune_verbose)
                    std::fprintf(stderr, "[xlf] tune %s: tile %dx%d nxb %d wres %d slots %d grid_all %d ew %d ts %d ns %d smem %d: %.1f us (model %.0f)\n",
                                 s.id.c_str(), t.tile_h, t.tile_w, t.nxb, t.wres, t.ring_slots, t.grid_all, t.epi_warps, t.tsets, t.nsplit, P->smem_bytes,
                                 ms * 1000.0f, c.model);
                if (ms < best_ms) {
                    if (bestP) cudaFree(const_cast<void*>(bestP->dev_copy));
                    best_ms = ms, best = t, bestP = std::move(P);
                } else {
                    cudaFree(const_cast<void*>(P->dev_copy));
                }
            }
        if (!bestP) continue;
        const float model_ms = -1.0f;
        (void)model_ms;
        cudaFree(const_cast<void*>(bparams_[i]->dev_copy));
        s = best;
        bparams_[i] = std::move(bestP);
        js << (first ? "" : ",") << "{\"id\":\"" << s.id << "\",\"tried\":" << tried << ",\"us\":" << best_ms * 1000.0f
           << ",\"tile\":[" << s.tile_h << "," << s.tile_w << "],\"nxb\":" << s.nxb << ",\"wres\":" << s.wres
           << ",\"ring_slots\":" << s.ring_slots << ",\"ring_chunk\":" << s.ring_chunk << ",\"grid_all\":" << s.grid_all << ",\"epi_warps\":" << s.epi_warps
           << ",\"tsets\":" << s.tsets << ",\"nsplit\":" << s.nsplit << ",\"smem_bytes\":" << s.smem_bytes << "}";
        first = false;
    }
    js << "]";
    cudaEventDestroy(e0), cudaEventDestroy(e1);
    cudaStreamDestroy(st);
    return js.str();
}

// Re-applies a tuning report (the JSON autotune returns) without measuring:
// the tuned plan as a reusable artifact (tune once per model / batch / GPU,
// then load).  Every entry must name a tensor-core fused step of this plan and
// give a feasible configuration; the report's format is the one autotune
// writes (flat objects, numeric fields, "id" string, "tile" [h, w]).  All
// entries are parsed and validated before anything changes: a bad report
// leaves the engine as it was.
void Engine::apply_tuning(const std::string& js) {
    // value position of "key" (after the colon; whitespace tolerated), or npos
    auto at = [](const std::string& obj, const std::string& key) -> size_t {
        const size_t k = obj.find("\"" + key + "\"");
        if (k == std::string::npos) return std::string::npos;
        const size_t c = obj.find(':', k + key.size() + 2);
        return c == std::string::npos ? c : c + 1;
    };
    auto num = [&](const std::string& obj, const std::string& key, int& out) {
        const size_t v = at(obj, key);
        if (v == std::string::npos) return false;
        out = std::atoi(obj.c_str() + v);
        return true;
    };
    std::vector<std::pair<size_t, StepSpec>> todo;
    std::vector<std::pair<size_t, std::array<int, 6>>> fire_todo;
    size_t pos = 0;
    while ((pos = js.find('{', pos)) != std::string::npos) {
        const size_t end = js.find('}', pos);
        if (end == std::string::npos) fail(ErrorKind::parse, "tuning report: unterminated object");
        const std::string obj = js.substr(pos, end - pos + 1);
        pos = end + 1;
        const size_t iv = at(obj, "id");
        const size_t is = iv == std::string::npos ? iv : obj.find('"', iv);
        const size_t ie = is == std::string::npos ? is : obj.find('"', is + 1);
        if (ie == std::string::npos) fail(ErrorKind::parse, "tuning report: entry without \"id\"");
        const std::string id = obj.substr(is + 1, ie - is - 1);
        size_t i = 0;
        while (i < plan_.steps.size() && plan_.steps[i].id != id) ++i;
        if (i < plan_.steps.size() && fires_[i]) {  // fire step: channel split and unit
            int ns = 0, G = 0, R = 0, sqs = -1, cb = 0, cps = 0;
            num(obj, "sqs", sqs), num(obj, "cb", cb), num(obj, "cps", cps);
            if (!num(obj, "nsplit", ns) || !num(obj, "G", G) || !num(obj, "R", R))
                fail(ErrorKind::parse, "tuning report: fire step '" + id + "' needs \"nsplit\", \"G\" and \"R\"");
            if (ns < 1 || G < 1 || R < 1) fail(ErrorKind::infeasible, "tuning report: configuration of step '" + id + "' is not feasible for this plan");
            if ((cb != 0 && cb != 64 && cb != 128) || cps < 0 || cps > 2) fail(ErrorKind::infeasible, "tuning report: configuration of step '" + id + "' is not feasible for this plan");
            fire_todo.push_back({i, {ns, G, R, sqs, cb, cps}});
            continue;
        }
        if (!tc_es_) {  // fp32 SIMT step: tile and register-blocked convs on / off
            if (i == plan_.steps.size() || plan_.steps[i].kind != StepSpec::FUSED || dws_[i])
                fail(ErrorKind::validation, "tuning report: no fp32 fused step '" + id + "'");
            StepSpec t = plan_.steps[i];
            const size_t tv = at(obj, "tile");
            const size_t tb = tv == std::string::npos ? tv : obj.find('[', tv);
            const size_t tc = tb == std::string::npos ? tb : obj.find(',', tb);
            if (tc == std::string::npos) fail(ErrorKind::parse, "tuning report: step '" + id + "' without \"tile\": [h, w]");
            t.tile_h = std::atoi(obj.c_str() + tb + 1), t.tile_w = std::atoi(obj.c_str() + tc + 1);
            num(obj, "rb", t.rb), num(obj, "threads", t.threads);
            const long long sm = t.tile_h < 1 || t.tile_w < 1 || (t.rb != 0 && t.rb != 1) || (t.threads != 256 && t.threads != 512)
                                     ? -1
                                     : fp32_layout_bytes(g_, t, t.tile_h, t.tile_w);
            if (sm < 0 || sm > 227 * 1024) fail(ErrorKind::infeasible, "tuning report: configuration of step '" + id + "' is not feasible for this plan");
            t.smem_bytes = int(sm);
            todo.emplace_back(i, t);
            continue;
        }
        if (i == plan_.steps.size() || !bparams_[i]) fail(ErrorKind::validation, "tuning report: no tensor-core fused step '" + id + "'");
        StepSpec t = plan_.steps[i];
        const size_t tv = at(obj, "tile");
        const size_t tb = tv == std::string::npos ? tv : obj.find('[', tv);
        const size_t tc = tb == std::string::npos ? tb : obj.find(',', tb);
        if (tc == std::string::npos) fail(ErrorKind::parse, "tuning report: step '" + id + "' without \"tile\": [h, w]");
        t.tile_h = std::atoi(obj.c_str() + tb + 1);
        t.tile_w = std::atoi(obj.c_str() + tc + 1);
        num(obj, "nxb", t.nxb), num(obj, "wres", t.wres), num(obj, "ring_slots", t.ring_slots), num(obj, "ring_chunk", t.ring_chunk);
        num(obj, "grid_all", t.grid_all), num(obj, "epi_warps", t.epi_warps), num(obj, "tsets", t.tsets), num(obj, "nsplit", t.nsplit);
        // layout_tc rejects staging / accumulator-set / ring values the kernel
        // cannot run (nxb, tsets in {1, 2}; 1 <= ring_slots <= kRingMax; a
        // ring slot holding at least one K step)
        BParams probe;
        const long long sm = layout_tc(g_, t, t.tile_h, t.tile_w, &probe, t.nxb, t.wres, t.ring_slots, t.tsets, t.ring_chunk, tc_es_, knobs_);
        if (sm < 0 || sm > kSmemBudgetTc || (t.epi_warps != 4 && t.epi_warps != 8) || (t.grid_all != 0 && t.grid_all != 1))
            fail(ErrorKind::infeasible, "tuning report: configuration of step '" + id + "' is not feasible for this plan");
        t.smem_bytes = int(sm);
        todo.emplace_back(i, t);
    }
    std::vector<std::unique_ptr<FireParams>> fire_built;
    for (auto& [i, c] : fire_todo) {
        fire_built.push_back(build_fire(plan_.steps[i], c[0], c[1], c[2], c[3], c[4], c[5]));
        if (!fire_built.back() || fire_built.back()->nsplit != c[0] || fire_built.back()->G != c[1] || fire_built.back()->R != c[2] ||
            (c[3] >= 0 && fire_built.back()->sq_stream != c[3]) || (c[4] > 0 && fire_built.back()->cb != c[4]) ||
            (c[5] > 0 && fire_built.back()->cps != c[5]))
            fail(ErrorKind::infeasible, "tuning report: configuration of step '" + plan_.steps[i].id + "' is not feasible for this plan");
    }
    // captured forwards and external-address descriptors hold the current configurations
    drop_derived();
    for (size_t k = 0; k < fire_todo.size(); ++k) {
        const size_t i = fire_todo[k].first;
        fires_[i] = std::move(fire_built[k]);
        StepSpec& t = plan_.steps[i];
        t.nsplit = fires_[i]->nsplit;
        t.tile_h = fires_[i]->G > 1 ? fires_[i]->G * fires_[i]->H : fires_[i]->R;
        t.smem_bytes = fires_[i]->smem_bytes;
    }
    if (!tc_es_) {
        for (auto& [i, t] : todo) {
            plan_.steps[i] = t;
            params_[i] = make_params(g_, plan_, t, allocs_, weights_);
        }
        return;
    }
    std::vector<std::unique_ptr<BParams>> built;
    for (auto& [i, t] : todo) built.push_back(build_bparams(t));
    for (size_t k = 0; k < todo.size(); ++k) {
        const size_t i = todo[k].first;
        retired_.push_back(const_cast<void*>(bparams_[i]->dev_copy));  // freed with the engine (never while a launch may read it)
        plan_.steps[i] = todo[k].second;
        bparams_[i] = std::move(built[k]);
    }
}

void Engine::drop_derived() {
    for (auto& [b, ge] : graphs_) cudaGraphExecDestroy(ge);
    graphs_.clear();
    for (auto& [key, x] : ext_sets_)
        for (auto& P : x->bp)
            if (P) retired_.push_back(const_cast<void*>(P->dev_copy));  // a queued launch may still read it
    ext_sets_.clear();
}

Engine::~Engine() {
    cudaSetDevice(device_);
    for (auto& [b, ge] : graphs_) cudaGraphExecDestroy(ge);
    for (float* p : allocs_) cudaFree(p);
    cudaFree(weights_);
    if (weights_tc_) cudaFree(weights_tc_);
    for (unsigned long long* p : traces_) cudaFree(p);
    for (auto& P : bparams_)
        if (P) cudaFree(const_cast<void*>(P->dev_copy));
    cudaFree(staging_);
    if (out_staging_) cudaFree(out_staging_);
    for (auto& [id, b] : gap_parts_) cudaFree(b.first);
    for (auto& [key, x] : ext_sets_)
        for (auto& P : x->bp)
            if (P) cudaFree(const_cast<void*>(P->dev_copy));
    for (void* p : retired_) cudaFree(p);
    for (auto& [k, p] : packed_) cudaFree(p);
    if (copy_in_) {
        cudaStreamDestroy(copy_in_), cudaStreamDestroy(copy_out_);
        for (cudaEvent_t ev : chunk_ev_) cudaEventDestroy(ev);
    }
    if (capture_) cudaStreamDestroy(capture_);
}

const TensorSlot& Engine::slot(const std::string& n) const {
    auto it = plan_.tensors.find(n);
    if (it == plan_.tensors.end()) fail(ErrorKind::validation, "no tensor '" + n + "'");
    if (!it->second.materialized) fail(ErrorKind::validation, "tensor '" + n + "' is a fused intermediate (never stored to HBM)");
    return it->second;
}

// A tensor the user may read back: materialised and in the user's layout (a
// graph input rewritten to space-to-depth holds 4C channels at half the
// resolution and is not the tensor the user passed in).
const TensorSlot& Engine::readable(const std::string& n) const {
    const TensorSlot& t = slot(n);
    if (s2d_ && n == g_.inputs[0].name)
        fail(ErrorKind::validation, "tensor '" + n + "' is held in the space-to-depth layout of the tensor-core plan; it cannot be read back");
    return t;
}

void Engine::set_input_nchw(const std::string& name, const float* d, int batch, cudaStream_t st) {
    if (batch < 1 || batch > max_batch_) fail(ErrorKind::validation, "batch out of range");
    if (!user_inputs_.count(name)) fail(ErrorKind::validation, "'" + name + "' is not a graph input");
    const TensorSlot& t = slot(name);
    void* dst = allocs_[size_t(t.alloc)];
    if (s2d_ && name == g_.inputs[0].name)
        cuda_check(launch_s2d_tc(tc_es_, d, 0, 0, dst, batch, in_shape_.channels, in_shape_.height, in_shape_.width, t.cstride, s2d_planar_, st),
                   "space-to-depth input");
    else if (tc_es_)
        cuda_check(launch_nchw_to_nhwc_tc(tc_es_, d, dst, batch, t.C, t.H, t.W, t.cstride, st), "nchw_to_nhwc");
    else
        cuda_check(launch_nchw_to_nhwc(d, allocs_[size_t(t.alloc)], batch, t.C, t.H, t.W, t.cstride, st), "nchw_to_nhwc");
}

void Engine::set_input_seeded(const std::string& name, uint64_t seed, uint64_t first_image, int batch, cudaStream_t st) {
    if (batch < 1 || batch > max_batch_) fail(ErrorKind::validation, "batch out of range");
    if (!user_inputs_.count(name)) fail(ErrorKind::validation, "'" + name + "' is not a graph input");
    const TensorSlot& t = slot(name);
    void* dst = allocs_[size_t(t.alloc)];
    if (s2d_ && name == g_.inputs[0].name)
        cuda_check(launch_s2d_tc(tc_es_, nullptr, seed, first_image, dst, batch, in_shape_.channels, in_shape_.height, in_shape_.width,
                                 t.cstride, s2d_planar_, st),
                   "seeded space-to-depth input");
    else if (tc_es_)
        cuda_check(launch_seeded_nhwc_tc(tc_es_, dst, seed, first_image, batch, t.C, t.H, t.W, t.cstride, st), "seeded fill");
    else
        cuda_check(launch_seeded_nhwc(allocs_[size_t(t.alloc)], seed, first_image, batch, t.C, t.H, t.W, t.cstride, st), "seeded fill");
}

// A tensor-core fused step over images [n0, n0 + count): the kernel, plus the
// reduction that finishes a conv + global-average-pool step.
void Engine::launch_tc_step(size_t i, int n0, int count, cudaStream_t st) {
    if (dws_[i]) {
        cuda_check(launch_dw(*dws_[i], n0, count, st), "depthwise (+ pointwise)");
        return;
    }
    if (stems_[i]) {
        cuda_check(launch_stem(*stems_[i], count, st, n0), "stem (conv + max-pool, tensor cores)");
        return;
    }
    if (fires_[i]) {
        cuda_check(launch_fire(*fires_[i], n0, count, st), "fire block (squeeze -> expand, tensor cores)");
        return;
    }
    if (pws_[i]) {
        const PwParams& P = *pws_[i];
        cuda_check(launch_pw(P, n0, count, st), "pointwise conv (tensor cores)");
        const StepSpec& s = plan_.steps[i];
        if (!s.gap_out.empty()) {
            const TensorSlot& t = slot(s.gap_out);
            const Layer& pool = *g_.find_layer(s.gap_out);
            const float scale = 1.0f / float(pool.pool->kernel * pool.pool->kernel);
            cuda_check(launch_pw_gap_finish(P, t.C, scale, allocs_[size_t(t.alloc)], t.cstride, t.coff, n0, count, st), "global average pool finish");
        }
        return;
    }
    const BParams& P = *bparams_[i];
    cuda_check(launch_fused_tc(P, count, st, n0), "fused block (tensor cores)");
    const StepSpec& s = plan_.steps[i];
    if (s.gap_out.empty()) return;
    const TensorSlot& t = slot(s.gap_out);
    const Layer& pool = *g_.find_layer(s.gap_out);
    const float scale = 1.0f / float(pool.pool->kernel * pool.pool->kernel);
    cuda_check(launch_gap_finish_tc(tc_es_, P.gap_part, P.grid_h * P.grid_w, P.gap_np_total, scale, allocs_[size_t(t.alloc)], t.cstride, t.coff,
                                    t.C, n0, count, st),
               "global average pool finish");
}

bool Engine::range_capable() const {
    if (!tc_es_ || g_.inputs.size() != 1) return false;
    for (size_t i = 0; i < plan_.steps.size(); ++i)
        if (plan_.steps[i].kind != StepSpec::FUSED || !(bparams_[i] || stems_[i] || pws_[i] || fires_[i] || dws_[i])) return false;
    return true;
}

// Images [n0, n0 + count) only (tensor-core plans made of fused kernels: the
// kernels take the image offset; see run_host).
void Engine::forward_range(int n0, int count, cudaStream_t st) {
    if (n0 < 0 || count < 1 || n0 + count > max_batch_) fail(ErrorKind::validation, "image range out of bounds");
    if (!range_capable()) fail(ErrorKind::validation, "forward_range needs a tensor-core plan of fused kernels only");
    const long long key = -(1LL + (long long)n0 * 65536 + count);  // negative keys: ranges (positive: whole batches)
    auto it = graphs_.find(key);
    if (it == graphs_.end()) {
        if (!capture_) cuda_check(cudaStreamCreateWithFlags(&capture_, cudaStreamNonBlocking), "capture stream");
        cudaGraph_t graph;
        cuda_check(cudaStreamBeginCapture(capture_, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            for (size_t i = 0; i < plan_.steps.size(); ++i) launch_tc_step(i, n0, count, capture_);
        } catch (...) {
            cudaStreamEndCapture(capture_, &graph);
            throw;
        }
        cuda_check(cudaStreamEndCapture(capture_, &graph), "end capture");
        cudaGraphExec_t exec;
        cuda_check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
        cudaGraphDestroy(graph);
        it = graphs_.emplace(key, exec).first;
    }
    cuda_check(cudaGraphLaunch(it->second, st), "graph launch");
}

void Engine::launch_step(size_t i, int batch, cudaStream_t st) {
    const StepSpec& s = plan_.steps[i];
    auto ptr = [&](const TensorSlot& t) { return static_cast<void*>(allocs_[size_t(t.alloc)]); };
    switch (s.kind) {
    case StepSpec::FUSED:
        if (dws_[i]) cuda_check(launch_dw(*dws_[i], 0, batch, st), "depthwise (+ pointwise)");
        else if (tc_es_) launch_tc_step(i, 0, batch, st);
        else cuda_check(launch_fused_fp32(params_[i], batch, prec_ == Precision::fp32_exact, st), "fused block");
        return;
    case StepSpec::CONCAT_COPY: {
        const TensorSlot& o = slot(s.layers[0]);
        int off = 0;
        for (const std::string& in : s.inputs) {
            const TensorSlot& t = slot(in);
            const long long px = (long long)batch * t.H * t.W;
            if (tc_es_)
                cuda_check(launch_concat_copy_tc(tc_es_, ptr(t), t.cstride, t.coff, ptr(o), o.cstride, o.coff + off, t.C, px, st), "concat");
            else
                cuda_check(launch_concat_copy(allocs_[size_t(t.alloc)], t.cstride, t.coff, allocs_[size_t(o.alloc)], o.cstride,
                                              o.coff + off, t.C, px, st),
                           "concat copy");
            off += t.C;
        }
        return;
    }
    case StepSpec::ADD:
    case StepSpec::RELU: {
        const TensorSlot& o = slot(s.layers[0]);
        const TensorSlot& a = slot(s.inputs[0]);
        const TensorSlot& b = s.kind == StepSpec::ADD ? slot(s.inputs[1]) : a;
        const int op = s.kind == StepSpec::ADD ? 0 : 1;
        const long long px = (long long)batch * o.H * o.W;
        if (tc_es_)
            cuda_check(launch_eltwise_tc(tc_es_, op, ptr(a), a.cstride, a.coff, ptr(b), b.cstride, b.coff, ptr(o), o.cstride, o.coff, o.C, px,
                                         st),
                       "eltwise");
        else
            cuda_check(launch_eltwise(op, allocs_[size_t(a.alloc)], a.cstride, a.coff, allocs_[size_t(b.alloc)], b.cstride, b.coff,
                                      allocs_[size_t(o.alloc)], o.cstride, o.coff, o.C, px, st),
                       "eltwise");
        return;
    }
    }
}

void Engine::run_step(int index, int batch, cudaStream_t st) {
    if (index < 0 || index >= num_steps()) fail(ErrorKind::validation, "step index out of range");
    if (batch < 1 || batch > max_batch_) fail(ErrorKind::validation, "batch out of range");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    launch_step(size_t(index), batch, st);
}

void Engine::forward(int batch, cudaStream_t st, bool use_graph) {
    if (batch < 1 || batch > max_batch_) fail(ErrorKind::validation, "batch out of range");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    if (!use_graph) {
        for (size_t i = 0; i < plan_.steps.size(); ++i) launch_step(i, batch, st);
        return;
    }
    auto it = graphs_.find(batch);
    if (it == graphs_.end()) {
        // Capture on the engine's own stream (the caller's may be the legacy
        // default stream, which cannot be captured); replay on the caller's.
        if (!capture_) cuda_check(cudaStreamCreateWithFlags(&capture_, cudaStreamNonBlocking), "capture stream");
        cudaGraph_t graph;
        cuda_check(cudaStreamBeginCapture(capture_, cudaStreamCaptureModeThreadLocal), "begin capture");
        try {
            for (size_t i = 0; i < plan_.steps.size(); ++i) launch_step(i, batch, capture_);
        } catch (...) {
            cudaStreamEndCapture(capture_, &graph);
            throw;
        }
        cuda_check(cudaStreamEndCapture(capture_, &graph), "end capture");
        cudaGraphExec_t exec;
        cuda_check(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
        cudaGraphDestroy(graph);
        it = graphs_.emplace(batch, exec).first;
    }
    cuda_check(cudaGraphLaunch(it->second, st), "graph launch");
}

// Caller-owned tensors: the allocation of each named tensor is replaced by the
// caller's address (the tensor must own its allocation: a concat view shares
// it with its siblings), the descriptors of every fused step are rebuilt
// against the substituted table once per distinct address set, and the steps
// are launched with the substituted table in place.
void Engine::forward_external(const std::vector<External>& ext, int batch, cudaStream_t st) {
    if (batch < 1 || batch > max_batch_) fail(ErrorKind::validation, "batch out of range");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    const int cpc = 16 / esz_;
    std::string key;
    for (size_t i = 0; i < stems_.size(); ++i)
        if ((stems_[i] || pws_[i]) && !ext.empty())
            fail(ErrorKind::validation, "caller-owned tensors are not supported by plans with stem / pointwise steps");
    for (const External& x : ext) {
        const TensorSlot& t = slot(x.name);
        if (s2d_ && x.name == g_.inputs[0].name)
            fail(ErrorKind::validation, "input '" + x.name + "' is read in space-to-depth layout by this plan; pass it as NCHW");
        const int cp = (t.C + cpc - 1) / cpc * cpc;
        if (!x.ptr || reinterpret_cast<uintptr_t>(x.ptr) % 16)
            fail(ErrorKind::validation, "tensor '" + x.name + "': NHWC address must be non-NULL and 16-byte aligned");
        if (x.cstride % cpc || x.coff % cpc || x.coff < 0 || x.coff + cp > x.cstride)
            fail(ErrorKind::validation, "tensor '" + x.name + "': channel pitch " + std::to_string(x.cstride) + " / offset " +
                                            std::to_string(x.coff) + " must be multiples of " + std::to_string(cpc) +
                                            " elements (16 bytes) holding " + std::to_string(cp) + " channels");
        int sharing = 0;
        for (const auto& [n, u] : plan_.tensors) sharing += u.materialized && u.alloc == t.alloc;
        if (sharing != 1) fail(ErrorKind::validation, "tensor '" + x.name + "' shares its allocation (a concat view) and cannot be bound alone");
        key += x.name + "@" + std::to_string(reinterpret_cast<uintptr_t>(x.ptr)) + "/" + std::to_string(x.cstride) + "/" +
               std::to_string(x.coff) + ";";
    }
    auto it = ext_sets_.find(key);
    if (it == ext_sets_.end()) {
        auto set = std::make_unique<ExtSet>();
        set->allocs = allocs_;
        set->tensors = plan_.tensors;
        for (const External& x : ext) {
            TensorSlot& t = set->tensors.at(x.name);
            set->allocs[size_t(t.alloc)] = static_cast<float*>(x.ptr);
            t.cstride = x.cstride, t.coff = x.coff;
        }
        std::swap(allocs_, set->allocs), std::swap(plan_.tensors, set->tensors);
        try {
            set->bp.resize(plan_.steps.size());
            set->fp.resize(plan_.steps.size());
            set->fr.resize(plan_.steps.size());
            set->dw.resize(plan_.steps.size());
            for (size_t i = 0; i < plan_.steps.size(); ++i) {
                const StepSpec& s = plan_.steps[i];
                if (s.kind != StepSpec::FUSED) continue;
                if (dws_[i]) {
                    set->dw[i] = build_dw(s);
                    if (!set->dw[i]) fail(ErrorKind::internal, "step " + s.id + ": depthwise descriptor for caller-owned tensors");
                } else if (fires_[i]) {  // same configuration, the caller's addresses
                    set->fr[i] = build_fire(s, fires_[i]->nsplit, fires_[i]->G, fires_[i]->R, fires_[i]->sq_stream, fires_[i]->cb, fires_[i]->cps);
                    if (!set->fr[i]) fail(ErrorKind::internal, "step " + s.id + ": fire kernel descriptor for caller-owned tensors");
                } else if (tc_es_) set->bp[i] = build_bparams(s);
                else set->fp[i] = make_params(g_, plan_, s, allocs_, weights_);
            }
        } catch (...) {
            std::swap(allocs_, set->allocs), std::swap(plan_.tensors, set->tensors);
            for (auto& P : set->bp)
                if (P) cudaFree(const_cast<void*>(P->dev_copy));
            throw;
        }
        std::swap(allocs_, set->allocs), std::swap(plan_.tensors, set->tensors);
        it = ext_sets_.emplace(key, std::move(set)).first;
    }
    ExtSet& x = *it->second;
    // launch with the substituted table (restored on every exit path)
    struct Swap {
        Engine* e;
        ExtSet* x;
        void flip() {
            std::swap(e->allocs_, x->allocs), std::swap(e->plan_.tensors, x->tensors);
            std::swap(e->bparams_, x->bp), std::swap(e->params_, x->fp), std::swap(e->fires_, x->fr), std::swap(e->dws_, x->dw);
        }
        ~Swap() { flip(); }
    } sw{this, &x};
    sw.flip();
    for (size_t i = 0; i < plan_.steps.size(); ++i) launch_step(i, batch, st);
}

void Engine::read_output_nchw(const std::string& name, float* d, int batch, cudaStream_t st) {
    if (batch < 1 || batch > max_batch_) fail(ErrorKind::validation, "batch out of range");
    const TensorSlot& t = readable(name);
    if (tc_es_)
        cuda_check(launch_nhwc_tc_to_nchw(tc_es_, allocs_[size_t(t.alloc)], t.cstride, t.coff, d, batch, t.C, t.H, t.W, st), "nhwc_to_nchw");
    else
        cuda_check(launch_nhwc_to_nchw(allocs_[size_t(t.alloc)], t.cstride, t.coff, d, batch, t.C, t.H, t.W, st), "nhwc_to_nchw");
}

size_t Engine::tensor_elements(const std::string& name) const {
    const TensorSlot& t = readable(name);
    return size_t(t.C) * t.H * t.W;
}

// End to end from host memory.  Tensor-core plans made only of fused kernels
// are pipelined over chunks of images: the H2D copy of chunk c+1 (copy
// stream) overlaps the layout conversion + forward of chunk c (caller's
// stream), and each chunk's result is read back as soon as it is ready
// (second copy stream), so the PCIe transfer -- the e2e bound for 224x224x3
// fp32 inputs -- hides the compute.  Other plans: H2D, forward, D2H in sequence.
void Engine::run_host(const float* h_in, int batch, const std::string& out_name, float* h_out, cudaStream_t st) {
    if (batch < 1 || batch > max_batch_) fail(ErrorKind::validation, "batch out of range");
    if (g_.inputs.size() != 1) fail(ErrorKind::validation, "run_host: graphs with exactly one input (use set_input per input)");
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    const GraphInput& in = g_.inputs[0];
    const size_t img_in = size_t(in_shape_.elements());  // user-facing NCHW input, per image
    const TensorSlot& t = readable(out_name);
    const size_t img_out = size_t(t.C) * t.H * t.W;
    if (img_out * batch > staging_floats_) fail(ErrorKind::validation, "output larger than the staging buffer");
    int chunks = std::min(knobs_.e2e_chunks, batch);
    if (!range_capable() || chunks == 1) {
        cuda_check(cudaMemcpyAsync(staging_, h_in, img_in * batch * 4, cudaMemcpyHostToDevice, st), "H2D input");
        set_input_nchw(in.name, staging_, batch, st);
        forward(batch, st, true);
        read_output_nchw(out_name, staging_, batch, st);
        cuda_check(cudaMemcpyAsync(h_out, staging_, img_out * batch * 4, cudaMemcpyDeviceToHost, st), "D2H output");
        cuda_check(cudaStreamSynchronize(st), "sync");
        return;
    }
    if (!copy_in_) {
        cuda_check(cudaStreamCreateWithFlags(&copy_in_, cudaStreamNonBlocking), "copy stream");
        cuda_check(cudaStreamCreateWithFlags(&copy_out_, cudaStreamNonBlocking), "copy stream");
        for (int k = 0; k < 2 * kMaxChunks; ++k) cuda_check(cudaEventCreateWithFlags(&chunk_ev_[k], cudaEventDisableTiming), "event");
        cuda_check(cudaMalloc(&out_staging_, staging_floats_ * 4), "cudaMalloc(output staging)");
    }
    chunks = std::min(chunks, int(kMaxChunks) - 1);
    // Chunk boundaries: the first and last chunks half size (the first H2D and
    // the last forward are the only stages nothing overlaps): chunks + 1
    // pieces of 1/2, 1, ..., 1, 1/2 (3.251 -> 3.226 ms per 256 images);
    // option e2e_ramp=0: equal chunks.
    std::vector<int> cut{0};
    const bool ramp = knobs_.e2e_ramp && chunks >= 2 && chunks + 1 <= batch;
    const int pieces = ramp ? chunks + 1 : chunks;
    for (int c = 1; c < pieces; ++c) {
        const double w = ramp ? (c - 0.5) / chunks : double(c) / chunks;  // cumulative share
        cut.push_back(std::max(cut.back() + 1, std::min(batch - (pieces - c), int(batch * w + 0.5))));
    }
    cut.push_back(batch);
    const TensorSlot& xin = slot(in.name);
    const size_t es = size_t(esz_);
    for (int c = 0; c < pieces; ++c) {
        const int n0 = cut[size_t(c)], n1 = cut[size_t(c) + 1], cnt = n1 - n0;
        float* dst = staging_ + size_t(n0) * img_in;
        cuda_check(cudaMemcpyAsync(dst, h_in + size_t(n0) * img_in, size_t(cnt) * img_in * 4, cudaMemcpyHostToDevice, copy_in_),
                   "H2D input chunk");
        cuda_check(cudaEventRecord(chunk_ev_[c], copy_in_), "event");
        cuda_check(cudaStreamWaitEvent(st, chunk_ev_[c], 0), "wait H2D");
        uint8_t* x = reinterpret_cast<uint8_t*>(allocs_[size_t(xin.alloc)]) + size_t(n0) * xin.H * xin.W * xin.cstride * es;
        if (s2d_)
            cuda_check(launch_s2d_tc(tc_es_, dst, 0, 0, x, cnt, in_shape_.channels, in_shape_.height, in_shape_.width, xin.cstride, s2d_planar_, st),
                       "space-to-depth input chunk");
        else
            cuda_check(launch_nchw_to_nhwc_tc(tc_es_, dst, x, cnt, xin.C, xin.H, xin.W, xin.cstride, st), "nchw_to_nhwc chunk");
        forward_range(n0, cnt, st);
        const uint8_t* o = reinterpret_cast<const uint8_t*>(allocs_[size_t(t.alloc)]) + size_t(n0) * t.H * t.W * t.cstride * es;
        cuda_check(launch_nhwc_tc_to_nchw(tc_es_, o, t.cstride, t.coff, out_staging_ + size_t(n0) * img_out, cnt, t.C, t.H, t.W, st),
                   "nhwc_to_nchw chunk");
        cuda_check(cudaEventRecord(chunk_ev_[kMaxChunks + c], st), "event");
        cuda_check(cudaStreamWaitEvent(copy_out_, chunk_ev_[kMaxChunks + c], 0), "wait chunk");
        cuda_check(cudaMemcpyAsync(h_out + size_t(n0) * img_out, out_staging_ + size_t(n0) * img_out, size_t(cnt) * img_out * 4,
                                   cudaMemcpyDeviceToHost, copy_out_),
                   "D2H output chunk");
    }
    cuda_check(cudaStreamSynchronize(copy_out_), "sync");
    cuda_check(cudaStreamSynchronize(st), "sync");
}

int Engine::launches_per_forward() const {
    int n = 0;
    for (const StepSpec& s : plan_.steps) n += s.kind == StepSpec::CONCAT_COPY ? int(s.inputs.size()) : s.gap_out.empty() ? 1 : 2;
    return n;
}

std::string Engine::describe_json() const {
    std::ostringstream os;
    os << "{\"precision\":\"" << to_string(prec_) << "\",\"max_batch\":" << max_batch_
       << ",\"launches_per_forward\":" << launches_per_forward() << ",\"plan\":" << describe_plan_json(g_, plan_) << "}";
    return os.str();
}

}  // namespace xlf

namespace xlf {

std::vector<unsigned long long> Engine::trace(int index) const {
    if (index < 0 || index >= num_steps()) fail(ErrorKind::validation, "step index out of range");
    if (const FireParams* F = fires_[size_t(index)].get(); F && F->trace) {
        std::vector<unsigned long long> out(size_t(3) * kFireTraceN * 2);
        cuda_check(cudaMemcpy(out.data(), F->trace, out.size() * 8, cudaMemcpyDeviceToHost), "trace D2H");
        return out;
    }
    const BParams* P = bparams_[size_t(index)].get();
    if (!P || !P->trace) fail(ErrorKind::validation, "no trace for this step (tensor-core steps of an engine created with option trace=1 only)");
    std::vector<unsigned long long> out(size_t(kTraceCtas) * kTraceEvents);
    cuda_check(cudaMemcpy(out.data(), P->trace, out.size() * 8, cudaMemcpyDeviceToHost), "trace D2H");
    return out;
}

}  // namespace xlf
