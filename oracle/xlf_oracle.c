/*
 * xlf_oracle.c -- CPU restatement of the xlfuse reference arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the
 * B200 product path.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The
 * product (paper_2007_06000_b200) never links, imports or calls it.
 *
 * Parity pinning: every function below is checked against the reference
 * library itself (oracle/_ref, compiled from /root/reference/proj/src by
 * oracle/Makefile) and against the committed golden vectors in
 * tests/golden/ (generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Arithmetic contract (matches the reference build: g++ -O2, x86-64
 * baseline ISA, so no FMA contraction; this file is compiled with
 * -ffp-contract=off to keep that):
 *   conv   : acc = 0; for ic, kh, kw (in that order): acc += w * x   (mul then add,
 *            out-of-image taps skipped); acc += bias; relu = (acc < 0 ? 0 : acc)
 *            -- reference.cpp:16-57 (conv_layer), order documented at reference.hpp:14-16
 *   pool   : zero padding for both max and avg; avg divides by kernel*kernel
 *            -- reference.cpp:59-88 (pool_layer)
 *   add    : a + b, concat: CHW append -- reference.cpp:103-121 (run_layer)
 *   stream : splitmix64, top 24 bits * 2^-24 - 0.5, seed 0 -> golden ratio
 *            -- tensor.cpp:19-29 (SeededStream)
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define XLO_GOLDEN 0x9e3779b97f4a7c15ULL

/* tensor.cpp:19-29.  Element i (0-based) of SeededStream(seed) is a pure
 * function of (seed, i): state after i+1 increments is seed' + (i+1)*phi. */
static inline float xlo_mix(uint64_t state) {
    uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    z = z ^ (z >> 31);
    return (float)(z >> 40) * (1.0f / 16777216.0f) - 0.5f;
}

void xlo_stream_fill(uint64_t seed, uint64_t first, float* out, size_t n) {
    uint64_t s = seed ? seed : XLO_GOLDEN;
    uint64_t state = s + (first + 1) * XLO_GOLDEN;
    for (size_t i = 0; i < n; ++i) {
        out[i] = xlo_mix(state);
        state += XLO_GOLDEN;
    }
}

/* seeded_weights uses a separate stream keyed by seed ^ 0xabcdef1234567890
 * (tensor.cpp:42-62); callers pass the already-xored seed through here. */
uint64_t xlo_weight_seed(uint64_t seed) { return seed ^ 0xabcdef1234567890ULL; }

static inline int out_dim(int in, int k, int pad, int stride) {
    return (in + 2 * pad - k) / stride + 1; /* graph.cpp:76-78 */
}

/* reference.cpp:16-57.  One image, CHW.  The outer loops are reordered for
 * cache friendliness; the per-output accumulation sequence (ic, kh, kw with
 * skipped out-of-image taps) is exactly the reference's. */
void xlo_conv(const float* in, int C, int H, int W,
              const float* filter, const float* bias,
              int Cout, int kh_, int kw_, int pad, int stride, int group, int relu,
              float* out) {
    const int Ho = out_dim(H, kh_, pad, stride);
    const int Wo = out_dim(W, kw_, pad, stride);
    const int cin_g = C / group, cout_g = Cout / group;
    for (int oc = 0; oc < Cout; ++oc) {
        const int grp = oc / cout_g;
        const float* wb = filter + (size_t)oc * cin_g * kh_ * kw_;
        for (int oy = 0; oy < Ho; ++oy) {
            for (int ox = 0; ox < Wo; ++ox) {
                float acc = 0.0f;
                for (int ic = 0; ic < cin_g; ++ic) {
                    const float* plane = in + (size_t)(grp * cin_g + ic) * H * W;
                    for (int kh = 0; kh < kh_; ++kh) {
                        const int iy = oy * stride - pad + kh;
                        if (iy < 0 || iy >= H) continue;
                        for (int kw = 0; kw < kw_; ++kw) {
                            const int ix = ox * stride - pad + kw;
                            if (ix < 0 || ix >= W) continue;
                            const float prod = wb[((size_t)ic * kh_ + kh) * kw_ + kw] * plane[(size_t)iy * W + ix];
                            acc = acc + prod;
                        }
                    }
                }
                if (bias) acc = acc + bias[oc];
                if (relu) acc = acc < 0.0f ? 0.0f : acc;
                out[((size_t)oc * Ho + oy) * Wo + ox] = acc;
            }
        }
    }
}

/* reference.cpp:59-88.  kind 0 = max, 1 = avg. */
void xlo_pool(const float* in, int C, int H, int W, int kind, int k, int stride, int pad,
              float* out) {
    const int Ho = out_dim(H, k, pad, stride), Wo = out_dim(W, k, pad, stride);
    for (int c = 0; c < C; ++c)
        for (int oy = 0; oy < Ho; ++oy)
            for (int ox = 0; ox < Wo; ++ox) {
                float best = -__builtin_inff();
                float sum = 0.0f;
                for (int kh = 0; kh < k; ++kh) {
                    const int iy = oy * stride - pad + kh;
                    for (int kw = 0; kw < k; ++kw) {
                        const int ix = ox * stride - pad + kw;
                        float v = 0.0f;
                        if (iy >= 0 && iy < H && ix >= 0 && ix < W) v = in[((size_t)c * H + iy) * W + ix];
                        best = (best < v) ? v : best; /* std::max(best, v) */
                        sum = sum + v;
                    }
                }
                out[((size_t)c * Ho + oy) * Wo + ox] = kind == 0 ? best : sum / (float)(k * k);
            }
}

/* reference.cpp:97-102 */
void xlo_relu(const float* in, float* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = in[i] < 0.0f ? 0.0f : in[i];
}

/* reference.cpp:103-110 */
void xlo_add(const float* a, const float* b, float* out, size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = a[i] + b[i];
}

/* reference.cpp:144-157: element-wise max_abs and max_rel with a 1e-6 floor. */
void xlo_compare(const float* a, const float* b, size_t n, double* max_abs, double* max_rel) {
    double ma = 0, mr = 0;
    for (size_t i = 0; i < n; ++i) {
        const double av = a[i], bv = b[i];
        const double d = av > bv ? av - bv : bv - av;
        double den = av < 0 ? -av : av;
        const double bb = bv < 0 ? -bv : bv;
        if (bb > den) den = bb;
        if (den < 1e-6) den = 1e-6;
        if (d > ma) ma = d;
        if (d / den > mr) mr = d / den;
    }
    *max_abs = ma;
    *max_rel = mr;
}
