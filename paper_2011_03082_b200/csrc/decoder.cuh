// decoder.cuh -- fused per-thread evaluator of the three CVAE decoders
// (mlp_forward, mlp.cpp:70-87; cvae_decode, cvae.cpp:93-98;
//  cvae_decode_sample / reparameterize, cvae.cpp:100-104, mlp.cpp:204-212;
//  decode_with_retry, scatter.cpp:44-58).
//
// Weights live in __constant__ memory (`c_weights`, one precision per translation
// unit). All lanes of a warp read the same weight at the same time, so every FMA takes its weight straight from the
// constant bank as an instruction operand: no loads, no shared-memory traffic.
// Shapes are the production architectures (CvaeSpec::production_default,
// cvae.cpp:51-58; Table 1) and fully unrolled at compile time:
//   LengthGen  4 -> 8 -> 8 -> 2    (112 MAC)
//   PathGen    8 -> 16 -> 16 -> 6  (480 MAC)
//   EventGen  12 -> 16 -> 16 -> 12 (640 MAC)
#pragma once

#include "common.cuh"
#include "rng.cuh"

namespace sstg {

template <int IN_, int W_, int P_OUT_, int LATENT_, int OFFSET_>
struct DecoderShape {
    static constexpr int IN = IN_, W = W_, P_OUT = P_OUT_, LATENT = LATENT_, P_IN = IN_ - LATENT_;
    static constexpr int OUT = 2 * P_OUT_;
    static constexpr int OFF_W0 = OFFSET_;
    static constexpr int OFF_B0 = OFF_W0 + W * IN;
    static constexpr int OFF_W1 = OFF_B0 + W;
    static constexpr int OFF_B1 = OFF_W1 + W * W;
    static constexpr int OFF_W2 = OFF_B1 + W;
    static constexpr int OFF_B2 = OFF_W2 + OUT * W;
    static constexpr int END = OFF_B2 + OUT;
    static constexpr int MACS = W * IN + W * W + OUT * W;
    // Row-pair layout (FP32 FFMA2 path, c_wpair in float2 units): pair (2k, 2k+1) of
    // every layer's rows side by side, W0 pairs [W/2][IN], b0 pairs, W1 [W/2][W], b1,
    // W2 [OUT/2][W], b2 -- the same weights, END - OFFSET floats.
    static constexpr int P_W0 = OFFSET_ / 2;
    static constexpr int P_B0 = P_W0 + (W / 2) * IN;
    static constexpr int P_W1 = P_B0 + W / 2;
    static constexpr int P_B1 = P_W1 + (W / 2) * W;
    static constexpr int P_W2 = P_B1 + W / 2;
    static constexpr int P_B2 = P_W2 + (OUT / 2) * W;
    static_assert(OFFSET_ % 2 == 0 && W % 2 == 0 && OUT % 2 == 0, "row pairs");
};

using LengthShape = DecoderShape<4, 8, 1, 2, 0>;
using PathShape = DecoderShape<8, 16, 3, 5, LengthShape::END>;
using EventShape = DecoderShape<12, 16, 6, 5, PathShape::END>;
constexpr int kTotalWeights = EventShape::END;  // 1332
static_assert(kTotalWeights == 1332, "production decoder parameter count");

// The including TU must declare, BEFORE including this header (one real type per TU):
//   __constant__ SST_REAL c_weights[1332];
// Host-side packing order of one decoder: W0, b0, W1, b1, W2, b2 (row-major W).

#ifdef SST_DECODER_PAIRS
// FP32: two rows per instruction (FFMA2 = two IEEE FP32 FMAs): the input broadcast, the
// row pair's weights adjacent in c_wpair. Each row's operation sequence -- bias, then
// acc = fma(w_c, in_c, acc) for c = 0, 1, ... -- is the scalar path's, so the results are
// bit-identical; the decoders issue ~40% fewer instructions.
SST_D unsigned long long f2_pack(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
SST_D void f2_unpack(unsigned long long v, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v)); }
SST_D unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// out[r] = b[r] + sum_c W[r][c] in[c] for the ROWS rows of one layer (pair layout at PW/PB)
template <int ROWS, int COLS, int PW, int PB>
SST_D void layer_pairs(const float (&in)[COLS], float (&out)[ROWS]) {
#pragma unroll
    for (int rp = 0; rp < ROWS / 2; ++rp) {
        const float2 b = c_wpair[PB + rp];
        unsigned long long acc = f2_pack(b.x, b.y);
#pragma unroll
        for (int c = 0; c < COLS; ++c) {
            const float2 w = c_wpair[PW + rp * COLS + c];
            acc = f2_fma(f2_pack(w.x, w.y), f2_pack(in[c], in[c]), acc);
        }
        f2_unpack(acc, out[2 * rp], out[2 * rp + 1]);
    }
}
#endif

// Decoder mean/log-variance: 2 softplus hidden layers + identity head
// (mlp.cpp:70-87), log-variance clamped to [-10, 10] (cvae.cpp:20-22).
template <class R, class S>
SST_D void decode_head(const R (&in)[S::IN], R (&mu)[S::P_OUT], R (&lv)[S::P_OUT]) {
#ifdef SST_DECODER_PAIRS
    if constexpr (sizeof(R) == 4) {
        float h0[S::W], h1[S::W], o[S::OUT];
        layer_pairs<S::W, S::IN, S::P_W0, S::P_B0>(in, h0);
#pragma unroll
        for (int r = 0; r < S::W; ++r) h0[r] = Real<R>::softplus(h0[r]);
        layer_pairs<S::W, S::W, S::P_W1, S::P_B1>(h0, h1);
#pragma unroll
        for (int r = 0; r < S::W; ++r) h1[r] = Real<R>::softplus(h1[r]);
        layer_pairs<S::OUT, S::W, S::P_W2, S::P_B2>(h1, o);
#pragma unroll
        for (int r = 0; r < S::P_OUT; ++r) {
            mu[r] = o[r];
            lv[r] = Real<R>::fmin_(R(10), Real<R>::fmax_(R(-10), o[S::P_OUT + r]));
        }
        return;
    }
#endif
    R h0[S::W], h1[S::W];
#pragma unroll
    for (int r = 0; r < S::W; ++r) {
        R acc = c_weights[S::OFF_B0 + r];
#pragma unroll
        for (int c = 0; c < S::IN; ++c) acc += c_weights[S::OFF_W0 + r * S::IN + c] * in[c];
        h0[r] = Real<R>::softplus(acc);
    }
#pragma unroll
    for (int r = 0; r < S::W; ++r) {
        R acc = c_weights[S::OFF_B1 + r];
#pragma unroll
        for (int c = 0; c < S::W; ++c) acc += c_weights[S::OFF_W1 + r * S::W + c] * h0[c];
        h1[r] = Real<R>::softplus(acc);
    }
#pragma unroll
    for (int r = 0; r < S::OUT; ++r) {
        R acc = c_weights[S::OFF_B2 + r];
#pragma unroll
        for (int c = 0; c < S::W; ++c) acc += c_weights[S::OFF_W2 + r * S::W + c] * h1[c];
        if (r < S::P_OUT) mu[r] = acc;
        else lv[r - S::P_OUT] = Real<R>::fmin_(R(10), Real<R>::fmax_(R(-10), acc));
    }
}

// decode_with_retry (scatter.cpp:44-58): z ~ N(0,I_L) then eps ~ N(0,I_P)
// (draw order of the reference), x = mu + exp(lv/2) * eps; one retry on a
// non-finite output. Returns false if still non-finite (the reference throws).
template <class R, class S>
SST_D bool decode_sample(const R (&cond)[S::P_IN], Rng& rng, R (&x)[S::P_OUT], uint32_t& count) {
#pragma unroll 1
    for (int attempt = 0; attempt < 2; ++attempt) {
        R in[S::IN];
        R nz[S::LATENT + S::P_OUT];  // z then eps, the reference's draw order
        rng.s = draw_normals<R>(rng.s, nz, S::LATENT + S::P_OUT);
#pragma unroll
        for (int i = 0; i < S::LATENT; ++i) in[i] = nz[i];
#pragma unroll
        for (int i = 0; i < S::P_IN; ++i) in[S::LATENT + i] = cond[i];
        ++count;
        R mu[S::P_OUT], lv[S::P_OUT];
        decode_head<R, S>(in, mu, lv);
        bool finite = true;
#pragma unroll
        for (int i = 0; i < S::P_OUT; ++i) {
            x[i] = mu[i] + Real<R>::exp_(R(0.5) * lv[i]) * nz[S::LATENT + i];
            finite = finite && Real<R>::isfinite_(x[i]);
        }
        if (finite) return true;
    }
    return false;
}

}  // namespace sstg
