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
};

using LengthShape = DecoderShape<4, 8, 1, 2, 0>;
using PathShape = DecoderShape<8, 16, 3, 5, LengthShape::END>;
using EventShape = DecoderShape<12, 16, 6, 5, PathShape::END>;
constexpr int kTotalWeights = EventShape::END;  // 1332
static_assert(kTotalWeights == 1332, "production decoder parameter count");

// The including TU must declare, BEFORE including this header (one real type per TU):
//   __constant__ SST_REAL c_weights[1332];
// Host-side packing order of one decoder: W0, b0, W1, b1, W2, b2 (row-major W).

// Decoder mean/log-variance: 2 softplus hidden layers + identity head
// (mlp.cpp:70-87), log-variance clamped to [-10, 10] (cvae.cpp:20-22).
template <class R, class S>
SST_D void decode_head(const R (&in)[S::IN], R (&mu)[S::P_OUT], R (&lv)[S::P_OUT]) {
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
