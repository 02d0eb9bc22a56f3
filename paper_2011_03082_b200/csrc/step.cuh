// step.cuh -- one factorized CVAE sphere step on one thread: the device form of
// sample_sphere_step (scatter.cpp:152-177) and everything below it:
//   rescale_sigma            scatter.cpp:34-38
//   sample_num_events        scatter.cpp:62-70   (LengthGen, N = round(exp(n~ ln n_ref)))
//   test_absorption          scatter.cpp:72-74 -> absorption_prob optics.cpp:62-67
//   sample_exit              scatter.cpp:76-91   (PathGen, clamp + unit-disk projection)
//   to_world / make_sphere_frame  scatter.cpp:93-129
//   sample_event             scatter.cpp:131-150 (EventGen, |X| < 1, W normalised)
//   representative_weight_sum optics.cpp:69-75
// RNG draws are consumed in exactly the reference order (7 / 24 / 46 draws for
// absorbed / survived / survived+event, plus retries).
//
// Requires the including TU to declare (before including):
//   __constant__ SST_REAL c_weights[1332];
//   __constant__ SST_REAL c_norm[6];  // per model {log1p(sigma_ref), log(n_ref)}
#pragma once

#include "common.cuh"
#include "decoder.cuh"
#include "rng.cuh"
#include "types.cuh"

namespace sstg {


// absorption_prob (optics.cpp:62-67) for n >= 1.
template <class R>
SST_D R absorption_p(uint32_t n, const MediumK<R>& m) {
    if (m.phi_is_one) return R(0);
    if (m.phi_is_zero) return R(1);
    return -Real<R>::expm1_(static_cast<R>(n) * m.log_phi);
}

// representative_weight_sum (optics.cpp:69-75) for n >= 1.
template <class R>
SST_D R lambda_weight(uint32_t n, const MediumK<R>& m) {
    if (m.phi_is_zero) return R(0);
    if (m.phi_is_one) return static_cast<R>(n);
    if (Real<R>::kIsDouble) {
        const R phi_n = Real<R>::exp_(static_cast<R>(n) * m.log_phi);
        return m.phi * (R(1) - phi_n) / (R(1) - m.phi);
    }
    return Real<R>::div_(m.phi * (-Real<R>::expm1_(static_cast<R>(n) * m.log_phi)), m.one_minus_phi);
}

// rotation_z(2 pi u) (vec3.hpp:75-78): returns (cos, sin).
template <class R>
SST_D void rot_angle(R u, R* c, R* s);
template <>
SST_D void rot_angle<double>(double u, double* c, double* s) {
    const double psi = kTwoPiD * u;
    *c = cos(psi);
    *s = sin(psi);
}
template <>
SST_D void rot_angle<float>(float u, float* c, float* s) {
    float sn, cs;  // psi - pi in [-pi, pi): MUFU range; sin/cos(psi) = -sin/cos(psi - pi)
    __sincosf(fmaf(6.28318530717958647692f, u, -3.14159265358979323846f), &sn, &cs);
    *c = -cs;
    *s = -sn;
}

// make_sphere_frame rotation: frame_to(w_in) * rotation_z(psi) (scatter.cpp:93-100).
template <class R>
SST_D M3<R> sphere_rotation(V3<R> w_in, R c, R s) {
    M3<R> f;
    onb(w_in, &f.c0, &f.c1);
    f.c2 = w_in;
    const V3<R> z0 = mk<R>(c, s, R(0)), z1 = mk<R>(-s, c, R(0)), z2 = mk<R>(R(0), R(0), R(1));
    return M3<R>{f * z0, f * z1, f * z2};
}

// sample_sphere_step. Returns false when a decoder stayed non-finite after its
// retry (the reference throws std::runtime_error there).
template <class R>
SST_D bool sphere_step(const MediumK<R>& m, V3<R> w_in, V3<R> center, R r, bool with_event,
                       Rng& rng, StepOut<R>& o, DecodeCount& dc) {
    o.absorbed = false;
    o.lambda = R(0);
    const R ss = m.sigma_t * r;                                   // rescale_sigma
    const R l1 = Real<R>::log1p_(Real<R>::fmax_(R(0), ss));       // normalize_sigma numerator
    R out[6];
    {  // sample_num_events
        R cond[2] = {Real<R>::div_(l1, c_norm[0]), m.g};
        R x[1];
        if (!decode_sample<R, LengthShape>(cond, rng, x, dc.l)) return false;
        const R nn = Real<R>::exp_(x[0] * c_norm[1]);
        o.n = !(nn < R(4e9)) ? 4000000000u
                             : static_cast<uint32_t>(Real<R>::fmax_(R(1), Real<R>::round_(nn)));
    }
    const R u = rng.uniform<R>();
    if (u < absorption_p(o.n, m)) {  // test_absorption
        o.absorbed = true;
        return true;
    }
    const R nf = static_cast<R>(o.n);
    R ct, al, be;
    bool projected = false;
    {  // sample_exit
        R cond[3] = {Real<R>::div_(l1, c_norm[2]), m.g,
                     Real<R>::div_(Real<R>::log_(Real<R>::fmax_(R(1), nf)), c_norm[3])};
        R x[3];
        if (!decode_sample<R, PathShape>(cond, rng, x, dc.p)) return false;
        ct = Real<R>::fmin_(R(1), Real<R>::fmax_(R(-1), x[0]));
        al = x[1];
        be = x[2];
        const R r2 = al * al + be * be;
        if (r2 > R(1)) {
            const R inv = R(1) / Real<R>::sqrt_(r2);
            al *= inv;
            be *= inv;
            projected = true;
        }
    }
    R cp, sp;
    rot_angle<R>(rng.uniform<R>(), &cp, &sp);
    const M3<R> rot = sphere_rotation(w_in, cp, sp);
    {  // to_world
        const R st = Real<R>::sqrt_(Real<R>::fmax_(R(0), R(1) - ct * ct));
        const V3<R> e_n = mk<R>(st, R(0), ct);
        o.exit_pos = center + (rot * e_n) * r;
        V3<R> e_b, b2;
        if (st < R(1e-9)) onb(e_n, &e_b, &b2);
        else e_b = normalize(cross(mk<R>(R(0), R(0), R(1)), e_n));
        const V3<R> e_t = cross(e_b, e_n);
        // Normal component sqrt(1 - a^2 - b^2) (scatter.cpp:124). After the unit-disk
        // projection it is 0 mathematically; FP64 keeps the reference's expression
        // (whose rounding leaves up to ~1.5e-8), FP32 uses the exact 0 because
        // sqrt(FP32 rounding) would inject ~3e-4 into grazing exits.
        R nc;
        if (Real<R>::kIsDouble) nc = Real<R>::sqrt_(Real<R>::fmax_(R(0), R(1) - al * al - be * be));
        else nc = projected ? R(0) : Real<R>::sqrt_(Real<R>::fmax_(R(0), R(1) - al * al - be * be));
        const V3<R> d = normalize(e_b * al + e_t * be + e_n * nc);
        o.exit_dir = rot * d;
    }
    if (with_event) {  // sample_event
        R cond[7] = {Real<R>::div_(l1, c_norm[4]), m.g, m.phi, ct, al, be,
                     Real<R>::div_(Real<R>::log_(Real<R>::fmax_(R(1), nf)), c_norm[5])};
        if (!decode_sample<R, EventShape>(cond, rng, out, dc.e)) return false;
        V3<R> X = mk<R>(out[0], out[1], out[2]);
        const R lx = Real<R>::sqrt_(dot(X, X));
        if (lx >= R(1)) X = X * (R(0.999) / lx);
        V3<R> W = mk<R>(out[3], out[4], out[5]);
        const R lw = Real<R>::sqrt_(dot(W, W));
        if (Real<R>::kIsDouble) W = lw > R(0) ? W / lw : mk<R>(R(0), R(0), R(1));
        else W = lw > R(0) ? W * Real<R>::div_(R(1), lw) : mk<R>(R(0), R(0), R(1));
        o.rep_pos = center + (rot * X) * r;
        o.rep_dir = rot * W;
        o.lambda = lambda_weight(o.n, m);
    }
    return true;
}

}  // namespace sstg
