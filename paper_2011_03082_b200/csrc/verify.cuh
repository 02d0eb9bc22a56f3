// verify.cuh -- on-device verification of two properties the fast paths rely on
// (tests/test_gpu_verify.py; C ABI sst_gpu_verify_culling / sst_gpu_nee_identity).
//
// 1. Conservativeness (acceptance 8, extended to every flight-culling
//    rule). Random free flights inside the media -- uniform in the SDF box and just
//    below the surface, where the rules are tight -- go through the PRODUCTION
//    predicates of the logic pass (same device functions, same precision build):
//    SDF safe radius, skip-grid radius, convex / two-ball end-point containment, the
//    convex end point's face-plane test (integrator.cuh end_inside_planes). Each
//    culled flight is checked against the exact FP64 geometry: brute force over every
//    triangle (Moller-Trumbore without epsilon on (0, t]), and every queried radius
//    against the exact point-mesh distance. Any hit is a violation.
// 2. NEE estimator identity (acceptance 7): on
//    brute-force unit-sphere walks, the single-representative estimate
//    Lambda * f(X_k), k ~ phi^k (the dataset generator's representative_k, which
//    produces EventGen's training targets) against the full per-event sum
//    sum_k phi^k f(X_k), with f a point-light NEE term (HG lobe x transmittance to
//    the sphere exit x inverse-square falloff).
#pragma once

#include "common.cuh"
#include "dataset.cuh"
#include "geom.cuh"
#include "integrator.cuh"
#include "rng.cuh"
#include "types.cuh"

namespace sstg {

namespace vfy {
struct D3 {
    double x, y, z;
};
SST_D D3 d3(double x, double y, double z) { return D3{x, y, z}; }
SST_D D3 sub(D3 a, D3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
SST_D D3 add(D3 a, D3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
SST_D D3 mul(D3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
SST_D double dt(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
SST_D D3 cr(D3 a, D3 b) { return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }

// Squared point-triangle distance (Ericson's region test, as mesh.cpp:199-233).
SST_D double pt_tri_d2(D3 p, D3 a, D3 ab, D3 ac) {
    const D3 b = add(a, ab), c = add(a, ac);
    const D3 ap = sub(p, a);
    const double d1 = dt(ab, ap), d2 = dt(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) return dt(ap, ap);
    const D3 bp = sub(p, b);
    const double d3v = dt(ab, bp), d4 = dt(ac, bp);
    if (d3v >= 0.0 && d4 <= d3v) return dt(bp, bp);
    const double vc = d1 * d4 - d3v * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3v <= 0.0) {
        const D3 q = sub(p, add(a, mul(ab, d1 / (d1 - d3v))));
        return dt(q, q);
    }
    const D3 cp = sub(p, c);
    const double d5 = dt(ab, cp), d6 = dt(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) return dt(cp, cp);
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const D3 q = sub(p, add(a, mul(ac, d2 / (d2 - d6))));
        return dt(q, q);
    }
    const double va = d3v * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3v) >= 0.0 && (d5 - d6) >= 0.0) {
        const double w = (d4 - d3v) / ((d4 - d3v) + (d5 - d6));
        const D3 q = sub(p, add(b, mul(sub(c, b), w)));
        return dt(q, q);
    }
    const double den = 1.0 / (va + vb + vc);
    const D3 q = sub(p, add(add(a, mul(ab, vb * den)), mul(ac, vc * den)));
    return dt(q, q);
}

// Exact segment test: does o + d s, s in (0, t], cross the triangle (no epsilon)?
SST_D bool seg_hits(D3 o, D3 d, double t, D3 a, D3 e1, D3 e2) {
    const D3 pv = cr(d, e2);
    const double det = dt(e1, pv);
    if (det == 0.0) return false;
    const double inv = 1.0 / det;
    const D3 tv = sub(o, a);
    const double u = dt(tv, pv) * inv;
    if (u < 0.0 || u > 1.0) return false;
    const D3 qv = cr(tv, e1);
    const double v = dt(d, qv) * inv;
    if (v < 0.0 || u + v > 1.0) return false;
    const double s = dt(e2, qv) * inv;
    return s > 0.0 && s <= t;
}
}  // namespace vfy

constexpr int kVfyTile = 64;

template <class R>
SST_D void verify_cull(const CullCheckArgs<R>& a) {
    __shared__ double tile[kVfyTile * 9];
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const DevScene<R>& sc = a.sc;
    bool active = i < a.n;
    Rng rng{rng_key(a.seed, 0x31, i, 0)};
    // ---- sample a flight start the logic pass would treat as inside object o
    int o = 0;
    V3<R> x = mk<R>(R(0), R(0), R(0));
    R v = R(1);
    bool in_grid = false;
    if (active) {
        if ((i & 1u) == 0u) {  // uniform in the object's SDF box (rejection on the SDF sign)
            o = static_cast<int>((i >> 1) % sc.n_objects);
            const ObjK<R>& ob = sc.objs[o];
            for (int tries = 0; tries < 32 && !(in_grid && v < R(0)); ++tries) {
                x = mk<R>(ob.sdf_origin[0] + rng.template uniform<R>() * ob.sdf_voxel * R(ob.dims[0]),
                          ob.sdf_origin[1] + rng.template uniform<R>() * ob.sdf_voxel * R(ob.dims[1]),
                          ob.sdf_origin[2] + rng.template uniform<R>() * ob.sdf_voxel * R(ob.dims[2]));
                v = sdf_raw(ob, x, &in_grid);
            }
        } else {  // just below the surface: a random triangle, depth 1e-6 .. 1e-1
            const uint32_t t = static_cast<uint32_t>(rng.template uniform<double>() * a.n_tris) % a.n_tris;
            const TriD& tr = a.tris[t];
            double bu = rng.template uniform<double>(), bv = rng.template uniform<double>();
            if (bu + bv > 1.0) {
                bu = 1.0 - bu;
                bv = 1.0 - bv;
            }
            const vfy::D3 e1 = vfy::d3(tr.e1[0], tr.e1[1], tr.e1[2]), e2 = vfy::d3(tr.e2[0], tr.e2[1], tr.e2[2]);
            const vfy::D3 n = vfy::cr(e1, e2);  // outward (winding enforced at upload)
            const double nl = sqrt(vfy::dt(n, n));
            const double depth = pow(10.0, -6.0 + 5.0 * rng.template uniform<double>());
            const vfy::D3 p = vfy::add(vfy::add(vfy::d3(tr.v0[0], tr.v0[1], tr.v0[2]), vfy::mul(e1, bu)),
                                       vfy::sub(vfy::mul(e2, bv), vfy::mul(n, depth / nl)));
            o = static_cast<int>(tr.obj);
            x = mk<R>(static_cast<R>(p.x), static_cast<R>(p.y), static_cast<R>(p.z));
            v = sdf_raw(sc.objs[o], x, &in_grid);
        }
        active = in_grid && !leaked(sc.objs[o], v, in_grid) && v <= R(0);
    }
    // ---- a flight: uniform direction, exponential length at the medium's density (or
    // uniform in [0, 0.3] for every fourth)
    const ObjK<R>& ob = sc.objs[o];
    V3<R> w = mk<R>(R(0), R(0), R(1));
    R t = R(0);
    bool cull_sdf = false, cull_skip = false, cull_end = false, cull_planes = false;
    R r_here = R(0), rs = R(0);
    if (active) {
        const double cz = 1.0 - 2.0 * rng.template uniform<double>();
        const double ph = kTwoPiD * rng.template uniform<double>();
        const double sz = sqrt(fmax(0.0, 1.0 - cz * cz));
        w = mk<R>(static_cast<R>(sz * cos(ph)), static_cast<R>(sz * sin(ph)), static_cast<R>(cz));
        const MediumK<R>& m = ob.med[static_cast<int>(i % 3u)];
        const R u = rng.template uniform<R>();
        if ((i & 3u) == 3u || !(m.sigma_t > R(0))) t = R(0.3) * u;
        else t = -Real<R>::div_(Real<R>::log_(R(1) - u), m.sigma_t);  // the logic pass's free path
        // the logic pass's culling rules (wavefront.cuh wf_logic_slot, flight start)
        r_here = v < R(0) ? -v : R(0);
        cull_sdf = t < r_here;
        if (!cull_sdf) {
            rs = skip_radius(ob, x);
            cull_skip = t < rs;
            if (!cull_skip && a.convex_end) {
                const int rule = flight_contained_rule(ob, x, w, t, Real<R>::fmax_(r_here, rs));
                cull_end = rule == kContainSdf;
                cull_planes = rule == kContainPlanes;
            }
        } else {
            rs = skip_radius(ob, x);
        }
    }
    // ---- exact FP64 ground truth: every triangle, tiled through shared memory
    const vfy::D3 xd = vfy::d3(x.x, x.y, x.z), wd = vfy::d3(w.x, w.y, w.z);
    const double td = static_cast<double>(t);
    double best = 1e300;
    bool hit = false;
    for (uint32_t base = 0; base < a.n_tris; base += kVfyTile) {
        const uint32_t nt = min(static_cast<uint32_t>(kVfyTile), a.n_tris - base);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < nt * 9; k += blockDim.x) {
            const TriD& tr = a.tris[base + k / 9];
            const int c = k % 9;
            tile[k] = c < 3 ? tr.v0[c] : (c < 6 ? tr.e1[c - 3] : tr.e2[c - 6]);
        }
        __syncthreads();
        if (!active) continue;
        for (uint32_t k = 0; k < nt; ++k) {
            const double* q = tile + 9 * k;
            const vfy::D3 A = vfy::d3(q[0], q[1], q[2]), E1 = vfy::d3(q[3], q[4], q[5]), E2 = vfy::d3(q[6], q[7], q[8]);
            best = fmin(best, vfy::pt_tri_d2(xd, A, E1, E2));
            hit = hit || vfy::seg_hits(xd, wd, td, A, E1, E2);
        }
    }
    unsigned long long c[kCvCount] = {};
    if (active) {
        const double dist = sqrt(best);
        c[kCvFlights] = 1;
        c[kCvCullSdf] = cull_sdf;
        c[kCvCullSkip] = cull_skip;
        c[kCvCullConvex] = cull_end && ob.convex;
        c[kCvCullTwoBall] = cull_end && !ob.convex;
        c[kCvViolSdf] = cull_sdf && hit;
        c[kCvViolSkip] = cull_skip && hit;
        c[kCvViolConvex] = cull_end && ob.convex && hit;
        c[kCvViolTwoBall] = cull_end && !ob.convex && hit;
        c[kCvCullPlanes] = cull_planes;
        c[kCvViolPlanes] = cull_planes && hit;
        c[kCvRadiusViol] = static_cast<double>(r_here) > dist;
        c[kCvSkipRadiusViol] = static_cast<double>(rs) > dist;
    }
#pragma unroll
    for (int k = 0; k < kCvCount; ++k) {
        const unsigned long long s = warp_sum(c[k]);
        if ((threadIdx.x & 31u) == 0 && s) atomicAdd(a.counts + k, s);
    }
}

// ------------------------------------------------------------------ NEE identity
// f(X, w): point-light NEE term from event X with incoming direction w in the unit
// sphere (sigma_t, g): hg(g, w . wl) exp(-sigma_t d_exit) / |L - X|^2.
template <class R>
SST_D double nee_f(const NeeIdentityArgs& a, V3<R> x, V3<R> w) {
    const double lx = a.light[0] - x.x, ly = a.light[1] - x.y, lz = a.light[2] - x.z;
    const double d2 = lx * lx + ly * ly + lz * lz, d = sqrt(d2);
    const V3<R> wl = mk<R>(static_cast<R>(lx / d), static_cast<R>(ly / d), static_cast<R>(lz / d));
    const double te = static_cast<double>(sphere_exit_t(x, wl));
    const double c = static_cast<double>(dot(w, wl));
    const double den = 1.0 + a.g * a.g - 2.0 * a.g * c;
    return kInv4PiD * (1.0 - a.g * a.g) / (den * sqrt(den)) * exp(-a.sigma_t * te) / d2;
}

// walk_sphere event loop (sphere_walk.cpp:34-49; dataset.cuh) from `s0`: returns N and,
// through `visit`, each event's position and incoming direction; stops after event
// `stop` (0 = run to the exit).
template <class R, class F>
SST_D uint32_t nee_walk(const NeeIdentityArgs& a, uint64_t s0, uint32_t stop, F&& visit) {
    Rng rng{s0};
    V3<R> pos = mk<R>(R(0), R(0), R(0)), inc = mk<R>(R(0), R(0), R(1));
    const R sig = static_cast<R>(a.sigma_t), g = static_cast<R>(a.g);
    uint32_t count = 1;  // the forced event at the centre
    visit(count, pos, inc);
    while (stop == 0 || count < stop) {
        const R u2 = rng.template uniform<R>();
        const R u1 = rng.template uniform<R>();
        const V3<R> dir = hg_sample(g, inc, u1, u2);
        const R step = -Real<R>::div_(Real<R>::log_(R(1) - rng.template uniform<R>()), sig);
        if (step >= sphere_exit_t(pos, dir) || count >= kMaxWalkEvents) break;
        pos = pos + dir * step;
        inc = dir;
        ++count;
        visit(count, pos, inc);
    }
    return count;
}

template <class R>
SST_D void nee_identity(const NeeIdentityArgs& a) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    double full = 0.0, single = 0.0;
    unsigned long long events = 0, res = 0;
    const bool active = i < a.walks;
    if (active) {
        const uint64_t s0 = rng_key(a.seed, 0x32, i, 0);
        // full per-event sum: sum_k phi^k f(X_k)
        double wk = 1.0, lambda = 0.0;
        const uint32_t n = nee_walk<R>(a, s0, 0u, [&](uint32_t, V3<R> x, V3<R> w) {
            wk *= a.phi;
            lambda += wk;
            full += wk * nee_f<R>(a, x, w);
        });
        events = n;
        // single representative: k ~ phi^k (the dataset generator's sampler), weight Lambda
        Rng pick{rng_key(a.seed, 0x33, i, 0)};
        for (uint32_t r = 0; r < a.resamples; ++r) {
            const uint32_t k = representative_k(a.phi, n, pick);
            double fk = 0.0;
            nee_walk<R>(a, s0, k, [&](uint32_t cnt, V3<R> x, V3<R> w) {
                if (cnt == k) fk = nee_f<R>(a, x, w);
            });
            single += lambda * fk;
            ++res;
        }
        single /= static_cast<double>(a.resamples);
    }
    const double dif = single - full;
    double v[3] = {full, single, dif * dif};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double s = warp_sum(v[k]);
        if ((threadIdx.x & 31u) == 0 && s != 0.0) atomicAdd(a.sums + k, s);
    }
    const unsigned long long cw = warp_sum(static_cast<unsigned long long>(active)), ce = warp_sum(events),
                             cr = warp_sum(res);
    if ((threadIdx.x & 31u) == 0) {
        if (cw) atomicAdd(a.counts + 0, cw);
        if (ce) atomicAdd(a.counts + 1, ce);
        if (cr) atomicAdd(a.counts + 2, cr);
    }
}

}  // namespace sstg
