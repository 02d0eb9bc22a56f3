// integrator.cuh -- the per-path loop of the two integrators as a
// persistent megakernel body. DESIGN.md "Integrator semantics" fixes the loop; the
// CPU oracle (oracle/sst_oracle.c trace_one, oracle/ref_shim.cpp trace_one) follows
// the same draw order, so FP64 paths reproduce the oracle draw for draw.
//
// Path state lives in registers for the whole path (no HBM round trips); a lane
// whose path ends fetches the next path id with one warp-aggregated atomic.
#pragma once

#include "common.cuh"
#ifdef SST_TRACE_DEBUG
#include <cstdio>
#endif
#include "geom.cuh"
#include "rng.cuh"
#include "step.cuh"
#include "types.cuh"

namespace sstg {


// hg_sample_cos (optics.cpp:33-39)
template <class R>
SST_D R hg_cos(R g, R u) {
    if (Real<R>::fabs_(g) < R(1e-4)) return R(1) - R(2) * u;
    const R s = Real<R>::div_(R(1) - g * g, R(1) + g - R(2) * g * u);
    const R c = Real<R>::div_(R(1) + g * g - s * s, R(2) * g);
    return c < R(-1) ? R(-1) : (c > R(1) ? R(1) : c);
}

// hg_sample (optics.cpp:41-48)
template <class R>
SST_D V3<R> hg_sample(R g, V3<R> w_in, R u1, R u2) {
    const R ct = hg_cos(g, u1);
    const R st = Real<R>::sqrt_(Real<R>::fmax_(R(0), R(1) - ct * ct));
    R cp, sp;
    rot_angle<R>(u2, &cp, &sp);
    V3<R> b1, b2;
    onb(w_in, &b1, &b2);
    return b1 * (st * cp) + b2 * (st * sp) + w_in * ct;
}

// hg_eval (optics.cpp:27-31)
template <class R>
SST_D R hg_eval(R g, R c) {
    const R denom = R(1) + g * g - R(2) * g * c;
    return Real<R>::div_(R(kInv4PiD) * (R(1) - g * g), denom * Real<R>::sqrt_(denom));
}

// Shadow-ray length of a directional light (beyond every scene; FP32-representable).
constexpr double kFarLight = 1e30;

// NEE toward the point light from p (in object obj, channel c) with incoming w:
// weight * Phi * hg(g, w.wl) * exp(-tau) / d^2.
template <class R>
SST_D R nee_term(const DevScene<R>& sc, const MediumK<R>& m, int c, V3<R> p, V3<R> w, R weight,
                 uint64_t& tri_tests, int own = -1) {
    if (sc.directional) {
        // E * hg(g, w.wl) * exp(-tau), tau over the in-medium part of the ray out to the
        // last boundary exit (closed meshes: every hit beyond it is an entry/exit pair).
        const RayK<R> ray = make_ray(p, sc.light_dir);
        const R tau = optical_depth(sc, ray, sc.t_min, R(kFarLight), c);
        return weight * sc.power[c] * hg_eval(m.g, dot(w, sc.light_dir)) * Real<R>::exp_(R(-1) * tau);
    }
    const V3<R> to_l = sc.light - p;
    const R d2 = dot(to_l, to_l);
    const R d = Real<R>::sqrt_(d2);
    const R inv_d = Real<R>::div_(R(1), d);  // FP64: IEEE 1/d (the reference divides; see below)
    const V3<R> wl = Real<R>::kIsDouble ? to_l / d : to_l * inv_d;
    RayK<R> ray;  // the light-grid path needs no slab reciprocals
    if (sc.grid_off) {
        ray.o = p;
        ray.d = wl;
    } else {
        ray = make_ray(p, wl);
    }
    const R tau = sc.grid_off ? optical_depth_grid(sc, ray, sc.t_min, d, c, tri_tests, own)
                              : optical_depth(sc, ray, sc.t_min, d, c);
    const R phase = hg_eval(m.g, dot(w, wl));
    if (Real<R>::kIsDouble) return weight * sc.power[c] * phase * Real<R>::exp_(R(-1) * tau) / d2;
    return weight * sc.power[c] * phase * Real<R>::exp_(R(-1) * tau) * (inv_d * inv_d);
}

template <class R>
struct PathLocal {
    V3<R> x, w;
    Rng rng;
    R L;
    R r_here;       // SDF radius at x (valid iff r_valid)
    uint64_t id;
    uint32_t seg, pixel;
    int obj;        // -1 outside every medium
    int skip;       // triangle to ignore on the next traversal (FP32 surface start)
    int cull;       // convex object just left: its subtree is culled on the next traversal
    uint8_t c;
    bool r_valid;
    bool pending;   // a sphere step is requested and waits for its warp batch
    bool tpend;     // a traversal is requested and waits for its warp batch (t_pend = flight)
    uint16_t waited, twaited;
    R t_pend;
};

// The path's exit state (trace_paths_ex): position and direction when it ended.
template <class R>
SST_D void write_exit_state(R* e, const PathLocal<R>& p) {
    e += 6 * p.id;
    e[0] = p.x.x;
    e[1] = p.x.y;
    e[2] = p.x.z;
    e[3] = p.w.x;
    e[4] = p.w.y;
    e[5] = p.w.z;
}

struct LaneStats {
    uint32_t paths = 0, absorbed = 0, escaped = 0, capped = 0, errors = 0;
    uint64_t seg = 0, sphere = 0, events = 0, shadow = 0;
    uint64_t traversals = 0, nodes = 0, tris = 0, lane_iters = 0, warp_iters = 0, shadow_tris = 0, wf_slots = 0;
    DecodeCount dc;
};

// Can the ray x + t d (t > 0) hit an object other than `skip_obj` (a convex object the
// ray is leaving)? False only if it misses every object's bounding sphere (radius grown
// past the test's rounding error): then no triangle can be hit, and a traversal would
// return a miss -- the test replaces it exactly.
template <class R>
SST_D bool ray_may_hit(const DevScene<R>& sc, V3<R> x, V3<R> d, int skip_obj) {
    for (uint32_t o = 0; o < sc.n_objects; ++o) {
        if (static_cast<int>(o) == skip_obj) continue;
        const ObjK<R>& ob = sc.objs[o];
        const V3<R> oc = mk<R>(ob.bsphere[0], ob.bsphere[1], ob.bsphere[2]) - x;
        const R b = dot(oc, d), r = ob.bsphere[3];
        if (b + r >= R(0) && dot(oc, oc) - b * b <= r * r) return true;
    }
    return false;
}

// Camera ray direction of (pixel, sample): jitter = the first two draws of the pixel
// stream (DESIGN.md camera model).
template <class R>
SST_D V3<R> camera_dir(const TraceArgs<R>& a, uint32_t pixel, uint32_t sample) {
    const DevScene<R>& sc = a.sc;
    Rng cam{rng_key(a.seed, 0x06, pixel, sample)};  // kRenderPixel
    const R jx = cam.uniform<R>();
    const R jy = cam.uniform<R>();
    const uint32_t px = pixel % sc.width, py = pixel / sc.width;
    const R sx = (R(2) * (static_cast<R>(px) + jx) / static_cast<R>(sc.width) - R(1)) * sc.tan_half * sc.aspect;
    const R sy = (R(1) - R(2) * (static_cast<R>(py) + jy) / static_cast<R>(sc.height)) * sc.tan_half;
    return normalize(sc.cam_fwd + sc.cam_right * sx + sc.cam_up * sy);
}

template <class R, bool EXPLICIT>
SST_D void path_init(const TraceArgs<R>& a, uint64_t id, PathLocal<R>& p) {
    if (a.keys) {  // camera pre-pass: the id-th path whose camera ray can hit the scene
        id = EXPLICIT ? static_cast<uint64_t>(a.keys[id])
                      : static_cast<uint64_t>(a.keys[id / 3]) * 3u + static_cast<uint32_t>(id % 3);
    }
    uint32_t pixel, sample, c;
    if (EXPLICIT) {
        pixel = a.pixel[id];
        sample = a.sample[id];
        c = a.channel[id];
    } else if (id <= 0xffffffffull) {  // id = (s_local * n_pix + pixel) * 3 + c (32-bit divisions)
        const uint32_t id32 = static_cast<uint32_t>(id), rest = id32 / 3u;
        c = id32 - 3u * rest;
        pixel = rest % a.n_pix;
        sample = a.sample_begin + rest / a.n_pix;
    } else {
        c = static_cast<uint32_t>(id % 3);
        const uint64_t rest = id / 3;
        pixel = static_cast<uint32_t>(rest % a.n_pix);
        sample = a.sample_begin + static_cast<uint32_t>(rest / a.n_pix);
    }
    const DevScene<R>& sc = a.sc;
    p.x = sc.cam_pos;
    p.w = camera_dir(a, pixel, sample);
    p.rng.s = rng_key(a.seed, 0x07, pixel, 3ull * sample + c);  // kRenderChannel
    p.L = R(0);
    p.id = id;
    p.seg = 0;
    p.pixel = pixel;
    p.obj = -1;
    p.skip = -1;
    p.cull = -1;
    p.c = static_cast<uint8_t>(c);
    p.r_valid = false;
    p.pending = false;
    p.waited = 0;
    p.tpend = false;
    p.twaited = 0;
    p.t_pend = R(0);
}

// A flight inside a CONVEX object whose end point is conservatively inside (stored SDF
// value < 0: the whole safe ball around it is in the medium) stays inside: the segment
// between two points of a convex set lies in it, so the traversal cannot find a leaving
// crossing (the start point is excluded by the skip triangle / t_min and the FP32
// orientation filter). FP32 only (FP64 keeps the reference's traversal of every flight).
// Any object: the safe balls at the two end points (radius r_x at the start -- the
// larger of the SDF and skip-grid bounds -- and the SDF safe radius at the end) cover the
// segment when r_x + r_y > t, so it cannot cross the surface either.
// Exact end-point containment for convex objects (FP32): the end point e lies in a
// boundary SDF voxel V that holds a point q inside the object (its centre, stored -0, or
// a corner -- checked against every face plane at upload); F_V = every face that can
// meet V. If e is strictly inside every plane of F_V, e is inside the object: otherwise
// the segment [q, e] (inside V) leaves the object through a face of F_V and e would be
// beyond that face's plane. A convex object then
// contains the whole flight [x, e] (x inside), so it cannot cross the surface --
// exactly the traversal's answer, without the traversal. The margin plane_eps (>> the
// FP32 error of the plane test) keeps end points on the surface on the traced side.
template <class R>
SST_D bool end_inside_planes(const ObjK<R>& ob, uint32_t vox, V3<R> e) {
    if constexpr (Real<R>::kIsDouble) {
        return false;
    } else {
        if (!ob.plane_off) return false;
        const uint32_t b = ldg_keep(ob.plane_off + vox), en = ldg_keep(ob.plane_off + vox + 1);
        if (b == en) return false;
        for (uint32_t k = b; k < en; ++k) {
            const float4 pl = ldg_keep(ob.planes + k);
            if (!(fmaf(pl.x, e.x, fmaf(pl.y, e.y, fmaf(pl.z, e.z, -pl.w))) < -ob.plane_eps)) return false;
        }
        return true;
    }
}

// Any closed object: a flight whose both ends lie in the same listed voxel V and strictly
// inside all of V's planes stays in the medium. Every point of the segment is then
// strictly inside those planes (an intersection of half-spaces is convex) and in V, so
// -- by the argument above, which needs no convexity: a point of V outside the object
// lies beyond the plane of the face through which [q, point] leaves last -- every point
// is interior: the segment meets no face.
template <class R>
SST_D bool seg_inside_planes(const ObjK<R>& ob, uint32_t vox, V3<R> x, V3<R> e) {
    if constexpr (Real<R>::kIsDouble) {
        return false;
    } else {
        if (!ob.plane_off) return false;
        const uint32_t b = ldg_keep(ob.plane_off + vox), en = ldg_keep(ob.plane_off + vox + 1);
        if (b == en) return false;
        for (uint32_t k = b; k < en; ++k) {
            const float4 pl = ldg_keep(ob.planes + k);
            if (!(fmaf(pl.x, e.x, fmaf(pl.y, e.y, fmaf(pl.z, e.z, -pl.w))) < -ob.plane_eps) ||
                !(fmaf(pl.x, x.x, fmaf(pl.y, x.y, fmaf(pl.z, x.z, -pl.w))) < -ob.plane_eps))
                return false;
        }
        return true;
    }
}

// Culling rule that decided a contained flight (verification counters).
enum : int { kContainNone = 0, kContainSdf = 1, kContainPlanes = 2 };
template <class R>
SST_D int flight_contained_rule(const ObjK<R>& ob, V3<R> x, V3<R> w, R t, R r_x) {
    if (Real<R>::kIsDouble) return kContainNone;
    bool in_grid;
    uint32_t vox = 0;
    const V3<R> e = x + w * t;
    const R v = sdf_raw(ob, e, &in_grid, &vox);
    if (!in_grid) return kContainNone;
    if (v < R(0) && (ob.convex || t < r_x - v)) return kContainSdf;
    if (ob.convex) return end_inside_planes(ob, vox, e) ? kContainPlanes : kContainNone;
    uint32_t vox_x;
    return sdf_voxel(ob, x, &vox_x) && vox_x == vox && seg_inside_planes(ob, vox, x, e) ? kContainPlanes
                                                                                        : kContainNone;
}
template <class R>
SST_D bool flight_contained(const ObjK<R>& ob, V3<R> x, V3<R> w, R t, R r_x) {
    return flight_contained_rule(ob, x, w, t, r_x) != kContainNone;
}

// A convex object's end point e strictly beyond one of its voxel's face planes (margin
// plane_eps) is outside the object: a convex object lies inside every face plane.
template <class R>
SST_D bool end_beyond_a_plane(const ObjK<R>& ob, uint32_t vox, V3<R> e) {
    if constexpr (Real<R>::kIsDouble) {
        return false;
    } else {
        if (!ob.plane_off) return false;
        const uint32_t b = ldg_keep(ob.plane_off + vox), en = ldg_keep(ob.plane_off + vox + 1);
        for (uint32_t k = b; k < en; ++k) {
            const float4 pl = ldg_keep(ob.planes + k);
            if (fmaf(pl.x, e.x, fmaf(pl.y, e.y, fmaf(pl.z, e.z, -pl.w))) > ob.plane_eps) return true;
        }
        return false;
    }
}

// Where a flight ends relative to its medium (wavefront logic pass, the end point's SDF
// value already loaded): kEndIn -- provably inside, no traversal (flight_contained);
// kEndOut -- a convex object's end point provably outside (off the grid, a voxel wholly
// outside, or beyond a face plane): the flight leaves the object; kEndUnknown.
enum : int { kEndUnknown = 0, kEndIn = 1, kEndOut = 2 };
template <class R>
SST_D int end_where(const ObjK<R>& ob, R v_end, bool in_grid, uint32_t vox, V3<R> x, V3<R> e, R t, R r_x) {
    if (Real<R>::kIsDouble) return kEndUnknown;
    if (!in_grid) return ob.convex ? kEndOut : kEndUnknown;  // the grid covers the mesh box
    if (v_end < R(0) && (ob.convex || t < r_x - v_end)) return kEndIn;
    if (ob.convex) {
        if (v_end > R(0)) return kEndOut;  // conservative SDF: the whole voxel is outside
        if (end_inside_planes(ob, vox, e)) return kEndIn;
        return end_beyond_a_plane(ob, vox, e) ? kEndOut : kEndUnknown;
    }
    uint32_t vox_x;
    return sdf_voxel(ob, x, &vox_x) && vox_x == vox && seg_inside_planes(ob, vox, x, e) ? kEndIn : kEndUnknown;
}

// FP32 leak detection: the conservative SDF value at x is > 0 (or x is off the grid)
// only if x is OUTSIDE the object -- a path that believes it is inside missed its
// exit crossing (non-watertight FP32 Moller-Trumbore at an edge). FP64 keeps the
// reference's semantics untouched.
template <class R>
SST_D bool leaked(const ObjK<R>& ob, R v, bool in_grid) {
    return !Real<R>::kIsDouble && (!in_grid || v > ob.sdf_voxel * R(1e-4));
}
// Recovery: continue as an outside ray from x (it re-enters or escapes), instead of
// random-walking in the void until absorbed (10^5+ events: a launch-long tail).
template <class R>
SST_D void recover_leak(PathLocal<R>& p, const ObjK<R>& ob) {
    p.cull = ob.convex ? p.obj : -1;
    p.obj = -1;
    p.skip = -1;
    p.r_valid = false;
}

// One iteration of the path loop, written as a fixed sequence of phases in which
// every expensive operation (BVH traversal, sphere step, NEE shadow traversal)
// has exactly ONE call site: the kernel is instruction-cache bound, and lanes of a
// warp that reached the same operation by different routes (e.g. NEE after a
// sphere step and NEE after a delta-tracking event) execute it together.
//   1. traversal : medium entry (outside) or free flight (inside, unless the
//                  conservative SDF ball already contains the whole flight)
//   2. resolve   : escape / enter / leave / collide
//   3. collision : one delta-tracking event, or a sphere-step REQUEST (ST, r > r_min)
//   4. sphere    : warp-regrouped: requested sphere steps wait until at least
//                  `sphere_batch` lanes (or every live lane) want one, so the
//                  ~3k-instruction CVAE step runs on a mostly full warp
//   5. NEE       : shadow ray toward the point light
// Returns -1 while the path lives, else its end code. `alive` lanes only.
template <class R, bool ST>
SST_D int path_advance(const TraceArgs<R>& a, PathLocal<R>& p, LaneStats& st, bool alive) {
    const DevScene<R>& sc = a.sc;
    int end = -1;
    const bool active = alive && !p.pending;  // lanes waiting for a sphere batch sit out 1-3
    // ---- 1. traversal
    bool trace = false, inside = false;
    R t_max = Real<R>::kInf, t_free = Real<R>::kInf;
    const ObjK<R>* ob = alive && p.obj >= 0 ? &sc.objs[p.obj] : nullptr;
    if (active) {
        inside = p.obj >= 0;
        if (inside && !p.tpend && !p.r_valid) {
            bool in_grid;
            const R v = sdf_raw(*ob, p.x, &in_grid);
            p.r_here = v < R(0) ? -v : R(0);
            p.r_valid = true;
            if (leaked(*ob, v, in_grid)) {
                recover_leak(p, *ob);
                inside = false;
            }
        }
        if (p.tpend) {  // flight drawn in an earlier iteration, traversal still pending
            t_free = p.t_pend;
            trace = true;
        } else if (inside) {
            const MediumK<R>& m = ob->med[p.c];
            if (m.sigma_t > R(0)) {  // sample_free_path (optics.cpp:55-60)
                const R u = p.rng.template uniform<R>();
                if (Real<R>::kIsDouble) t_free = -Real<R>::log1p_(-u) / m.sigma_t;
                else t_free = -Real<R>::div_(Real<R>::log_(R(1) - u), m.sigma_t);
            }
            // A flight shorter than a conservative distance to the surface cannot
            // reach the boundary: skip the traversal (exact). Bounds: the scene SDF
            // radius and, when that is too coarse, the finer skip grid.
            trace = !(t_free < p.r_here);
            if (trace) {
                const R rs = skip_radius(*ob, p.x);
                trace = !(t_free < rs);
                if (trace && a.convex_end)
                    trace = !flight_contained(*ob, p.x, p.w, t_free, Real<R>::fmax_(p.r_here, rs));
            }
        } else {
            trace = ray_may_hit(sc, p.x, p.w, p.cull);  // else a miss (escape) without traversal
        }
        if (inside) t_max = t_free;
    }
    // Traversals are regrouped per warp like sphere steps (trace_batch > 0): a lane
    // whose flight needs the BVH parks it (t_pend) while lanes with culled flights keep
    // iterating, until enough lanes (or every live lane) wait.
    if (a.trace_batch > 0) {
        if (active && trace && !p.tpend) {
            p.tpend = true;
            p.t_pend = t_free;
            p.twaited = 0;
        }
        const unsigned tp = __ballot_sync(0xffffffffu, alive && p.tpend);
        if (tp) {
            const unsigned live = __ballot_sync(0xffffffffu, alive);
            const unsigned sp = __ballot_sync(0xffffffffu, alive && p.pending);
            const bool starving = __any_sync(0xffffffffu, alive && p.tpend && p.twaited >= 32);
            const bool go = __popc(tp) >= a.trace_batch || (live & ~(tp | sp)) == 0u || starving;
            if (alive && p.tpend) {
                if (go) {
                    p.tpend = false;
                } else {
                    ++p.twaited;
                    trace = false;
                }
            }
        }
    }
    else if (active) p.tpend = false;  // resumed wavefront slot: its queued traversal runs now
    const bool proceed = active && !p.tpend;  // this lane's flight is resolved this iteration
    bool hit = false;
    R t_hit = R(0);
    Hit h{0, 0};
    if (trace && proceed) {
        const RayK<R> ray = make_ray(p.x, p.w);
        const int want = Real<R>::kIsDouble ? 0 : (inside ? -1 : 1);
        // an in-medium flight starts at its object's subtree (disjoint objects, FP32)
        hit = intersect_nearest(sc, ray, p.skip >= 0 ? sc.surf_eps : sc.t_min, t_max, p.skip, p.cull, want,
                                &t_hit, &h, st.nodes, st.tris, inside ? ob->bvh_root : 0);
        ++st.traversals;
    }
#ifdef SST_TRACE_DEBUG
    if (active) printf("[gpu] seg=%u obj=%d x=(%.17g,%.17g,%.17g) w=(%.17g,%.17g,%.17g) trace=%d tfree=%.17g hit=%d thit=%.17g rhere=%.17g\n",
                       p.seg, p.obj, (double)p.x.x, (double)p.x.y, (double)p.x.z, (double)p.w.x, (double)p.w.y, (double)p.w.z,
                       (int)trace, (double)t_free, (int)hit, (double)t_hit, (double)p.r_here);
#endif
    // ---- 2. resolve
    bool collide = false;
    if (proceed) {
        if (!inside) {
            if (!hit) {
                p.L += sc.bg[p.c];
                end = kEndEscaped;
            } else {  // medium entry (index-matched boundary)
                p.x = p.x + p.w * t_hit;
                p.obj = static_cast<int>(h.obj);
                p.cull = -1;
                p.skip = Real<R>::kIsDouble ? -1 : static_cast<int>(h.tri);
                p.r_valid = false;
            }
        } else if (hit) {  // leaves the medium
            p.x = p.x + p.w * t_hit;
            p.cull = ob->convex ? p.obj : -1;
            p.obj = -1;
            p.skip = Real<R>::kIsDouble ? -1 : static_cast<int>(h.tri);
        } else {  // collision
            p.skip = -1;
            p.x = p.x + p.w * t_free;
            p.r_valid = false;
            if (p.seg >= (ST ? sc.cap_st : sc.cap_pt)) {
                p.L = R(0);  // dropped
                end = kEndCapped;
            } else {
                ++p.seg;
                collide = true;
            }
        }
    }
    // ---- 3. collision
    bool nee = false;
    V3<R> nee_p, nee_w;
    R nee_wt = R(1);
    bool event = collide;
    if (ST && collide) {
        bool in_grid;
        const R v = sdf_raw(*ob, p.x, &in_grid);
        p.r_here = v < R(0) ? -v : R(0);
        p.r_valid = true;
        if (leaked(*ob, v, in_grid)) {  // not in the medium: no event here
            recover_leak(p, *ob);
            collide = false;
            event = false;
        }
#ifdef SST_TRACE_DEBUG
        printf("[gpu]   collide r=%.17g r_min=%.17g\n", (double)p.r_here, (double)ob->med[p.c].r_min);
#endif
        if (p.r_here > ob->med[p.c].r_min) {
            p.pending = true;
            p.waited = 0;
            event = false;
        }
    }
    if (event) {  // delta-tracking event: roulette, NEE, HG scatter
        ++st.events;
        const MediumK<R>& m = ob->med[p.c];
        if (!((p.rng.next() >> 11) < m.survive_below)) {  // u < phi, bit-exact
            end = kEndAbsorbed;
        } else {
            nee = a.nee != 0;
            nee_p = p.x;
            nee_w = p.w;  // incoming direction (NEE draws no random numbers)
            const R u1 = p.rng.template uniform<R>();
            const R u2 = p.rng.template uniform<R>();
            p.w = hg_sample(m.g, p.w, u1, u2);
        }
    }
    // ---- 4. sphere steps, regrouped per warp
    if (ST) {
        const unsigned pend = __ballot_sync(0xffffffffu, alive && p.pending);
        if (pend) {
            const unsigned live = __ballot_sync(0xffffffffu, alive && end < 0);
            const bool starving = __any_sync(0xffffffffu, alive && p.pending && p.waited >= 64);
            const unsigned tpend = __ballot_sync(0xffffffffu, alive && p.tpend);
            const bool go = __popc(pend) >= a.sphere_batch || (live & ~(pend | tpend)) == 0u || starving;
            if (alive && p.pending) {
                if (!go) {
                    ++p.waited;
                } else {
                    p.pending = false;
                    ++st.sphere;
                    StepOut<R> o;
                    const MediumK<R>& m = ob->med[p.c];
                    if (!sphere_step(m, p.w, p.x, p.r_here, a.nee != 0, p.rng, o, st.dc)) {
                        p.L = R(0);
                        end = kEndError;
                    } else if (o.absorbed) {
                        end = kEndAbsorbed;
                    } else {
                        nee = a.nee != 0;
                        nee_p = o.rep_pos;
                        nee_w = o.rep_dir;
                        nee_wt = o.lambda;
                        p.x = o.exit_pos;
                        p.w = o.exit_dir;
                        p.r_valid = false;
                    }
                }
            }
        }
    }
    // ---- 5. NEE
    if (nee) {
        const uint64_t t0 = st.tris;
        p.L += nee_term(sc, ob->med[p.c], p.c, nee_p, nee_w, nee_wt, st.tris,
                        ob->convex ? static_cast<int>(ob - sc.objs) : -1);
        st.shadow_tris += st.tris - t0;
        ++st.shadow;
    }
    return end;
}

template <class T>
SST_D T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Wavefront slot -> path state (wavefront.cuh).
template <class R>
SST_D void load_slot(const WfPool<R>& q, uint32_t s, PathLocal<R>& p, uint32_t* phase, const V3<R>& cam,
                     bool need_tpend, bool fold);

template <class R, bool ST, bool EXPLICIT>
SST_D void trace_persistent(const TraceArgs<R>& a) {
    const unsigned lane = threadIdx.x & 31u;
    PathLocal<R> p;
    bool alive = false, exhausted = false;
    LaneStats st;
    for (;;) {
        const unsigned need = __ballot_sync(0xffffffffu, !alive && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            unsigned long long base = 0;
            if (static_cast<int>(lane) == leader) base = atomicAdd(a.work, static_cast<unsigned long long>(__popc(need)));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (!alive && !exhausted) {
                const uint64_t my = base + __popc(need & ((1u << lane) - 1u));
                if (a.resume) {  // hand-off of the wavefront pool's live slots
                    if (my < a.pool.counts[kQResume]) {
                        uint32_t phase;  // the slot's staged NEE contributions are added here
                        load_slot(a.pool, a.pool.q_live[my], p, &phase, a.sc.cam_pos, true, true);
                        if (phase >= 4u) {  // kPhEnded(Escaped): absorbed / escaped once those were in
                            if (phase == 5u) p.L += a.sc.bg[p.c];
                            a.radiance[p.id] = p.L;
                            if (a.segments) a.segments[p.id] = p.seg;
                            if (a.exit_state) write_exit_state(a.exit_state, p);
                            ++st.paths;
                            st.seg += p.seg;
                            st.absorbed += phase == 4u;
                            st.escaped += phase == 5u;
                        } else {
                            alive = true;
                        }
                    } else {
                        exhausted = true;
                    }
                } else if (my < a.n_paths) {
                    path_init<R, EXPLICIT>(a, my, p);
                    alive = true;
                } else {
                    exhausted = true;
                }
            }
        }
        if (!__any_sync(0xffffffffu, alive)) {
            if (__all_sync(0xffffffffu, exhausted)) break;
            continue;  // every fetched slot had already ended (hand-off): fetch again
        }
        st.lane_iters += alive;
        st.warp_iters += lane == 0;
        const int end = path_advance<R, ST>(a, p, st, alive);
        if (alive && end >= 0) {
            a.radiance[p.id] = p.L;
            if (a.segments) a.segments[p.id] = p.seg;
            if (a.exit_state) write_exit_state(a.exit_state, p);
            ++st.paths;
            st.seg += p.seg;
            st.escaped += end == kEndEscaped;
            st.absorbed += end == kEndAbsorbed;
            st.capped += end == kEndCapped;
            st.errors += end == kEndError;
            alive = false;
        }
    }
    unsigned long long v[kStCount] = {st.paths, st.seg, st.sphere, st.events, st.dc.l, st.dc.p,
                                      st.dc.e, st.absorbed, st.escaped, st.capped, st.errors, st.shadow,
                                      st.traversals, st.nodes, st.tris, st.lane_iters, st.warp_iters,
                                      st.shadow_tris, st.wf_slots};
    unsigned long long* dst = a.stats + static_cast<size_t>(blockIdx.x % kStCopies) * kStCount;
#pragma unroll
    for (int k = 0; k < kStCount; ++k) {
        const unsigned long long s = warp_sum(v[k]);
        if (lane == 0 && s) atomicAdd(dst + k, s);
    }
}

}  // namespace sstg
