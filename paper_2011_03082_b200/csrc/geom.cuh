// geom.cuh -- software ray traversal (B200 has no RT cores) and the SDF lookup.
//
//   BVH2 with both child boxes stored in the parent (64 B FP32 node = 4 x LDG.128),
//   near-child-first traversal, per-ray inverse direction.
//   Triangle test: Moller-Trumbore with the operation order of bvh.cpp:11-27.
//   intersect_nearest  ~ Bvh::intersect      (bvh.cpp:115-148)
//   optical_depth      ~ Bvh::intersect_all + in-medium toggling (bvh.cpp:150-179,
//                        SPEC.md:597), restated order-free: for closed outward-oriented
//                        meshes the in-medium length of object j on [0, d] from a
//                        start inside j is sum_hits(j) sign * t with sign = +1 when the
//                        ray leaves (det < 0 in Moller-Trumbore) and -1 when it enters.
//                        No hit list, no sort.
//   sdf_radius         ~ query_safe_radius   (sdf.cpp:60-69)
#pragma once

#include "common.cuh"
#include "step.cuh"
#include "types.cuh"

namespace sstg {


// --------------------------------------------------------------- SDF lookup
template <class R>
SST_D R sdf_raw(const ObjK<R>& o, V3<R> p, bool* inside_grid, uint32_t* vox = nullptr) {
    R rx, ry, rz;
    if (Real<R>::kIsDouble) {  // (point - origin) / voxel_size, sdf.cpp:61
        rx = (p.x - o.sdf_origin[0]) / o.sdf_voxel;
        ry = (p.y - o.sdf_origin[1]) / o.sdf_voxel;
        rz = (p.z - o.sdf_origin[2]) / o.sdf_voxel;
    } else {
        rx = (p.x - o.sdf_origin[0]) * o.sdf_inv_voxel;
        ry = (p.y - o.sdf_origin[1]) * o.sdf_inv_voxel;
        rz = (p.z - o.sdf_origin[2]) * o.sdf_inv_voxel;
    }
    *inside_grid = false;
    if (rx < R(0) || ry < R(0) || rz < R(0)) return R(0);
    const uint32_t x = static_cast<uint32_t>(rx), y = static_cast<uint32_t>(ry),
                   z = static_cast<uint32_t>(rz);
    if (x >= o.dims[0] || y >= o.dims[1] || z >= o.dims[2]) return R(0);
    *inside_grid = true;
    const uint32_t k = (z * o.dims[1] + y) * o.dims[0] + x;
    if (vox) *vox = k;
    return static_cast<R>(ldg_keep(o.sdf + k));
}

// The SDF voxel of p (sdf_raw's index arithmetic, no load); false off the grid.
template <class R>
SST_D bool sdf_voxel(const ObjK<R>& o, V3<R> p, uint32_t* vox) {
    const R rx = (p.x - o.sdf_origin[0]) * o.sdf_inv_voxel;
    const R ry = (p.y - o.sdf_origin[1]) * o.sdf_inv_voxel;
    const R rz = (p.z - o.sdf_origin[2]) * o.sdf_inv_voxel;
    if (rx < R(0) || ry < R(0) || rz < R(0)) return false;
    const uint32_t x = static_cast<uint32_t>(rx), y = static_cast<uint32_t>(ry), z = static_cast<uint32_t>(rz);
    if (x >= o.dims[0] || y >= o.dims[1] || z >= o.dims[2]) return false;
    *vox = (z * o.dims[1] + y) * o.dims[0] + x;
    return true;
}

// query_safe_radius: -v inside (v < 0), else 0; 0 outside the grid.
template <class R>
SST_D R sdf_radius(const ObjK<R>& o, V3<R> p) {
    bool in;
    const R v = sdf_raw(o, p, &in);
    return v < R(0) ? -v : R(0);
}

// Conservative distance-to-surface bound from the fine skip grid (0 outside it).
template <class R>
SST_D R skip_radius(const ObjK<R>& o, V3<R> p) {
    if (!o.skip) return R(0);
    const R rx = (p.x - o.sdf_origin[0]) * o.skip_inv_voxel;
    const R ry = (p.y - o.sdf_origin[1]) * o.skip_inv_voxel;
    const R rz = (p.z - o.sdf_origin[2]) * o.skip_inv_voxel;
    if (rx < R(0) || ry < R(0) || rz < R(0)) return R(0);
    const uint32_t x = static_cast<uint32_t>(rx), y = static_cast<uint32_t>(ry), z = static_cast<uint32_t>(rz);
    if (x >= o.skip_dims[0] || y >= o.skip_dims[1] || z >= o.skip_dims[2]) return R(0);
    const uint8_t q = ldg_keep(o.skip + (static_cast<size_t>(z) * o.skip_dims[1] + y) * o.skip_dims[0] + x);
    return static_cast<R>(q) * o.skip_unit;
}

// --------------------------------------------------------------- ray setup
template <class R>
struct RayK {
    V3<R> o, d, inv;
    V3<R> oi;  // FP32: o * inv, so each slab plane is one FFMA (t = lo * inv - oi)
};

template <class R>
SST_D RayK<R> make_ray(V3<R> o, V3<R> d) {
    RayK<R> r;
    r.o = o;
    r.d = d;
    if (Real<R>::kIsDouble) {  // bvh.cpp:91 computes 1/dir per axis (inf allowed)
        r.inv = mk<R>(R(1) / d.x, R(1) / d.y, R(1) / d.z);
        r.oi = r.o;
    } else {
        const float e = 1e-20f;
        r.inv = mk<R>(__fdividef(1.0f, fabsf(d.x) > e ? d.x : copysignf(e, d.x)),
                      __fdividef(1.0f, fabsf(d.y) > e ? d.y : copysignf(e, d.y)),
                      __fdividef(1.0f, fabsf(d.z) > e ? d.z : copysignf(e, d.z)));
        r.oi = mk<R>(o.x * r.inv.x, o.y * r.inv.y, o.z * r.inv.z);
    }
    return r;
}

// Traversal stacks: registers/local memory (megakernel), or shared memory with a
// per-thread stride (wavefront trace kernel: no local-memory traffic through L2).
template <class R, int N>
struct LocalStack {
    int n[N];
    R t[N];
    SST_D int& node(int i) { return n[i]; }
    SST_D R& dist(int i) { return t[i]; }
};
template <class R>
struct SharedStack {
    int* n;
    R* t;
    int stride;
    SST_D int& node(int i) { return n[i * stride]; }
    SST_D R& dist(int i) { return t[i * stride]; }
};

// Three-input FP32 min / max (sm_100: one FMNMX3 instead of two FMNMX).
SST_D float max3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
SST_D float min3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// slab_hit (bvh.cpp:88-101) returning the entry distance.
template <class R>
SST_D bool slab(const RayK<R>& r, R lox, R hix, R loy, R hiy, R loz, R hiz, R t_min, R t_max,
                R* t_enter) {
    R t0 = t_min, t1 = t_max;
    if constexpr (!Real<R>::kIsDouble) {  // FP32: branch-free min/max (inv is finite, no NaN);
        // one FFMA per plane -- its rounding (<= 1 ulp of t) is covered by the outward
        // box padding of the FP32 nodes (host.cpp down/up, ~2e-7 relative)
        const R nx = fmaf(lox, r.inv.x, -r.oi.x), fx = fmaf(hix, r.inv.x, -r.oi.x);
        const R ny = fmaf(loy, r.inv.y, -r.oi.y), fy = fmaf(hiy, r.inv.y, -r.oi.y);
        const R nz = fmaf(loz, r.inv.z, -r.oi.z), fz = fmaf(hiz, r.inv.z, -r.oi.z);
        t0 = max3f(fmaxf(t0, fminf(nx, fx)), fminf(ny, fy), fminf(nz, fz));
        t1 = min3f(fminf(t1, fmaxf(nx, fx)), fmaxf(ny, fy), fmaxf(nz, fz));
        *t_enter = t0;
        return t0 <= t1;
    }
    R n = (lox - r.o.x) * r.inv.x, f = (hix - r.o.x) * r.inv.x;
    if (n > f) { const R t = n; n = f; f = t; }
    t0 = Real<R>::fmax_(t0, n);
    t1 = Real<R>::fmin_(t1, f);
    n = (loy - r.o.y) * r.inv.y;
    f = (hiy - r.o.y) * r.inv.y;
    if (n > f) { const R t = n; n = f; f = t; }
    t0 = Real<R>::fmax_(t0, n);
    t1 = Real<R>::fmin_(t1, f);
    n = (loz - r.o.z) * r.inv.z;
    f = (hiz - r.o.z) * r.inv.z;
    if (n > f) { const R t = n; n = f; f = t; }
    t0 = Real<R>::fmax_(t0, n);
    t1 = Real<R>::fmin_(t1, f);
    *t_enter = t0;
    return t0 <= t1;
}

// Moller-Trumbore (bvh.cpp:11-27). Returns t (> t_min, < t_max) or a negative
// value on a miss; *det_out receives det (sign = crossing direction).
template <class R>
SST_D R ray_tri(const RayK<R>& r, V3<R> v0, V3<R> e1, V3<R> e2, R t_min, R t_max, R* det_out) {
    const V3<R> pvec = cross(r.d, e2);
    const R det = dot(e1, pvec);
    *det_out = det;
    if (Real<R>::fabs_(det) < R(1e-14)) return R(-1);
    const R inv_det = Real<R>::div_(R(1), det);  // FP32: MUFU reciprocal (2 ulp); FP64: IEEE
    const V3<R> tvec = r.o - v0;
    const R u = dot(tvec, pvec) * inv_det;
    if (u < R(0) || u > R(1)) return R(-1);
    const V3<R> qvec = cross(tvec, e1);
    const R v = dot(r.d, qvec) * inv_det;
    if (v < R(0) || u + v > R(1)) return R(-1);
    const R t = dot(e2, qvec) * inv_det;
    if (t <= t_min || t >= t_max) return R(-1);
    return t;
}

template <class R>
SST_D void load_node(const void* nodes, int i, R (&b)[12], int& c0, int& c1, int& o0, int& o1);
template <>
SST_D void load_node<float>(const void* nodes, int i, float (&b)[12], int& c0, int& c1, int& o0, int& o1) {
    const NodeF* n = static_cast<const NodeF*>(nodes) + i;
    const float4 a = ldg_keep(&n->a), bb = ldg_keep(&n->b), c = ldg_keep(&n->c);
    const int4 d = ldg_keep(&n->d);
    // b = lo0x hi0x lo0y hi0y lo0z hi0z | lo1x hi1x lo1y hi1y lo1z hi1z
    b[0] = a.x; b[1] = a.y; b[2] = a.z; b[3] = a.w; b[4] = c.x; b[5] = c.y;
    b[6] = bb.x; b[7] = bb.y; b[8] = bb.z; b[9] = bb.w; b[10] = c.z; b[11] = c.w;
    c0 = d.x;
    c1 = d.y;
    o0 = d.z;
    o1 = d.w;
}
template <>
SST_D void load_node<double>(const void* nodes, int i, double (&b)[12], int& c0, int& c1, int& o0, int& o1) {
    const NodeD* n = static_cast<const NodeD*>(nodes) + i;
    b[0] = n->lo0[0]; b[1] = n->hi0[0]; b[2] = n->lo0[1]; b[3] = n->hi0[1]; b[4] = n->lo0[2]; b[5] = n->hi0[2];
    b[6] = n->lo1[0]; b[7] = n->hi1[0]; b[8] = n->lo1[1]; b[9] = n->hi1[1]; b[10] = n->lo1[2]; b[11] = n->hi1[2];
    c0 = n->c0;
    c1 = n->c1;
    o0 = n->pad0;
    o1 = n->pad1;
}

template <class R>
SST_D void load_tri(const void* tris, uint32_t i, V3<R>& v0, V3<R>& e1, V3<R>& e2, uint32_t& obj,
                    uint32_t& id);
template <>
SST_D void load_tri<float>(const void* tris, uint32_t i, V3<float>& v0, V3<float>& e1,
                           V3<float>& e2, uint32_t& obj, uint32_t& id) {
    const TriF* t = static_cast<const TriF*>(tris) + i;
    const float4 a = ldg_keep(&t->v0o), b = ldg_keep(&t->e1i), c = ldg_keep(&t->e2);
    v0 = mk(a.x, a.y, a.z);
    e1 = mk(b.x, b.y, b.z);
    e2 = mk(c.x, c.y, c.z);
    obj = __float_as_uint(a.w);
    id = __float_as_uint(b.w);
}
template <>
SST_D void load_tri<double>(const void* tris, uint32_t i, V3<double>& v0, V3<double>& e1,
                            V3<double>& e2, uint32_t& obj, uint32_t& id) {
    const TriD* t = static_cast<const TriD*>(tris) + i;
    v0 = mk(t->v0[0], t->v0[1], t->v0[2]);
    e1 = mk(t->e1[0], t->e1[1], t->e1[2]);
    e2 = mk(t->e2[0], t->e2[1], t->e2[2]);
    obj = t->obj;
    id = t->id;
}


// Nearest hit with t in (t_min, t_max), ignoring triangle `skip` (FP32
// self-intersection guard for rays leaving a surface; -1 = none).
//
// While-while traversal with postponed leaves (Aila & Laine 2009): a lane that
// reaches a leaf parks it and keeps descending interior nodes until every lane
// of the (active) warp holds a leaf, then the leaves are intersected together --
// interior-node work and triangle work each run on mostly full warps.
constexpr int kDone = 0x7fffffff;

// want_sign: +1 accept only entering crossings (det > 0), -1 only leaving ones,
// 0 any. FP32 rays use it (a ray outside every medium can only enter, a flight
// inside can only leave): with outward-wound meshes this rejects the spurious
// re-hits of neighbouring triangles that FP32 rounding produces at surfaces.
// Traversal state of one ray. round() = one while-while round: interior nodes until
// this lane holds a leaf and every active lane does (or is done), then the parked
// leaf (and a leaf the traversal sits on). The wavefront trace kernel drives rounds
// directly so that lanes whose ray finished take a new ray between rounds.
template <class R>
struct Trav {
    int node;    // interior (>= 0), leaf (< 0) or kDone
    int leaf;    // postponed leaf (< 0) or 0 = none
    int sp;
    R t_best;
    bool found;
    Hit hit;
    SST_D void init(R t_max, int root = 0) {
        node = root;
        leaf = 0;
        sp = 0;
        t_best = t_max;
        found = false;
        hit = Hit{0, 0};
    }
    SST_D bool done() const { return node == kDone && leaf == 0; }

    template <class Stack>
    SST_D int pop(Stack& stk) {
        while (sp > 0) {
            --sp;
            if (stk.dist(sp) <= t_best) return stk.node(sp);
        }
        return kDone;
    }

    template <class Stack>
    SST_D void round(const DevScene<R>& sc, const RayK<R>& ray, R t_min, int skip, int cull_obj, int want_sign,
                     uint64_t& n_nodes, uint64_t& n_tris, Stack& stk) {
        // interior nodes until this lane holds a leaf and all lanes do
        while (node != kDone && node >= 0) {
            R b[12];
            int c0, c1, o0, o1;
            load_node<R>(sc.nodes, node, b, c0, c1, o0, o1);
            ++n_nodes;
            R t0, t1;
            const bool h0 = slab(ray, b[0], b[1], b[2], b[3], b[4], b[5], t_min, t_best, &t0) &&
                            (cull_obj < 0 || o0 != cull_obj);
            const bool h1 = slab(ray, b[6], b[7], b[8], b[9], b[10], b[11], t_min, t_best, &t1) &&
                            (cull_obj < 0 || o1 != cull_obj);
            if (h0 && h1) {
                const bool first0 = t0 <= t1;
                stk.node(sp) = first0 ? c1 : c0;
                stk.dist(sp) = first0 ? t1 : t0;
                ++sp;
                node = first0 ? c0 : c1;
            } else if (h0) {
                node = c0;
            } else if (h1) {
                node = c1;
            } else {
                node = pop(stk);
            }
            if (node < 0 && leaf == 0) {  // park the leaf, keep descending
                leaf = node;
                node = pop(stk);
            }
            if (!__any_sync(__activemask(), leaf == 0)) break;
        }
        // intersect the parked leaf (and any leaf the traversal is sitting on)
        while (leaf < 0) {
            const uint32_t code = static_cast<uint32_t>(~leaf);
            const uint32_t first = code >> 3, count = code & 7u;
            n_tris += count;
            for (uint32_t i = first; i < first + count; ++i) {
                V3<R> v0, e1, e2;
                uint32_t obj, id;
                load_tri<R>(sc.tris, i, v0, e1, e2, obj, id);
                R det;
                const R t = ray_tri(ray, v0, e1, e2, t_min, t_best, &det);
                const bool orient = want_sign == 0 || (want_sign > 0 ? det > R(0) : det < R(0));
                if (t >= R(0) && static_cast<int>(id) != skip && orient) {
                    t_best = t;
                    hit.tri = id;
                    hit.obj = obj;
                    found = true;
                }
            }
            leaf = 0;
            if (node != kDone && node < 0) {
                leaf = node;
                node = pop(stk);
            }
        }
    }
};

template <class R, class Stack>
SST_D bool intersect_nearest_s(const DevScene<R>& sc, const RayK<R>& ray, R t_min, R t_max, int skip,
                               int cull_obj, int want_sign, R* t_hit, Hit* hit, uint64_t& n_nodes,
                               uint64_t& n_tris, Stack& stk, int root = 0) {
    Trav<R> tr;
    tr.init(t_max, root);
    while (!tr.done()) tr.round(sc, ray, t_min, skip, cull_obj, want_sign, n_nodes, n_tris, stk);
    *t_hit = tr.t_best;
    if (tr.found) *hit = tr.hit;
    return tr.found;
}

template <class R>
SST_D bool intersect_nearest(const DevScene<R>& sc, const RayK<R>& ray, R t_min, R t_max, int skip,
                             int cull_obj, int want_sign, R* t_hit, Hit* hit, uint64_t& n_nodes,
                             uint64_t& n_tris, int root = 0) {
    LocalStack<R, kStack> stk;
    return intersect_nearest_s(sc, ray, t_min, t_max, skip, cull_obj, want_sign, t_hit, hit, n_nodes, n_tris, stk,
                               root);
}

// Optical depth along [0, t_max] from a point inside a medium (order-free signed sum;
// see header). sigma(obj) = objs[obj].med[c].sigma_t.
template <class R>
SST_D R optical_depth(const DevScene<R>& sc, const RayK<R>& ray, R t_min, R t_max, int c) {
    int stack_n[kStack];
    int sp = 0;
    int cur = 0;
    R tau = R(0);
    for (;;) {
        if (cur >= 0) {
            R b[12];
            int c0, c1, o0, o1;
            load_node<R>(sc.nodes, cur, b, c0, c1, o0, o1);
            R t0, t1;
            const bool h0 = slab(ray, b[0], b[1], b[2], b[3], b[4], b[5], t_min, t_max, &t0);
            const bool h1 = slab(ray, b[6], b[7], b[8], b[9], b[10], b[11], t_min, t_max, &t1);
            if (h0 && h1) {
                stack_n[sp++] = c1;
                cur = c0;
                continue;
            }
            if (h0) { cur = c0; continue; }
            if (h1) { cur = c1; continue; }
        } else {
            const uint32_t leaf = static_cast<uint32_t>(~cur);
            const uint32_t first = leaf >> 3, count = leaf & 7u;
            for (uint32_t i = first; i < first + count; ++i) {
                V3<R> v0, e1, e2;
                uint32_t obj, id;
                load_tri<R>(sc.tris, i, v0, e1, e2, obj, id);
                R det;
                const R t = ray_tri(ray, v0, e1, e2, t_min, t_max, &det);
                if (t >= R(0)) {
                    const R sig = sc.objs[obj].med[c].sigma_t;
                    tau += det < R(0) ? sig * t : -(sig * t);
                }
            }
        }
        if (sp == 0) return tau;
        cur = stack_n[--sp];
    }
}

// ---------------------------------------------------------------- camera tiles
// Nearest entering hit of a camera ray from its pixel tile's triangle list (FP32;
// DevScene::cam_off): the same Moller-Trumbore test and acceptance as the BVH leaves.
template <class R>
SST_D bool camera_tile_hit(const DevScene<R>& sc, const RayK<R>& ray, R t_min, R* t_best, uint32_t* tri,
                           uint32_t* obj, uint64_t& n_tris) {
    const R z = dot(ray.d, sc.cam_fwd);
    const R px = (Real<R>::div_(dot(ray.d, sc.cam_right), z) / (sc.tan_half * sc.aspect) + R(1)) * R(0.5) *
                 static_cast<R>(sc.width);
    const R py = (R(1) - Real<R>::div_(dot(ray.d, sc.cam_up), z) / sc.tan_half) * R(0.5) * static_cast<R>(sc.height);
    int tx = static_cast<int>(px) / static_cast<int>(sc.cam_tile), ty = static_cast<int>(py) / static_cast<int>(sc.cam_tile);
    tx = tx < 0 ? 0 : (tx >= static_cast<int>(sc.cam_tiles_x) ? static_cast<int>(sc.cam_tiles_x) - 1 : tx);
    ty = ty < 0 ? 0 : (ty >= static_cast<int>(sc.cam_tiles_y) ? static_cast<int>(sc.cam_tiles_y) - 1 : ty);
    const uint32_t tile = static_cast<uint32_t>(ty) * sc.cam_tiles_x + static_cast<uint32_t>(tx);
    const uint32_t b = ldg_keep(sc.cam_off + tile), e = ldg_keep(sc.cam_off + tile + 1);
    n_tris += e - b;
    bool found = false;
    for (uint32_t k = b; k < e; ++k) {
        V3<R> v0, e1, e2;
        uint32_t o, id;
        load_tri<R>(sc.cam_tris, k, v0, e1, e2, o, id);
        R det;
        const R t = ray_tri(ray, v0, e1, e2, t_min, *t_best, &det);
        if (t >= R(0) && det > R(0)) {
            *t_best = t;
            *tri = id;
            *obj = o;
            found = true;
        }
    }
    return found;
}

// ---------------------------------------------------------------- light grid
// Cube-map cell of a direction (faces +x,-x,+y,-y,+z,-z; (s,t) = minor/|major|).
// Shared by the device lookup and the build kernel (cell centres).
template <class R>
SST_HD uint32_t cube_cell(R x, R y, R z, uint32_t res) {
    const R ax = x < R(0) ? -x : x, ay = y < R(0) ? -y : y, az = z < R(0) ? -z : z;
    uint32_t face;
    R s, t, m;
    if (ax >= ay && ax >= az) {
        face = x > R(0) ? 0u : 1u;
        m = ax; s = y; t = z;
    } else if (ay >= az) {
        face = y > R(0) ? 2u : 3u;
        m = ay; s = x; t = z;
    } else {
        face = z > R(0) ? 4u : 5u;
        m = az; s = x; t = y;
    }
    const R fs = (Real<R>::div_(s, m) + R(1)) * R(0.5) * static_cast<R>(res);
    const R ft = (Real<R>::div_(t, m) + R(1)) * R(0.5) * static_cast<R>(res);
    int i = static_cast<int>(fs), j = static_cast<int>(ft);
    i = i < 0 ? 0 : (i >= static_cast<int>(res) ? static_cast<int>(res) - 1 : i);
    j = j < 0 ? 0 : (j >= static_cast<int>(res) ? static_cast<int>(res) - 1 : j);
    return (face * res + static_cast<uint32_t>(j)) * res + static_cast<uint32_t>(i);
}

// Optical depth along [0, t_max] from p toward the point light using the light
// grid: the same Moller-Trumbore tests as the BVH path on a conservative
// candidate set (every triangle whose footprint seen from the light overlaps the
// cell of this direction), so the hit set is identical -- without pointer chasing.
// own: the convex object the ray starts in (-1: none / unknown).
template <class R>
SST_D R optical_depth_grid(const DevScene<R>& sc, const RayK<R>& ray, R t_min, R t_max, int c,
                           uint64_t& n_tris, int own = -1) {
    const uint32_t cell = cube_cell<R>(-ray.d.x, -ray.d.y, -ray.d.z, sc.grid_res);
    const uint32_t b = ldg_keep(sc.grid_off + cell);
    uint32_t e = ldg_keep(sc.grid_off + cell + 1);
    if (!Real<R>::kIsDouble && sc.grid_split && own >= 0) {
        const uint32_t sp = ldg_keep(sc.grid_split + cell);
        if (static_cast<int>(sp >> 24) == own) e = b + (sp & 0xffffffu);  // skip own back faces
    }
    n_tris += e - b;
    R tau = R(0);
    const bool direct = !Real<R>::kIsDouble && sc.grid_tris;  // cell's triangles stored contiguously
    for (uint32_t k = b; k < e; ++k) {
        V3<R> v0, e1, e2;
        R sig;
        if constexpr (!Real<R>::kIsDouble) {
            if (direct) {  // the copy carries sigma_t per channel in its .w words (k_grid_sigma)
                const TriF* tr = static_cast<const TriF*>(sc.grid_tris) + k;
                const float4 p = ldg_keep(&tr->v0o), q = ldg_keep(&tr->e1i), r = ldg_keep(&tr->e2);
                v0 = mk(p.x, p.y, p.z);
                e1 = mk(q.x, q.y, q.z);
                e2 = mk(r.x, r.y, r.z);
                sig = c == 0 ? p.w : (c == 1 ? q.w : r.w);
            }
        }
        if (!direct) {
            uint32_t obj, id;
            load_tri<R>(sc.tris, ldg_keep(sc.grid_tri + k), v0, e1, e2, obj, id);
            sig = sc.objs[obj].med[c].sigma_t;
        }
        R det;
        const R t = ray_tri(ray, v0, e1, e2, t_min, t_max, &det);
        if (t >= R(0)) tau += det < R(0) ? sig * t : -(sig * t);
    }
    return tau;
}

}  // namespace sstg
