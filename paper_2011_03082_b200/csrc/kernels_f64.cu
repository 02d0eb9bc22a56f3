// kernels_f64.cu -- FP64 parity instantiation (compiled with -fmad=false so every
// product/sum rounds like the reference's x86-64 FP64 code), plus the exact SDF
// build kernel.
#include <cstdint>

#define SST_REAL double
#define SST_NS f64

__constant__ double c_weights[1332];
__constant__ double c_norm[6];

#include "kernels_impl.cuh"

namespace sstg {

namespace {

struct D3 {
    double x, y, z;
};
__device__ __forceinline__ D3 d3(double x, double y, double z) { return D3{x, y, z}; }
__device__ __forceinline__ D3 sub(D3 a, D3 b) { return d3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ D3 add(D3 a, D3 b) { return d3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ D3 mul(D3 a, double s) { return d3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ double dt(D3 a, D3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ D3 cr(D3 a, D3 b) {
    return d3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// point_triangle_distance_squared (mesh.cpp:199-233), same operation order.
__device__ double pt_tri_d2(D3 p, D3 a, D3 b, D3 c) {
    const D3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
    const double d1 = dt(ab, ap), d2 = dt(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) { const D3 q = sub(p, a); return dt(q, q); }
    const D3 bp = sub(p, b);
    const double d3v = dt(ab, bp), d4 = dt(ac, bp);
    if (d3v >= 0.0 && d4 <= d3v) { const D3 q = sub(p, b); return dt(q, q); }
    const double vc = d1 * d4 - d3v * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3v <= 0.0) {
        const double v = d1 / (d1 - d3v);
        const D3 q = sub(p, add(a, mul(ab, v)));
        return dt(q, q);
    }
    const D3 cp = sub(p, c);
    const double d5 = dt(ab, cp), d6 = dt(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) { const D3 q = sub(p, c); return dt(q, q); }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double w = d2 / (d2 - d6);
        const D3 q = sub(p, add(a, mul(ac, w)));
        return dt(q, q);
    }
    const double va = d3v * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3v) >= 0.0 && (d5 - d6) >= 0.0) {
        const double w = (d4 - d3v) / ((d4 - d3v) + (d5 - d6));
        const D3 q = sub(p, add(b, mul(sub(c, b), w)));
        return dt(q, q);
    }
    const double denom = 1.0 / (va + vb + vc);
    const double v = vb * denom, w = vc * denom;
    const D3 q = sub(p, add(add(a, mul(ab, v)), mul(ac, w)));
    return dt(q, q);
}

// ray_triangle (bvh.cpp:11-27) with t_min 1e-9, t_max 1e300 (Bvh::inside).
__device__ bool mt_hit(D3 o, D3 d, D3 a, D3 b, D3 c) {
    const D3 e1 = sub(b, a), e2 = sub(c, a);
    const D3 pvec = cr(d, e2);
    const double det = dt(e1, pvec);
    if (fabs(det) < 1e-14) return false;
    const double inv_det = 1.0 / det;
    const D3 tvec = sub(o, a);
    const double u = dt(tvec, pvec) * inv_det;
    if (u < 0.0 || u > 1.0) return false;
    const D3 qvec = cr(tvec, e1);
    const double v = dt(d, qvec) * inv_det;
    if (v < 0.0 || u + v > 1.0) return false;
    const double t = dt(e2, qvec) * inv_det;
    return !(t <= 1e-9 || t >= 1e300);
}

constexpr int kSdfTile = 128;

// One voxel per thread; triangles staged through shared memory in tiles. The min
// distance and the hit parity do not depend on traversal order, so brute force
// over all triangles reproduces the reference's BVH-pruned build bit for bit.
__global__ void __launch_bounds__(128) k_sdf_build(SdfBuildArgs a) {
    __shared__ double tile[kSdfTile * 9];
    const uint64_t nvox = static_cast<uint64_t>(a.dims[0]) * a.dims[1] * a.dims[2];
    const uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const bool active = v < nvox;
    const uint32_t x = active ? static_cast<uint32_t>(v % a.dims[0]) : 0;
    const uint32_t y = active ? static_cast<uint32_t>((v / a.dims[0]) % a.dims[1]) : 0;
    const uint32_t z = active ? static_cast<uint32_t>(v / (static_cast<uint64_t>(a.dims[0]) * a.dims[1])) : 0;
    // voxel_center (sdf.hpp:29-32)
    const D3 c = add(d3(a.origin[0], a.origin[1], a.origin[2]),
                     d3((x + 0.5) * a.voxel, (y + 0.5) * a.voxel, (z + 0.5) * a.voxel));
    const D3 dirs[3] = {d3(a.dirs[0], a.dirs[1], a.dirs[2]), d3(a.dirs[3], a.dirs[4], a.dirs[5]),
                        d3(a.dirs[6], a.dirs[7], a.dirs[8])};
    double best = 1e300, wind = 0.0;
    uint32_t hits[3] = {0, 0, 0};
    for (uint32_t base = 0; base < a.n_tris; base += kSdfTile) {
        const uint32_t n = min(static_cast<uint32_t>(kSdfTile), a.n_tris - base);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < n * 9; k += blockDim.x) tile[k] = a.tri_vertices[base * 9ull + k];
        __syncthreads();
        if (!active) continue;
        for (uint32_t t = 0; t < n; ++t) {
            const double* q = tile + 9 * t;
            const D3 A = d3(q[0], q[1], q[2]), B = d3(q[3], q[4], q[5]), C = d3(q[6], q[7], q[8]);
            best = fmin(best, pt_tri_d2(c, A, B, C));
            if (a.watertight) {
                for (int k = 0; k < 3; ++k) hits[k] += mt_hit(c, dirs[k], A, B, C);
            } else {  // winding_number (bvh.cpp:219-232)
                const D3 pa = sub(A, c), pb = sub(B, c), pc = sub(C, c);
                const double la = sqrt(dt(pa, pa)), lb = sqrt(dt(pb, pb)), lc = sqrt(dt(pc, pc));
                const double num = dt(pa, cr(pb, pc));
                const double den = la * lb * lc + dt(pa, pb) * lc + dt(pb, pc) * la + dt(pc, pa) * lb;
                wind += 2.0 * atan2(num, den);
            }
        }
    }
    if (!active) return;
    bool inside;
    if (a.watertight) {
        const int votes = (hits[0] & 1) + (hits[1] & 1) + (hits[2] & 1);
        inside = votes >= 2;
    } else {
        inside = wind / (4.0 * 3.14159265358979323846) > 0.5;
    }
    const double d = sqrt(best);
    const double cons = fmax(0.0, d - a.half_diagonal);
    a.values[v] = static_cast<float>(inside ? -cons : cons);
}

__global__ void __launch_bounds__(128) k_skip_build(SkipBuildArgs a) {
    __shared__ double tile[kSdfTile * 9];
    const uint64_t nvox = static_cast<uint64_t>(a.dims[0]) * a.dims[1] * a.dims[2];
    const uint64_t v = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    const bool active = v < nvox;
    const uint32_t x = active ? static_cast<uint32_t>(v % a.dims[0]) : 0;
    const uint32_t y = active ? static_cast<uint32_t>((v / a.dims[0]) % a.dims[1]) : 0;
    const uint32_t z = active ? static_cast<uint32_t>(v / (static_cast<uint64_t>(a.dims[0]) * a.dims[1])) : 0;
    const D3 c = add(d3(a.origin[0], a.origin[1], a.origin[2]),
                     d3((x + 0.5) * a.voxel, (y + 0.5) * a.voxel, (z + 0.5) * a.voxel));
    double best = 1e300;
    for (uint32_t base = 0; base < a.n_tris; base += kSdfTile) {
        const uint32_t n = min(static_cast<uint32_t>(kSdfTile), a.n_tris - base);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < n * 9; k += blockDim.x) tile[k] = a.tri_vertices[base * 9ull + k];
        __syncthreads();
        if (!active) continue;
        for (uint32_t t = 0; t < n; ++t) {
            const double* q = tile + 9 * t;
            best = fmin(best, pt_tri_d2(c, d3(q[0], q[1], q[2]), d3(q[3], q[4], q[5]), d3(q[6], q[7], q[8])));
        }
    }
    if (!active) return;
    // 0.999: margin against the float rounding of positions at lookup time
    const double cons = fmax(0.0, 0.999 * sqrt(best) - a.half_diagonal);
    a.values[v] = static_cast<uint8_t>(fmin(255.0, floor(cons / a.unit)));
}

constexpr int kGridTile = 128;

// Exact test of a (projected) triangle against a cube-map cell. Directions are
// projected gnomonically onto the cell's face plane (great circles -> straight
// lines), so the spherical triangle becomes a 2D triangle and the cell a square:
// separating-axis test with padding. Returns -1 when a vertex is not strictly in
// front of the face (caller keeps the cone result).
__device__ int tri_cell_overlap(const double* q, int face, double s0, double s1, double t0, double t1,
                                double pad) {
    const int major = face >> 1;
    const double sign = (face & 1) ? -1.0 : 1.0;
    const int ia = major == 0 ? 1 : 0, ib = major == 2 ? 1 : 2;
    double ps[3], pt[3];
    for (int c = 0; c < 3; ++c) {
        const double* d = q + 6 + 3 * c;
        const double m = sign * d[major];
        if (!(m > 1e-3)) return -1;
        ps[c] = d[ia] / m;
        pt[c] = d[ib] / m;
    }
    s0 -= pad; s1 += pad; t0 -= pad; t1 += pad;
    if (fmax(ps[0], fmax(ps[1], ps[2])) < s0 || fmin(ps[0], fmin(ps[1], ps[2])) > s1) return 0;
    if (fmax(pt[0], fmax(pt[1], pt[2])) < t0 || fmin(pt[0], fmin(pt[1], pt[2])) > t1) return 0;
    for (int e = 0; e < 3; ++e) {
        const int i = e, j = (e + 1) % 3, k = (e + 2) % 3;
        const double nx = -(pt[j] - pt[i]), ny = ps[j] - ps[i];
        const double side = nx * (ps[k] - ps[i]) + ny * (pt[k] - pt[i]);
        if (fabs(side) < 1e-14) continue;  // degenerate (edge-on) projection: keep
        // the square is separated if all four corners are strictly on the far side
        bool sep = true;
        for (int cc = 0; cc < 4 && sep; ++cc) {
            const double cs = (cc & 1) ? s1 : s0, ct = (cc & 2) ? t1 : t0;
            const double v = nx * (cs - ps[i]) + ny * (ct - pt[i]);
            sep = side > 0 ? v < 0 : v > 0;
        }
        if (sep) return 0;
    }
    return 1;
}

// Light grid build: one cube-map cell per thread. A triangle is listed in a cell
// when the cell's bounding cone overlaps the triangle's cone AND (where the
// projection is valid) the exact 2D test on the cell's face passes.
__global__ void __launch_bounds__(128) k_light_grid(LightGridArgs a) {
    __shared__ double tile[kGridTile * kCapStride];
    const uint32_t ncell = 6u * a.res * a.res;
    const uint32_t cell = blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = cell < ncell;
    double cx = 0, cy = 0, cz = 1, cr = 1, sr = 0, r = 0, s0 = 0, s1 = 0, t0 = 0, t1 = 0;
    int face = 0;
    if (active) {
        face = static_cast<int>(cell / (a.res * a.res));
        const uint32_t rem = cell % (a.res * a.res);
        const uint32_t j = rem / a.res, i = rem % a.res;
        auto dir = [&](double s, double t, double* o) {
            double v[3];
            switch (face) {
                case 0: v[0] = 1; v[1] = s; v[2] = t; break;
                case 1: v[0] = -1; v[1] = s; v[2] = t; break;
                case 2: v[0] = s; v[1] = 1; v[2] = t; break;
                case 3: v[0] = s; v[1] = -1; v[2] = t; break;
                case 4: v[0] = s; v[1] = t; v[2] = 1; break;
                default: v[0] = s; v[1] = t; v[2] = -1; break;
            }
            const double l = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            o[0] = v[0] / l; o[1] = v[1] / l; o[2] = v[2] / l;
        };
        const double h = 1.0 / a.res;
        s0 = i * 2.0 * h - 1.0;
        s1 = s0 + 2.0 * h;
        t0 = j * 2.0 * h - 1.0;
        t1 = t0 + 2.0 * h;
        const double sc = 0.5 * (s0 + s1), tc = 0.5 * (t0 + t1);
        double c[3];
        dir(sc, tc, c);
        double mind = 1.0;
        for (int k = 0; k < 4; ++k) {
            double q[3];
            dir(sc + ((k & 1) ? h : -h), tc + ((k & 2) ? h : -h), q);
            mind = fmin(mind, c[0] * q[0] + c[1] * q[1] + c[2] * q[2]);
        }
        r = acos(fmax(-1.0, fmin(1.0, mind))) + a.eps;
        cx = c[0]; cy = c[1]; cz = c[2];
        cr = cos(r); sr = sin(r);
    }
    const double pad = 2.0 * a.eps;  // face-plane units: |d(s,t)/d angle| >= 1
    const uint32_t base_out = (a.fill && active) ? a.offsets[cell] : 0;
    uint32_t count = 0;
    for (uint32_t base = 0; base < a.n_tris; base += kGridTile) {
        const uint32_t n = min(static_cast<uint32_t>(kGridTile), a.n_tris - base);
        __syncthreads();
        for (uint32_t k = threadIdx.x; k < n * kCapStride; k += blockDim.x)
            tile[k] = a.caps[static_cast<uint64_t>(base) * kCapStride + k];
        __syncthreads();
        if (!active) continue;
        for (uint32_t t = 0; t < n; ++t) {
            const double* q = tile + kCapStride * t;
            bool hit;
            if (r + q[3] >= 3.14159265358979323846) hit = true;
            else hit = cx * q[0] + cy * q[1] + cz * q[2] >= cr * q[4] - sr * q[5];
            if (hit && q[3] < 3.0) hit = tri_cell_overlap(q, face, s0, s1, t0, t1, pad) != 0;
            if (hit) {
                if (a.fill) a.lists[base_out + count] = base + t;
                ++count;
            }
        }
    }
    if (active && !a.fill) a.counts[cell] = count;
}

__global__ void k_gather_tris(const uint32_t* __restrict__ idx, const TriF* __restrict__ tris, uint64_t n,
                              TriF* __restrict__ out) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[k] = tris[idx[k]];
}

// The light grid's FP32 triangle copies carry their object's extinction per channel in
// the three .w words (v0.w, e1.w, e2.w) instead of object / triangle ids: a shadow ray's
// hit needs sigma_t and nothing else, and reading it from the record saves the dependent
// ObjK load (geom.cuh optical_depth_grid).
__global__ void k_grid_sigma(TriF* __restrict__ t, uint64_t n, const ObjK<float>* __restrict__ objs) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const ObjK<float>& o = objs[__float_as_uint(t[k].v0o.w)];
        t[k].v0o.w = o.med[0].sigma_t;
        t[k].e1i.w = o.med[1].sigma_t;
        t[k].e2.w = o.med[2].sigma_t;
    }
}

}  // namespace

cudaError_t launch_grid_sigma(TriF* tris, uint64_t n, const ObjK<float>* objs, cudaStream_t s) {
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k_grid_sigma<<<static_cast<unsigned>(blocks), 256, 0, s>>>(tris, n, objs);
    return cudaGetLastError();
}

cudaError_t launch_gather_tris(const uint32_t* idx, const TriF* tris, uint64_t n, TriF* out, cudaStream_t s) {
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148ull * 16);
    k_gather_tris<<<static_cast<unsigned>(blocks), 256, 0, s>>>(idx, tris, n, out);
    return cudaGetLastError();
}

cudaError_t launch_skip_build(const SkipBuildArgs& a, cudaStream_t s) {
    const uint64_t nvox = static_cast<uint64_t>(a.dims[0]) * a.dims[1] * a.dims[2];
    k_skip_build<<<static_cast<unsigned>((nvox + 127) / 128), 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_light_grid(const LightGridArgs& a, cudaStream_t s) {
    const uint32_t ncell = 6u * a.res * a.res;
    k_light_grid<<<(ncell + 127) / 128, 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sdf_build(const SdfBuildArgs& a, cudaStream_t s) {
    const uint64_t nvox = static_cast<uint64_t>(a.dims[0]) * a.dims[1] * a.dims[2];
    const unsigned grid = static_cast<unsigned>((nvox + 127) / 128);
    k_sdf_build<<<grid, 128, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace sstg
