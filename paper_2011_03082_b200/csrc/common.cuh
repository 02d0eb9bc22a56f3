// common.cuh -- precision traits and small vector math for the sm_100a kernels.
//
// Every kernel is instantiated twice:
//   float  : the production path (fast MUFU transcendentals where the parity
//            tolerance allows, see Real<float> below);
//   double : the parity mode, compiled in its own translation unit with
//            -fmad=false so the arithmetic matches the FP64 reference
//            (vec3.hpp / optics.cpp / scatter.cpp operation order) except for the
//            last-ulp differences of CUDA's libm vs glibc.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#define SST_HD __host__ __device__ __forceinline__
#define SST_D __device__ __forceinline__

namespace sstg {

// Scene gathers (SDF / skip grids, BVH nodes, triangles, light grid: ~16 MB, read at
// random by every kernel) carry an L2 evict_last priority, so the pool's multi-GB
// SoA streams do not evict them between kernels (SST_L2_KEEP=0: plain __ldg). No
// persisting set-aside is configured: measured on C5, a 16 MB set-aside changed
// nothing, 32 MB made the logic pass 25% slower and 64 MB 2.2x slower (the pool
// streams lose that L2 capacity), while the hint alone took logic 83 -> 78 ms.
#ifndef SST_L2_KEEP
#define SST_L2_KEEP 1
#endif
SST_D uint64_t l2_keep_policy() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
SST_D float ldg_keep(const float* a) {
    if (!SST_L2_KEEP) return __ldg(a);
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(l2_keep_policy()));
    return v;
}
SST_D uint32_t ldg_keep(const uint32_t* a) {
    if (!SST_L2_KEEP) return __ldg(a);
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(l2_keep_policy()));
    return v;
}
SST_D uint8_t ldg_keep(const uint8_t* a) {
    if (!SST_L2_KEEP) return __ldg(a);
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u8 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(l2_keep_policy()));
    return static_cast<uint8_t>(v);
}
SST_D float4 ldg_keep(const float4* a) {
    if (!SST_L2_KEEP) return __ldg(a);
    float4 v;
    asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
        : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
        : "l"(a), "l"(l2_keep_policy()));
    return v;
}
SST_D int4 ldg_keep(const int4* a) {
    if (!SST_L2_KEEP) return __ldg(a);
    int4 v;
    asm("ld.global.nc.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(a), "l"(l2_keep_policy()));
    return v;
}

template <class R>
struct Real;

template <>
struct Real<float> {
    static constexpr bool kIsDouble = false;
    // Free-flight epsilon for rays leaving a surface (FP32 self-intersection guard).
    static constexpr float kSurfaceEps = 2e-6f;
    static constexpr float kInf = 3e38f;
    // MUFU square root (sqrt.approx, ~1 ulp): FP32 statistical parity, FP64 stays IEEE
    SST_D static float sqrt_(float x) {
        float r;
        asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
        return r;
    }
    SST_D static float exp_(float x) { return __expf(x); }
    SST_D static float log_(float x) { return __logf(x); }
    SST_D static float log1p_(float x) { return log1pf(x); }
    SST_D static float expm1_(float x) { return expm1f(x); }
    SST_D static float cos_(float x) { return __cosf(x); }
    SST_D static void sincos_(float x, float* s, float* c) { __sincosf(x, s, c); }
    SST_D static float round_(float x) { return roundf(x); }
    SST_D static float fmax_(float a, float b) { return fmaxf(a, b); }
    SST_D static float fmin_(float a, float b) { return fminf(a, b); }
    SST_D static float fabs_(float a) { return fabsf(a); }
    SST_D static float rcp_(float a) { return __frcp_rn(a); }
    SST_D static float div_(float a, float b) { return __fdividef(a, b); }
    // softplus(x) = max(x,0) + log1p(exp(-|x|)) (mlp.cpp:60-62); 1 + e is exact to
    // 2^-24 absolute, so the MUFU log is within ~1e-7 absolute of log1p.
    SST_D static float softplus(float x) { return fmaxf(x, 0.0f) + __logf(1.0f + __expf(-fabsf(x))); }
    // Uniform in [0,1) from a 64-bit draw: top 24 bits (rng.hpp:31 keeps 53).
    SST_D static float uniform(uint64_t bits) {
        return static_cast<float>(static_cast<uint32_t>(bits >> 40)) * 0x1.0p-24f;
    }
    SST_D static bool isfinite_(float x) { return isfinite(x); }
};

template <>
struct Real<double> {
    static constexpr bool kIsDouble = true;
    static constexpr double kSurfaceEps = 0.0;
    static constexpr double kInf = 1e300;
    SST_D static double sqrt_(double x) { return sqrt(x); }
    SST_D static double exp_(double x) { return exp(x); }
    SST_D static double log_(double x) { return log(x); }
    SST_D static double log1p_(double x) { return log1p(x); }
    SST_D static double expm1_(double x) { return expm1(x); }
    SST_D static double cos_(double x) { return cos(x); }
    SST_D static void sincos_(double x, double* s, double* c) { *s = sin(x); *c = cos(x); }
    SST_D static double round_(double x) { return round(x); }
    SST_D static double fmax_(double a, double b) { return fmax(a, b); }
    SST_D static double fmin_(double a, double b) { return fmin(a, b); }
    SST_D static double fabs_(double a) { return fabs(a); }
    SST_D static double rcp_(double a) { return 1.0 / a; }
    SST_D static double div_(double a, double b) { return a / b; }
    SST_D static double softplus(double x) { return fmax(x, 0.0) + log1p(exp(-fabs(x))); }
    SST_D static double uniform(uint64_t bits) {
        return static_cast<double>(bits >> 11) * 0x1.0p-53;
    }
    SST_D static bool isfinite_(double x) { return isfinite(x); }
};

template <class R>
struct V3 {
    R x, y, z;
};

template <class R>
SST_HD V3<R> mk(R x, R y, R z) { return V3<R>{x, y, z}; }
template <class R>
SST_HD V3<R> operator+(V3<R> a, V3<R> b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
template <class R>
SST_HD V3<R> operator-(V3<R> a, V3<R> b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
template <class R>
SST_HD V3<R> operator*(V3<R> a, R s) { return {a.x * s, a.y * s, a.z * s}; }
template <class R>
SST_HD V3<R> operator/(V3<R> a, R s) { return {a.x / s, a.y / s, a.z / s}; }
template <class R>
SST_HD R dot(V3<R> a, V3<R> b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
template <class R>
SST_HD V3<R> cross(V3<R> a, V3<R> b) {
    return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <class R>
SST_D V3<R> normalize(V3<R> v) {
    const R len = Real<R>::sqrt_(dot(v, v));
    if (Real<R>::kIsDouble) return {v.x / len, v.y / len, v.z / len};
    const R inv = Real<R>::div_(R(1), len);
    return {v.x * inv, v.y * inv, v.z * inv};
}
template <class R>
SST_HD R comp(V3<R> v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }

// orthonormal_basis (vec3.hpp:53-59): (b1, b2, n) right-handed.
template <class R>
SST_D void onb(V3<R> n, V3<R>* b1, V3<R>* b2) {
    const R sign = copysign(R(1), n.z);
    const R a = Real<R>::div_(R(-1), sign + n.z);  // |sign + n.z| >= 1
    const R b = n.x * n.y * a;
    *b1 = mk<R>(R(1) + sign * n.x * n.x * a, sign * b, -sign * n.x);
    *b2 = mk<R>(b, sign + n.y * n.y * a, -n.y);
}

// Column-major 3x3 (vec3.hpp:62-83).
template <class R>
struct M3 {
    V3<R> c0, c1, c2;
};
template <class R>
SST_D V3<R> operator*(const M3<R>& m, V3<R> v) { return m.c0 * v.x + m.c1 * v.y + m.c2 * v.z; }

constexpr double kTwoPiD = 6.28318530717958647692;
constexpr double kInv4PiD = 0.07957747154594766788;

}  // namespace sstg
