// rng.cuh -- device port of the reference's counter-based RandomStream
// (rng.hpp:15-50). Bit-exact on the 64-bit draws: state += 0x9E3779B97F4A7C15,
// draw = splitmix64 finalizer(state). The state after construction is one u64,
// so a path's stream is (key -> state) plus the running state in a register.
//
// Why not Philox: the reference's stream is splitmix64; GPU/CPU draw-for-draw
// identity (the parity contract) requires the same generator.
#pragma once

#include "common.cuh"

namespace sstg {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

SST_HD uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// RandomStream(seed, s1, s2, s3) constructor (rng.hpp:17-23).
SST_HD uint64_t rng_key(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t s3) {
    uint64_t s = mix64(seed);
    s = mix64(s ^ (s1 + 0x9E3779B97F4A7C15ULL));
    s = mix64(s ^ (s2 + 0xBF58476D1CE4E5B9ULL));
    s = mix64(s ^ (s3 + 0x94D049BB133111EBULL));
    return s;
}

struct Rng {
    uint64_t s;
    SST_D uint64_t next() {
        s += kGolden;
        return mix64(s);
    }
    // uniform() (rng.hpp:31): [0,1).
    template <class R>
    SST_D R uniform() { return Real<R>::uniform(next()); }
    // normal() (rng.hpp:36-40): Box-Muller cosine branch, u1 drawn first.
    template <class R>
    SST_D R normal();
};

template <>
SST_D double Rng::normal<double>() {
    const double u1 = 1.0 - uniform<double>();
    const double u2 = uniform<double>();
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

template <>
SST_D float Rng::normal<float>() {
    const float u1 = 1.0f - uniform<float>();  // exact: 24-bit grid, (0, 1]
    const float u2 = uniform<float>();
    // cos(2 pi u) = -cos(2 pi u - pi): keeps the MUFU argument in [-pi, pi).
    const float c = -__cosf(fmaf(6.28318530717958647692f, u2, -3.14159265358979323846f));
    return sqrtf(-2.0f * __logf(u1)) * c;
}

// n consecutive normal() draws (one out-of-line copy of Box-Muller for every
// decoder instead of 22 inlined copies: the render kernel is I-cache bound).
template <class R>
__device__ __noinline__ uint64_t draw_normals(uint64_t s, R* out, int n) {
    Rng r{s};
#pragma unroll 1
    for (int i = 0; i < n; ++i) out[i] = r.normal<R>();
    return r.s;
}

}  // namespace sstg
