// dataset.cuh -- config 4: CVAE training-data generation on the GPU (the reference's
// generate_dataset, dataset.cpp:40-92, over walk_sphere / parameterize_exit /
// sample_representative, sphere_walk.cpp:22-102).
//
// One lane = one sample (persistent warps, warp-aggregated work fetching, like the
// render kernel). The reference stores the full event list of a walk (up to 1e6
// events) to pick the representative event k AFTER the walk (k depends on N and a
// draw taken after the walk). Here the walk runs twice from the same RNG state:
// pass 1 counts N and finds the exit, pass 2 replays it up to event k -- identical
// arithmetic, so the replayed event is the stored one, without any event storage.
// Draw order follows the reference as compiled (g++ x86-64): hg_sample's two
// uniform() arguments are evaluated right to left, i.e. u2 first (pinned by the
// golden vectors, see oracle/sst_oracle.c SO_HG_ARG_ORDER_RTL).
#pragma once

#include "common.cuh"
#include "integrator.cuh"
#include "rng.cuh"
#include "types.cuh"

namespace sstg {


template <class R>
struct WalkLane {
    Rng rng;
    uint64_t s_walk;      // RNG state at walk start (for the replay)
    uint64_t idx;
    V3<R> pos, inc;       // current position / incoming direction
    V3<R> exit_pos, exit_dir;
    R sigma, g;
    double sigma_d, g_d, phi_d;
    uint32_t n, k, count;
    uint8_t pass;         // 1 = counting walk, 2 = replay to event k
    bool vacuum;
};

constexpr uint32_t kMaxWalkEvents = 1000000u;  // sphere_walk.hpp:35

// sphere_exit_t (sphere_walk.cpp:14-18), radius 1.
template <class R>
SST_D R sphere_exit_t(V3<R> pos, V3<R> dir) {
    const R b = dot(pos, dir);
    const R c = dot(pos, pos) - R(1);
    return -b + Real<R>::sqrt_(Real<R>::fmax_(R(0), b * b - c));
}

template <class R>
SST_D void walk_begin(WalkLane<R>& w) {
    w.rng.s = w.s_walk;
    w.pos = mk<R>(R(0), R(0), R(0));
    w.inc = mk<R>(R(0), R(0), R(1));
    w.count = 1;  // the forced event at the centre
}

template <class R>
SST_D void write_sample(const DatasetArgs& a, const WalkLane<R>& w) {
    // parameterize_exit (sphere_walk.cpp:52-73): w_in = (0,0,1), radius 1
    const V3<R> w_in = mk<R>(R(0), R(0), R(1));
    const V3<R> x_hat = w.exit_pos;
    const R ct = dot(w_in, x_hat);
    V3<R> e_b, b2;
    if (Real<R>::fabs_(ct) > R(1) - R(1e-9)) onb(x_hat, &e_b, &b2);
    else e_b = normalize(cross(w_in, x_hat));
    const V3<R> e_t = cross(e_b, x_hat);
    // rotate the representative by -psi_exit (dataset.cpp:71-74)
    const double psi = atan2(static_cast<double>(w.exit_pos.y), static_cast<double>(w.exit_pos.x));
    const R c = static_cast<R>(cos(-psi)), s = static_cast<R>(sin(-psi));
    const M3<R> undo{mk<R>(c, s, R(0)), mk<R>(-s, c, R(0)), mk<R>(R(0), R(0), R(1))};
    const V3<R> xs = undo * w.pos, ws = undo * w.inc;
    TrainingSampleDev o;
    o.sigma_t = static_cast<float>(w.sigma_d);
    o.g = static_cast<float>(w.g_d);
    o.phi = static_cast<float>(w.phi_d);
    o.n_events = w.n;
    o.cos_theta = static_cast<float>(ct);
    o.alpha = static_cast<float>(dot(w.exit_dir, e_b));
    o.beta = static_cast<float>(dot(w.exit_dir, e_t));
    o.rep_position[0] = static_cast<float>(xs.x);
    o.rep_position[1] = static_cast<float>(xs.y);
    o.rep_position[2] = static_cast<float>(xs.z);
    o.rep_direction[0] = static_cast<float>(ws.x);
    o.rep_direction[1] = static_cast<float>(ws.y);
    o.rep_direction[2] = static_cast<float>(ws.z);
    a.out[w.idx - a.first] = o;
}

// sample_representative (sphere_walk.cpp:75-102): event k in [1, n] with P(k) ~ phi^k
// (uniform for phi = 1, k = 1 for phi = 0), one FP64 uniform draw.
SST_D uint32_t representative_k(double phi, uint64_t n, Rng& rng) {
    uint64_t k = 1;
    if (phi <= 0.0) {
        k = 1;
    } else if (phi >= 1.0) {
        const uint64_t t = static_cast<uint64_t>(rng.template uniform<double>() * static_cast<double>(n));
        k = 1 + (n - 1 < t ? n - 1 : t);
    } else {
        const double u = rng.template uniform<double>();
        const double phi_n = exp(static_cast<double>(n) * log(phi));
        const double target = 1.0 - u * (1.0 - phi_n);
        k = static_cast<uint64_t>(ceil(log(target) / log(phi)));
        k = k < 1 ? 1 : (k > n ? n : k);
    }
    return static_cast<uint32_t>(k);
}

template <class R>
SST_D void dataset_persistent(const DatasetArgs& a) {
    const unsigned lane = threadIdx.x & 31u;
    WalkLane<R> w;
    bool alive = false, exhausted = false;
    unsigned long long ev1 = 0, ev2 = 0, nmax = 0;
    for (;;) {
        const unsigned need = __ballot_sync(0xffffffffu, !alive && !exhausted);
        if (need) {
            const int leader = __ffs(need) - 1;
            unsigned long long base = 0;
            if (static_cast<int>(lane) == leader) base = atomicAdd(a.work, static_cast<unsigned long long>(__popc(need)));
            base = __shfl_sync(0xffffffffu, base, leader);
            if (!alive && !exhausted) {
                const uint64_t my = base + __popc(need & ((1u << lane) - 1u));
                if (my < a.n) {
                    // per-sample stream and material draws (dataset.cpp:59-63), in FP64
                    w.idx = a.first + my;
                    w.rng.s = rng_key(a.seed, 0x01, w.idx, 0);  // kDataset
                    w.sigma_d = a.s_lo + w.rng.template uniform<double>() * (a.s_hi - a.s_lo);
                    const double gg = a.g_lo + w.rng.template uniform<double>() * (a.g_hi - a.g_lo);
                    w.g_d = fmin(1.0 - 1e-6, fmax(-(1.0 - 1e-6), gg));
                    if (a.phi_kind == 0) w.phi_d = 1.0 - pow(10.0, a.phi_a + w.rng.template uniform<double>() * (a.phi_b - a.phi_a));
                    else if (a.phi_kind == 1) w.phi_d = a.phi_a;
                    else w.phi_d = a.phi_a + w.rng.template uniform<double>() * (a.phi_b - a.phi_a);
                    w.sigma = static_cast<R>(w.sigma_d);
                    w.g = static_cast<R>(w.g_d);
                    w.vacuum = w.sigma_d <= 1e-6;  // kVacuumSigmaT
                    w.s_walk = w.rng.s;
                    walk_begin(w);
                    w.pass = 1;
                    alive = true;
                } else {
                    exhausted = true;
                }
            }
        }
        if (!__any_sync(0xffffffffu, alive)) break;
        if (!alive) continue;
        if (w.pass == 2 && w.count == w.k) {  // replay reached the representative
            write_sample(a, w);
            alive = false;
            continue;
        }
        // one event of walk_sphere (sphere_walk.cpp:34-49)
        const R u2 = w.rng.template uniform<R>();
        const R u1 = w.rng.template uniform<R>();
        const V3<R> dir = hg_sample(w.g, w.inc, u1, u2);
        R step;
        if (w.vacuum) step = R(2);
        else if (Real<R>::kIsDouble) step = -Real<R>::log1p_(-w.rng.template uniform<R>()) / w.sigma;
        else step = -Real<R>::div_(Real<R>::log_(R(1) - w.rng.template uniform<R>()), w.sigma);
        const R t_exit = sphere_exit_t(w.pos, dir);
        if (w.vacuum || step >= t_exit) {
            // pass 2 never gets here (k <= N)
            w.exit_pos = w.pos + dir * t_exit;
            w.exit_dir = dir;
            w.n = w.count;
            ev1 += w.count;
            nmax = nmax > w.count ? nmax : w.count;
            w.k = representative_k(w.phi_d, w.count, w.rng);
            walk_begin(w);  // replay from the walk's first draw
            w.pass = 2;
            if (w.k == 1) {
                write_sample(a, w);
                alive = false;
            }
            continue;
        }
        w.pos = w.pos + dir * step;
        w.inc = dir;
        ++w.count;
        if (w.pass == 2) ++ev2;
        if (w.pass == 1 && w.count > kMaxWalkEvents) {  // the reference throws
            atomicOr(a.error, 1);
            alive = false;
        }
    }
    const unsigned long long s1 = warp_sum(ev1), s2 = warp_sum(ev2);
    unsigned long long m = nmax;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long v = __shfl_xor_sync(0xffffffffu, m, o);
        m = m > v ? m : v;
    }
    if (lane == 0) {
        if (s1) atomicAdd(a.stats + 0, s1);
        if (s2) atomicAdd(a.stats + 1, s2);
        atomicMax(a.stats + 2, m);
    }
}

}  // namespace sstg
