// kernels_impl.cuh -- kernel bodies instantiated once per precision.
// Included by kernels_f32.cu (SST_REAL=float, SST_NS=f32) and kernels_f64.cu
// (SST_REAL=double, SST_NS=f64, compiled with -fmad=false).
#pragma once

#include "dataset.cuh"
#include "integrator.cuh"
#include "wavefront.cuh"
#include "verify.cuh"
#include "launch.h"

namespace sstg {
namespace SST_NS {

using R = SST_REAL;

// ---------------------------------------------------------------------------
// Batch of independent sphere steps (the parity unit; C ABI
// sst_gpu_sphere_step_batch). One thread per step.
__global__ void __launch_bounds__(128) k_step_batch(StepBatchArgs a) {
    DecodeCount dc;
    bool err = false;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < a.n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const double phi = a.phi[i];
        MediumK<R> m;
        m.sigma_t = static_cast<R>(a.sigma_t[i]);
        m.g = static_cast<R>(a.g[i]);
        m.phi = static_cast<R>(phi);
        m.phi_is_one = phi >= 1.0;
        m.phi_is_zero = phi <= 0.0;
        m.one_minus_phi = static_cast<R>(1.0 - phi);
        m.log_phi = (phi > 0.0 && phi < 1.0) ? static_cast<R>(log(phi)) : R(0);
        const V3<R> w = mk<R>(a.w_in[3 * i], a.w_in[3 * i + 1], a.w_in[3 * i + 2]);
        const V3<R> c = mk<R>(a.center[3 * i], a.center[3 * i + 1], a.center[3 * i + 2]);
        const bool we = a.with_event ? a.with_event[i] != 0 : a.with_event_default != 0;
        Rng rng{a.rng_state[i]};
        StepOut<R> o;
        o.n = 1;
        const bool ok = sphere_step(m, w, c, static_cast<R>(a.r[i]), we, rng, o, dc);
        err |= !ok;
        a.rng_state[i] = rng.s;
        a.absorbed[i] = o.absorbed;
        a.n_events[i] = o.n;
        const bool ex = ok && !o.absorbed;
        const bool rep = ex && we;
        const V3<R> z = mk<R>(R(0), R(0), R(0));
        const V3<R> ep = ex ? o.exit_pos : z, ed = ex ? o.exit_dir : z;
        const V3<R> rp = rep ? o.rep_pos : z, rd = rep ? o.rep_dir : z;
        a.exit_pos[3 * i] = ep.x; a.exit_pos[3 * i + 1] = ep.y; a.exit_pos[3 * i + 2] = ep.z;
        a.exit_dir[3 * i] = ed.x; a.exit_dir[3 * i + 1] = ed.y; a.exit_dir[3 * i + 2] = ed.z;
        a.rep_pos[3 * i] = rp.x; a.rep_pos[3 * i + 1] = rp.y; a.rep_pos[3 * i + 2] = rp.z;
        a.rep_dir[3 * i] = rd.x; a.rep_dir[3 * i + 1] = rd.y; a.rep_dir[3 * i + 2] = rd.z;
        a.has_rep[i] = rep;
        a.lambda[i] = rep ? static_cast<double>(o.lambda) : 0.0;
    }
    const unsigned long long l = warp_sum<unsigned long long>(dc.l);
    const unsigned long long p = warp_sum<unsigned long long>(dc.p);
    const unsigned long long e = warp_sum<unsigned long long>(dc.e);
    if ((threadIdx.x & 31) == 0) {
        if (l) atomicAdd(a.counters + 0, l);
        if (p) atomicAdd(a.counters + 1, p);
        if (e) atomicAdd(a.counters + 2, e);
    }
    if (err) atomicOr(a.error, 1);
}

// ---------------------------------------------------------------------------
// Persistent path-tracing megakernel (PT or ST; render ids or explicit keys).
// Minimum resident one-warp blocks per SM (register cap) per integrator; tuning knobs.
#ifndef SST_ST_MIN_BLOCKS
#define SST_ST_MIN_BLOCKS 16
#endif
#ifndef SST_PT_MIN_BLOCKS
#define SST_PT_MIN_BLOCKS 24
#endif
template <bool ST, bool EXPLICIT>
__global__ void __launch_bounds__(kTraceBlock, ST ? SST_ST_MIN_BLOCKS : SST_PT_MIN_BLOCKS) k_trace(TraceArgs<R> a) {
    trace_persistent<R, ST, EXPLICIT>(a);
}

// ---------------------------------------------------------------------------
// Wavefront integrator kernels (wavefront.cuh). Persistent grid-stride kernels sized
// to the resident capacity (SM count x blocks per SM) so per-block stat flushes stay few.
#ifndef SST_WF_BLOCK
#define SST_WF_BLOCK 128
#endif
constexpr int kWfBlock = SST_WF_BLOCK;
// Minimum resident blocks per SM (register caps) of the wavefront kernels; tuning knobs.
#ifndef SST_WF_LOGIC_BLOCKS
#define SST_WF_LOGIC_BLOCKS 7
#endif
#ifndef SST_WF_TRACE_BLOCKS
#define SST_WF_TRACE_BLOCKS 1
#endif
#ifndef SST_WF_SPHERE_BLOCKS
#define SST_WF_SPHERE_BLOCKS 4
#endif
template <bool ST, bool EX>
__global__ void __launch_bounds__(kWfBlock, SST_WF_LOGIC_BLOCKS) k_wf_logic(TraceArgs<R> a) { wf_logic<R, ST, EX>(a, a.pool); }
template <bool EX>
__global__ void __launch_bounds__(kWfBlock) k_wf_gen(TraceArgs<R> a) { wf_gen<R, EX>(a, a.pool); }
__global__ void __launch_bounds__(kWfBlock, SST_WF_TRACE_BLOCKS) k_wf_trace(TraceArgs<R> a) { wf_trace<R>(a, a.pool); }
__global__ void __launch_bounds__(kWfBlock, SST_WF_SPHERE_BLOCKS) k_wf_sphere(TraceArgs<R> a) { wf_sphere<R>(a, a.pool); }
#ifndef SST_WF_SHADOW_BLOCKS
#define SST_WF_SHADOW_BLOCKS 10
#endif
__global__ void __launch_bounds__(kWfBlock, SST_WF_SHADOW_BLOCKS) k_wf_shadow(TraceArgs<R> a, int with_sphere) {
    wf_shadow<R>(a, a.pool, with_sphere != 0);
}
__global__ void __launch_bounds__(kWfBlock) k_wf_compact(TraceArgs<R> a) { wf_compact<R>(a.pool); }
__global__ void __launch_bounds__(kWfBlock) k_wf_init(TraceArgs<R> a) { wf_init<R>(a.pool); }
__global__ void k_wf_reset(TraceArgs<R> a) { wf_reset<R>(a.pool); }
template <bool EX>
__global__ void __launch_bounds__(kWfBlock) k_wf_cam_filter(TraceArgs<R> a, uint32_t n_keys, uint32_t* list,
                                                            uint32_t* hdr, uint8_t* cls_of, int pass) {
    wf_cam_filter<R, EX>(a, n_keys, list, hdr, cls_of, pass);
}

// ---------------------------------------------------------------------------
// Config 4: training-data generation (persistent, one sample per lane).
__global__ void __launch_bounds__(kTraceBlock) k_dataset(DatasetArgs a) { dataset_persistent<R>(a); }

// ---------------------------------------------------------------------------
// Film accumulation: deterministic fixed-order FP64 sums over the slab's samples.
// radiance[s * stride + k], k = pixel * 3 + channel (Image layout, image.hpp:13-29).
__global__ void k_film(const R* __restrict__ radiance, uint64_t stride, uint32_t n_samples,
                       double* __restrict__ sum, double* __restrict__ sumsq) {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < stride;
         k += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        double s = 0.0, q = 0.0;
        for (uint32_t j = 0; j < n_samples; ++j) {
            const double v = static_cast<double>(radiance[j * stride + k]);
            s += v;
            q += v * v;
        }
        sum[k] += s;
        sumsq[k] += q;
    }
}

static int g_sms = 0;
static int sm_count() {
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    }
    return g_sms;
}

cudaError_t upload_constants(const double* weights1332, const double* norms6, cudaStream_t s) {
    R w[kTotalWeights];
    R n[6];
    for (int i = 0; i < kTotalWeights; ++i) w[i] = static_cast<R>(weights1332[i]);
    for (int i = 0; i < 6; ++i) n[i] = static_cast<R>(norms6[i]);
    cudaError_t e = cudaMemcpyToSymbolAsync(c_weights, w, sizeof w, 0, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyToSymbolAsync(c_norm, n, sizeof n, 0, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
#ifdef SST_DECODER_PAIRS
    float2 wp[kTotalWeights / 2];
    auto pack = [&](auto shape) {
        using S = decltype(shape);
        auto layer = [&](int rows, int cols, int off_w, int off_b, int p_w, int p_b) {
            for (int rp = 0; rp < rows / 2; ++rp) {
                for (int c = 0; c < cols; ++c)
                    wp[p_w + rp * cols + c] = make_float2(static_cast<float>(w[off_w + 2 * rp * cols + c]),
                                                          static_cast<float>(w[off_w + (2 * rp + 1) * cols + c]));
                wp[p_b + rp] = make_float2(static_cast<float>(w[off_b + 2 * rp]), static_cast<float>(w[off_b + 2 * rp + 1]));
            }
        };
        layer(S::W, S::IN, S::OFF_W0, S::OFF_B0, S::P_W0, S::P_B0);
        layer(S::W, S::W, S::OFF_W1, S::OFF_B1, S::P_W1, S::P_B1);
        layer(S::OUT, S::W, S::OFF_W2, S::OFF_B2, S::P_W2, S::P_B2);
    };
    pack(LengthShape{});
    pack(PathShape{});
    pack(EventShape{});
    e = cudaMemcpyToSymbolAsync(c_wpair, wp, sizeof wp, 0, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
#endif
    return cudaStreamSynchronize(s);  // the host staging arrays live on this stack
}

cudaError_t launch_step_batch(const StepBatchArgs& a, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    const int block = 128;
    const uint64_t need = (a.n + block - 1) / block;
    const int grid = static_cast<int>(need < 1u << 20 ? need : 1u << 20);
    k_step_batch<<<grid, block, 0, s>>>(a);
    return cudaGetLastError();
}

template <bool ST, bool EX>
static cudaError_t launch_trace_t(const TraceArgs<R>& a, cudaStream_t s) {
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_trace<ST, EX>, kTraceBlock, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    uint64_t grid = static_cast<uint64_t>(sm_count()) * blocks_per_sm;
    const uint64_t warps_needed = (a.n_paths + 31) / 32;
    const uint64_t max_grid = (warps_needed * 32 + kTraceBlock - 1) / kTraceBlock;
    if (grid > max_grid) grid = max_grid;
    if (grid < 1) grid = 1;
    k_trace<ST, EX><<<static_cast<unsigned>(grid), kTraceBlock, 0, s>>>(a);
    return cudaGetLastError();
}

template <class K>
static unsigned wf_grid(K kernel, uint32_t items, size_t smem = 0) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kWfBlock, smem);
    if (per_sm < 1) per_sm = 1;
    uint64_t g = static_cast<uint64_t>(sm_count()) * per_sm;
    const uint64_t need = (static_cast<uint64_t>(items) + kWfBlock - 1) / kWfBlock;
    if (g > need) g = need;
    return static_cast<unsigned>(g < 1 ? 1 : g);
}

cudaError_t launch_wf_cam_filter(const TraceArgs<R>& a, bool explicit_keys, uint32_t n_keys, uint32_t* list,
                                 uint32_t* count, cudaStream_t s) {
    if (n_keys == 0) return cudaSuccess;
    uint8_t* cls_of = reinterpret_cast<uint8_t*>(list + n_keys);  // per-key class, after the list
    for (int pass = 0; pass < 2; ++pass) {  // classify + count, then scatter
        if (explicit_keys)
            k_wf_cam_filter<true><<<wf_grid(k_wf_cam_filter<true>, n_keys), kWfBlock, 0, s>>>(a, n_keys, list, count,
                                                                                              cls_of, pass);
        else
            k_wf_cam_filter<false><<<wf_grid(k_wf_cam_filter<false>, n_keys), kWfBlock, 0, s>>>(a, n_keys, list, count,
                                                                                                cls_of, pass);
    }
    return cudaGetLastError();
}

cudaError_t launch_wf_init(const TraceArgs<R>& a, cudaStream_t s) {
    k_wf_init<<<wf_grid(k_wf_init, a.pool.cap), kWfBlock, 0, s>>>(a);
    return cudaGetLastError();
}

// One wavefront iteration (a.pool.q_in/q_out set by the caller; queue counters cleared first).
// side != null (and no per-kernel timing): after the logic pass the iteration forks --
// generation + trace on s, sphere steps + shadow rays on `side` (they touch disjoint
// slots, records and counters; see wavefront.cuh) -- and joins before the next one.
// live_hint: an upper bound on the live slots (the pool size while it is full; during
// the drain the last live count the host read): grids shrink with the drain, so the
// late iterations do not pay for scheduling thousands of idle blocks.
cudaError_t launch_wf_iteration(const TraceArgs<R>& a, bool st, bool explicit_keys, cudaStream_t s,
                                cudaEvent_t* ev, cudaStream_t side, cudaEvent_t fork, cudaEvent_t join,
                                uint32_t live_hint) {
    static unsigned g_logic[2][2] = {}, g_gen[2] = {}, g_trace = 0, g_sphere = 0, g_shadow = 0;
    static uint32_t cap_seen = 0, depth_seen = 0;
    const size_t trace_smem = wf_trace_smem<R>(a.sc.bvh_depth, kWfBlock);
    if (cap_seen != a.pool.cap || depth_seen != a.sc.bvh_depth) {  // grids depend on pool size and BVH depth
        cap_seen = a.pool.cap;
        depth_seen = a.sc.bvh_depth;
        cudaFuncSetAttribute(k_wf_trace, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(trace_smem));
        g_logic[0][0] = wf_grid(k_wf_logic<false, false>, a.pool.cap);
        g_logic[0][1] = wf_grid(k_wf_logic<false, true>, a.pool.cap);
        g_logic[1][0] = wf_grid(k_wf_logic<true, false>, a.pool.cap);
        g_logic[1][1] = wf_grid(k_wf_logic<true, true>, a.pool.cap);
        g_gen[0] = wf_grid(k_wf_gen<false>, a.pool.cap);
        g_gen[1] = wf_grid(k_wf_gen<true>, a.pool.cap);
        g_trace = wf_grid(k_wf_trace, a.pool.cap, trace_smem);
        g_sphere = wf_grid(k_wf_sphere, a.pool.cap);
        g_shadow = wf_grid(k_wf_shadow, a.pool.cap);
    }
    // ev (optional, 7 events): brackets reset | logic | gen | trace | sphere | shadow
    auto mark = [&](int k) {
        if (ev) cudaEventRecord(ev[k], s);
    };
    mark(0);
    k_wf_reset<<<1, 32, 0, s>>>(a);
    mark(1);
    const unsigned need = static_cast<unsigned>((static_cast<uint64_t>(live_hint) + kWfBlock - 1) / kWfBlock);
    auto fit = [need](unsigned g) { return need < g ? (need > 0 ? need : 1u) : g; };
    const bool draining = live_hint < a.pool.cap;  // supply exhausted: nothing to generate
    const unsigned gl = fit(g_logic[st][explicit_keys]);
    const unsigned gs = fit(g_sphere), gh = fit(g_shadow), gt = fit(g_trace);
    const unsigned gg0 = draining ? 1u : g_gen[0], gg1 = draining ? 1u : g_gen[1];
    if (st) {
        if (explicit_keys) k_wf_logic<true, true><<<gl, kWfBlock, 0, s>>>(a);
        else k_wf_logic<true, false><<<gl, kWfBlock, 0, s>>>(a);
    } else {
        if (explicit_keys) k_wf_logic<false, true><<<gl, kWfBlock, 0, s>>>(a);
        else k_wf_logic<false, false><<<gl, kWfBlock, 0, s>>>(a);
    }
    mark(2);
    const bool concurrent = side && !ev && (st || a.nee);
    cudaStream_t s2 = s;
    if (concurrent) {
        cudaEventRecord(fork, s);
        cudaStreamWaitEvent(side, fork, 0);
        s2 = side;
    }
    if (concurrent) {  // sphere + shadow first on the side stream
        if (st) k_wf_sphere<<<gs, kWfBlock, 0, s2>>>(a);
        if (a.nee) k_wf_shadow<<<gh, kWfBlock, 0, s2>>>(a, 1);
    }
    if (explicit_keys) k_wf_gen<true><<<gg1, kWfBlock, 0, s>>>(a);
    else k_wf_gen<false><<<gg0, kWfBlock, 0, s>>>(a);
    mark(3);
    k_wf_trace<<<gt, kWfBlock, trace_smem, s>>>(a);
    mark(4);
    if (concurrent && a.nee) k_wf_shadow<<<gh, kWfBlock, 0, s>>>(a, 0);  // shares the logic records
    if (concurrent) {
        cudaEventRecord(join, side);
        cudaStreamWaitEvent(s, join, 0);
        return cudaGetLastError();
    }
    if (st) k_wf_sphere<<<gs, kWfBlock, 0, s>>>(a);
    mark(5);
    if (a.nee) k_wf_shadow<<<gh, kWfBlock, 0, s>>>(a, 1);
    mark(6);
    return cudaGetLastError();
}

// Hand-off: compact the live slots and finish them in the megakernel.
cudaError_t launch_wf_finish(const TraceArgs<R>& a, bool st, bool explicit_keys, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(a.pool.counts + kQResume, 0, sizeof(uint32_t), s);
    if (e != cudaSuccess) return e;
    k_wf_compact<<<wf_grid(k_wf_compact, a.pool.cap), kWfBlock, 0, s>>>(a);
    e = cudaMemsetAsync(a.pool.resume_work, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    TraceArgs<R> r = a;
    r.resume = 1;
    r.work = a.pool.resume_work;
    r.n_paths = a.pool.cap;  // upper bound on live slots: sizes the grid
    return launch_trace(r, st, explicit_keys, s);
}

cudaError_t launch_trace(const TraceArgs<R>& a, bool st, bool explicit_keys, cudaStream_t s) {
    if (a.n_paths == 0) return cudaSuccess;
    if (st) return explicit_keys ? launch_trace_t<true, true>(a, s) : launch_trace_t<true, false>(a, s);
    return explicit_keys ? launch_trace_t<false, true>(a, s) : launch_trace_t<false, false>(a, s);
}

cudaError_t launch_dataset(const DatasetArgs& a, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    static int blocks_per_sm = 0;
    if (!blocks_per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_dataset, kTraceBlock, 0);
        if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    uint64_t grid = static_cast<uint64_t>(sm_count()) * blocks_per_sm;
    const uint64_t max_grid = (a.n + kTraceBlock - 1) / kTraceBlock;
    if (grid > max_grid) grid = max_grid;
    k_dataset<<<static_cast<unsigned>(grid), kTraceBlock, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_film(const R* radiance, uint64_t stride, uint32_t n_samples, double* sum,
                        double* sumsq, cudaStream_t s) {
    const int block = 256;
    uint64_t grid = (stride + block - 1) / block;
    if (grid > 65535u * 16u) grid = 65535u * 16u;
    k_film<<<static_cast<unsigned>(grid), block, 0, s>>>(radiance, stride, n_samples, sum, sumsq);
    return cudaGetLastError();
}

// Verification kernels (verify.cuh): the culling rules of this precision build against
// exact FP64 geometry, and the NEE estimator identity.
__global__ void __launch_bounds__(128) k_verify_cull(CullCheckArgs<R> a) { verify_cull<R>(a); }
__global__ void __launch_bounds__(128) k_nee_identity(NeeIdentityArgs a) { nee_identity<R>(a); }

cudaError_t launch_verify_cull(const CullCheckArgs<R>& a, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    k_verify_cull<<<static_cast<unsigned>((a.n + 127) / 128), 128, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_nee_identity(const NeeIdentityArgs& a, cudaStream_t s) {
    if (a.walks == 0) return cudaSuccess;
    k_nee_identity<<<static_cast<unsigned>((a.walks + 127) / 128), 128, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace SST_NS
}  // namespace sstg
