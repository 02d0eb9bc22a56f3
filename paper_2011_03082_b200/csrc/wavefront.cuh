// wavefront.cuh -- the per-path loop of integrator.cuh as a wavefront over a pool of
// path slots whose state lives in HBM/L2 as structure-of-arrays (16-byte vectors,
// coalesced 128-bit loads and stores), with one stream-compacted queue per
// expensive operation:
//
//   k_wf_logic   every live slot: resolve the last traversal, collision (delta-
//                tracking event / sphere-step request), path end (slot -> free queue),
//                next free flight; pushes the slot onto AT MOST ONE of the queues
//                below (block-aggregated atomics)
//   k_wf_gen     free queue: new paths (camera ray + RNG key) with consecutive ids,
//                straight onto the trace queue
//   k_wf_trace   trace queue: nearest-hit BVH traversal (medium entry / free flight)
//   k_wf_sphere  sphere queue: the CVAE sphere step (ST); survivors push NEE
//   k_wf_shadow  shadow queue: NEE shadow ray (light grid) + radiance update
//
// Every kernel runs its operation on full warps drawn from the whole pool, instead of
// the 5-10 lanes per warp that reach the same phase of the megakernel's loop
// (ncu: 7.3 threads/instruction, 40% of lane-iterations waiting for a sphere batch).
// The per-path operation sequence -- and therefore every RNG draw and every result --
// is exactly the megakernel's (integrator.cuh path_advance): paths are keyed, so the
// iteration structure does not matter. When the pool has drained below a threshold
// (the long-path tail) the remaining slots are handed to the register-resident
// megakernel (trace_persistent in resume mode), which finishes them without
// per-iteration launch costs.
#pragma once

#include <cooperative_groups.h>

#include "integrator.cuh"

namespace sstg {

namespace cg = cooperative_groups;

// Slot phases (meta.w bits 11-12).
enum : uint32_t { kPhEmpty = 0, kPhFlight = 1, kPhTrace = 2, kPhSphere = 3 };
// meta.w packing: obj+1 (bits 0-7), channel (8-9), r_valid (10), phase (11-12),
// cull+1 (16-23).
SST_D uint32_t pack_meta(int obj, int c, bool r_valid, uint32_t phase, int cull) {
    return static_cast<uint32_t>(obj + 1) | (static_cast<uint32_t>(c) << 8) |
           (static_cast<uint32_t>(r_valid) << 10) | (phase << 11) | (static_cast<uint32_t>(cull + 1) << 16);
}
SST_D uint32_t meta_phase(uint32_t m) { return (m >> 11) & 3u; }
// meta.w bit 13: a path fresh from the generation kernel whose position / direction
// live only in its camera-ray trace record (xl / wr were not written; L = 0).
constexpr uint32_t kMetaFresh = 1u << 13;
// NEE mailbox (types.cuh kNeeChain): meta.w bits 24-27 = number of staged NEE records
// whose contributions the slot's next logic visit adds to L (in event order); bit 14 /
// bit 15 = the path was absorbed / escaped after staging some: the next visit adds them,
// then ends it.
constexpr uint32_t kMetaEndAbsorbed = 1u << 14;
constexpr uint32_t kMetaEndEscaped = 1u << 15;
constexpr uint32_t kMetaEnded = kMetaEndAbsorbed | kMetaEndEscaped;
constexpr int kMetaPendShift = 24;
SST_D uint32_t meta_pending(uint32_t m) { return (m >> kMetaPendShift) & 0xfu; }
// Transient phases returned by load_slot for a slot whose path already ended (absorbed /
// escaped) once its staged contributions are in.
constexpr uint32_t kPhEnded = 4, kPhEndedEscaped = 5;
// Integer payloads carried in the spare lane of a record vector.
template <class R>
SST_D R int_bits(int v) {
    if constexpr (sizeof(R) == 4) return __int_as_float(v);
    else return __longlong_as_double(static_cast<long long>(v));
}
template <class R>
SST_D int bits_int(R v) {
    if constexpr (sizeof(R) == 4) return __float_as_int(v);
    else return static_cast<int>(__double_as_longlong(v));
}
SST_D int meta_obj(uint32_t m) { return static_cast<int>(m & 0xffu) - 1; }
SST_D int meta_c(uint32_t m) { return static_cast<int>((m >> 8) & 3u); }

// The slot's mailbox entries, loaded as one vector (issued with the slot state, before
// the pending count is known: most visits have some).
template <class R>
struct Mailbox {
    R v[kNeeChain];
};
template <class R>
SST_D Mailbox<R> load_mailbox(const WfPool<R>& q, uint32_t s) {
    Mailbox<R> mb;
    const R* src = q.nee_res + static_cast<size_t>(s) * kNeeChain;
    if constexpr (sizeof(R) == 4 && kNeeChain == 2) {
        const float2 t = *reinterpret_cast<const float2*>(src);
        mb.v[0] = t.x;
        mb.v[1] = t.y;
    } else if constexpr (sizeof(R) == 4 && kNeeChain == 4) {
        const float4 t = *reinterpret_cast<const float4*>(src);
        mb.v[0] = t.x;
        mb.v[1] = t.y;
        mb.v[2] = t.z;
        mb.v[3] = t.w;
    } else {
#pragma unroll
        for (uint32_t i = 0; i < kNeeChain; ++i) mb.v[i] = src[i];
    }
    return mb;
}

// A slot's position + radiance and direction + safe radius; SST_SLOT_PAIR keeps both in
// one 32-byte sector (the sphere kernel's slots are scattered: ~11% of the pool per pass).
#ifndef SST_SLOT_PAIR
#define SST_SLOT_PAIR 1
#endif
template <class R>
SST_D Q4<R>& slot_xl(const WfPool<R>& q, uint32_t s) {
    return SST_SLOT_PAIR ? q.xl[2u * s] : q.xl[s];
}
template <class R>
SST_D Q4<R>& slot_wr(const WfPool<R>& q, uint32_t s) {
    return SST_SLOT_PAIR ? q.xl[2u * s + 1u] : q.wr[s];
}

// need_tpend: the queued flight length is only stored while a traversal is queued and
// only the megakernel hand-off reads it from the slot (the logic pass takes it from the
// traversal result: a miss leaves t_hit = t_max = the flight length).
// fold: add the contributions of the slot's staged NEE records (the logic visit and the
// megakernel hand-off; never the sphere kernel, which runs while they are computed).
template <class R>
SST_D void load_slot_from(const WfPool<R>& q, uint32_t s, const uint4 m, PathLocal<R>& p, uint32_t* phase,
                          const V3<R>& sc_cam_pos, bool need_tpend, bool fold, const Mailbox<R>* mb = nullptr) {
    const Q4<R> xl = slot_xl(q, s), wr = slot_wr(q, s);
    p.x = mk<R>(xl.x, xl.y, xl.z);
    p.L = xl.w;
    p.w = mk<R>(wr.x, wr.y, wr.z);
    p.r_here = wr.w;
    p.t_pend = Real<R>::kInf;
    // meta.z: the skip triangle, or -- while a traversal is queued -- the record's trace-
    // queue position (the record carries the skip triangle and the flight length; only
    // the megakernel hand-off reads them back: a logic visit takes the traversal result)
    const bool queued = meta_phase(m.w) == kPhTrace;
    p.skip = queued ? -1 : static_cast<int>(m.z);
    if (need_tpend && queued && !(m.w & kMetaFresh)) {  // the slot's own trace record
        p.t_pend = q.trs_o[s].w;
        p.skip = bits_int<R>(q.trs_d[s].w);
    }
    if (m.w & kMetaFresh) {  // camera ray: the state is in the trace record
        const Q4<R> d = q.tr_cam[m.z];
        p.x = sc_cam_pos;
        p.w = mk<R>(d.x, d.y, d.z);
        p.L = R(0);
        p.r_here = R(0);
    }
    p.rng.s = q.rng[s];
    p.id = m.x;
    p.seg = m.y;
    p.obj = meta_obj(m.w);
    p.c = static_cast<uint8_t>(meta_c(m.w));
    p.r_valid = (m.w >> 10) & 1u;
    *phase = meta_phase(m.w);
    p.cull = static_cast<int>((m.w >> 16) & 0xffu) - 1;
    p.pending = *phase == kPhSphere;
    p.tpend = *phase == kPhTrace;
    p.waited = 0;
    p.twaited = 0;
    p.pixel = 0;
    if (fold) {
        const uint32_t k = meta_pending(m.w);
        if (mb) {
#pragma unroll
            for (uint32_t i = 0; i < kNeeChain; ++i)
                if (i < k) p.L += mb->v[i];
        } else {
            for (uint32_t i = 0; i < k; ++i) p.L += q.nee_res[s * kNeeChain + i];
        }
        if (m.w & kMetaEnded) *phase = (m.w & kMetaEndEscaped) ? kPhEndedEscaped : kPhEnded;
    }
}

template <class R>
SST_D void load_slot(const WfPool<R>& q, uint32_t s, PathLocal<R>& p, uint32_t* phase, const V3<R>& cam,
                     bool need_tpend, bool fold) {
    load_slot_from(q, s, q.meta[s], p, phase, cam, need_tpend, fold);
}

// pending: staged NEE records not yet added to L; flags: kMetaEndAbsorbed. A slot that
// queues a traversal stores its meta after the queue append (slot_meta with z = the
// record's position; store_state here).
template <class R>
SST_D void store_state(const WfPool<R>& q, uint32_t s, const PathLocal<R>& p) {
    slot_xl(q, s) = Q4<R>{p.x.x, p.x.y, p.x.z, p.L};
    slot_wr(q, s) = Q4<R>{p.w.x, p.w.y, p.w.z, p.r_here};
    q.rng[s] = p.rng.s;
}
template <class R>
SST_D uint4 slot_meta(const PathLocal<R>& p, uint32_t z, uint32_t phase, uint32_t pending = 0u, uint32_t flags = 0u) {
    return make_uint4(static_cast<uint32_t>(p.id), p.seg, z,
                      pack_meta(p.obj, p.c, p.r_valid, phase, p.cull) | (pending << kMetaPendShift) | flags);
}
template <class R>
SST_D void store_slot(const WfPool<R>& q, uint32_t s, const PathLocal<R>& p, uint32_t phase, uint32_t pending = 0u,
                      uint32_t flags = 0u) {
    store_state(q, s, p);
    q.meta[s] = slot_meta(p, static_cast<uint32_t>(p.skip), phase, pending, flags);
}

// NEE record idx: point + weight, direction + obj | channel << 8. SST_NEE_PAIR keeps the two
// halves of a record adjacent (one 32-byte sector in FP32) instead of in two arrays: a slot
// stages ~2 of its 4 records per visit, so the split layout wrote and read half-used
// sectors in both arrays (C5: shadow 27.9 -> 26.4, sphere 21.7 -> 20.1 ms per slab).
// The pool carves nee_p and nee_w back to back: the 2 x (cap x kNeeChain) paired entries
// fit in their span.
#ifndef SST_NEE_PAIR
#define SST_NEE_PAIR 1
#endif
template <class R>
SST_D Q4<R>& nee_rec_p(const WfPool<R>& q, uint32_t idx) {
    return SST_NEE_PAIR ? q.nee_p[2u * idx] : q.nee_p[idx];
}
template <class R>
SST_D Q4<R>& nee_rec_w(const WfPool<R>& q, uint32_t idx) {
    return SST_NEE_PAIR ? q.nee_p[2u * idx + 1u] : q.nee_w[idx];
}

// Staged NEE record i of slot s.
template <class R>
SST_D void put_nee(const WfPool<R>& q, uint32_t s, uint32_t i, V3<R> x, V3<R> w, R weight, int obj, int c) {
    const uint32_t idx = s * kNeeChain + i;
    nee_rec_p(q, idx) = Q4<R>{x.x, x.y, x.z, weight};
    nee_rec_w(q, idx) = Q4<R>{w.x, w.y, w.z, int_bits<R>(obj | (c << 8))};
}

SST_D void set_phase(uint4* meta, uint32_t s, uint32_t phase) {
    uint32_t w = meta[s].w;
    w = (w & ~(3u << 11)) | (phase << 11);
    meta[s].w = w;
}

// TMA bulk prefetch of [p, p + bytes) into L2 (no registers, no completion to wait
// for): the pool's SoA streams are read a known distance ahead.
SST_D void l2_prefetch(const void* p, size_t bytes) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
    if (e > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"(static_cast<uint32_t>(e - a))
                     : "memory");
}

// Records [j, j + n) of a trace / shadow queue (bounded by the queue length).
#ifndef SST_WF_PREFETCH_AHEAD
#define SST_WF_PREFETCH_AHEAD 32768
#endif
template <class R>
SST_D void prefetch_trace(const WfPool<R>& q, uint32_t j, uint32_t n, uint32_t len) {
    j += SST_WF_PREFETCH_AHEAD;
    if (j >= len) return;
    if (n > len - j) n = len - j;
    l2_prefetch(q.q_trace + j, n * sizeof(uint32_t));  // logic entries (their records are gathered)
    l2_prefetch(q.tr_o + j, n * sizeof(Q4<R>));         // camera records
    l2_prefetch(q.tr_d + j, n * sizeof(Q4<R>));
    l2_prefetch(q.tr_f + j, n * sizeof(uint32_t));
}
template <class R>
SST_D void prefetch_shadow(const WfPool<R>& q, uint32_t j, uint32_t n, uint32_t len) {
    j += SST_WF_PREFETCH_AHEAD;
    if (j >= len) return;
    if (n > len - j) n = len - j;
    l2_prefetch(q.q_shadow + j, n * sizeof(uint32_t));
}

// Per-thread counters flushed once per thread block (warp sums -> shared -> one
// atomic per counter per block, spread over kStCopies copies of the stats array).
template <int N>
SST_D void flush_counts(unsigned long long* stats, const unsigned long long (&v)[N]) {
    __shared__ unsigned long long sh[kStCount];
    for (int k = threadIdx.x; k < kStCount; k += blockDim.x) sh[k] = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const unsigned long long s = warp_sum(v[k]);
        if ((threadIdx.x & 31u) == 0 && s) atomicAdd(&sh[k], s);
    }
    __syncthreads();
    unsigned long long* dst = stats + static_cast<size_t>(blockIdx.x % kStCopies) * kStCount;
    for (int k = threadIdx.x; k < N; k += blockDim.x)
        if (sh[k]) atomicAdd(dst + k, sh[k]);
}

// Per-thread counters of one wavefront launch: a thread handles tens of slots per launch,
// so 32 bits suffice (the logic pass is register-bound; 64-bit counters cost it ~9 more).
struct WfStats {
    uint32_t paths = 0, absorbed = 0, escaped = 0, capped = 0, errors = 0;
    uint32_t seg = 0, sphere = 0, events = 0, lane_iters = 0, wf_slots = 0;
    DecodeCount dc;
};
SST_D void flush_lane_stats(unsigned long long* stats, const WfStats& st) {
    unsigned long long v[kStCount] = {};
    v[kStPaths] = st.paths;
    v[kStSegments] = st.seg;
    v[kStSphere] = st.sphere;
    v[kStEvents] = st.events;
    v[kStDecL] = st.dc.l;
    v[kStDecP] = st.dc.p;
    v[kStDecE] = st.dc.e;
    v[kStAbsorbed] = st.absorbed;
    v[kStEscaped] = st.escaped;
    v[kStCapped] = st.capped;
    v[kStErrors] = st.errors;
    v[kStLaneIters] = st.lane_iters;
    v[kStWfSlots] = st.wf_slots;
    flush_counts<kStCount>(stats, v);
}

SST_D void flush_lane_stats(unsigned long long* stats, const LaneStats& st) {
    const unsigned long long v[kStCount] = {st.paths, st.seg, st.sphere, st.events, st.dc.l, st.dc.p,
                                            st.dc.e, st.absorbed, st.escaped, st.capped, st.errors, st.shadow,
                                            st.traversals, st.nodes, st.tris, st.lane_iters, st.warp_iters,
                                            st.shadow_tris, st.wf_slots};
    flush_counts<kStCount>(stats, v);
}

// Path end: the radiance (and segment count) of path p.id, end statistics.
template <class R, class Stats>
SST_D void finish_path(const TraceArgs<R>& a, const PathLocal<R>& p, int end, Stats& st) {
    a.radiance[p.id] = p.L;
    if (a.segments) a.segments[p.id] = p.seg;
    if (a.exit_state) write_exit_state(a.exit_state, p);
    ++st.paths;
    st.seg += p.seg;
    st.escaped += end == kEndEscaped;
    st.absorbed += end == kEndAbsorbed;
    st.capped += end == kEndCapped;
    st.errors += end == kEndError;
}

// Block-aggregated queue append: every thread of the block calls it (uniformly);
// threads with `want` get consecutive positions. One global atomic per block.
SST_D void block_push(bool want, uint32_t value, uint32_t* counter, uint32_t* queue) {
    __shared__ uint32_t wcount[32];
    __shared__ uint32_t base;
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const unsigned nw = (blockDim.x + 31u) >> 5;
    const unsigned b = __ballot_sync(0xffffffffu, want);
    if (lane == 0) wcount[warp] = __popc(b);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (unsigned i = 0; i < nw; ++i) {
            const uint32_t c = wcount[i];
            wcount[i] = tot;
            tot += c;
        }
        base = tot ? atomicAdd(counter, tot) : 0u;
    }
    __syncthreads();
    if (want) queue[base + wcount[warp] + __popc(b & ((1u << lane) - 1u))] = value;
    __syncthreads();  // wcount/base are reused by the next call
}

// N block-aggregated appends in one pass (2 barriers, one global atomic per
// non-empty queue per block): queue j receives `value` from the threads with want[j].
template <int N>
SST_D void block_pushn(const bool (&want)[N], uint32_t value, uint32_t* const (&counter)[N],
                       uint32_t* const (&queue)[N], uint32_t (&pos)[N]) {
    __shared__ uint32_t wc[8][33];
    __shared__ uint32_t qbase[8];
    static_assert(N <= 8, "queues");
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const unsigned nw = (blockDim.x + 31u) >> 5;
    unsigned b[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        b[j] = __ballot_sync(0xffffffffu, want[j]);
        if (lane == 0) wc[j][warp] = __popc(b[j]);
    }
    __syncthreads();
    if (threadIdx.x < N && counter[threadIdx.x]) {
        const int j = threadIdx.x;
        uint32_t tot = 0;
        for (unsigned i = 0; i < nw; ++i) {
            const uint32_t c = wc[j][i];
            wc[j][i] = tot;
            tot += c;
        }
        qbase[j] = tot ? atomicAdd(counter[j], tot) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < N; ++j) {
        pos[j] = qbase[j] + wc[j][warp] + __popc(b[j] & ((1u << lane) - 1u));
        if (want[j] && queue[j]) queue[j][pos[j]] = value;
    }
    __syncthreads();
}

// block_pushn plus one COUNTED queue: the calling thread appends cnt consecutive
// entries first, first + 1, ... (its chained NEE records) at consecutive positions.
template <int N>
SST_D void block_pushn_counted(const bool (&want)[N], uint32_t value, uint32_t* const (&counter)[N],
                               uint32_t* const (&queue)[N], uint32_t (&pos)[N], uint32_t cnt, uint32_t first,
                               uint32_t* ccounter, uint32_t* cqueue, uint32_t parity) {
    // double-buffered by call parity: a call's writes never meet the previous call's
    // reads, so no trailing barrier (every thread passed this call's two barriers before
    // the buffer comes round again)
    __shared__ uint32_t wcb[2][8][33];
    __shared__ uint32_t qbaseb[2][8];
    uint32_t(&wc)[8][33] = wcb[parity & 1u];
    uint32_t(&qbase)[8] = qbaseb[parity & 1u];
    static_assert(N + 1 <= 8, "queues");
    const unsigned lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const unsigned nw = (blockDim.x + 31u) >> 5;
    unsigned b[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
        b[j] = __ballot_sync(0xffffffffu, want[j]);
        if (lane == 0) wc[j][warp] = __popc(b[j]);
    }
    uint32_t incl = cnt;  // warp inclusive scan of the counted queue
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= static_cast<unsigned>(o)) incl += t;
    }
    if (lane == 31) wc[N][warp] = incl;
    __syncthreads();
    if (threadIdx.x <= N && (threadIdx.x == N ? ccounter != nullptr : counter[threadIdx.x] != nullptr)) {
        const int j = threadIdx.x;
        uint32_t tot = 0;
        for (unsigned i = 0; i < nw; ++i) {
            const uint32_t c = wc[j][i];
            wc[j][i] = tot;
            tot += c;
        }
        qbase[j] = tot ? atomicAdd(j == N ? ccounter : counter[j], tot) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < N; ++j) {
        pos[j] = qbase[j] + wc[j][warp] + __popc(b[j] & ((1u << lane) - 1u));
        if (want[j] && queue[j]) queue[j][pos[j]] = value;
    }
    const uint32_t at = qbase[N] + wc[N][warp] + incl - cnt;
    for (uint32_t i = 0; i < cnt; ++i) cqueue[at + i] = first + i;
}

// Warp-granular work stealing over a queue of n items: returns the next item index
// for this lane (>= n when the queue is exhausted for the whole warp).
SST_D uint32_t warp_fetch(uint32_t* cursor) {
    uint32_t base = 0;
    if ((threadIdx.x & 31u) == 0) base = atomicAdd(cursor, 32u);
    return __shfl_sync(0xffffffffu, base, 0) + (threadIdx.x & 31u);
}

// Warp-aggregated append from divergent code.
SST_D uint32_t warp_push(uint32_t value, uint32_t* counter, uint32_t* queue) {
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(counter, g.size());
    base = g.shfl(base, 0);
    queue[base + g.thread_rank()] = value;
    return base + g.thread_rank();
}

// Queue record written after the block push (the position is known only then):
// trace -- a = origin, b = direction, t = t_max, u = skip, v = (cull + 1) | inside << 8;
template <class R>
struct WfRec {
    V3<R> a, b;
    R t;
    int u;
    uint32_t v;
};

template <class R>
SST_D void put_trace(const WfPool<R>& q, uint32_t j, const WfRec<R>& r) {
    q.tr_o[j] = Q4<R>{r.a.x, r.a.y, r.a.z, r.t};
    q.tr_d[j] = Q4<R>{r.b.x, r.b.y, r.b.z, int_bits<R>(r.u)};
    q.tr_f[j] = r.v;
}

enum : int { kEmitNone = 0, kEmitTrace = 1, kEmitSphere = 2, kEmitFree = 4 };

// Paths of the launch the wavefront generates (after the camera pre-pass, if any).
template <class R, bool EX>
SST_D uint64_t wf_n_paths(const TraceArgs<R>& a) {
    return a.keys ? static_cast<uint64_t>(*a.keys_count) * (EX ? 1u : 3u) : a.n_paths;
}

// ------------------------------------------------------------------ k_wf_cam_filter
// Camera pre-pass: a camera ray that misses every object's (error-grown) bounding sphere
// misses every triangle, so its paths escape at the camera exactly as a traversal miss
// ends them (radiance = background, 0 segments, exit state = camera + direction); they
// are finished here and never occupy a pool slot (C5: ~76% of the frame is background).
// The other keys are compacted into `list` (block-aggregated, count in *count).
template <class R>
SST_D bool camera_ray_may_hit(const DevScene<R>& sc, V3<R> d) {
    return ray_may_hit(sc, sc.cam_pos, d, -1);
}

// Keys are grouped by the cost class of the costliest object their ray may enter
// (ObjK::cost_class, 0 = densest medium first): expensive paths are generated first, so
// the pool's drain -- exposed at the end of a launch -- holds the cheap ones. Two passes:
// pass 0 finishes the misses and counts the classes (hdr[1 + c]); pass 1 scatters each
// kept key behind the classes before it (cursors hdr[1 + kCostClasses + c]), reading the
// class pass 0 stored per key (cls_of). hdr[0] = the total.
constexpr uint32_t kCostClasses = 4;
template <class R>
SST_D uint32_t camera_ray_class(const DevScene<R>& sc, V3<R> d) {
    uint32_t cls = kCostClasses;  // none: the ray misses every bounding sphere
    for (uint32_t o = 0; o < sc.n_objects; ++o) {
        const ObjK<R>& ob = sc.objs[o];
        const V3<R> oc = mk<R>(ob.bsphere[0], ob.bsphere[1], ob.bsphere[2]) - sc.cam_pos;
        const R b = dot(oc, d), r = ob.bsphere[3];
        if (b + r >= R(0) && dot(oc, oc) - b * b <= r * r) cls = min(cls, ob.cost_class);
    }
    return cls;
}

template <class R, bool EX>
SST_D void wf_cam_filter(const TraceArgs<R>& a, uint32_t n_keys, uint32_t* list, uint32_t* hdr, uint8_t* cls_of,
                         int pass) {
    const DevScene<R>& sc = a.sc;
    unsigned long long done = 0;
    __shared__ uint32_t base_cls[kCostClasses];
    if (pass == 1 && threadIdx.x == 0) {
        uint32_t acc = 0;
        for (uint32_t c = 0; c < kCostClasses; ++c) {
            base_cls[c] = acc;
            acc += hdr[1 + c];
        }
    }
    __syncthreads();
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x; base < n_keys; base += stride) {  // block-uniform
        const uint32_t k = base + threadIdx.x;
        uint32_t cls = kCostClasses;
        if (k < n_keys && pass == 1) cls = cls_of[k];  // pass 0's class of this key
        if (k < n_keys && pass == 0) {
            const uint32_t pixel = EX ? a.pixel[k] : k % a.n_pix;
            const uint32_t sample = EX ? a.sample[k] : a.sample_begin + k / a.n_pix;
            const V3<R> d = camera_dir(a, pixel, sample);
            cls = camera_ray_class(sc, d);
            cls_of[k] = static_cast<uint8_t>(cls);
            if (cls == kCostClasses) {
                const uint32_t n_ch = EX ? 1u : 3u;
                for (uint32_t j = 0; j < n_ch; ++j) {
                    const uint64_t id = EX ? k : 3ull * k + j;
                    const uint32_t c = EX ? a.channel[k] : j;
                    a.radiance[id] = sc.bg[c];
                    if (a.segments) a.segments[id] = 0u;
                    if (a.exit_state) {
                        R* e = a.exit_state + 6 * id;
                        e[0] = sc.cam_pos.x, e[1] = sc.cam_pos.y, e[2] = sc.cam_pos.z;
                        e[3] = d.x, e[4] = d.y, e[5] = d.z;
                    }
                }
                done += n_ch;
            }
        }
        const bool want[kCostClasses] = {cls == 0u, cls == 1u, cls == 2u, cls == 3u};
        uint32_t pos[kCostClasses];
        if (pass == 0) {
            uint32_t* const ctr[kCostClasses] = {hdr + 1, hdr + 2, hdr + 3, hdr + 4};
            uint32_t* const qs[kCostClasses] = {nullptr, nullptr, nullptr, nullptr};
            block_pushn<kCostClasses>(want, k, ctr, qs, pos);
        } else {
            uint32_t* const ctr[kCostClasses] = {hdr + 5, hdr + 6, hdr + 7, hdr + 8};
            uint32_t* const qs[kCostClasses] = {nullptr, nullptr, nullptr, nullptr};
            block_pushn<kCostClasses>(want, k, ctr, qs, pos);
            if (cls < kCostClasses) list[base_cls[cls] + pos[cls]] = k;
        }
    }
    if (pass == 0) {
        unsigned long long v[kStCount] = {};
        v[kStPaths] = done;
        v[kStEscaped] = done;
        flush_counts<kStCount>(a.stats, v);
    } else if (blockIdx.x == 0 && threadIdx.x == 0) {
        uint32_t tot = 0;
        for (uint32_t c = 0; c < kCostClasses; ++c) tot += hdr[1 + c];
        hdr[0] = tot;
    }
}

// ------------------------------------------------------------------ k_wf_logic
// The non-traversal part of path_advance for one slot, run until the slot needs a
// traversal, a sphere step or a shadow ray (at most one per iteration), or its path
// ends. Operation order per path is path_advance's.
template <class R, bool ST, bool EX>
SST_D int wf_logic_slot(const TraceArgs<R>& a, const WfPool<R>& q, uint32_t s, const uint4 mt, unsigned m,
                        WfStats& st, bool* live, uint32_t* nrec_out) {
    // m: the lanes of this warp calling (converged). The loop below has no break /
    // continue / return inside: every stage is an if-block that all lanes of the warp
    // reach together, so lanes that got to a collision by different routes (after a
    // traversal, or after a flight that needed none) run it in ONE warp pass.
    const DevScene<R>& sc = a.sc;
    PathLocal<R> p;
    const Mailbox<R> mb = load_mailbox(q, s);
    uint32_t phase = meta_phase(mt.w);
    *live = false;
    *nrec_out = 0u;
    ++st.wf_slots;
    const bool ended = (mt.w & kMetaEnded) != 0u;
    m = __ballot_sync(m, phase != kPhEmpty && !ended);
    // ended in k_wf_sphere (which runs concurrently with the generation kernel and so
    // does not touch the free queue): free it now if new paths remain
    if (phase == kPhEmpty) return *a.work < wf_n_paths<R, EX>(a) ? kEmitFree : kEmitNone;
    if (ended) {  // absorbed / escaped after staging NEE records: add them, then it ends
        load_slot_from(q, s, mt, p, &phase, sc.cam_pos, false, true, &mb);
        if (mt.w & kMetaEndEscaped) p.L += sc.bg[p.c];
        finish_path(a, p, (mt.w & kMetaEndEscaped) ? kEndEscaped : kEndAbsorbed, st);
        q.meta[s] = make_uint4(0u, 0u, 0u, pack_meta(-1, 0, false, kPhEmpty, -1));
        return kEmitFree;
    }
    // the traversal result (and a fresh path's camera record) at the slot's trace-queue
    // position, issued with the slot loads
    uint2 hi = make_uint2(0u, 0u);
    R t_hit = R(0);
    if (phase == kPhTrace) {
        hi = q.hinfo[mt.z];
        t_hit = q.thit[mt.z];
    }
    load_slot_from(q, s, mt, p, &phase, sc.cam_pos, false, true, &mb);
    ++st.lane_iters;
    int emit = kEmitNone;
    int end = -1;
    bool run = true;
    bool bg_pending = false;  // an escape decided without its exit: background not yet added
    uint32_t nrec = 0u;  // NEE records staged by this visit (the mailbox)
#pragma unroll 1
    for (int guard = 0; guard < 4 + 2 * static_cast<int>(kNeeChain); ++guard) {
        if (!__any_sync(m, run)) break;
        bool collide = false;
        R t_free = Real<R>::kInf;
        // FP32: a flight that collides without a traversal hands its end point and the SDF
        // value there (gathered for the culling tests) to the collision stage
        bool have_end = false, in_end = false;
        R v_end = R(1);
        V3<R> x_end = p.x;
        if (run && phase == kPhTrace) {
            // ---- resolve (path_advance phase 2) with the traversal result
            const bool hit = (hi.y >> 31) != 0u;
            if (p.obj < 0) {
                if (!hit) {
                    p.L += sc.bg[p.c];
                    end = kEndEscaped;
                } else {  // medium entry (index-matched boundary)
                    p.x = p.x + p.w * t_hit;
                    p.obj = static_cast<int>(hi.y & 0x7fffffffu);
                    p.cull = -1;
                    p.skip = Real<R>::kIsDouble ? -1 : static_cast<int>(hi.x);
                    p.r_valid = false;
                    phase = kPhFlight;
                }
            } else if (hit) {  // leaves the medium
                p.x = p.x + p.w * t_hit;
                p.cull = sc.objs[p.obj].convex ? p.obj : -1;
                p.obj = -1;
                p.skip = Real<R>::kIsDouble ? -1 : static_cast<int>(hi.x);
                phase = kPhFlight;
            } else {
                t_free = t_hit;  // a miss leaves t_best = t_max = the queued flight length
                collide = true;
            }
        }
        if (run && end < 0 && !collide && phase == kPhFlight) {
            // ---- flight start (path_advance phase 1); a path that just crossed a
            // boundary starts its next flight in the same pass as the others
            bool inside = p.obj >= 0;
            bool trace = true;
            if (inside) {
                const ObjK<R>& ob = sc.objs[p.obj];
                const MediumK<R>& m = ob.med[p.c];
                // The free-path draw (on a copy of the stream, committed only if the path
                // is still inside) and the three gathers of the culling tests -- SDF at x,
                // skip grid at x, SDF at the flight's end -- are issued together: one
                // L2 round trip instead of three dependent ones. Same draws, same tests.
                Rng r2 = p.rng;
                R t_c = Real<R>::kInf;
                if (m.sigma_t > R(0)) {  // sample_free_path (optics.cpp:55-60)
                    const R u = r2.template uniform<R>();
                    if (Real<R>::kIsDouble) t_c = -Real<R>::log1p_(-u) / m.sigma_t;
                    else t_c = -Real<R>::div_(Real<R>::log_(R(1) - u), m.sigma_t);
                }
                bool in_grid = true;
                R v = R(0);
                uint32_t vox_end = 0;
                x_end = p.x + p.w * t_c;
                if (!p.r_valid) v = sdf_raw(ob, p.x, &in_grid);
                // with the safe radius known, a flight inside it needs no skip-grid gather
                const bool gather = !p.r_valid || !(t_c < p.r_here);
                R rs = R(0);
                if (gather) rs = skip_radius(ob, p.x);
                if (!Real<R>::kIsDouble && m.sigma_t > R(0)) {
                    v_end = sdf_raw(ob, x_end, &in_end, &vox_end);
                    have_end = true;
                }
                if (!p.r_valid) {
                    p.r_here = v < R(0) ? -v : R(0);
                    p.r_valid = true;
                    if (leaked(ob, v, in_grid)) {
                        recover_leak(p, ob);
                        inside = false;
                    }
                }
                if (inside) {
                    p.rng = r2;
                    t_free = t_c;
                    trace = !(t_free < p.r_here);
                    if (trace) {
                        trace = !(t_free < rs);
                        if (trace && a.convex_end) {
                            const int where = end_where(ob, v_end, in_end, vox_end, p.x, x_end, t_free,
                                                        Real<R>::fmax_(p.r_here, rs));
                            trace = where != kEndIn;
                            // The flight certainly leaves the convex object; if its ray misses
                            // every other object's bounding sphere, so does the ray continuing
                            // from the exit point (a sub-ray): the path escapes. Without an
                            // exit-state output the exit point itself is never needed.
                            // (The background is added once the visit's staged NEE
                            // contributions are in: the reference's order of additions.)
                            if (where == kEndOut && !a.exit_state && !ray_may_hit(sc, p.x, p.w, p.obj)) {
                                end = kEndEscaped;
                                bg_pending = true;
                                trace = false;
                            }
                        }
                    }
                }
            }
            if (!inside && !ray_may_hit(sc, p.x, p.w, p.cull)) {
                // an outside ray that misses every bounding sphere escapes (a traversal
                // miss): the path ends in this visit, without a trace round trip
                p.L += sc.bg[p.c];
                end = kEndEscaped;
                trace = false;
            }
            if (trace) {
                p.t_pend = t_free;
                phase = kPhTrace;
                emit = kEmitTrace;
                q.trs_o[s] = Q4<R>{p.x.x, p.x.y, p.x.z, t_free};
                q.trs_d[s] = Q4<R>{p.w.x, p.w.y, p.w.z, int_bits<R>(p.skip)};
                q.trs_f[s] = static_cast<uint32_t>(p.cull + 1) | (static_cast<uint32_t>(inside) << 8) |
                        (inside ? static_cast<uint32_t>(p.obj + 1) << 16 : 0u);
                run = false;
            } else if (end < 0) {
                collide = true;  // the flight stays inside: collision without traversal
            }
        }
        __syncwarp(m);
        if (run && collide) {
            // ---- collision (path_advance phases 2-3)
            const ObjK<R>& ob = sc.objs[p.obj];
            p.skip = -1;
            p.x = have_end ? x_end : p.x + p.w * t_free;
            p.r_valid = false;
            if (p.seg >= (ST ? sc.cap_st : sc.cap_pt)) {
                p.L = R(0);  // dropped
                end = kEndCapped;
            } else {
                ++p.seg;
                bool event = true;
                phase = kPhFlight;
                if (ST) {
                    bool in_grid = in_end;
                    const R v = have_end ? v_end : sdf_raw(ob, p.x, &in_grid);
                    p.r_here = v < R(0) ? -v : R(0);
                    p.r_valid = true;
                    if (leaked(ob, v, in_grid)) {  // not in the medium: next pass flies from here
                        recover_leak(p, ob);
                        event = false;
                    }
                    if (p.r_here > ob.med[p.c].r_min) {
                        phase = kPhSphere;
                        emit = kEmitSphere;
                        run = false;
                        event = false;
                    }
                }
                if (event) {
                    ++st.events;
                    const MediumK<R>& m = ob.med[p.c];
                    if (!((p.rng.next() >> 11) < m.survive_below)) {  // u < phi, bit-exact
                        end = kEndAbsorbed;
                    } else {
                        if (a.nee) {  // NEE with the incoming direction (no draws), staged
                            put_nee(q, s, nrec, p.x, p.w, R(1), p.obj, static_cast<int>(p.c));
                            ++nrec;
                        }
                        const R u1 = p.rng.template uniform<R>();
                        const R u2 = p.rng.template uniform<R>();
                        p.w = hg_sample(m.g, p.w, u1, u2);
                        // the next event chains into this visit until the mailbox is full
                        if (a.nee && nrec >= kNeeChain) run = false;
                    }
                }
            }
        }
        if (end >= 0) run = false;
    }
    if (end >= 0) {
        if ((end == kEndAbsorbed || end == kEndEscaped) && nrec > 0u) {
            // its staged contributions arrive next pass (then an escape adds the background)
            store_slot(q, s, p, kPhFlight, nrec, end == kEndAbsorbed ? kMetaEndAbsorbed : kMetaEndEscaped);
            *live = true;
            *nrec_out = nrec;
            return kEmitNone;
        }
        if (bg_pending) p.L += sc.bg[p.c];
        finish_path(a, p, end, st);  // capped: L = 0, the staged records do not matter
        q.meta[s] = make_uint4(0u, 0u, 0u, pack_meta(-1, 0, false, kPhEmpty, -1));
        return kEmitFree;
    }
    *live = true;
    *nrec_out = nrec;
    // a queued traversal's meta.z (its queue position) is patched after the append
    store_slot(q, s, p, phase, nrec);
    return emit;
}

// Processes the input list of live slots (all slots on the first iteration); slots
// still live afterwards form the output list (stream compaction), so drained slots
// cost nothing in later iterations.
// Processes the input list of live slots (all slots on the first iteration); slots
// still live afterwards form the output list (stream compaction), so drained slots
// cost nothing in later iterations.
template <class R, bool ST, bool EX>
SST_D void wf_logic(const TraceArgs<R>& a, const WfPool<R>& q) {
    WfStats st;
    // q_in == null: every slot in slot order (while the pool is full: coalesced SoA
    // accesses); otherwise the compacted list of the previous iteration (drain)
    const uint32_t n_in = q.q_in ? q.counts[q.cnt_in] : q.cap;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x; base < n_in; base += stride) {  // block-uniform
        const uint32_t i = base + threadIdx.x;
#ifndef SST_WF_NO_PREFETCH
        if (!q.q_in && threadIdx.x == 0 && base + stride < n_in) {  // slot order: this block's next chunk
            const uint32_t nb = base + stride, cnt = min(blockDim.x, n_in - nb);
            l2_prefetch(q.meta + nb, cnt * sizeof(uint4));
            if (SST_SLOT_PAIR) {
                l2_prefetch(&slot_xl(q, nb), 2u * cnt * sizeof(Q4<R>));
            } else {
                l2_prefetch(q.xl + nb, cnt * sizeof(Q4<R>));
                l2_prefetch(q.wr + nb, cnt * sizeof(Q4<R>));
            }
            l2_prefetch(q.rng + nb, cnt * sizeof(uint64_t));
        }
#endif
        int emit = kEmitNone;
        bool live = false;
        uint32_t nrec = 0u;
        const uint32_t s = i < n_in ? (q.q_in ? q.q_in[i] : i) : 0u;
        const unsigned m = __ballot_sync(0xffffffffu, i < n_in);
        if (i < n_in) emit = wf_logic_slot<R, ST, EX>(a, q, s, q.meta[s], m, st, &live, &nrec);
        const bool want[4] = {live, emit == kEmitTrace, emit == kEmitSphere, emit == kEmitFree};
        uint32_t* const ctr[4] = {q.counts + q.cnt_out, q.counts + kQTrace, ST ? q.counts + kQSphere : nullptr,
                                  q.counts + kQFree};
        uint32_t* const qs[4] = {q.q_out, q.q_trace, q.q_sphere, q.q_free};
        uint32_t pos[4];
        // the staged NEE records of the visit go onto the shadow queue as record indices
        block_pushn_counted<4>(want, s, ctr, qs, pos, nrec, s * kNeeChain, q.counts + kQShadow, q.q_shadow,
                               base / stride);
        if (emit == kEmitTrace) q.meta[s].z = pos[1];  // the traversal's queue position
    }
    flush_lane_stats(a.stats, st);
}

// ------------------------------------------------------------------ k_wf_gen
// New paths into the free slots: entry i of the free queue gets path id work + i, the
// camera ray is set up (path_init) and queued for its first traversal at trace
// position T + i and live-list position L + i (T, L = the logic pass's final counts):
// every position is known up front, so there are no atomics and no barriers. The last
// block to finish advances the path counter and the two queue counts and empties the
// free queue (slots left over once the ids run out stay empty).
template <class R, bool EX>
SST_D void wf_gen(const TraceArgs<R>& a, const WfPool<R>& q) {
    const uint32_t n_free = q.counts[kQFree];
    const uint64_t base = *a.work;
    const uint64_t n_paths = wf_n_paths<R, EX>(a);
    const uint64_t left = base < n_paths ? n_paths - base : 0;
    const uint32_t n_new = static_cast<uint32_t>(left < n_free ? left : n_free);
    const uint32_t t0 = q.counts[kQTrace], l0 = q.counts[q.cnt_out];
    // The three channel paths of a (pixel, sample) share one camera ray (the camera
    // stream is keyed by pixel and sample only): ids are consecutive, so entry i
    // (channel c_i = id % 3) shares the record of entry max(i - c_i, 0), and only those
    // owner entries are traced -- one traversal instead of three, identical results.
    const uint32_t c0 = EX ? 0u : static_cast<uint32_t>(base % 3), k0 = (3u - c0) % 3u;
    auto rank = [&](uint32_t i) -> uint32_t {  // trace position of owner entry i
        if (EX) return i;
        if (c0 == 0u) return i / 3u;
        return i == 0u ? 0u : 1u + (i - k0) / 3u;
    };
    const uint32_t n_own = EX ? n_new
                              : (n_new == 0u ? 0u
                                             : (c0 == 0u ? (n_new + 2u) / 3u
                                                         : 1u + (n_new > k0 ? (n_new - k0 + 2u) / 3u : 0u)));
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_new; i += stride) {
        const uint32_t s = q.q_free[i];
        PathLocal<R> p;
        path_init<R, EX>(a, base + i, p);
        // only the id/flags and the RNG go to the slot (scattered stores); position and
        // direction stay in the camera-ray record (kMetaFresh, load_slot)
        q.rng[s] = p.rng.s;
        const uint32_t ci = EX ? 0u : (c0 + i) % 3u;
        const uint32_t owner = i >= ci ? i - ci : 0u;
        const uint32_t j = t0 + rank(owner);
        q.meta[s] = make_uint4(static_cast<uint32_t>(p.id), 0u, j, pack_meta(-1, p.c, false, kPhTrace, -1) | kMetaFresh);
        if (owner == i) {
            WfRec<R> rec;
            rec.a = p.x;
            rec.b = p.w;
            rec.t = Real<R>::kInf;
            rec.u = -1;
            rec.v = 1u << 9;  // no cull, outside, camera ray
            put_trace(q, j, rec);
        }
        q.q_out[l0 + i] = s;
    }
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(q.counts + kQTicket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        *a.work = base + n_new;
        q.counts[kQTraceLogic] = t0;
        q.counts[kQTrace] = t0 + n_own;
        q.counts[q.cnt_out] = l0 + n_new;
        q.counts[kQFree] = 0u;
        q.counts[kQTicket] = 0u;
    }
}

// Pool start: every slot empty (the first logic pass puts them on the free queue).
template <class R>
SST_D void wf_init(const WfPool<R>& q) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < q.cap; s += gridDim.x * blockDim.x)
        q.meta[s] = make_uint4(0u, 0u, 0u, pack_meta(-1, 0, false, kPhEmpty, -1));
    if (blockIdx.x == 0 && threadIdx.x < kQCount) q.counts[threadIdx.x] = 0u;
}

// Iteration start: queue lengths and the output live count to zero.
template <class R>
SST_D void wf_reset(const WfPool<R>& q) {
    if (threadIdx.x < 3 || (threadIdx.x >= kQFetchTrace && threadIdx.x <= kQFetchShadow) || threadIdx.x == kQShadowS ||
        threadIdx.x == kQFetchShadowS)
        q.counts[threadIdx.x] = 0u;
    if (threadIdx.x == 3) q.counts[q.cnt_out] = 0u;
}

// ------------------------------------------------------------------ k_wf_trace
// Traversal stacks live in dynamic shared memory ([entry][thread], conflict-free),
// sc.bvh_depth + 1 entries per thread (wf_trace_smem bytes per block).
template <class R>
SST_HD size_t wf_trace_smem(uint32_t bvh_depth, int block) {
    return static_cast<size_t>(bvh_depth + 1) * block * (sizeof(int) + sizeof(R));
}

template <class R>
SST_D void wf_trace(const TraceArgs<R>& a, const WfPool<R>& q) {
    const DevScene<R>& sc = a.sc;
    uint64_t nodes = 0, tris = 0, trav = 0;
    extern __shared__ __align__(16) unsigned char wf_smem[];
    const uint32_t entries = sc.bvh_depth + 1;
    SharedStack<R> stk{reinterpret_cast<int*>(wf_smem) + threadIdx.x,
                       reinterpret_cast<R*>(wf_smem + static_cast<size_t>(entries) * blockDim.x * sizeof(int)) +
                           threadIdx.x,
                       static_cast<int>(blockDim.x)};
    // Persistent lanes with ray refill (Aila & Laine): rays run while-while rounds;
    // when at least kTraceRefill lanes of the warp have finished their ray (or all
    // have), they take new rays from the queue together, so a warp never idles until
    // its slowest ray is done.
#ifndef SST_TRACE_REFILL
#define SST_TRACE_REFILL 16
#endif
    constexpr int kTraceRefill = SST_TRACE_REFILL;
    const uint32_t n = q.counts[kQTrace], n_logic = q.counts[kQTraceLogic];
    const unsigned lane = threadIdx.x & 31u;
    bool have = false, exhausted = false;
    uint32_t s = 0;
    int skip = -1, cull = -1, want = 0;
    bool cam = false;  // camera ray: its direction is copied next to the result
    R t_min = R(0);
    RayK<R> ray;
    Trav<R> tr;
    tr.init(R(0));
    tr.node = kDone;
    for (;;) {
        const unsigned idle = __ballot_sync(0xffffffffu, !have);
        if (!exhausted && (__popc(idle) >= kTraceRefill || idle == 0xffffffffu)) {
            uint32_t base = 0;
            if (lane == 0) {
                base = atomicAdd(q.counts + kQFetchTrace, static_cast<uint32_t>(__popc(idle)));
#ifndef SST_WF_NO_PREFETCH
                prefetch_trace(q, base, static_cast<uint32_t>(__popc(idle)), n);
#endif
            }
            base = __shfl_sync(0xffffffffu, base, 0);
            if (base >= n) {
                exhausted = true;
            } else if (!have) {
                const uint32_t i = base + __popc(idle & ((1u << lane) - 1u));
                if (i < n) {
                    s = i;  // results go to the record's queue position
                    Q4<R> o, d;
                    uint32_t f;
                    if (i < n_logic) {  // a logic flight: its slot's record
                        const uint32_t sl = q.q_trace[i];
                        o = q.trs_o[sl], d = q.trs_d[sl], f = q.trs_f[sl];
                    } else {  // a camera ray: the generation kernel's record
                        o = q.tr_o[i], d = q.tr_d[i], f = q.tr_f[i];
                    }
                    skip = bits_int<R>(d.w);
                    cull = static_cast<int>(f & 0xffu) - 1;
                    const bool inside = (f >> 8) & 1u;
                    cam = (f >> 9) & 1u;
                    ray = make_ray(mk<R>(o.x, o.y, o.z), mk<R>(d.x, d.y, d.z));
                    want = Real<R>::kIsDouble ? 0 : (inside ? -1 : 1);
                    t_min = skip >= 0 ? sc.surf_eps : sc.t_min;
                    if (cam && sc.cam_off) {  // camera ray: its pixel tile's list, no traversal
                        R t_best = o.w;
                        uint32_t tri = 0u, obj = 0u;
                        const bool found = camera_tile_hit(sc, ray, t_min, &t_best, &tri, &obj, tris);
                        q.tr_cam[s] = Q4<R>{ray.d.x, ray.d.y, ray.d.z, R(0)};
                        q.thit[s] = t_best;
                        q.hinfo[s] = make_uint2(found ? tri : 0u, (found ? obj : 0u) | (found ? 0x80000000u : 0u));
                        ++trav;
                    } else {
                        // an in-medium flight starts at its object's subtree (disjoint objects, FP32)
                        tr.init(o.w, inside ? sc.objs[static_cast<int>(f >> 16) - 1].bvh_root : 0);
                        have = true;
                    }
                }
            }
        }
        if (__ballot_sync(0xffffffffu, have) == 0u) {
            if (exhausted) break;
            continue;
        }
        if (have) {
            tr.round(sc, ray, t_min, skip, cull, want, nodes, tris, stk);
            if (tr.done()) {
                if (cam) q.tr_cam[s] = Q4<R>{ray.d.x, ray.d.y, ray.d.z, R(0)};
                q.thit[s] = tr.t_best;
                q.hinfo[s] = make_uint2(tr.found ? tr.hit.tri : 0u,
                                        (tr.found ? tr.hit.obj : 0u) | (tr.found ? 0x80000000u : 0u));
                ++trav;
                have = false;
            }
        }
    }
    unsigned long long v[kStCount] = {};
    v[kStTraversals] = trav;
    v[kStNodes] = nodes;
    v[kStTriTests] = tris;
    flush_counts<kStCount>(a.stats, v);
}

// ------------------------------------------------------------------ k_wf_sphere
template <class R>
SST_D void wf_sphere(const TraceArgs<R>& a, const WfPool<R>& q) {
    const DevScene<R>& sc = a.sc;
    WfStats st;
    const uint32_t n = q.counts[kQSphere];
    for (;;) {
        const uint32_t i = warp_fetch(q.counts + kQFetchSphere);
        if (i - (threadIdx.x & 31u) >= n) break;  // warp-uniform
        if (i >= n) continue;
        const uint32_t s = q.q_sphere[i];
        PathLocal<R> p;
        uint32_t phase;
        const uint4 mt = q.meta[s];
        // the records the logic visit staged before this step are computed meanwhile
        // (their shadow launch runs concurrently): stay pending, this step's record follows
        load_slot_from(q, s, mt, p, &phase, sc.cam_pos, false, false);
        uint32_t pend = meta_pending(mt.w);
        ++st.sphere;
        StepOut<R> o;
        const MediumK<R>& m = sc.objs[p.obj].med[p.c];
        int end = -1;
        if (!sphere_step(m, p.w, p.x, p.r_here, a.nee != 0, p.rng, o, st.dc)) {
            p.L = R(0);
            end = kEndError;
        } else if (o.absorbed) {
            end = kEndAbsorbed;
        } else {
            if (a.nee) {
                // sphere-step NEE records go onto the shadow queue from the back (their own
                // counter): the logic pass's records can be consumed concurrently
                put_nee(q, s, pend, o.rep_pos, o.rep_dir, o.lambda, p.obj, static_cast<int>(p.c));
                cg::coalesced_group g = cg::coalesced_threads();
                uint32_t base = 0;
                if (g.thread_rank() == 0) base = atomicAdd(q.counts + kQShadowS, g.size());
                const uint32_t j = q.cap * (kNeeChain + 1u) - 1u - (g.shfl(base, 0) + g.thread_rank());
                q.q_shadow[j] = s * kNeeChain + pend;
                ++pend;
            }
            p.x = o.exit_pos;
            p.w = o.exit_dir;
            p.r_valid = false;
        }
        if (end == kEndAbsorbed && pend > 0u) {  // earlier staged contributions: next pass ends it
            store_slot(q, s, p, kPhFlight, pend, kMetaEndAbsorbed);
        } else if (end >= 0) {  // the slot goes back to the free queue in the next logic pass
            finish_path(a, p, end, st);
            q.meta[s] = make_uint4(0u, 0u, 0u, pack_meta(-1, 0, false, kPhEmpty, -1));
        } else {
            store_slot(q, s, p, kPhFlight, pend);
        }
    }
    flush_lane_stats(a.stats, st);
}

// ------------------------------------------------------------------ k_wf_shadow
// One staged NEE record (index idx = slot * kNeeChain + i): shadow ray through the light
// grid; the contribution goes to the record's mailbox entry (the slot adds it next pass).
template <class R>
SST_D void shadow_rec(const TraceArgs<R>& a, const WfPool<R>& q, uint32_t idx, const Q4<R>& np, const Q4<R>& nw,
                      uint64_t& tris) {
    const DevScene<R>& sc = a.sc;
    const int oc = bits_int<R>(nw.w);
    const int obj = oc & 0xff, c = oc >> 8;
    q.nee_res[idx] =
        nee_term(sc, sc.objs[obj].med[c], c, mk<R>(np.x, np.y, np.z), mk<R>(nw.x, nw.y, nw.z), np.w, tris,
                 sc.objs[obj].convex ? obj : -1);
}

// Records [0, n) of one shadow range (queue position pos(i)) by work stealing in grabs
// of 32 * kShadowGrab items per warp, processed one after another: the grab's single
// atomic on the shared cursor is what matters (950M shadow rays per C5 slab -- at one
// same-address atomic per 32 rays the cursor's L2 atomic throughput showed as 16% of the
// kernel's stall samples). Measured (Gseg/s): grab 1: 7.79, 2: 8.00, 4: 8.03, 8: 8.01;
// loading each lane's next record while its current ray is traced cost more registers
// than it saved (grab 2: 7.95, grab 4: 7.87).
#ifndef SST_SHADOW_GRAB
#define SST_SHADOW_GRAB 4
#endif
constexpr uint32_t kShadowGrab = SST_SHADOW_GRAB;
constexpr uint32_t kNoRec = 0xffffffffu;
template <class R, class Pos>
SST_D void shadow_range(const TraceArgs<R>& a, const WfPool<R>& q, uint32_t* cursor, uint32_t n, Pos pos,
                        bool prefetch, uint64_t& tris, uint64_t& shadow) {
    const unsigned lane = threadIdx.x & 31u;
    for (;;) {
        uint32_t base = 0;
        if (lane == 0) {
            base = atomicAdd(cursor, 32u * kShadowGrab);
#ifndef SST_WF_NO_PREFETCH
            if (prefetch) prefetch_shadow(q, base, 32u * kShadowGrab, n);
#endif
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if (base >= n) break;  // warp-uniform
#pragma unroll 1
        for (uint32_t j = 0; j < kShadowGrab; ++j) {
            const uint32_t i = base + 32u * j + lane;
            if (i - lane >= n) break;  // warp-uniform
            if (i >= n) continue;
            const uint32_t idx = q.q_shadow[pos(i)];
            if (idx == kNoRec) continue;
            shadow_rec(a, q, idx, nee_rec_p(q, idx), nee_rec_w(q, idx), tris);
            ++shadow;
        }
    }
}

// The logic pass's NEE records (front of the arrays, counts[kQShadow]) are consumed by
// work stealing; with_sphere: then the sphere steps' records (back of the arrays,
// counts[kQShadowS]). In a concurrent iteration a logic-only launch follows the trace
// kernel on the job stream and a full one follows the sphere kernel on the side stream,
// so whichever stream runs out of work first takes more of the shared queue.
template <class R>
SST_D void wf_shadow(const TraceArgs<R>& a, const WfPool<R>& q, bool with_sphere) {
    uint64_t tris = 0, shadow = 0;
    shadow_range(a, q, q.counts + kQFetchShadow, q.counts[kQShadow], [](uint32_t i) { return i; }, true, tris,
                 shadow);
    if (with_sphere) {
        const uint32_t back = q.cap * (kNeeChain + 1u) - 1u;
        shadow_range(a, q, q.counts + kQFetchShadowS, q.counts[kQShadowS], [back](uint32_t i) { return back - i; },
                     false, tris, shadow);
    }
    unsigned long long v[kStCount] = {};
    v[kStShadow] = shadow;
    v[kStTriTests] = tris;
    v[kStShadowTris] = tris;
    flush_counts<kStCount>(a.stats, v);
}

// Live slots (phase != empty) -> q_live, count in counts[kQResume] (hand-off list).
template <class R>
SST_D void wf_compact(const WfPool<R>& q) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x; base < q.cap; base += stride) {
        const uint32_t s = base + threadIdx.x;
        const bool live = s < q.cap && meta_phase(q.meta[s].w) != kPhEmpty;
        block_push(live, s, q.counts + kQResume, q.q_live);
    }
}

}  // namespace sstg
