// types.cuh -- plain data shared by the host API (api.cu) and the kernel TUs.
#pragma once

#include "common.cuh"

namespace sstg {

// Per-medium constants, precomputed on the host in double (so FP32 kernels see
// correctly rounded log(phi) and 1-phi, not their float cancellations).
template <class R>
struct MediumK {
    R sigma_t, g, phi;
    R log_phi;        // log(phi)   (0 < phi < 1)
    R one_minus_phi;  // 1 - phi
    R r_min;          // sphere-step threshold
    uint64_t survive_below;  // roulette: survive iff (draw >> 11) < ceil(phi * 2^53): bit-exact u < phi
    uint32_t phi_is_one, phi_is_zero;
};

template <class R>
struct StepOut {
    bool absorbed;
    uint32_t n;
    V3<R> exit_pos, exit_dir, rep_pos, rep_dir;
    R lambda;
};

struct DecodeCount {
    uint32_t l = 0, p = 0, e = 0;
};

// FP32 node: a = (lo0.x, hi0.x, lo0.y, hi0.y), b = (lo1.x, hi1.x, lo1.y, hi1.y),
//            c = (lo0.z, hi0.z, lo1.z, hi1.z), d = (child0, child1, -, -)
// child >= 0: interior node index; child < 0: leaf, ~child = (first << 3) | count.
struct alignas(16) NodeF {
    float4 a, b, c;
    int4 d;  // child0, child1, object of child0 subtree, object of child1 subtree (-1 mixed)
};
struct alignas(16) NodeD {
    double lo0[3], hi0[3], lo1[3], hi1[3];
    int32_t c0, c1, pad0, pad1;
};
// Triangles in leaf order. FP32: v0.xyz + object id, e1.xyz + triangle id, e2.xyz.
struct alignas(16) TriF {
    float4 v0o, e1i, e2;
};
struct alignas(16) TriD {
    double v0[3], e1[3], e2[3];
    uint32_t obj, id;
};

template <class R>
struct ObjK {
    MediumK<R> med[3];
    R sdf_origin[3];
    R sdf_voxel;
    R sdf_inv_voxel;
    uint32_t dims[3];
    const float* sdf;
    // Acceleration-only skip grid (2x the SDF resolution, same origin): per voxel a
    // lower bound on the distance from ANY point of the voxel to this object's
    // surface, in units of skip_unit (uint8, floor-quantised). Never changes results:
    // it only proves that a free flight cannot reach the boundary.
    const uint8_t* skip;
    R skip_inv_voxel, skip_unit;
    uint32_t skip_dims[3];
    uint32_t convex;  // closed convex mesh: a ray leaving it cannot hit it again
    // FP32, convex objects: per boundary SDF voxel (stored value +-0) that holds a point
    // inside the object (the centre, or a corner), the planes (unit outward normal,
    // offset) of every face that can meet the voxel, CSR (plane_off[v] .. plane_off[v +
    // 1]); a point of such a voxel strictly inside all of them is inside the object
    // (integrator.cuh end_inside_planes). Null: no lists.
    const uint32_t* plane_off;
    const float4* planes;
    float plane_eps;  // required margin below every plane
    int32_t bvh_root;  // FP32 in-medium traversals start here (host.h FlatBvh::obj_root); 0 = root
    // Bounding sphere (centre, radius grown by the FP error of the camera-ray test): a
    // camera ray that misses it misses every triangle of the object (wf_cam_filter).
    R bsphere[4];
    // Rank of the object's medium density among the scene's objects (0 = densest, capped
    // at kCostClasses - 1): the camera pre-pass generates paths into dense media first.
    uint32_t cost_class;
};

template <class R>
struct DevScene {
    const void* nodes;
    const void* tris;
    const ObjK<R>* objs;
    uint32_t n_objects;
    V3<R> light;
    V3<R> light_dir;  // directional light (unit, toward the light); used iff directional
    int directional;
    R power[3], bg[3];
    V3<R> cam_pos, cam_fwd, cam_right, cam_up;
    R tan_half, aspect;
    uint32_t width, height;
    R t_min, surf_eps;
    uint32_t cap_pt, cap_st;
    // Light-space culling grid for NEE shadow rays: a cube map over directions
    // from the point light; cell c lists (leaf-order) triangles whose angular
    // footprint overlaps it: grid_tri[grid_off[c] .. grid_off[c+1]). Null = use the BVH.
    const uint32_t* grid_off;
    const uint32_t* grid_tri;
    const void* grid_tris;  // FP32: TriF records in list order (grid_tri gathered); null in FP64
    // Per cell: the list holds the faces that face the light first, then the ones facing
    // away grouped by object; grid_split[c] = count of the former | (the single object
    // owning all of the latter, 0xff if mixed) << 24. A shadow ray from inside a convex
    // object never crosses that object's faces that face away from the light (FP32: those
    // tests are skipped when they are the whole back part). Null: test the whole list.
    const uint32_t* grid_split;
    // FP32 camera tiles (cam_tile x cam_tile pixels): per tile the triangles facing the
    // camera whose projection (grown by a pixel) meets it, as contiguous TriF records
    // (CSR cam_off over cam_tiles_x * cam_tiles_y tiles). A camera ray's nearest entering
    // hit is among its tile's list: the trace kernel answers camera rays from it instead
    // of the BVH. Null: BVH.
    const uint32_t* cam_off;
    const void* cam_tris;
    uint32_t cam_tile, cam_tiles_x, cam_tiles_y;
    uint32_t grid_res;
    uint32_t bvh_depth;  // FlatBvh::max_depth (traversal stack bound)
};

// Traversal stack capacity (entries); scenes whose BVH is deeper are rejected at upload.
constexpr int kStack = 48;

struct Hit {
    uint32_t tri, obj;
};

enum : int { kEndEscaped = 0, kEndAbsorbed = 1, kEndCapped = 2, kEndError = 3 };

// Stats slots (device u64 array).
enum : int {
    kStPaths = 0, kStSegments, kStSphere, kStEvents, kStDecL, kStDecP, kStDecE, kStAbsorbed,
    kStEscaped, kStCapped, kStErrors, kStShadow,
    // work counters (profiling): nearest-hit traversals, interior nodes visited,
    // triangle tests (nearest + shadow), live-lane iterations, warp iterations
    kStTraversals, kStNodes, kStTriTests, kStLaneIters, kStWarpIters,
    kStShadowTris,  // triangle tests of NEE shadow rays (also in kStTriTests)
    kStWfSlots,     // wavefront logic-pass slot visits
    kStCount
};

// Stats are kept in kStCopies interleaved copies ([copy][kStCount]) so the per-block
// flushes of the short wavefront kernels do not serialise on one address.
constexpr int kStCopies = 64;

// Wavefront path pool (wavefront.cuh): per-slot path state as structure-of-arrays of
// 16-byte vectors (FP32; 32 bytes for FP64), plus the per-operation slot queues.
template <class R>
struct alignas(4 * sizeof(R)) Q4 {
    R x, y, z, w;
};
// counts[]: queue lengths, the two ping-pong live-slot lists, the hand-off list.
// kQFetch*: work-stealing cursors of the trace / sphere / shadow kernels.
enum : int {
    kQTrace = 0, kQSphere = 1, kQShadow = 2, kQLiveA = 3, kQLiveB = 4, kQResume = 5,
    kQFetchTrace = 6, kQFetchSphere = 7, kQFetchShadow = 8,
    kQFree = 9,     // slots whose path ended (generation input)
    kQTicket = 10,  // last-block detection of the generation kernel
    kQShadowS = 11,       // sphere-step NEE records (stored from the back of the shadow arrays)
    kQFetchShadowS = 12,  // their work-stealing cursor
    kQTraceLogic = 13,    // trace entries [0, n) are the logic pass's (slot records), the rest camera records
    kQCount = 14
};
// NEE mailbox (wavefront.cuh): a logic visit chains up to kNeeChain delta-tracking
// events; their NEE records are staged per slot at s * kNeeChain + i, the shadow kernel
// writes each contribution to nee_res at the same index, and the slot's next visit adds
// them to its radiance in event order. With traversals frequent (round 2 start) 2
// measured best on C5 (3: +6%, 4: +10% logic time -- a warp runs as long as its longest
// chain, and traversals cut chains anyway); once the exact flight culling removed 85% of
// the traversals, the mailbox became what ends most visits: 2 / 3 / 4 / 5 / 6 give
// 6.86 / 7.06 / 7.20 / 7.07 / 6.93 Gseg/s.
#ifndef SST_NEE_CHAIN
#define SST_NEE_CHAIN 4
#endif
constexpr uint32_t kNeeChain = SST_NEE_CHAIN;
static_assert(kNeeChain >= 1 && kNeeChain <= 15, "pending count lives in 4 meta bits");

template <class R>
struct WfPool {
    uint32_t cap;     // slots
    Q4<R>* xl;        // position, radiance
    Q4<R>* wr;        // direction, SDF radius at the position
    uint64_t* rng;    // RandomStream state
    uint4* meta;      // path id, segments, skip triangle (while a traversal is queued: its
                      // trace-queue position), packed obj/channel/flags/phase/cull
    // Trace queue as contiguous ray records (indexed by queue position, written by
    // the logic / generation kernels, read coalesced by k_wf_trace), and the
    // traversal results at the same positions (read by the next logic pass).
    Q4<R>* tr_o;      // origin, t_max
    Q4<R>* tr_d;      // direction, skip triangle (int bits)
    uint32_t* tr_f;   // (cull + 1) | inside << 8 | camera ray << 9
    // A flight the logic pass queues is written to its slot's record (trs_*, slot-indexed)
    // the moment it is decided -- no record held in registers until the queue append --
    // and the trace queue entry q_trace[j] names the slot; positions [counts[kQTraceLogic],
    // counts[kQTrace]) hold the generation kernel's camera records (tr_*, position-indexed).
    Q4<R>* trs_o;
    Q4<R>* trs_d;
    uint32_t* trs_f;
    uint32_t* q_trace;
    // Direction of a camera ray, copied by the trace kernel next to its result (a fresh
    // path reads it there in the next logic pass, which overwrites the records).
    Q4<R>* tr_cam;
    R* thit;          // traversal result: distance
    uint2* hinfo;     // traversal result: triangle, object | found << 31
    // NEE records staged per slot ([cap * kNeeChain], index s * kNeeChain + i); the
    // shadow queue q_shadow ([cap * (kNeeChain + 1)]) holds record indices: the logic
    // records from the front, the sphere steps' records from the back.
    Q4<R>* nee_p;     // NEE record: point, weight
    Q4<R>* nee_w;     // NEE record: direction, obj | channel << 8 (int bits)
    R* nee_res;       // contribution of each record (written by k_wf_shadow)
    uint32_t *q_sphere, *q_shadow, *q_live;
    uint32_t *q_la, *q_lb;  // ping-pong lists of live slots (logic input / output)
    uint32_t* q_free;       // free slots (path ended), refilled by the generation kernel
    uint32_t* q_in;         // this iteration's input list (q_la or q_lb), count counts[cnt_in]
    uint32_t* q_out;        // output list, count counts[cnt_out]
    int cnt_in, cnt_out;
    uint32_t* counts;  // [kQCount]
    unsigned long long* resume_work;  // path counter of the megakernel hand-off
};

template <class R>
struct TraceArgs {
    DevScene<R> sc;
    int nee;
    uint64_t seed;
    uint64_t n_paths;
    uint32_t n_pix;
    uint32_t sample_begin;
    const uint32_t* pixel;   // explicit-key mode (trace_paths); null for render
    const uint32_t* sample;
    const uint8_t* channel;
    R* radiance;             // [n_paths]
    uint32_t* segments;      // [n_paths] or null
    R* exit_state;           // [6 n_paths] final position, direction (trace_paths_ex) or null
    unsigned long long* work;   // path-id counter
    unsigned long long* stats;  // [kStCount]
    int sphere_batch;           // warp regrouping threshold for sphere steps (lanes)
    int trace_batch;            // warp regrouping threshold for BVH traversals (0 = off)
    WfPool<R> pool;             // wavefront pool (wavefront.cuh)
    int resume;                 // megakernel resumes the pool's live slots (q_live) instead of new ids
    int convex_end;             // FP32: skip traversals of flights that end inside a convex object
    // Camera pre-pass (wavefront.cuh wf_cam_filter): the camera keys whose ray can hit an
    // object's bounding sphere, compacted; path id i maps to key keys[i / 3] (render) or
    // keys[i] (explicit keys). Null: ids are keys. keys_count: their number (device).
    const uint32_t* keys;
    const uint32_t* keys_count;
};

// TrainingSample (dataset.hpp:17-27): the SSWK record, 52 bytes, no padding.
struct TrainingSampleDev {
    float sigma_t, g, phi;
    uint32_t n_events;
    float cos_theta, alpha, beta;
    float rep_position[3];
    float rep_direction[3];
};
static_assert(sizeof(TrainingSampleDev) == 52, "TrainingSample layout");

// Arguments of the dataset kernel (dataset.cuh).
struct DatasetArgs {
    uint64_t n, first;
    double s_lo, s_hi, g_lo, g_hi;
    int phi_kind;
    double phi_a, phi_b;
    uint64_t seed;
    TrainingSampleDev* out;          // [n]
    unsigned long long* work;        // sample counter
    unsigned long long* stats;       // [0] events (pass 1), [1] replayed events, [2] max N
    int* error;                      // walk exceeded 1e6 events (the reference throws)
};

// Arguments of the sphere-step batch kernel (C ABI sst_gpu_sphere_step_batch).
struct StepBatchArgs {
    uint64_t n;
    const double *sigma_t, *g, *phi, *w_in, *center, *r;
    const uint8_t* with_event;
    int with_event_default;
    uint64_t* rng_state;
    uint8_t* absorbed;
    uint32_t* n_events;
    double *exit_pos, *exit_dir;
    uint8_t* has_rep;
    double *rep_pos, *rep_dir, *lambda;
    unsigned long long* counters;  // [3] length, path, event
    int* error;
};

// Verification kernels (verify.cuh).
// counters of k_verify_cull (sst_cull_report order)
enum : int {
    kCvFlights = 0, kCvCullSdf, kCvCullSkip, kCvCullConvex, kCvCullTwoBall, kCvViolSdf, kCvViolSkip,
    kCvViolConvex, kCvViolTwoBall, kCvRadiusViol, kCvSkipRadiusViol, kCvCullPlanes, kCvViolPlanes, kCvCount
};

template <class R>
struct CullCheckArgs {
    DevScene<R> sc;
    const TriD* tris;  // FP64 triangles (leaf order) of the uploaded scene
    uint32_t n_tris;
    uint64_t n, seed;
    int convex_end;
    unsigned long long* counts;  // [kCvCount]
};

struct NeeIdentityArgs {
    uint64_t walks;
    uint32_t resamples;
    double sigma_t, g, phi;
    double light[3];
    uint64_t seed;
    double* sums;                // [0] sum F, [1] sum S, [2] sum (S - F)^2
    unsigned long long* counts;  // [0] walks, [1] events, [2] resamples
};

}  // namespace sstg
