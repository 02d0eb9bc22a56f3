// api.cu -- implementation of the C ABI (include/sst_gpu.h, include/sst_host.h).
//
// Host C++ around the kernels: contexts, uploads (models -> __constant__, scene ->
// BVH/SDF/medium tables in HBM), launches, error mapping. No exception crosses the
// boundary; there is no CPU fallback -- without a CUDA device every compute entry
// fails with SST_E_CUDA.
#include <cuda_runtime.h>
#include <zlib.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <thread>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/sst_gpu.h"
#include "../../include/sst_host.h"
#include "host.h"
#include "launch.h"
#include "train.h"
#include "rng.cuh"
#include "types.cuh"

using namespace sstg;

namespace {

thread_local std::string g_last_error;

#define CK(expr)                                                                                \
    do {                                                                                        \
        const cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                                  \
            throw CudaFailure(std::string(#expr) + ": " + cudaGetErrorString(e_));              \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return SST_OK;
    } catch (const InvalidArgument& e) {
        g_last_error = e.what();
        return SST_E_INVALID_ARGUMENT;
    } catch (const DomainError& e) {
        g_last_error = e.what();
        return SST_E_DOMAIN;
    } catch (const CudaFailure& e) {
        g_last_error = e.what();
        return SST_E_CUDA;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return SST_E_RUNTIME;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SST_E_RUNTIME;
    }
}

// Grow-only device scratch buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void reserve(size_t n) {
        if (n <= bytes) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        CK(cudaMalloc(&p, n));
        bytes = n;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

// Function-local device buffer: released on every exit path (including CK throws).
struct ScopedBuf : DevBuf {
    ScopedBuf() = default;
    ScopedBuf(const ScopedBuf&) = delete;
    ScopedBuf& operator=(const ScopedBuf&) = delete;
    ~ScopedBuf() { release(); }
};

struct ObjectHost {
    double sdf_origin[3];
    double sdf_voxel;
    uint32_t dims[3];
    std::vector<float> sdf;
    sst_medium media[3];
    // acceleration-only skip grid (types.cuh ObjK::skip)
    std::vector<uint8_t> skip;
    double skip_voxel = 0.0, skip_unit = 0.0;
    uint32_t skip_dims[3] = {0, 0, 0};
    bool convex = false;
    // FP32 end-point face-plane lists (types.cuh ObjK::plane_off / planes), convex only
    std::vector<uint32_t> plane_off;
    std::vector<float> planes;  // 4 per plane: unit outward normal, offset
    float plane_eps = 0.0f;
    double bsphere[4] = {0, 0, 0, 0};  // bounding sphere of the vertices (centre, radius)
};

}  // namespace

namespace sstg {
// A wavefront render launch in flight (api.cu WfJob): the host drives its iterations
// in batches; render calls return while a job drains so consecutive calls overlap.
struct WfJobBase {
    virtual ~WfJobBase() = default;
    // Reads completed batches and keeps two in flight; the oldest job may finish (hand-
    // off + film). block: wait for this job's oldest batch. Returns 2 finished, 1
    // progressed, 0 idle.
    virtual int advance(bool may_finish, bool block) = 0;
    virtual bool supply_done() const = 0;
    const void* slot = nullptr;
};
}  // namespace sstg

struct sst_gpu_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int precision = SST_PREC_F32;
    uint64_t serial = 0;

    bool models = false;
    HostModel host_models[3];
    bool have_model[3] = {false, false, false};  // decoders staged for install (train_model)
    std::vector<double> weights;
    double norms[6] = {};
    uint64_t model_gen = 0;
    uint64_t weights_fp = 0;  // fingerprint of (weights, norms): equal weights share the constant bank

    bool scene = false;
    uint64_t scene_bytes = 0, scene_bytes_grid = 0;
    uint64_t grid_list_n = 0;  // light-grid list entries
    uint32_t n_nodes = 0, n_tris = 0;
    std::vector<ObjectHost> objects;
    std::vector<uint64_t> object_fp;  // fingerprint of objects[o] (re-upload of the same object: no copy)
    sst_scene_desc desc{};
    DevBuf nodes32, tris32, nodes64, tris64, objs32, objs64, grid_off, grid_tri, grid_split;
    DevBuf grid_tris32;  // FP32 triangle records in light-grid list order (grid_tri gathered)
    DevBuf cam_off, cam_idx, cam_tris32;  // camera tiles (types.cuh DevScene::cam_off)
    uint32_t cam_tiles_x = 0, cam_tiles_y = 0;
    uint64_t cam_list_n = 0;
    uint32_t grid_res = 0;
    std::vector<DevBuf> sdf_dev, skip_dev, plane_off_dev, planes_dev;
    DevScene<float> sc32{};
    DevScene<double> sc64{};

    DevBuf radiance, segments, work, stats, error, film_sum, film_sq, keys_pix, keys_smp, keys_ch;
    // pinned staging for host-film readback (grow-only; cudaFreeHost on destroy)
    double* film_pin = nullptr;
    size_t film_pin_n = 0;
    cudaEvent_t film_pin_ev[8] = {};
    DevBuf step_in, step_out;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;

    // Derived-structure caches keyed by content fingerprints (FNV-1a), the way the
    // reference caches SDFs (load_or_build_sdf, sdf.cpp:103-119): per-object SDF /
    // skip grid / convexity, and the scene BVH + light grid. Re-uploading an
    // unchanged scene recomputes nothing but still copies everything to the device.
    std::map<uint64_t, ObjectHost> obj_cache;
    // The BVH is keyed by the geometry alone; the light grid by (geometry, light
    // position), so a re-upload that moves only the light -- or any directional-light
    // upload -- keeps the BVH.
    struct SceneCache {
        uint64_t geo_fp = 0, grid_fp = 0;
        bool have_bvh = false;
        FlatBvh bvh;
        std::vector<uint32_t> grid_off, grid_tri, grid_split;
        uint32_t grid_res = 0;
        uint64_t cam_fp = 0;  // camera tiles of (geometry, camera): lists kept for re-uploads
        std::vector<uint32_t> cam_off, cam_idx;
        uint32_t cam_tiles_x = 0, cam_tiles_y = 0;
    } scene_cache;

    // Render pipeline: chunks of a render call rotate over kSlots streams so the
    // long-path tail of one persistent launch overlaps the next launch's bulk.
    // Film accumulations stay in chunk order (event chain) -> deterministic sums.
    static constexpr int kSlots = 5;
    struct Slot {
        cudaStream_t s = nullptr;
        DevBuf rad, work;
        cudaEvent_t film_done = nullptr;
        // wavefront pool (wavefront.cuh) + pinned queue counters read by the host loop
        DevBuf wf;
        DevBuf keys;  // camera pre-pass: [16 u32 header] + compacted key list (wf_cam_filter)
        uint32_t* wf_host = nullptr;  // [2][kQCount]
        cudaEvent_t wf_ev[2] = {nullptr, nullptr};
        // concurrent half of a wavefront iteration (sphere + shadow) and its fork/join
        cudaStream_t side = nullptr;
        cudaEvent_t wf_fork = nullptr, wf_join = nullptr;
    } slots[kSlots];
    // Wavefront integrator: SST_WAVEFRONT=0 megakernel only, 1 wavefront for the sphere
    // tracer only, 2 (default) also for the delta-tracking path tracer (C5 PT+NEE 1.42x,
    // C3 sigma_t=160 1.44x the megakernel since the session-3 wavefront work; the long-path
    // tail still goes to the megakernel). Pool slots per launch, hand-off when live slots
    // <= min(pool / 8, wf_tail), iterations per host check. wf_tail: with the flight and
    // camera culling the drain iterations stay cheaper than the megakernel down to ~16K
    // live paths (C5, 10-slab runs: 512K 5.94, 128K 6.03, 32K 6.13, 16K 6.15, 2K 6.14
    // Gseg/s; synchronous calls unchanged).
    int wavefront = 2;
    uint32_t wf_pool = 1u << 23;
    uint32_t wf_tail = 1u << 14;
    uint64_t wf_chunk = 1ull << 28;  // paths per render launch (radiance scratch)
    int wf_batch = 4;
    bool wf_concurrent = true;  // SST_WF_CONCURRENT=0: one stream per iteration
    bool cam_filter = true;     // SST_CAM_FILTER=0: every camera ray through the wavefront
    int convex_end = 1;         // SST_CONVEX_END=0: trace every flight the SDF/skip bounds do not cull
    // launches with fewer paths use the megakernel (the wavefront's per-iteration costs
    // dominate below ~3e5 paths: tools/small_render_crossover.py); SST_WF_MIN_PATHS
    uint64_t wf_min_paths = 327680;
    std::deque<std::unique_ptr<WfJobBase>> jobs;  // FIFO: finishes (and films) in launch order
    // per-kernel device timing (sst_gpu_kernel_timing)
    bool ktime = false;
    double kt_ms[SST_KT_COUNT] = {};
    uint64_t kt_n[SST_KT_COUNT] = {};
    cudaEvent_t kt_ev[8] = {};
    int next_slot = 0;
    cudaEvent_t ev_start = nullptr, last_film = nullptr;
    bool timing_open = false;
    int sphere_batch = 16;  // SST_SPHERE_BATCH overrides (tuning)
    int trace_batch = 0;    // SST_TRACE_BATCH overrides (tuning; 0 = traversals never wait)
};

namespace {

// Decoder weights live in per-device __constant__ memory (FFMA operands, decoder.cuh).
// Contexts on one device share it: the owner record says whose weights are resident.
// Every launch that reads the weights first calls ensure_constants() and keeps the
// returned lock until the launch is enqueued, so no other thread can swap the bank
// in between. A swap to DIFFERENT weights first waits for every launch already
// enqueued on the device (cudaDeviceSynchronize) -- some may belong to another
// context's asynchronous renders -- and a context that lost the bank re-takes it
// (same protocol) before its next launch, including the later iterations of its
// draining wavefront jobs.
std::recursive_mutex g_const_mu;
struct ConstOwner {
    const sst_gpu_ctx* ctx;
    uint64_t gen;
    uint64_t weights_fp;
};
std::map<int, ConstOwner> g_const_owner;  // device -> resident weights
uint64_t g_serial = 0;

uint64_t fnv(const void* data, size_t n, uint64_t h = 0xCBF29CE484222325ULL) {
    const auto* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) {
        h ^= p[i];
        h *= 0x100000001B3ULL;
    }
    return h;
}

void require_device(sst_gpu_ctx* ctx) {
    if (!ctx) throw InvalidArgument("null context");
    CK(cudaSetDevice(ctx->device));
}

using ConstLock = std::unique_lock<std::recursive_mutex>;

ConstLock ensure_constants(sst_gpu_ctx* ctx) {
    if (!ctx->models) throw InvalidArgument("no models uploaded (sst_gpu_upload_models / sst_gpu_load_models_dir)");
    ConstLock lk(g_const_mu);
    auto it = g_const_owner.find(ctx->device);
    if (it != g_const_owner.end()) {
        ConstOwner& o = it->second;
        if (o.ctx == ctx && o.gen == ctx->model_gen) return lk;
        if (o.weights_fp == ctx->weights_fp) {  // the same weights are resident: nothing to copy
            o = {ctx, ctx->model_gen, ctx->weights_fp};
            return lk;
        }
        CK(cudaDeviceSynchronize());  // launches that read the resident weights have finished
    }
    CK(f32::upload_constants(ctx->weights.data(), ctx->norms, ctx->stream));
    CK(f64::upload_constants(ctx->weights.data(), ctx->norms, ctx->stream));
    g_const_owner[ctx->device] = {ctx, ctx->model_gen, ctx->weights_fp};
    return lk;
}

void join_slots(sst_gpu_ctx* ctx);

void set_models(sst_gpu_ctx* ctx, const HostModel (&m)[3]) {
    join_slots(ctx);  // in-flight renders read the decoder constants
    std::vector<double> w;
    double norms[6];
    pack_models(m, w, norms);
    for (int k = 0; k < 3; ++k) {
        ctx->host_models[k] = m[k];
        ctx->have_model[k] = true;
    }
    ctx->weights = std::move(w);
    std::memcpy(ctx->norms, norms, sizeof norms);
    ctx->weights_fp = fnv(ctx->norms, sizeof ctx->norms, fnv(ctx->weights.data(), ctx->weights.size() * sizeof(double)));
    ctx->models = true;
    ctx->model_gen = ++g_serial;
}

void validate_medium(const sst_medium& m) {  // MediumParams::validate (optics.cpp:21-25)
    if (!(m.sigma_t >= 0.0)) throw DomainError("sigma_t must be >= 0");
    if (!(m.g > -1.0 && m.g < 1.0)) throw DomainError("HG anisotropy g must lie in (-1, 1)");
    if (!(m.phi >= 0.0 && m.phi <= 1.0)) throw DomainError("albedo phi must lie in [0, 1]");
}

template <class R>
MediumK<R> medium_constants(const sst_medium& m, double r_min) {
    MediumK<R> k{};
    k.sigma_t = static_cast<R>(m.sigma_t);
    k.g = static_cast<R>(m.g);
    k.phi = static_cast<R>(m.phi);
    k.log_phi = (m.phi > 0.0 && m.phi < 1.0) ? static_cast<R>(std::log(m.phi)) : R(0);
    k.one_minus_phi = static_cast<R>(1.0 - m.phi);
    k.r_min = static_cast<R>(r_min > 3e38 && !std::is_same<R, double>::value ? 3e38 : r_min);
    // u < phi with u = (x >> 11) * 2^-53  <=>  (x >> 11) < ceil(phi * 2^53)
    k.survive_below = static_cast<uint64_t>(std::ceil(m.phi * 9007199254740992.0));
    k.phi_is_one = m.phi >= 1.0;
    k.phi_is_zero = m.phi <= 0.0;
    return k;
}

double r_min_of(const sst_scene_desc& d, const ObjectHost& o, int c) {
    if (d.r_min > 0.0) return d.r_min;
    const double s = o.media[c].sigma_t;
    if (!(s > 0.0)) return 1e300;
    return std::fmax(2.0 / s, 1.5 * o.sdf_voxel);
}

// build_sdf geometry (sdf.cpp:20-38) + exact FP64 GPU evaluation.
void build_sdf_gpu(sst_gpu_ctx* ctx, const sst_object_desc& od, ObjectHost& oh, bool watertight) {
    const uint32_t res = od.sdf_resolution ? od.sdf_resolution : 64;
    if (res < 8) throw InvalidArgument("build_sdf: resolution must be >= 8");
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (uint32_t i = 0; i < od.n_vertices; ++i)
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::fmin(lo[a], od.positions[3 * i + a]);
            hi[a] = std::fmax(hi[a], od.positions[3 * i + a]);
        }
    const double ext[3] = {hi[0] - lo[0], hi[1] - lo[1], hi[2] - lo[2]};
    const double me = std::fmax(ext[0], std::fmax(ext[1], ext[2]));
    if (!(me > 0.0)) throw InvalidArgument("build_sdf: empty mesh bounds");
    SdfBuildArgs a{};
    a.voxel = me / res;
    for (int k = 0; k < 3; ++k) {
        a.origin[k] = lo[k] - a.voxel;
        a.dims[k] = static_cast<uint32_t>(std::ceil(ext[k] / a.voxel - 1e-9)) + 2;
    }
    a.half_diagonal = 0.5 * std::sqrt(3.0) * a.voxel;
    const double raw[3][3] = {{0.5380, 0.1123, 0.8354}, {-0.8312, 0.3052, 0.4643}, {0.1710, -0.9364, 0.3063}};
    for (int k = 0; k < 3; ++k) {
        const double len = std::sqrt(raw[k][0] * raw[k][0] + raw[k][1] * raw[k][1] + raw[k][2] * raw[k][2]);
        for (int j = 0; j < 3; ++j) a.dirs[3 * k + j] = raw[k][j] / len;
    }
    a.watertight = watertight ? 1 : 0;
    a.n_tris = od.n_triangles;
    std::vector<double> tv(9ull * od.n_triangles);
    for (uint32_t t = 0; t < od.n_triangles; ++t)
        for (int c = 0; c < 3; ++c)
            for (int k = 0; k < 3; ++k) tv[9ull * t + 3 * c + k] = od.positions[3ull * od.triangles[3 * t + c] + k];
    const size_t nvox = static_cast<size_t>(a.dims[0]) * a.dims[1] * a.dims[2];
    ScopedBuf dtv, dval;
    dtv.reserve(tv.size() * sizeof(double));
    dval.reserve(nvox * sizeof(float));
    CK(cudaMemcpyAsync(dtv.p, tv.data(), tv.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    a.tri_vertices = dtv.as<double>();
    a.values = dval.as<float>();
    CK(launch_sdf_build(a, ctx->stream));
    oh.sdf.resize(nvox);
    CK(cudaMemcpyAsync(oh.sdf.data(), dval.p, nvox * sizeof(float), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    dtv.release();
    dval.release();
    for (int k = 0; k < 3; ++k) {
        oh.sdf_origin[k] = a.origin[k];
        oh.dims[k] = a.dims[k];
    }
    oh.sdf_voxel = a.voxel;
}

// Triangle / axis-aligned box overlap (separating axes: the box normals, the triangle
// normal, the 9 edge cross products; Akenine-Moller), box centre c and half size e.
bool tri_box_overlap(const std::array<std::array<double, 3>, 3>& t, const double (&c)[3], double e) {
    double v[3][3];
    for (int i = 0; i < 3; ++i)
        for (int a = 0; a < 3; ++a) v[i][a] = t[i][a] - c[a];
    auto sep = [&](const double (&ax)[3]) {
        const double r = e * (std::fabs(ax[0]) + std::fabs(ax[1]) + std::fabs(ax[2]));
        double lo = 1e300, hi = -1e300;
        for (int i = 0; i < 3; ++i) {
            const double p = v[i][0] * ax[0] + v[i][1] * ax[1] + v[i][2] * ax[2];
            lo = std::fmin(lo, p);
            hi = std::fmax(hi, p);
        }
        return lo > r || hi < -r;
    };
    for (int a = 0; a < 3; ++a) {
        double ax[3] = {0, 0, 0};
        ax[a] = 1.0;
        if (sep(ax)) return false;
    }
    double ed[3][3];
    for (int i = 0; i < 3; ++i)
        for (int a = 0; a < 3; ++a) ed[i][a] = v[(i + 1) % 3][a] - v[i][a];
    const double nn[3] = {ed[0][1] * ed[1][2] - ed[0][2] * ed[1][1], ed[0][2] * ed[1][0] - ed[0][0] * ed[1][2],
                          ed[0][0] * ed[1][1] - ed[0][1] * ed[1][0]};
    if (sep(nn)) return false;
    for (int i = 0; i < 3; ++i)
        for (int a = 0; a < 3; ++a) {
            double u[3] = {0, 0, 0};
            u[a] = 1.0;
            const double ax[3] = {u[1] * ed[i][2] - u[2] * ed[i][1], u[2] * ed[i][0] - u[0] * ed[i][2],
                                  u[0] * ed[i][1] - u[1] * ed[i][0]};
            if (sep(ax)) return false;
        }
    return true;
}

// Face-plane lists of an object (integrator.cuh end_inside_planes): for every SDF
// voxel whose stored value is -0 (centre inside, within half a diagonal of the surface),
// or +0 with a corner strictly inside the (convex) object, the planes of the faces that
// meet the voxel (separating-axis test on the voxel grown by 1e-6: a superset of the
// faces crossing it is all the containment argument needs); a listed voxel no face
// meets is wholly inside and gets one always-satisfied plane. tv[first, first + n): the
// object's outward-wound triangles.
void build_plane_lists(ObjectHost& oh, const std::vector<std::array<std::array<double, 3>, 3>>& tv, size_t first,
                       size_t n) {
    oh.plane_off.clear();
    oh.planes.clear();
    const uint32_t nx = oh.dims[0], ny = oh.dims[1], nz = oh.dims[2];
    const size_t nvox = static_cast<size_t>(nx) * ny * nz;
    const double h = oh.sdf_voxel;
    // eligible voxels: centre inside (stored -0), or centre outside (+0) with a corner
    // strictly inside the object (decided below) -- either gives a point of V inside it
    std::vector<uint8_t> elig(nvox, 0);
    // (non-convex objects: centre-inside voxels only -- "inside every face plane" is the
    // inside test of a convex object alone)
    for (size_t k = 0; k < nvox; ++k)
        elig[k] = oh.sdf[k] == 0.0f ? (std::signbit(oh.sdf[k]) ? 1 : (oh.convex ? 2 : 0)) : 0;
    auto eligible = [&](size_t k) { return elig[k] != 0; };
    struct Pl {
        double n[3], d;
    };
    std::vector<Pl> pl(n);
    double scale = 0.0;
    for (size_t t = 0; t < n; ++t) {
        const auto& c = tv[first + t];
        const double e1[3] = {c[1][0] - c[0][0], c[1][1] - c[0][1], c[1][2] - c[0][2]};
        const double e2[3] = {c[2][0] - c[0][0], c[2][1] - c[0][1], c[2][2] - c[0][2]};
        double nn[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
        const double l = std::sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]);
        if (!(l > 0.0)) {  // degenerate: no area, never crossed
            pl[t] = Pl{{0, 0, 0}, 0};
            continue;
        }
        for (double& v : nn) v /= l;
        pl[t] = Pl{{nn[0], nn[1], nn[2]}, nn[0] * c[0][0] + nn[1] * c[0][1] + nn[2] * c[0][2]};
        for (int a = 0; a < 3; ++a)
            for (int k = 0; k < 3; ++k) scale = std::fmax(scale, std::fabs(c[a][k]));
    }
    // candidate (voxel, face) pairs, counted then filled (CSR)
    std::vector<uint32_t> cnt(nvox + 1, 0);
    auto for_pairs = [&](auto&& fn) {
        for (size_t t = 0; t < n; ++t) {
            const Pl& p = pl[t];
            if (p.n[0] == 0.0 && p.n[1] == 0.0 && p.n[2] == 0.0) continue;
            const auto& c = tv[first + t];
            int lo[3], hi[3];
            for (int a = 0; a < 3; ++a) {
                const double mn = std::fmin(c[0][a], std::fmin(c[1][a], c[2][a]));
                const double mx = std::fmax(c[0][a], std::fmax(c[1][a], c[2][a]));
                lo[a] = std::max(0, static_cast<int>(std::floor((mn - oh.sdf_origin[a]) / h)) - 1);
                hi[a] = std::min(static_cast<int>(oh.dims[a]) - 1, static_cast<int>(std::floor((mx - oh.sdf_origin[a]) / h)) + 1);
            }
            for (int z = lo[2]; z <= hi[2]; ++z)
                for (int y = lo[1]; y <= hi[1]; ++y)
                    for (int x = lo[0]; x <= hi[0]; ++x) {
                        const size_t k = (static_cast<size_t>(z) * ny + y) * nx + x;
                        if (!eligible(k)) continue;
                        const double cc[3] = {oh.sdf_origin[0] + (x + 0.5) * h, oh.sdf_origin[1] + (y + 0.5) * h,
                                              oh.sdf_origin[2] + (z + 0.5) * h};
                        // the triangle meets the voxel (slightly grown): separating-axis test
                        if (tri_box_overlap(c, cc, 0.5 * h * (1.0 + 1e-6) + 1e-12 * scale)) fn(k, t);
                    }
        }
    };
    {  // +0 voxels: keep those with a corner strictly inside every face plane
        for_pairs([&](size_t k, size_t) { ++cnt[k + 1]; });
        for (size_t k = 0; k < nvox; ++k) cnt[k + 1] += cnt[k];
        std::vector<uint32_t> cand(cnt[nvox]), fill(cnt.begin(), cnt.end() - 1);
        for_pairs([&](size_t k, size_t t) { cand[fill[k]++] = static_cast<uint32_t>(t); });
        const double m = 1e-9 * std::fmax(scale, 1.0);
        auto inside = [&](const double* q, const uint32_t* b, const uint32_t* e) {
            for (const uint32_t* t = b; t != e; ++t) {
                const Pl& p = pl[*t];
                if (!(p.n[0] * q[0] + p.n[1] * q[1] + p.n[2] * q[2] - p.d < -m)) return false;
            }
            return true;
        };
        std::vector<uint32_t> all;
        for (size_t t = 0; t < n; ++t)
            if (pl[t].n[0] != 0.0 || pl[t].n[1] != 0.0 || pl[t].n[2] != 0.0) all.push_back(static_cast<uint32_t>(t));
        for (uint32_t z = 0; z < nz; ++z)
            for (uint32_t y = 0; y < ny; ++y)
                for (uint32_t x = 0; x < nx; ++x) {
                    const size_t k = (static_cast<size_t>(z) * ny + y) * nx + x;
                    if (elig[k] != 2) continue;
                    bool ok = false;
                    for (int c = 0; c < 8 && !ok; ++c) {
                        const double q[3] = {oh.sdf_origin[0] + (x + (c & 1)) * h, oh.sdf_origin[1] + (y + ((c >> 1) & 1)) * h,
                                             oh.sdf_origin[2] + (z + ((c >> 2) & 1)) * h};
                        // nearby planes first (cheap rejection), then every face plane
                        ok = inside(q, cand.data() + cnt[k], cand.data() + cnt[k + 1]) &&
                             inside(q, all.data(), all.data() + all.size());
                    }
                    elig[k] = ok ? 1 : 0;
                }
        std::fill(cnt.begin(), cnt.end(), 0u);
    }
    for_pairs([&](size_t k, size_t) { ++cnt[k + 1]; });
    // an eligible voxel that no face meets lies wholly inside (it holds an interior point
    // and the surface does not enter it): one always-satisfied plane (0, 0, 0, 1)
    std::vector<uint8_t> inner(nvox, 0);
    for (size_t k = 0; k < nvox; ++k)
        if (elig[k] && cnt[k + 1] == 0) inner[k] = 1, cnt[k + 1] = 1;
    for (size_t k = 0; k < nvox; ++k) cnt[k + 1] += cnt[k];
    oh.plane_off = cnt;
    oh.planes.resize(4 * static_cast<size_t>(cnt[nvox]));
    std::vector<uint32_t> fill(cnt.begin(), cnt.end() - 1);
    for_pairs([&](size_t k, size_t t) {
        float* q = oh.planes.data() + 4 * static_cast<size_t>(fill[k]++);
        for (int a = 0; a < 3; ++a) q[a] = static_cast<float>(pl[t].n[a]);
        q[3] = static_cast<float>(pl[t].d);
    });
    for (size_t k = 0; k < nvox; ++k)
        if (inner[k]) {
            float* q = oh.planes.data() + 4 * static_cast<size_t>(fill[k]++);
            q[0] = q[1] = q[2] = 0.0f;
            q[3] = 1.0f;
        }
    // margin: far above the FP32 error of n.e - d at this coordinate scale (~1e-7 x scale)
    oh.plane_eps = static_cast<float>(1e-4 * h + 4e-6 * std::fmax(scale, 1.0));
}

// Fine skip grid of one object (2x the SDF resolution over the SDF's box).
void build_skip_gpu(sst_gpu_ctx* ctx, const sst_object_desc& od, ObjectHost& oh) {
    SkipBuildArgs a{};
    a.voxel = 0.5 * oh.sdf_voxel;
    a.half_diagonal = 0.5 * std::sqrt(3.0) * a.voxel;
    a.unit = a.voxel / 8.0;
    for (int k = 0; k < 3; ++k) {
        a.origin[k] = oh.sdf_origin[k];
        a.dims[k] = 2 * oh.dims[k];
    }
    a.n_tris = od.n_triangles;
    std::vector<double> tv(9ull * od.n_triangles);
    for (uint32_t t = 0; t < od.n_triangles; ++t)
        for (int c = 0; c < 3; ++c)
            for (int k = 0; k < 3; ++k) tv[9ull * t + 3 * c + k] = od.positions[3ull * od.triangles[3 * t + c] + k];
    const size_t nvox = static_cast<size_t>(a.dims[0]) * a.dims[1] * a.dims[2];
    ScopedBuf dtv, dval;
    dtv.reserve(tv.size() * sizeof(double));
    dval.reserve(nvox);
    CK(cudaMemcpyAsync(dtv.p, tv.data(), tv.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    a.tri_vertices = dtv.as<double>();
    a.values = dval.as<uint8_t>();
    CK(launch_skip_build(a, ctx->stream));
    oh.skip.resize(nvox);
    CK(cudaMemcpyAsync(oh.skip.data(), dval.p, nvox, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    oh.skip_voxel = a.voxel;
    oh.skip_unit = a.unit;
    for (int k = 0; k < 3; ++k) oh.skip_dims[k] = a.dims[k];
}

constexpr uint32_t kCamTile = 8;  // camera tile size in pixels (build_camera_tiles)

template <class R>
void fill_devscene(sst_gpu_ctx* ctx, DevScene<R>& sc, const DevBuf& nodes, const DevBuf& tris, DevBuf& objs) {
    const sst_scene_desc& d = ctx->desc;
    std::vector<ObjK<R>> ok(ctx->objects.size());
    for (size_t o = 0; o < ctx->objects.size(); ++o) {
        const ObjectHost& oh = ctx->objects[o];
        for (int c = 0; c < 3; ++c) ok[o].med[c] = medium_constants<R>(oh.media[c], r_min_of(d, oh, c));
        for (int a = 0; a < 3; ++a) {
            ok[o].sdf_origin[a] = static_cast<R>(oh.sdf_origin[a]);
            ok[o].dims[a] = oh.dims[a];
        }
        ok[o].sdf_voxel = static_cast<R>(oh.sdf_voxel);
        ok[o].sdf_inv_voxel = static_cast<R>(1.0 / oh.sdf_voxel);
        ok[o].sdf = ctx->sdf_dev[o].as<float>();
        const char* no_skip = std::getenv("SST_NO_SKIP_GRID");
        const bool use_skip = !oh.skip.empty() && !(no_skip && no_skip[0] == '1');
        ok[o].skip = use_skip ? ctx->skip_dev[o].as<uint8_t>() : nullptr;
        ok[o].skip_inv_voxel = static_cast<R>(oh.skip_voxel > 0 ? 1.0 / oh.skip_voxel : 0.0);
        ok[o].skip_unit = static_cast<R>(oh.skip_unit);
        for (int a = 0; a < 3; ++a) ok[o].skip_dims[a] = oh.skip_dims[a];
        ok[o].convex = oh.convex ? 1u : 0u;
        {  // density rank (camera pre-pass ordering)
            auto dens = [](const ObjectHost& q) {
                return std::fmax(q.media[0].sigma_t, std::fmax(q.media[1].sigma_t, q.media[2].sigma_t));
            };
            uint32_t rank = 0;
            for (const ObjectHost& q : ctx->objects) rank += dens(q) > dens(oh);
            ok[o].cost_class = std::min<uint32_t>(rank, 3u);
        }
        {  // bounding sphere, radius grown past the FP error of ray_may_hit (|centre - origin|^2
           // * 1e-7 for an origin at the camera or anywhere within the objects' span)
            double span2 = 0.0;
            for (const ObjectHost& q : ctx->objects) {
                double dc2 = 0.0, dq2 = 0.0;
                for (int k = 0; k < 3; ++k) {
                    dc2 += (oh.bsphere[k] - d.cam_position[k]) * (oh.bsphere[k] - d.cam_position[k]);
                    dq2 += (oh.bsphere[k] - q.bsphere[k]) * (oh.bsphere[k] - q.bsphere[k]);
                }
                const double dq = std::sqrt(dq2) + q.bsphere[3] + oh.bsphere[3];
                span2 = std::fmax(span2, std::fmax(dc2, dq * dq));
            }
            const double r = oh.bsphere[3];
            for (int k = 0; k < 3; ++k) ok[o].bsphere[k] = static_cast<R>(oh.bsphere[k]);
            ok[o].bsphere[3] = static_cast<R>(r * (1.0 + 1e-3) + 1e-5 * span2 / std::fmax(r, 1e-3) + 1e-5);
        }
        {
            const char* e = std::getenv("SST_NO_PLANES");
            const bool use = std::is_same<R, float>::value && !oh.plane_off.empty() && !(e && e[0] == '1');
            ok[o].plane_off = use ? ctx->plane_off_dev[o].as<uint32_t>() : nullptr;
            ok[o].planes = use ? ctx->planes_dev[o].as<float4>() : nullptr;
            ok[o].plane_eps = oh.plane_eps;
        }
        {
            const auto& roots = ctx->scene_cache.bvh.obj_root;
            const char* e = std::getenv("SST_OBJ_ROOT");
            const bool use = std::is_same<R, float>::value && !(e && e[0] == '0');
            ok[o].bvh_root = use && o < roots.size() && roots[o] >= 0 ? roots[o] : 0;
        }
    }
    objs.reserve(ok.size() * sizeof(ObjK<R>));
    CK(cudaMemcpyAsync(objs.p, ok.data(), ok.size() * sizeof(ObjK<R>), cudaMemcpyHostToDevice, ctx->stream));
    sc.nodes = nodes.p;
    sc.tris = tris.p;
    sc.bvh_depth = ctx->scene_cache.bvh.max_depth;
    sc.objs = objs.as<ObjK<R>>();
    sc.n_objects = static_cast<uint32_t>(ok.size());
    // Camera basis in double (DESIGN.md camera model), then rounded.
    auto v = [](const double* p) { return std::array<double, 3>{p[0], p[1], p[2]}; };
    auto sub = [](std::array<double, 3> a, std::array<double, 3> b) {
        return std::array<double, 3>{a[0] - b[0], a[1] - b[1], a[2] - b[2]};
    };
    auto cross = [](std::array<double, 3> a, std::array<double, 3> b) {
        return std::array<double, 3>{a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    };
    auto norm = [](std::array<double, 3> a) {
        const double l = std::sqrt(a[0] * a[0] + a[1] * a[1] + a[2] * a[2]);
        return std::array<double, 3>{a[0] / l, a[1] / l, a[2] / l};
    };
    const auto fwd = norm(sub(v(d.cam_look_at), v(d.cam_position)));
    const auto right = norm(cross(fwd, v(d.cam_up)));
    const auto up = cross(right, fwd);
    auto tor = [](std::array<double, 3> a) { return mk<R>(R(a[0]), R(a[1]), R(a[2])); };
    sc.cam_pos = tor(v(d.cam_position));
    sc.cam_fwd = tor(fwd);
    sc.cam_right = tor(right);
    sc.cam_up = tor(up);
    sc.tan_half = static_cast<R>(std::tan(d.cam_vfov_deg * 3.14159265358979323846 / 360.0));
    sc.aspect = static_cast<R>(static_cast<double>(d.width) / static_cast<double>(d.height));
    sc.width = d.width;
    sc.height = d.height;
    sc.light = tor(v(d.light_position));
    sc.directional = d.light_kind == 1;
    {
        const double* ld = d.light_direction;
        const double n = std::sqrt(ld[0] * ld[0] + ld[1] * ld[1] + ld[2] * ld[2]);
        sc.light_dir = sc.directional ? mk<R>(R(ld[0] / n), R(ld[1] / n), R(ld[2] / n)) : mk<R>(R(0), R(0), R(1));
    }
    for (int c = 0; c < 3; ++c) {
        sc.power[c] = static_cast<R>(d.light_power[c]);
        sc.bg[c] = static_cast<R>(d.background[c]);
    }
    // Surface self-intersection guard for FP32 (relative to the scene extent).
    double ext = 1.0;
    for (const auto& oh : ctx->objects)
        for (int a = 0; a < 3; ++a) ext = std::fmax(ext, std::fabs(oh.sdf_origin[a]) + oh.dims[a] * oh.sdf_voxel);
    sc.t_min = static_cast<R>(1e-9);
    sc.surf_eps = std::is_same<R, double>::value ? static_cast<R>(1e-9) : static_cast<R>(2e-6 * ext);
    sc.cap_pt = d.max_pt_events ? d.max_pt_events : 1000000u;
    sc.cap_st = d.max_st_steps ? d.max_st_steps : 100000u;
    const char* no_grid = std::getenv("SST_NO_LIGHT_GRID");
    const bool use_grid = ctx->grid_res && !sc.directional && !(no_grid && no_grid[0] == '1');
    sc.grid_off = use_grid ? ctx->grid_off.as<uint32_t>() : nullptr;
    sc.grid_tri = use_grid ? ctx->grid_tri.as<uint32_t>() : nullptr;
    sc.grid_tris = use_grid && std::is_same<R, float>::value ? ctx->grid_tris32.p : nullptr;
    {
        const char* e = std::getenv("SST_NO_CAM_TILES");
        const bool use = std::is_same<R, float>::value && ctx->cam_off.p && !(e && e[0] == '1');
        sc.cam_off = use ? ctx->cam_off.as<uint32_t>() : nullptr;
        sc.cam_tris = use ? ctx->cam_tris32.p : nullptr;
        sc.cam_tile = kCamTile;
        sc.cam_tiles_x = ctx->cam_tiles_x;
        sc.cam_tiles_y = ctx->cam_tiles_y;
    }
    {
        const char* e = std::getenv("SST_NO_GRID_SPLIT");
        sc.grid_split = use_grid && std::is_same<R, float>::value && !(e && e[0] == '1') ? ctx->grid_split.as<uint32_t>()
                                                                                          : nullptr;
    }
    sc.grid_res = ctx->grid_res;
}

// Light-space culling grid for NEE shadow rays (see types.cuh DevScene::grid_*).
// Per triangle: the cone from the light that contains it (axis = mean vertex
// direction, half angle = max vertex angle + padding); cells overlap-tested on the
// GPU in FP64 (count pass, host prefix sum, fill pass).
void build_camera_tile_lists(const sst_scene_desc* d, const std::vector<std::array<std::array<double, 3>, 3>>& tv,
                             const FlatBvh& bvh, std::vector<uint32_t>& off, std::vector<uint32_t>& idx,
                             uint32_t& tiles_x, uint32_t& tiles_y);

// Camera tiles (types.cuh DevScene::cam_off): per kCamTile x kCamTile pixel tile, the
// leaf-order triangles that face the camera (a camera ray can only enter them: FP32 outside
// rays accept entering crossings only) whose projected bounding box, grown by one pixel,
// meets the tile. A triangle reaching behind the camera goes into every tile.
void build_camera_tiles(sst_gpu_ctx* ctx, const sst_scene_desc* d,
                        const std::vector<std::array<std::array<double, 3>, 3>>& tv, const FlatBvh& bvh) {
    auto& cache = ctx->scene_cache;
    uint64_t fp = fnv(d->cam_position, sizeof d->cam_position, cache.geo_fp);
    fp = fnv(d->cam_look_at, sizeof d->cam_look_at, fp);
    fp = fnv(d->cam_up, sizeof d->cam_up, fp);
    fp = fnv(&d->cam_vfov_deg, sizeof d->cam_vfov_deg, fp);
    fp = fnv(&d->width, sizeof d->width, fp);
    fp = fnv(&d->height, sizeof d->height, fp);
    if (cache.cam_fp != fp || cache.cam_off.empty()) {
        cache.cam_fp = 0;
        build_camera_tile_lists(d, tv, bvh, cache.cam_off, cache.cam_idx, cache.cam_tiles_x, cache.cam_tiles_y);
        cache.cam_fp = fp;
    }
    const auto& off = cache.cam_off;
    const auto& idx = cache.cam_idx;
    ctx->cam_off.reserve(off.size() * sizeof(uint32_t));
    ctx->cam_idx.reserve(std::max<size_t>(idx.size(), 1) * sizeof(uint32_t));
    ctx->cam_tris32.reserve(std::max<size_t>(idx.size(), 1) * sizeof(TriF));
    CK(cudaMemcpyAsync(ctx->cam_off.p, off.data(), off.size() * sizeof(uint32_t), cudaMemcpyHostToDevice, ctx->stream));
    if (!idx.empty())
        CK(cudaMemcpyAsync(ctx->cam_idx.p, idx.data(), idx.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           ctx->stream));
    ctx->cam_tiles_x = cache.cam_tiles_x;
    ctx->cam_tiles_y = cache.cam_tiles_y;
    ctx->cam_list_n = idx.size();
}

void build_camera_tile_lists(const sst_scene_desc* d, const std::vector<std::array<std::array<double, 3>, 3>>& tv,
                             const FlatBvh& bvh, std::vector<uint32_t>& off, std::vector<uint32_t>& idx,
                             uint32_t& tiles_x, uint32_t& tiles_y) {
    auto sub = [](const double* a, const double* b) { return std::array<double, 3>{a[0] - b[0], a[1] - b[1], a[2] - b[2]}; };
    auto cross = [](std::array<double, 3> a, std::array<double, 3> b) {
        return std::array<double, 3>{a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    };
    auto dot = [](std::array<double, 3> a, std::array<double, 3> b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; };
    auto norm = [&](std::array<double, 3> a) {
        const double l = std::sqrt(dot(a, a));
        return std::array<double, 3>{a[0] / l, a[1] / l, a[2] / l};
    };
    const auto fwd = norm(sub(d->cam_look_at, d->cam_position));
    const auto right = norm(cross(fwd, std::array<double, 3>{d->cam_up[0], d->cam_up[1], d->cam_up[2]}));
    const auto up = cross(right, fwd);
    const double tan_half = std::tan(d->cam_vfov_deg * 3.14159265358979323846 / 360.0);
    const double aspect = static_cast<double>(d->width) / static_cast<double>(d->height);
    const uint32_t nx = (d->width + kCamTile - 1) / kCamTile, ny = (d->height + kCamTile - 1) / kCamTile;
    const uint32_t n = bvh.n_tris;
    std::vector<std::vector<uint32_t>> tiles(static_cast<size_t>(nx) * ny);
    for (uint32_t k = 0; k < n; ++k) {
        const auto& t = tv[bvh.order[k]];
        std::array<double, 3> c[3];
        for (int i = 0; i < 3; ++i) c[i] = {t[i][0], t[i][1], t[i][2]};
        const auto nn = cross(std::array<double, 3>{c[1][0] - c[0][0], c[1][1] - c[0][1], c[1][2] - c[0][2]},
                              std::array<double, 3>{c[2][0] - c[0][0], c[2][1] - c[0][1], c[2][2] - c[0][2]});
        const auto to_cam = sub(d->cam_position, c[0].data());
        const double f = dot(nn, to_cam);
        if (f < -1e-9 * std::sqrt(dot(nn, nn) * dot(to_cam, to_cam))) continue;  // clearly faces away
        double x0 = 1e300, x1 = -1e300, y0 = 1e300, y1 = -1e300;
        bool behind = false;
        for (int i = 0; i < 3; ++i) {
            const auto q = sub(c[i].data(), d->cam_position);
            const double z = dot(q, fwd);
            if (!(z > 1e-9)) {
                behind = true;
                break;
            }
            const double px = (dot(q, right) / z / (tan_half * aspect) + 1.0) * 0.5 * d->width;
            const double py = (1.0 - dot(q, up) / z / tan_half) * 0.5 * d->height;
            x0 = std::fmin(x0, px), x1 = std::fmax(x1, px), y0 = std::fmin(y0, py), y1 = std::fmax(y1, py);
        }
        int tx0 = 0, tx1 = static_cast<int>(nx) - 1, ty0 = 0, ty1 = static_cast<int>(ny) - 1;
        if (!behind) {
            tx0 = std::max(tx0, static_cast<int>(std::floor((x0 - 1.0) / kCamTile)));
            tx1 = std::min(tx1, static_cast<int>(std::floor((x1 + 1.0) / kCamTile)));
            ty0 = std::max(ty0, static_cast<int>(std::floor((y0 - 1.0) / kCamTile)));
            ty1 = std::min(ty1, static_cast<int>(std::floor((y1 + 1.0) / kCamTile)));
        }
        for (int y = ty0; y <= ty1; ++y)
            for (int x = tx0; x <= tx1; ++x) tiles[static_cast<size_t>(y) * nx + x].push_back(k);
    }
    off.assign(tiles.size() + 1, 0);
    idx.clear();
    for (size_t i = 0; i < tiles.size(); ++i) {
        off[i] = static_cast<uint32_t>(idx.size());
        idx.insert(idx.end(), tiles[i].begin(), tiles[i].end());
    }
    off[tiles.size()] = static_cast<uint32_t>(idx.size());
    tiles_x = nx;
    tiles_y = ny;
}

void build_light_grid(sst_gpu_ctx* ctx, const sst_scene_desc* d,
                      const std::vector<std::array<std::array<double, 3>, 3>>& tv, const std::vector<uint32_t>& tobj,
                      const FlatBvh& bvh) {
    const uint32_t n = bvh.n_tris;
    uint32_t res = n <= 4096 ? 256u : 512u;
    if (const char* e = std::getenv("SST_LIGHT_GRID_RES")) res = static_cast<uint32_t>(std::max(8, std::atoi(e)));
    const double pad = 2e-5;
    std::vector<double> caps(static_cast<size_t>(kCapStride) * n);
    for (uint32_t k = 0; k < n; ++k) {
        const auto& t = tv[bvh.order[k]];
        double dir[3][3], ax[3] = {0, 0, 0};
        for (int c = 0; c < 3; ++c) {
            double v[3], l = 0;
            for (int a = 0; a < 3; ++a) {
                v[a] = t[c][a] - d->light_position[a];
                l += v[a] * v[a];
            }
            l = std::sqrt(l);
            for (int a = 0; a < 3; ++a) {
                dir[c][a] = l > 0 ? v[a] / l : 0.0;
                ax[a] += dir[c][a];
            }
        }
        const double al = std::sqrt(ax[0] * ax[0] + ax[1] * ax[1] + ax[2] * ax[2]);
        double alpha = 3.14159265358979323846;
        if (al > 1e-6) {
            for (int a = 0; a < 3; ++a) ax[a] /= al;
            double mind = 1.0;
            for (int c = 0; c < 3; ++c)
                mind = std::fmin(mind, ax[0] * dir[c][0] + ax[1] * dir[c][1] + ax[2] * dir[c][2]);
            alpha = std::acos(std::fmax(-1.0, std::fmin(1.0, mind))) + pad;
            // a cap contains the geodesic triangle only below a hemisphere
            if (alpha > 1.5) alpha = 3.14159265358979323846;
        }
        double* q = caps.data() + static_cast<size_t>(kCapStride) * k;
        q[0] = ax[0];
        q[1] = ax[1];
        q[2] = ax[2];
        q[3] = alpha;
        q[4] = std::cos(alpha);
        q[5] = std::sin(alpha);
        for (int c = 0; c < 3; ++c)
            for (int a = 0; a < 3; ++a) q[6 + 3 * c + a] = dir[c][a];
    }
    const uint32_t ncell = 6u * res * res;
    ScopedBuf dcaps, dcounts;
    dcaps.reserve(caps.size() * sizeof(double));
    dcounts.reserve(ncell * sizeof(uint32_t));
    CK(cudaMemcpyAsync(dcaps.p, caps.data(), caps.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    LightGridArgs a{};
    a.caps = dcaps.as<double>();
    a.n_tris = n;
    a.res = res;
    a.eps = pad;
    a.counts = dcounts.as<uint32_t>();
    a.fill = 0;
    CK(launch_light_grid(a, ctx->stream));
    std::vector<uint32_t> counts(ncell), offsets(ncell + 1);
    CK(cudaMemcpyAsync(counts.data(), dcounts.p, ncell * sizeof(uint32_t), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    uint64_t total = 0;
    for (uint32_t c = 0; c < ncell; ++c) {
        offsets[c] = static_cast<uint32_t>(total);
        total += counts[c];
    }
    offsets[ncell] = static_cast<uint32_t>(total);
    if (total >= (1ull << 31)) throw InvalidArgument("light grid too large");
    ctx->grid_off.reserve(offsets.size() * sizeof(uint32_t));
    ctx->grid_tri.reserve(std::max<uint64_t>(total, 1) * sizeof(uint32_t));
    CK(cudaMemcpyAsync(ctx->grid_off.p, offsets.data(), offsets.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                       ctx->stream));
    a.fill = 1;
    a.offsets = ctx->grid_off.as<uint32_t>();
    a.lists = ctx->grid_tri.as<uint32_t>();
    CK(launch_light_grid(a, ctx->stream));
    ctx->scene_cache.grid_off = offsets;
    ctx->scene_cache.grid_tri.resize(total);
    if (total) CK(cudaMemcpyAsync(ctx->scene_cache.grid_tri.data(), ctx->grid_tri.p, total * sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    {
        // Each cell's list: faces whose normal points toward the light first (list order
        // kept), then the faces pointing away, grouped by object (stable). grid_split =
        // front count | (the one object owning every back face, else 0xff) << 24.
        std::vector<int8_t> back(n, 0);
        for (uint32_t k = 0; k < n; ++k) {
            const auto& t = tv[bvh.order[k]];
            double e1[3], e2[3], to_l[3];
            for (int a = 0; a < 3; ++a) {
                e1[a] = t[1][a] - t[0][a];
                e2[a] = t[2][a] - t[0][a];
                to_l[a] = d->light_position[a] - t[0][a];
            }
            const double nn[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                                  e1[0] * e2[1] - e1[1] * e2[0]};
            const double f = nn[0] * to_l[0] + nn[1] * to_l[1] + nn[2] * to_l[2];
            const double scale = std::sqrt(nn[0] * nn[0] + nn[1] * nn[1] + nn[2] * nn[2]) *
                                 std::sqrt(to_l[0] * to_l[0] + to_l[1] * to_l[1] + to_l[2] * to_l[2]);
            back[k] = f < -1e-9 * scale ? 1 : 0;  // clearly facing away (the light is behind its plane)
        }
        auto& lst = ctx->scene_cache.grid_tri;
        std::vector<uint32_t> split(ncell, 0xffu << 24), tmp, bk;
        for (uint32_t c = 0; c < ncell; ++c) {
            const uint32_t b = offsets[c], e = offsets[c + 1];
            tmp.clear();
            bk.clear();
            for (uint32_t k = b; k < e; ++k)
                if (!back[lst[k]]) tmp.push_back(lst[k]);
            const uint32_t nf = static_cast<uint32_t>(tmp.size());
            for (uint32_t k = b; k < e; ++k)
                if (back[lst[k]]) bk.push_back(lst[k]);
            std::stable_sort(bk.begin(), bk.end(), [&](uint32_t x, uint32_t y) {
                return tobj[bvh.order[x]] < tobj[bvh.order[y]];
            });
            uint32_t owner = 0xffu;
            if (!bk.empty() && tobj[bvh.order[bk.front()]] == tobj[bvh.order[bk.back()]] &&
                tobj[bvh.order[bk.front()]] < 0xffu)
                owner = tobj[bvh.order[bk.front()]];
            tmp.insert(tmp.end(), bk.begin(), bk.end());
            std::copy(tmp.begin(), tmp.end(), lst.begin() + b);
            split[c] = (nf < (1u << 24) ? nf : 0xffffffu) | (nf < (1u << 24) ? owner << 24 : 0xffu << 24);
        }
        if (total) CK(cudaMemcpyAsync(ctx->grid_tri.p, lst.data(), total * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                      ctx->stream));
        ctx->scene_cache.grid_split = split;
        ctx->grid_split.reserve(split.size() * sizeof(uint32_t));
        CK(cudaMemcpyAsync(ctx->grid_split.p, split.data(), split.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    ctx->scene_cache.grid_res = res;
    ctx->grid_res = res;
    ctx->scene_bytes_grid = (offsets.size() + total + ncell) * sizeof(uint32_t);  // offsets, lists, split
    ctx->grid_list_n = total;
}

void ensure_film_staging(sst_gpu_ctx* ctx, uint64_t n);

template <class Lap>
void upload_scene_body(sst_gpu_ctx* ctx, const sst_scene_desc* d, bool directional, Lap& lap);

void upload_scene(sst_gpu_ctx* ctx, const sst_scene_desc* d) {
    const bool tdbg = std::getenv("SST_DEBUG_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t_start = now();
    auto lap = [&](const char* what) {
        if (tdbg)
            std::fprintf(stderr, "[upload_scene] %-14s %8.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(now() - t_start).count());
    };
    if (!d || d->n_objects == 0 || !d->objects) throw InvalidArgument("scene has no objects");
    if (d->width == 0 || d->height == 0) throw InvalidArgument("camera resolution must be >= 1x1");
    if (!(d->cam_vfov_deg > 0.0 && d->cam_vfov_deg < 180.0)) throw InvalidArgument("camera fov out of range");
    if (d->light_kind > 1) throw InvalidArgument("light_kind must be 0 (point) or 1 (directional)");
    const bool directional = d->light_kind == 1;
    if (directional && !(d->light_direction[0] * d->light_direction[0] + d->light_direction[1] * d->light_direction[1] +
                             d->light_direction[2] * d->light_direction[2] > 0.0))
        throw InvalidArgument("directional light needs a non-zero light_direction");
    // From here on the previous scene's host objects may be moved into this upload;
    // a failure past this point leaves NO scene (never a half-moved one).
    try {
        upload_scene_body(ctx, d, directional, lap);
    } catch (...) {
        ctx->scene = false;
        ctx->objects.clear();
        ctx->object_fp.clear();
        throw;
    }
}

template <class Lap>
void upload_scene_body(sst_gpu_ctx* ctx, const sst_scene_desc* d, bool directional, Lap& lap) {
    std::vector<ObjectHost> objs(d->n_objects);
    std::vector<uint64_t> objs_fp(d->n_objects, 0);
    std::vector<uint64_t> prev_fp;
    prev_fp.swap(ctx->object_fp);  // a failed upload leaves no reusable objects behind
    std::vector<std::array<std::array<double, 3>, 3>> tv;
    std::vector<uint32_t> tobj;
    for (uint32_t o = 0; o < d->n_objects; ++o) {
        const sst_object_desc& od = d->objects[o];
        if (!od.positions || !od.triangles || od.n_triangles == 0) throw InvalidArgument("object has no geometry");
        for (int c = 0; c < 3; ++c) {
            validate_medium(od.media[c]);
            objs[o].media[c] = od.media[c];
        }
        std::vector<std::array<uint32_t, 3>> tri(od.n_triangles);
        for (uint32_t t = 0; t < od.n_triangles; ++t)
            for (int c = 0; c < 3; ++c) {
                const uint32_t vi = od.triangles[3 * t + c];
                if (vi >= od.n_vertices) throw InvalidArgument("triangle index out of range");
                tri[t][c] = vi;
            }
        // Orientation: the order-free optical depth needs outward winding; flip an
        // inward-wound (negative signed volume) mesh.
        double vol = 0.0;
        for (const auto& t : tri) {
            const double* a = od.positions + 3 * t[0];
            const double* b = od.positions + 3 * t[1];
            const double* c = od.positions + 3 * t[2];
            vol += a[0] * (b[1] * c[2] - b[2] * c[1]) - a[1] * (b[0] * c[2] - b[2] * c[0]) +
                   a[2] * (b[0] * c[1] - b[1] * c[0]);
        }
        const bool flip = vol < 0.0;
        for (const auto& t : tri) {
            std::array<std::array<double, 3>, 3> corners;
            for (int c = 0; c < 3; ++c)
                for (int k = 0; k < 3; ++k) corners[c][k] = od.positions[3 * t[c] + k];
            if (flip) std::swap(corners[1], corners[2]);
            tv.push_back(corners);
            tobj.push_back(o);
        }
        uint64_t ofp = fnv(od.positions, 3ull * od.n_vertices * sizeof(double));
        ofp = fnv(od.triangles, 3ull * od.n_triangles * sizeof(uint32_t), ofp);
        ofp = fnv(&od.sdf_resolution, sizeof od.sdf_resolution, ofp);
        if (od.sdf_values) {
            ofp = fnv(od.sdf_origin, sizeof od.sdf_origin, ofp);
            ofp = fnv(&od.sdf_voxel, sizeof od.sdf_voxel, ofp);
            ofp = fnv(od.sdf_dims, sizeof od.sdf_dims, ofp);
            ofp = fnv(od.sdf_values, static_cast<size_t>(od.sdf_dims[0]) * od.sdf_dims[1] * od.sdf_dims[2] * sizeof(float), ofp);
        }
        objs_fp[o] = ofp;
        if (o < ctx->objects.size() && o < prev_fp.size() && prev_fp[o] == ofp) {
            // the same object as the previous upload: take its host copy over (no 3 MB copy)
            const sst_medium media[3] = {objs[o].media[0], objs[o].media[1], objs[o].media[2]};
            objs[o] = std::move(ctx->objects[o]);
            for (int c = 0; c < 3; ++c) objs[o].media[c] = media[c];
            continue;
        }
        if (auto it = ctx->obj_cache.find(ofp); it != ctx->obj_cache.end()) {
            const sst_medium media[3] = {objs[o].media[0], objs[o].media[1], objs[o].media[2]};
            objs[o] = it->second;
            for (int c = 0; c < 3; ++c) objs[o].media[c] = media[c];
            continue;
        }
        if (od.sdf_values) {
            if (!(od.sdf_voxel > 0.0) || !od.sdf_dims[0] || !od.sdf_dims[1] || !od.sdf_dims[2])
                throw InvalidArgument("SDF grid has empty dims or voxel size");
            const size_t n = static_cast<size_t>(od.sdf_dims[0]) * od.sdf_dims[1] * od.sdf_dims[2];
            objs[o].sdf.assign(od.sdf_values, od.sdf_values + n);
            for (int a = 0; a < 3; ++a) {
                objs[o].sdf_origin[a] = od.sdf_origin[a];
                objs[o].dims[a] = od.sdf_dims[a];
            }
            objs[o].sdf_voxel = od.sdf_voxel;
        } else {
            build_sdf_gpu(ctx, od, objs[o], is_watertight(tri));
        }
        objs[o].convex = is_convex(od.positions, od.n_vertices, tri);
        // the fine skip grid only pays for non-convex objects: a convex object's face-plane
        // lists decide the flights it would cull exactly (C5: 8.04 -> 8.33 Gseg/s without
        // it; C3 bumpy sphere sigma_t = 160: 4.27 vs 4.44 ms/spp with it)
        if (!objs[o].convex) build_skip_gpu(ctx, od, objs[o]);
        build_plane_lists(objs[o], tv, tv.size() - od.n_triangles, od.n_triangles);
        {  // bounding sphere: box centre, farthest referenced vertex
            double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
            for (const auto& t : tri)
                for (uint32_t vi : t)
                    for (int k = 0; k < 3; ++k) {
                        lo[k] = std::fmin(lo[k], od.positions[3 * vi + k]);
                        hi[k] = std::fmax(hi[k], od.positions[3 * vi + k]);
                    }
            double r2 = 0.0;
            for (int k = 0; k < 3; ++k) objs[o].bsphere[k] = 0.5 * (lo[k] + hi[k]);
            for (const auto& t : tri)
                for (uint32_t vi : t) {
                    double d2 = 0.0;
                    for (int k = 0; k < 3; ++k) {
                        const double dk = od.positions[3 * vi + k] - objs[o].bsphere[k];
                        d2 += dk * dk;
                    }
                    r2 = std::fmax(r2, d2);
                }
            objs[o].bsphere[3] = std::sqrt(r2);
        }
        if (ctx->obj_cache.size() >= 64) ctx->obj_cache.clear();
        ctx->obj_cache[ofp] = objs[o];
    }
    lap("objects");
    uint64_t gfp = fnv(tv.data(), tv.size() * sizeof(tv[0]));
    gfp = fnv(tobj.data(), tobj.size() * sizeof(uint32_t), gfp);
    const uint64_t lfp = fnv(d->light_position, sizeof d->light_position, gfp);
    auto& cache = ctx->scene_cache;
    const bool bvh_cached = cache.have_bvh && cache.geo_fp == gfp;
    if (!bvh_cached) {
        cache = sst_gpu_ctx::SceneCache{};
        FlatBvh b = build_bvh(tv, tobj);
        if (b.max_depth + 1 > static_cast<uint32_t>(kStack))
            throw InvalidArgument("BVH deeper than the traversal stack (" + std::to_string(kStack) + ")");
        cache.bvh = std::move(b);
        cache.geo_fp = gfp;
        cache.have_bvh = true;
    }
    const bool cached = !directional && cache.grid_fp == lfp && cache.grid_res;
    if (directional) {  // no light-space grid (it is a cube map around a point light)
        ctx->grid_res = 0;
        ctx->scene_bytes_grid = 0;
        ctx->grid_list_n = 0;
    } else if (!cached) {
        cache.grid_fp = 0;
        build_light_grid(ctx, d, tv, tobj, cache.bvh);
        cache.grid_fp = lfp;
    } else {  // copy the cached light grid to the device (inputs travel every upload)
        const auto& sc = ctx->scene_cache;
        ctx->grid_off.reserve(sc.grid_off.size() * sizeof(uint32_t));
        ctx->grid_tri.reserve(std::max<size_t>(sc.grid_tri.size(), 1) * sizeof(uint32_t));
        CK(cudaMemcpyAsync(ctx->grid_off.p, sc.grid_off.data(), sc.grid_off.size() * sizeof(uint32_t),
                           cudaMemcpyHostToDevice, ctx->stream));
        ctx->grid_split.reserve(std::max<size_t>(sc.grid_split.size(), 1) * sizeof(uint32_t));
        if (!sc.grid_split.empty())
            CK(cudaMemcpyAsync(ctx->grid_split.p, sc.grid_split.data(), sc.grid_split.size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
        if (!sc.grid_tri.empty())
            CK(cudaMemcpyAsync(ctx->grid_tri.p, sc.grid_tri.data(), sc.grid_tri.size() * sizeof(uint32_t),
                               cudaMemcpyHostToDevice, ctx->stream));
        ctx->grid_res = sc.grid_res;
        ctx->scene_bytes_grid = (sc.grid_off.size() + sc.grid_tri.size() + sc.grid_split.size()) * sizeof(uint32_t);
        ctx->grid_list_n = sc.grid_tri.size();
    }
    const FlatBvh& bvh = ctx->scene_cache.bvh;
    lap(bvh_cached ? (cached ? "bvh+grid(hit)" : "bvh(hit)") : "bvh+grid(build)");
    // upload
    ctx->objects = std::move(objs);
    ctx->object_fp = std::move(objs_fp);
    ctx->desc = *d;
    ctx->desc.objects = nullptr;
    auto up = [&](DevBuf& b, const std::vector<uint8_t>& src) {
        b.reserve(src.size());
        CK(cudaMemcpyAsync(b.p, src.data(), src.size(), cudaMemcpyHostToDevice, ctx->stream));
    };
    up(ctx->nodes32, bvh.nodes_f32);
    up(ctx->tris32, bvh.tris_f32);
    up(ctx->nodes64, bvh.nodes_f64);
    up(ctx->tris64, bvh.tris_f64);
    // device grids are reused across uploads (grow-only) -- no cudaFree/cudaMalloc per frame
    if (ctx->sdf_dev.size() < ctx->objects.size()) {
        ctx->sdf_dev.resize(ctx->objects.size());
        ctx->skip_dev.resize(ctx->objects.size());
        ctx->plane_off_dev.resize(ctx->objects.size());
        ctx->planes_dev.resize(ctx->objects.size());
    }
    for (size_t o = 0; o < ctx->objects.size(); ++o) {
        const auto& s = ctx->objects[o].sdf;
        ctx->sdf_dev[o].reserve(s.size() * sizeof(float));
        CK(cudaMemcpyAsync(ctx->sdf_dev[o].p, s.data(), s.size() * sizeof(float), cudaMemcpyHostToDevice, ctx->stream));
        const auto& k = ctx->objects[o].skip;
        ctx->skip_dev[o].reserve(std::max<size_t>(k.size(), 1));
        if (!k.empty()) CK(cudaMemcpyAsync(ctx->skip_dev[o].p, k.data(), k.size(), cudaMemcpyHostToDevice, ctx->stream));
        const auto& po = ctx->objects[o].plane_off;
        const auto& pp = ctx->objects[o].planes;
        ctx->plane_off_dev[o].reserve(std::max<size_t>(po.size(), 1) * sizeof(uint32_t));
        ctx->planes_dev[o].reserve(std::max<size_t>(pp.size(), 4) * sizeof(float));
        if (!po.empty())
            CK(cudaMemcpyAsync(ctx->plane_off_dev[o].p, po.data(), po.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               ctx->stream));
        if (!pp.empty())
            CK(cudaMemcpyAsync(ctx->planes_dev[o].p, pp.data(), pp.size() * sizeof(float), cudaMemcpyHostToDevice,
                               ctx->stream));
    }
    uint64_t bytes = bvh.nodes_f32.size() + bvh.tris_f32.size() + bvh.nodes_f64.size() + bvh.tris_f64.size();
    for (const auto& o : ctx->objects)
        bytes += o.sdf.size() * sizeof(float) + o.skip.size() + o.plane_off.size() * sizeof(uint32_t) +
                 o.planes.size() * sizeof(float);
    bytes += ctx->scene_bytes_grid;
    bytes += ctx->objects.size() * (sizeof(ObjK<float>) + sizeof(ObjK<double>));
    ctx->scene_bytes = bytes;
    ctx->n_nodes = bvh.n_nodes;
    ctx->n_tris = bvh.n_tris;
    lap("copies queued");
    {  // FP32 shadow rays read each light-grid cell's triangles contiguously (no index hop)
        const uint64_t n_list = ctx->grid_res ? ctx->grid_list_n : 0;
        ctx->grid_tris32.reserve(std::max<uint64_t>(n_list, 1) * sizeof(TriF));
        if (n_list)
            CK(launch_gather_tris(ctx->grid_tri.as<uint32_t>(), ctx->tris32.as<TriF>(), n_list,
                                  ctx->grid_tris32.as<TriF>(), ctx->stream));
        // (h2d bytes: the gathered records are built on the device from uploaded data)
        build_camera_tiles(ctx, d, tv, bvh);
        if (ctx->cam_list_n)
            CK(launch_gather_tris(ctx->cam_idx.as<uint32_t>(), ctx->tris32.as<TriF>(), ctx->cam_list_n,
                                  ctx->cam_tris32.as<TriF>(), ctx->stream));
        bytes += (ctx->cam_list_n + static_cast<uint64_t>(ctx->cam_tiles_x) * ctx->cam_tiles_y + 1) * 4;
        ctx->scene_bytes = bytes;
    }
    fill_devscene<float>(ctx, ctx->sc32, ctx->nodes32, ctx->tris32, ctx->objs32);
    if (ctx->grid_res && ctx->grid_list_n)  // after the FP32 ObjK upload (same stream)
        CK(launch_grid_sigma(ctx->grid_tris32.as<TriF>(), ctx->grid_list_n, ctx->objs32.as<ObjK<float>>(),
                             ctx->stream));
    fill_devscene<double>(ctx, ctx->sc64, ctx->nodes64, ctx->tris64, ctx->objs64);
    CK(cudaStreamSynchronize(ctx->stream));
    lap("done");
    ctx->scene = true;
    // host-film renders of this frame read back through pinned staging: allocate it (and
    // the device film sums) now rather than inside the first render call
    ensure_film_staging(ctx, 3ull * d->width * d->height);
    ctx->film_sum.reserve(3ull * d->width * d->height * sizeof(double));
    ctx->film_sq.reserve(3ull * d->width * d->height * sizeof(double));
}

template <class R>
const DevScene<R>& scene_of(const sst_gpu_ctx* ctx) {
    if constexpr (std::is_same<R, float>::value) return ctx->sc32;
    else return ctx->sc64;
}

constexpr uint64_t kChunkPaths = 1ull << 24;  // radiance scratch per launch

// Kernel timing: events around launches on their own stream (synchronous; only
// while sst_gpu_kernel_timing is enabled).
void kt_begin(sst_gpu_ctx* ctx, cudaStream_t s) {
    if (!ctx->ktime) return;
    if (!ctx->kt_ev[0])
        for (auto& e : ctx->kt_ev) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(ctx->kt_ev[0], s));
}
void kt_end(sst_gpu_ctx* ctx, cudaStream_t s, int kind) {
    if (!ctx->ktime) return;
    CK(cudaEventRecord(ctx->kt_ev[1], s));
    CK(cudaEventSynchronize(ctx->kt_ev[1]));
    float ms = 0.0f;
    CK(cudaEventElapsedTime(&ms, ctx->kt_ev[0], ctx->kt_ev[1]));
    ctx->kt_ms[kind] += ms;
    ++ctx->kt_n[kind];
}

bool use_wavefront(const sst_gpu_ctx* ctx, bool st) { return ctx->wavefront >= 2 || (ctx->wavefront == 1 && st); }

// Sizes of the wavefront pool's arrays for `cap` slots (carve_pool order).
constexpr int kPoolArrays = 25;
template <class R>
size_t pool_layout(uint32_t cap, size_t (&off)[kPoolArrays]) {
    const size_t n = cap, nk = n * kNeeChain;
    const size_t sizes[] = {n * sizeof(Q4<R>), n * sizeof(Q4<R>), n * 8, n * 16, n * sizeof(R),
                            n * 8, nk * sizeof(Q4<R>), nk * sizeof(Q4<R>), n * 4, (nk + n) * 4, n * 4,
                            kQCount * 4, 8, n * 4, n * 4, n * 4,
                            n * sizeof(Q4<R>), n * sizeof(Q4<R>), n * 4, n * sizeof(Q4<R>), nk * sizeof(R),
                            n * sizeof(Q4<R>), n * sizeof(Q4<R>), n * 4, n * 4};
    static_assert(sizeof(sizes) / sizeof(sizes[0]) == kPoolArrays, "pool arrays");
    size_t total = 0;
    int k = 0;
    for (size_t b : sizes) {
        off[k++] = total;
        total += (b + 255) & ~size_t(255);
    }
    return total;
}

// Carves the wavefront pool of `cap` slots out of the slot's device buffer.
template <class R>
WfPool<R> carve_pool(sst_gpu_ctx::Slot& sl, uint32_t cap) {
    size_t off[kPoolArrays];
    sl.wf.reserve(pool_layout<R>(cap, off));
    char* base = sl.wf.as<char>();
    WfPool<R> q{};
    q.cap = cap;
    q.xl = reinterpret_cast<Q4<R>*>(base + off[0]);
    q.wr = reinterpret_cast<Q4<R>*>(base + off[1]);
    q.rng = reinterpret_cast<uint64_t*>(base + off[2]);
    q.meta = reinterpret_cast<uint4*>(base + off[3]);
    q.thit = reinterpret_cast<R*>(base + off[4]);
    q.hinfo = reinterpret_cast<uint2*>(base + off[5]);
    q.nee_p = reinterpret_cast<Q4<R>*>(base + off[6]);
    q.nee_w = reinterpret_cast<Q4<R>*>(base + off[7]);  // contiguous with nee_p: the paired layout
                                                        // (SST_NEE_PAIR) uses both as one array
    q.q_sphere = reinterpret_cast<uint32_t*>(base + off[8]);
    q.q_shadow = reinterpret_cast<uint32_t*>(base + off[9]);
    q.q_live = reinterpret_cast<uint32_t*>(base + off[10]);
    q.counts = reinterpret_cast<uint32_t*>(base + off[11]);
    q.resume_work = reinterpret_cast<unsigned long long*>(base + off[12]);
    q.q_la = reinterpret_cast<uint32_t*>(base + off[13]);
    q.q_lb = reinterpret_cast<uint32_t*>(base + off[14]);
    q.q_free = reinterpret_cast<uint32_t*>(base + off[15]);
    q.tr_o = reinterpret_cast<Q4<R>*>(base + off[16]);
    q.tr_d = reinterpret_cast<Q4<R>*>(base + off[17]);
    q.tr_f = reinterpret_cast<uint32_t*>(base + off[18]);
    q.tr_cam = reinterpret_cast<Q4<R>*>(base + off[19]);
    q.nee_res = reinterpret_cast<R*>(base + off[20]);
    q.trs_o = reinterpret_cast<Q4<R>*>(base + off[21]);
    q.trs_d = reinterpret_cast<Q4<R>*>(base + off[22]);
    q.trs_f = reinterpret_cast<uint32_t*>(base + off[23]);
    q.q_trace = reinterpret_cast<uint32_t*>(base + off[24]);
    return q;
}

// Wavefront render of one launch's paths (wavefront.cuh): batches of iterations of
// reset -> logic -> gen -> trace -> sphere -> shadow over a pool of path slots until
// the live slots drop to min(pool/8, wf_tail), then the megakernel finishes the tail
// and on_finish (the film accumulation) is enqueued. The host keeps two batches in
// flight and reads the live count of each as it completes (no bubble).
template <class R>
struct WfJob final : WfJobBase {
    sst_gpu_ctx* ctx;
    sst_gpu_ctx::Slot* sl;
    TraceArgs<R> a;
    bool st, ex;
    cudaStream_t stream;
    uint32_t cap = 0, thresh = 0;
    int batch = 1;
    uint64_t it = 0, k = 0, nread = 0;  // iterations and batches launched, batches read
    bool full = true;                   // pool full (path supply left): logic walks all slots in order
    uint32_t live_hint = 0;             // last live count read while draining (upper bound)
    bool supply = false, done = false;
    int out_last[2] = {kQLiveA, kQLiveA};
    std::function<void()> on_finish;
    bool log = false;
    std::chrono::steady_clock::time_point t0;

    bool supply_done() const override { return supply; }

    void launch_batch() {
        ConstLock lk;  // sphere steps read the decoder constants (ensure_constants)
        if (st) lk = ensure_constants(ctx);
        for (int b = 0; b < batch; ++b, ++it) {
            const bool even = (it & 1) == 0;  // live lists ping-pong: A -> B -> A ...
            a.pool.q_in = full ? nullptr : (even ? a.pool.q_la : a.pool.q_lb);
            a.pool.q_out = even ? a.pool.q_lb : a.pool.q_la;
            a.pool.cnt_in = even ? kQLiveA : kQLiveB;
            a.pool.cnt_out = even ? kQLiveB : kQLiveA;
            cudaEvent_t* ev = nullptr;
            if (ctx->ktime) {
                if (!ctx->kt_ev[0])
                    for (auto& e : ctx->kt_ev) CK(cudaEventCreate(&e));
                ev = ctx->kt_ev;
            }
            cudaStream_t side = ctx->wf_concurrent ? sl->side : nullptr;
            const uint32_t hint = full ? cap : live_hint;
            if constexpr (std::is_same<R, float>::value)
                CK(f32::launch_wf_iteration(a, st, ex, stream, ev, side, sl->wf_fork, sl->wf_join, hint));
            else CK(f64::launch_wf_iteration(a, st, ex, stream, ev, side, sl->wf_fork, sl->wf_join, hint));
            if (ev) {  // reset | logic | gen | trace | sphere | shadow
                CK(cudaEventSynchronize(ev[6]));
                static const int kinds[6] = {SST_KT_WF_RESET, SST_KT_WF_LOGIC, SST_KT_WF_GEN, SST_KT_WF_TRACE,
                                             SST_KT_WF_SPHERE, SST_KT_WF_SHADOW};
                for (int j = 0; j < 6; ++j) {
                    float ms = 0.0f;
                    CK(cudaEventElapsedTime(&ms, ev[j], ev[j + 1]));
                    ctx->kt_ms[kinds[j]] += ms;
                    ++ctx->kt_n[kinds[j]];
                }
            }
        }
        out_last[k & 1] = a.pool.cnt_out;
        CK(cudaMemcpyAsync(sl->wf_host + (k & 1) * kQCount, a.pool.counts, kQCount * sizeof(uint32_t),
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaEventRecord(sl->wf_ev[k & 1], stream));
        ++k;
    }

    int advance(bool may_finish, bool block) override {
        bool progressed = false;
        while (nread < k && !done) {
            const cudaEvent_t e = sl->wf_ev[nread & 1];
            if (block && !progressed) {
                CK(cudaEventSynchronize(e));
            } else {
                const cudaError_t q = cudaEventQuery(e);
                if (q == cudaErrorNotReady) break;
                CK(q);
            }
            const uint32_t* h = sl->wf_host + (nread & 1) * kQCount;
            const uint32_t live = h[out_last[nread & 1]];
            if (log)
                std::fprintf(stderr, "[wf] batch %llu live %u trace %u sphere %u shadow %u t %.3f ms\n",
                             static_cast<unsigned long long>(nread), live, h[kQTrace], h[kQSphere], h[kQShadow],
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
            ++nread;
            progressed = true;
            // generation refills every free slot while ids remain: live < cap means the
            // supply is exhausted (the pool drains from here)
            if (live < cap) full = false, supply = true;
            live_hint = live;
            if (live <= thresh) done = true;
        }
        if (done) {
            if (!may_finish) return progressed ? 1 : 0;
            ConstLock lk;
            if (st) lk = ensure_constants(ctx);
            kt_begin(ctx, stream);
            if constexpr (std::is_same<R, float>::value) CK(f32::launch_wf_finish(a, st, ex, stream));
            else CK(f64::launch_wf_finish(a, st, ex, stream));
            kt_end(ctx, stream, SST_KT_WF_TAIL);
            if (on_finish) on_finish();
            return 2;
        }
        while (k - nread < 2) {  // two batches in flight (the pinned count buffers are double)
            launch_batch();
            progressed = true;
        }
        return progressed ? 1 : 0;
    }
};

// Advances every active job (only the oldest may finish). block: wait on the oldest.
bool pump_jobs(sst_gpu_ctx* ctx, bool block) {
    bool any = false;
    for (size_t i = 0; i < ctx->jobs.size();) {
        const int r = ctx->jobs[i]->advance(i == 0, block && i == 0);
        if (r == 2) {  // only the front finishes
            ctx->jobs.pop_front();
            any = true;
            continue;  // the next job is the front now
        }
        any |= r != 0;
        ++i;
    }
    return any;
}

// Drives every job to completion (sync points: stats, host films, uploads, destroy).
void drain_jobs(sst_gpu_ctx* ctx) {
    while (!ctx->jobs.empty()) pump_jobs(ctx, true);
}

// Waits until no job uses render slot sl (slots are reused round robin).
void wait_slot(sst_gpu_ctx* ctx, const sst_gpu_ctx::Slot* sl) {
    for (;;) {
        bool busy = false;
        for (const auto& j : ctx->jobs) busy |= j->slot == sl;
        if (!busy) return;
        if (!pump_jobs(ctx, false)) pump_jobs(ctx, true);
    }
}

template <class R>
void run_wavefront(sst_gpu_ctx* ctx, TraceArgs<R>& a, bool st, bool explicit_keys, sst_gpu_ctx::Slot& sl,
                   cudaStream_t stream, std::function<void()> on_finish, bool sync) {
    auto job = std::make_unique<WfJob<R>>();
    WfJob<R>& j = *job;
    j.ctx = ctx;
    j.sl = &sl;
    j.slot = &sl;
    j.st = st;
    j.ex = explicit_keys;
    j.stream = stream;
    j.cap = static_cast<uint32_t>(std::max<uint64_t>(32, std::min<uint64_t>(a.n_paths, ctx->wf_pool)));
    a.pool = carve_pool<R>(sl, j.cap);
    a.keys = nullptr;
    a.keys_count = nullptr;
    if (ctx->cam_filter && a.sc.n_objects <= 64 && (explicit_keys || a.n_paths % 3 == 0)) {
        // camera pre-pass: paths whose camera ray misses every bounding sphere end here
        const uint64_t n_keys = explicit_keys ? a.n_paths : a.n_paths / 3;
        sl.keys.reserve(64 + 5 * n_keys);  // header, list, per-key class byte
        uint32_t* cnt = sl.keys.as<uint32_t>();  // header: total, class counts, class cursors
        CK(cudaMemsetAsync(cnt, 0, 64, stream));
        kt_begin(ctx, stream);  // timed as generation work
        if constexpr (std::is_same<R, float>::value)
            CK(f32::launch_wf_cam_filter(a, explicit_keys, static_cast<uint32_t>(n_keys), cnt + 16, cnt, stream));
        else CK(f64::launch_wf_cam_filter(a, explicit_keys, static_cast<uint32_t>(n_keys), cnt + 16, cnt, stream));
        kt_end(ctx, stream, SST_KT_WF_GEN);
        a.keys = cnt + 16;
        a.keys_count = cnt;
    }
    j.a = a;
    if (!sl.wf_host) {
        CK(cudaMallocHost(&sl.wf_host, 2 * kQCount * sizeof(uint32_t)));
        for (auto& e : sl.wf_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if constexpr (std::is_same<R, float>::value) CK(f32::launch_wf_init(j.a, stream));
    else CK(f64::launch_wf_init(j.a, stream));
    j.thresh = std::max<uint32_t>(1, std::min<uint32_t>(j.cap / 8, ctx->wf_tail));
    j.batch = std::max(1, ctx->wf_batch);
    j.on_finish = std::move(on_finish);
    j.log = std::getenv("SST_WF_TRACE") != nullptr;
    j.t0 = std::chrono::steady_clock::now();
    ctx->jobs.push_back(std::move(job));
    if (sync) {
        drain_jobs(ctx);
        return;
    }
    // asynchronous call: drive every job until this one's path supply is exhausted;
    // its drain continues under later calls (overlapping their launches) or a sync point
    for (;;) {
        bool mine = false;
        for (const auto& q : ctx->jobs) mine |= q.get() == &j;
        if (!mine || j.supply) return;
        if (!pump_jobs(ctx, false)) std::this_thread::yield();
    }
}

template <class R>
void run_trace(sst_gpu_ctx* ctx, const DevScene<R>& sc, bool st, bool explicit_keys, int nee,
               uint64_t seed, uint64_t n_paths, uint32_t n_pix, uint32_t sample_begin,
               const uint32_t* pix, const uint32_t* smp, const uint8_t* ch, R* radiance,
               uint32_t* segments, unsigned long long* work, cudaStream_t stream,
               sst_gpu_ctx::Slot* wf, std::function<void()> on_finish, bool sync, R* exit_state = nullptr) {
    TraceArgs<R> a{};
    a.exit_state = exit_state;
    a.sc = sc;
    a.nee = nee;
    a.seed = seed;
    a.n_paths = n_paths;
    a.n_pix = n_pix;
    a.sample_begin = sample_begin;
    a.pixel = pix;
    a.sample = smp;
    a.channel = ch;
    a.radiance = radiance;
    a.segments = segments;
    a.work = work;
    a.stats = ctx->stats.as<unsigned long long>();
    a.sphere_batch = ctx->sphere_batch;
    a.trace_batch = ctx->trace_batch;
    a.convex_end = ctx->convex_end;
    CK(cudaMemsetAsync(a.work, 0, sizeof(unsigned long long), stream));
    if (wf && use_wavefront(ctx, st) && n_paths >= ctx->wf_min_paths && n_paths < (1ull << 32) &&
        ctx->desc.n_objects < 250) {
        run_wavefront<R>(ctx, a, st, explicit_keys, *wf, stream, std::move(on_finish), sync);
        return;
    }
    ConstLock lk;
    if (st) lk = ensure_constants(ctx);
    kt_begin(ctx, stream);
    if constexpr (std::is_same<R, float>::value) CK(f32::launch_trace(a, st, explicit_keys, stream));
    else CK(f64::launch_trace(a, st, explicit_keys, stream));
    kt_end(ctx, stream, SST_KT_MEGAKERNEL);
    if (on_finish) on_finish();
}

void read_stats(sst_gpu_ctx* ctx, sst_path_stats* out) {
    unsigned long long all[kStCopies * kStCount];
    CK(cudaMemcpyAsync(all, ctx->stats.p, sizeof all, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    unsigned long long v[kStCount] = {};
    for (int c = 0; c < kStCopies; ++c)
        for (int k = 0; k < kStCount; ++k) v[k] += all[c * kStCount + k];
    if (v[kStErrors]) {
        CK(cudaMemsetAsync(ctx->stats.p, 0, sizeof all, ctx->stream));
        // the reference throws std::runtime_error (scatter.cpp:56)
        if (out) {
            out->errors += v[kStErrors];
        }
        throw RuntimeError("decoder produced non-finite output twice (" + std::to_string(v[kStErrors]) + " paths)");
    }
    if (!out) return;
    out->paths += v[kStPaths];
    out->segments += v[kStSphere] + v[kStEvents];
    out->sphere_steps += v[kStSphere];
    out->pt_events += v[kStEvents];
    out->decodes_length += v[kStDecL];
    out->decodes_path += v[kStDecP];
    out->decodes_event += v[kStDecE];
    out->absorbed += v[kStAbsorbed];
    out->escaped += v[kStEscaped];
    out->capped += v[kStCapped];
    out->shadow_rays += v[kStShadow];
    out->traversals += v[kStTraversals];
    out->node_visits += v[kStNodes];
    out->triangle_tests += v[kStTriTests];
    out->lane_iterations += v[kStLaneIters];
    out->warp_iterations += v[kStWarpIters];
    out->shadow_triangle_tests += v[kStShadowTris];
    out->wavefront_slot_visits += v[kStWfSlots];
}

void check_render_ready(sst_gpu_ctx* ctx, int integrator) {
    if (!ctx->scene) throw InvalidArgument("no scene uploaded (sst_gpu_upload_scene)");
    if (integrator != SST_INTEGRATOR_PT && integrator != SST_INTEGRATOR_ST) throw InvalidArgument("unknown integrator");
    if (integrator == SST_INTEGRATOR_ST) ensure_constants(ctx);
}

void ensure_pipeline(sst_gpu_ctx* ctx) {
    if (ctx->ev_start) return;
    for (auto& sl : ctx->slots) {
        CK(cudaStreamCreateWithFlags(&sl.s, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&sl.side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&sl.film_done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sl.wf_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&sl.wf_join, cudaEventDisableTiming));
        sl.work.reserve(sizeof(unsigned long long));
        // the wavefront's pinned count buffers: cudaMallocHost on a slot's first job
        // (mid-pipeline, e.g. inside a timed stretch of asynchronous calls) stalls it
        CK(cudaMallocHost(&sl.wf_host, 2 * kQCount * sizeof(uint32_t)));
        for (auto& e : sl.wf_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&ctx->ev_start, cudaEventDisableTiming));
    CK(cudaEventCreate(&ctx->ev0));
    CK(cudaEventCreate(&ctx->ev1));
    ctx->stats.reserve(kStCopies * kStCount * sizeof(unsigned long long));
    CK(cudaMemsetAsync(ctx->stats.p, 0, kStCopies * kStCount * sizeof(unsigned long long), ctx->stream));
}

// Makes ctx->stream wait for every render slot (no host synchronisation).
void join_slots(sst_gpu_ctx* ctx) {
    drain_jobs(ctx);
    if (!ctx->ev_start) return;
    for (auto& sl : ctx->slots) CK(cudaStreamWaitEvent(ctx->stream, sl.film_done, 0));
}

// Joins, synchronises and moves the accumulated device counters (and the device
// time since the first unread call) into *out; resets the accumulators.
void collect_stats(sst_gpu_ctx* ctx, sst_path_stats* out) {
    ensure_pipeline(ctx);
    join_slots(ctx);
    float ms = 0.0f;
    if (ctx->timing_open) CK(cudaEventRecord(ctx->ev1, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->timing_open) {
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->timing_open = false;
    }
    if (out) out->device_ms += ms;
    read_stats(ctx, out);
    CK(cudaMemsetAsync(ctx->stats.p, 0, kStCopies * kStCount * sizeof(unsigned long long), ctx->stream));
}

void readback_films(sst_gpu_ctx* ctx, const double* dsum, const double* dsq, uint64_t n, double* film_sum,
                    double* film_sq);

template <class R>
void render_impl(sst_gpu_ctx* ctx, int integrator, int nee, uint32_t spp_total, uint32_t s0, uint32_t s1,
                 uint64_t seed, double* film_sum, double* film_sq, int ptr_kind, sst_path_stats* stats) {
    (void)spp_total;
    const DevScene<R>& sc = scene_of<R>(ctx);
    const uint32_t n_pix = ctx->desc.width * ctx->desc.height;
    const uint64_t per_sample = 3ull * n_pix;
    const uint32_t n_samples = s1 - s0;
    // chunk: <= 2^24 paths, and at least ~8 chunks per call when the call is big
    // enough (>= 2^20 paths per chunk) so the long-path tail of one launch overlaps
    // the next ones on the pipeline slots
    uint64_t target = std::min<uint64_t>(kChunkPaths, std::max<uint64_t>(per_sample * n_samples / 8, 1ull << 20));
    if (const char* e = std::getenv("SST_CHUNK_PATHS")) target = std::max<uint64_t>(1, std::strtoull(e, nullptr, 10));
    // wavefront: one pool drain per chunk, so chunks are as large as the radiance
    // scratch allows (2^28 paths = 1 GiB FP32): the long-path tail is paid once
    if (use_wavefront(ctx, integrator == SST_INTEGRATOR_ST)) target = ctx->wf_chunk;
    uint32_t chunk = static_cast<uint32_t>(std::max<uint64_t>(1, target / per_sample));
    if (chunk > n_samples) chunk = n_samples;
    ensure_pipeline(ctx);
    const bool sync = ptr_kind == SST_PTR_HOST || stats != nullptr;
    double* dsum = film_sum;
    double* dsq = film_sq;
    if (ptr_kind == SST_PTR_HOST) {
        ctx->film_sum.reserve(per_sample * sizeof(double));
        ctx->film_sq.reserve(per_sample * sizeof(double));
        dsum = ctx->film_sum.as<double>();
        dsq = ctx->film_sq.as<double>();
        CK(cudaMemsetAsync(dsum, 0, per_sample * sizeof(double), ctx->stream));
        CK(cudaMemsetAsync(dsq, 0, per_sample * sizeof(double), ctx->stream));
    }
    if (!ctx->timing_open) {
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        ctx->timing_open = true;
    }
    // Pipeline slots of this call: asynchronous calls rotate over all kSlots (their
    // drains overlap later calls); a synchronous call uses slots 0 .. (its chunk count
    // - 1) only, so a one-chunk host-film render keeps ONE slot's buffers resident.
    const uint32_t n_chunks = (n_samples + chunk - 1) / chunk;
    const int n_slots = sync ? static_cast<int>(std::min<uint32_t>(sst_gpu_ctx::kSlots, n_chunks))
                             : sst_gpu_ctx::kSlots;
    if (use_wavefront(ctx, integrator == SST_INTEGRATOR_ST)) {
        // The slots this call may use get their radiance scratch and wavefront pool now
        // (grow-only): a slot first used later -- e.g. inside a timed or
        // latency-sensitive stretch of calls -- would otherwise cudaFree/cudaMalloc
        // (device-synchronising) mid-pipeline.
        size_t off[kPoolArrays];
        const uint64_t cap = std::max<uint64_t>(32, std::min<uint64_t>(per_sample * chunk, ctx->wf_pool));
        const size_t pool = pool_layout<R>(static_cast<uint32_t>(cap), off);
        const size_t keys = 64 + 5 * (per_sample * chunk / 3 + 1);  // camera pre-pass list + classes
        bool grow = false;
        for (int k = 0; k < n_slots; ++k) {
            const auto& s2 = ctx->slots[k];
            grow |= s2.rad.bytes < per_sample * chunk * sizeof(R) || s2.wf.bytes < pool ||
                    (ctx->cam_filter && s2.keys.bytes < keys);
        }
        if (grow) {
            drain_jobs(ctx);
            for (int k = 0; k < n_slots; ++k) {
                ctx->slots[k].rad.reserve(per_sample * chunk * sizeof(R));
                ctx->slots[k].wf.reserve(pool);
                if (ctx->cam_filter) ctx->slots[k].keys.reserve(keys);
            }
        }
    }
    CK(cudaEventRecord(ctx->ev_start, ctx->stream));
    int sync_slot = 0;
    for (uint32_t s = s0; s < s1; s += chunk) {
        const uint32_t ns = std::min(chunk, s1 - s);
        int slot_index;
        if (sync) {
            slot_index = sync_slot;
            sync_slot = (sync_slot + 1) % n_slots;
        } else {
            slot_index = ctx->next_slot;
            ctx->next_slot = (ctx->next_slot + 1) % sst_gpu_ctx::kSlots;
        }
        auto& sl = ctx->slots[slot_index];
        wait_slot(ctx, &sl);  // a job still draining on this slot owns its buffers
        sl.rad.reserve(per_sample * chunk * sizeof(R));
        CK(cudaStreamWaitEvent(sl.s, ctx->ev_start, 0));
        // film accumulation of this chunk, enqueued once its paths are done; films
        // chain in chunk order (jobs finish FIFO) -> deterministic sums
        auto film = [ctx, &sl, per_sample, ns, dsum, dsq]() {
            if (ctx->last_film) CK(cudaStreamWaitEvent(sl.s, ctx->last_film, 0));
            kt_begin(ctx, sl.s);
            if constexpr (std::is_same<R, float>::value) CK(f32::launch_film(sl.rad.as<R>(), per_sample, ns, dsum, dsq, sl.s));
            else CK(f64::launch_film(sl.rad.as<R>(), per_sample, ns, dsum, dsq, sl.s));
            kt_end(ctx, sl.s, SST_KT_FILM);
            CK(cudaEventRecord(sl.film_done, sl.s));
            ctx->last_film = sl.film_done;
        };
        run_trace<R>(ctx, sc, integrator == SST_INTEGRATOR_ST, false, nee, seed, per_sample * ns, n_pix, s,
                     nullptr, nullptr, nullptr, sl.rad.as<R>(), nullptr, sl.work.as<unsigned long long>(), sl.s,
                     &sl, film, sync);
    }
    if (!sync) return;  // asynchronous device-pointer call: sst_gpu_read_stats collects
    join_slots(ctx);
    if (ptr_kind == SST_PTR_HOST) readback_films(ctx, dsum, dsq, per_sample, film_sum, film_sq);
    collect_stats(ctx, stats);
}

// Host films accumulate the call's device sums: the D2H copies go through a pinned
// staging buffer in pieces, and each piece is added (by a few host threads) while the
// next one is in flight.
// Pinned staging for n film entries (sum + sum of squares); grow-only.
void ensure_film_staging(sst_gpu_ctx* ctx, uint64_t n) {
    if (ctx->film_pin_n < 2 * n) {
        if (ctx->film_pin) CK(cudaFreeHost(ctx->film_pin));
        ctx->film_pin = nullptr;
        ctx->film_pin_n = 0;
        CK(cudaMallocHost(&ctx->film_pin, 2 * n * sizeof(double)));
        ctx->film_pin_n = 2 * n;
    }
}

void readback_films(sst_gpu_ctx* ctx, const double* dsum, const double* dsq, uint64_t n, double* film_sum,
                    double* film_sq) {
    ensure_film_staging(ctx, n);
    if (!ctx->film_pin_ev[0])
        for (auto& e : ctx->film_pin_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    constexpr int kPieces = 8;
    const uint64_t piece = (n + kPieces - 1) / kPieces;
    double* hs = ctx->film_pin;
    double* hq = ctx->film_pin + n;
    for (int k = 0; k < kPieces; ++k) {
        const uint64_t b = std::min<uint64_t>(n, k * piece), e = std::min<uint64_t>(n, b + piece);
        if (e > b) {
            CK(cudaMemcpyAsync(hs + b, dsum + b, (e - b) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaMemcpyAsync(hq + b, dsq + b, (e - b) * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        }
        CK(cudaEventRecord(ctx->film_pin_ev[k], ctx->stream));
    }
    const unsigned nt = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    for (int k = 0; k < kPieces; ++k) {
        CK(cudaEventSynchronize(ctx->film_pin_ev[k]));
        const uint64_t b = std::min<uint64_t>(n, k * piece), e = std::min<uint64_t>(n, b + piece);
        auto add = [&](uint64_t lo, uint64_t hi) {
            for (uint64_t i = lo; i < hi; ++i) {
                film_sum[i] += hs[i];
                film_sq[i] += hq[i];
            }
        };
        if (e - b < (1u << 16) || nt == 1) {
            add(b, e);
            continue;
        }
        std::vector<std::thread> th;
        const uint64_t part = (e - b + nt - 1) / nt;
        for (unsigned t = 0; t < nt; ++t) {
            const uint64_t lo = b + std::min<uint64_t>(e - b, t * part), hi = b + std::min<uint64_t>(e - b, (t + 1) * part);
            if (hi > lo) th.emplace_back(add, lo, hi);
        }
        for (auto& t : th) t.join();
    }
}

template <class R>
void trace_paths_impl(sst_gpu_ctx* ctx, int integrator, int nee, uint64_t seed, uint64_t n,
                      const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                      double* radiance, uint32_t* segments, double* exit_state, sst_path_stats* stats) {
    const DevScene<R>& sc = scene_of<R>(ctx);
    const uint32_t n_pix = ctx->desc.width * ctx->desc.height;
    for (uint64_t i = 0; i < n; ++i) {
        if (pixel[i] >= n_pix) throw InvalidArgument("pixel index out of range");
        if (channel[i] > 2) throw InvalidArgument("channel must be 0, 1 or 2");
    }
    ensure_pipeline(ctx);
    collect_stats(ctx, nullptr);  // drain (and discard) counters of earlier asynchronous calls
    ctx->keys_pix.reserve(n * 4);
    ctx->keys_smp.reserve(n * 4);
    ctx->keys_ch.reserve(n);
    ctx->radiance.reserve(n * sizeof(R));
    ctx->segments.reserve(n * 4);
    ctx->work.reserve(sizeof(unsigned long long));
    ScopedBuf dexit;
    if (exit_state) dexit.reserve(6 * n * sizeof(R));
    CK(cudaEventRecord(ctx->ev0, ctx->stream));
    ctx->timing_open = true;
    CK(cudaMemcpyAsync(ctx->keys_pix.p, pixel, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->keys_smp.p, sample, n * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->keys_ch.p, channel, n, cudaMemcpyHostToDevice, ctx->stream));
    run_trace<R>(ctx, sc, integrator == SST_INTEGRATOR_ST, true, nee, seed, n, n_pix, 0,
                 ctx->keys_pix.as<uint32_t>(), ctx->keys_smp.as<uint32_t>(), ctx->keys_ch.as<uint8_t>(),
                 ctx->radiance.as<R>(), ctx->segments.as<uint32_t>(), ctx->work.as<unsigned long long>(),
                 ctx->stream, &ctx->slots[0], nullptr, true, exit_state ? dexit.as<R>() : nullptr);
    std::vector<R> rad(n);
    CK(cudaMemcpyAsync(rad.data(), ctx->radiance.p, n * sizeof(R), cudaMemcpyDeviceToHost, ctx->stream));
    if (segments) CK(cudaMemcpyAsync(segments, ctx->segments.p, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
    std::vector<R> ex(exit_state ? 6 * n : 0);
    if (exit_state) CK(cudaMemcpyAsync(ex.data(), dexit.p, 6 * n * sizeof(R), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    for (uint64_t i = 0; i < n; ++i) radiance[i] = static_cast<double>(rad[i]);
    for (uint64_t i = 0; i < ex.size(); ++i) exit_state[i] = static_cast<double>(ex[i]);
    collect_stats(ctx, stats);
}

}  // namespace

namespace {
template <class R>
void verify_culling_impl(sst_gpu_ctx* ctx, uint64_t n, uint64_t seed, sst_cull_report* out) {
    ScopedBuf cnt;
    cnt.reserve(kCvCount * sizeof(unsigned long long));
    CK(cudaMemsetAsync(cnt.p, 0, kCvCount * sizeof(unsigned long long), ctx->stream));
    CullCheckArgs<R> a{};
    a.sc = scene_of<R>(ctx);
    a.tris = ctx->tris64.as<TriD>();
    a.n_tris = ctx->n_tris;
    a.n = n;
    a.seed = seed;
    a.convex_end = ctx->convex_end;
    a.counts = cnt.as<unsigned long long>();
    if constexpr (std::is_same<R, float>::value) CK(f32::launch_verify_cull(a, ctx->stream));
    else CK(f64::launch_verify_cull(a, ctx->stream));
    unsigned long long h[kCvCount];
    CK(cudaMemcpyAsync(h, cnt.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    out->flights = h[kCvFlights];
    out->culled_sdf = h[kCvCullSdf];
    out->culled_skip = h[kCvCullSkip];
    out->culled_endpoint_convex = h[kCvCullConvex];
    out->culled_endpoint_twoball = h[kCvCullTwoBall];
    out->violations_sdf = h[kCvViolSdf];
    out->violations_skip = h[kCvViolSkip];
    out->violations_endpoint_convex = h[kCvViolConvex];
    out->violations_endpoint_twoball = h[kCvViolTwoBall];
    out->radius_violations = h[kCvRadiusViol];
    out->skip_radius_violations = h[kCvSkipRadiusViol];
    out->culled_endpoint_planes = h[kCvCullPlanes];
    out->violations_endpoint_planes = h[kCvViolPlanes];
}
}  // namespace

// =========================================================================== C ABI
extern "C" {

int sst_gpu_abi_version(void) { return SST_GPU_ABI_VERSION; }

const char* sst_gpu_last_error(void) { return g_last_error.c_str(); }

uint64_t sst_rng_init(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t s3) {
    return rng_key(seed, s1, s2, s3);
}

int sst_gpu_create(int device, sst_gpu_ctx** out) {
    return guarded([&] {
        if (!out) throw InvalidArgument("null output pointer");
        *out = nullptr;
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess || n == 0)
            throw CudaFailure(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                              "); this library has no CPU fallback");
        if (device < 0 || device >= n) throw InvalidArgument("device ordinal out of range");
        CK(cudaSetDevice(device));
        cudaDeviceProp prop;
        CK(cudaGetDeviceProperties(&prop, device));
        if (prop.major < 10)
            throw CudaFailure(std::string("device ") + prop.name + " is not sm_100 (B200); kernels are built for sm_100a only");
        auto ctx = std::make_unique<sst_gpu_ctx>();
        ctx->device = device;
        CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->serial = ++g_serial;
        if (const char* e = std::getenv("SST_SPHERE_BATCH")) ctx->sphere_batch = std::max(1, std::atoi(e));
        if (const char* e = std::getenv("SST_TRACE_BATCH")) ctx->trace_batch = std::max(0, std::atoi(e));
        if (const char* e = std::getenv("SST_WAVEFRONT")) ctx->wavefront = std::atoi(e);
        if (const char* e = std::getenv("SST_WF_POOL")) ctx->wf_pool = static_cast<uint32_t>(std::max(32, std::atoi(e)));
        if (const char* e = std::getenv("SST_WF_TAIL")) ctx->wf_tail = static_cast<uint32_t>(std::max(1, std::atoi(e)));
        if (const char* e = std::getenv("SST_WF_BATCH")) ctx->wf_batch = std::max(1, std::atoi(e));
        if (const char* e = std::getenv("SST_WF_CONCURRENT")) ctx->wf_concurrent = std::atoi(e) != 0;
        if (const char* e = std::getenv("SST_CAM_FILTER")) ctx->cam_filter = std::atoi(e) != 0;
        if (const char* e = std::getenv("SST_CONVEX_END")) ctx->convex_end = std::atoi(e) != 0;
        if (const char* e = std::getenv("SST_WF_MIN_PATHS")) ctx->wf_min_paths = std::strtoull(e, nullptr, 10);
        if (const char* e = std::getenv("SST_WF_CHUNK")) ctx->wf_chunk = std::max<uint64_t>(1024, std::strtoull(e, nullptr, 10));
        *out = ctx.release();
    });
}

void sst_gpu_destroy(sst_gpu_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    try {
        drain_jobs(ctx);
    } catch (...) {
        ctx->jobs.clear();
    }
    cudaStreamSynchronize(ctx->stream);
    {
        // the weights stay resident (other contexts with equal weights may be reading
        // them): forget only the owner, so a later swap still waits for the device
        const ConstLock lk(g_const_mu);
        auto it = g_const_owner.find(ctx->device);
        if (it != g_const_owner.end() && it->second.ctx == ctx) it->second.ctx = nullptr;
    }
    for (DevBuf* b : {&ctx->nodes32, &ctx->tris32, &ctx->nodes64, &ctx->tris64, &ctx->objs32, &ctx->objs64, &ctx->grid_off, &ctx->grid_tri, &ctx->grid_split, &ctx->grid_tris32, &ctx->cam_off, &ctx->cam_idx, &ctx->cam_tris32,
                      &ctx->radiance, &ctx->segments, &ctx->work, &ctx->stats, &ctx->error, &ctx->film_sum,
                      &ctx->film_sq, &ctx->keys_pix, &ctx->keys_smp, &ctx->keys_ch, &ctx->step_in, &ctx->step_out})
        b->release();
    for (auto& b : ctx->sdf_dev) b.release();
    for (auto& b : ctx->skip_dev) b.release();
    for (auto& b : ctx->plane_off_dev) b.release();
    for (auto& b : ctx->planes_dev) b.release();
    for (auto& e : ctx->kt_ev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->film_pin_ev)
        if (e) cudaEventDestroy(e);
    if (ctx->film_pin) cudaFreeHost(ctx->film_pin);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->ev_start) cudaEventDestroy(ctx->ev_start);
    for (auto& sl : ctx->slots) {
        if (sl.s) cudaStreamSynchronize(sl.s);
        sl.rad.release();
        sl.work.release();
        sl.wf.release();
        sl.keys.release();
        if (sl.wf_host) cudaFreeHost(sl.wf_host);
        for (auto& e : sl.wf_ev)
            if (e) cudaEventDestroy(e);
        if (sl.film_done) cudaEventDestroy(sl.film_done);
        if (sl.wf_fork) cudaEventDestroy(sl.wf_fork);
        if (sl.wf_join) cudaEventDestroy(sl.wf_join);
        if (sl.side) cudaStreamDestroy(sl.side);
        if (sl.s) cudaStreamDestroy(sl.s);
    }
    cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int sst_gpu_set_precision(sst_gpu_ctx* ctx, int precision) {
    return guarded([&] {
        if (!ctx) throw InvalidArgument("null context");
        if (precision != SST_PREC_F32 && precision != SST_PREC_F64) throw InvalidArgument("precision must be SST_PREC_F32 or SST_PREC_F64");
        ctx->precision = precision;
    });
}

int sst_gpu_get_device(const sst_gpu_ctx* ctx) { return ctx ? ctx->device : -1; }

void* sst_gpu_stream(sst_gpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int sst_gpu_synchronize(sst_gpu_ctx* ctx) {
    return guarded([&] {
        require_device(ctx);
        join_slots(ctx);
        CK(cudaStreamSynchronize(ctx->stream));
    });
}

int sst_gpu_kernel_timing(sst_gpu_ctx* ctx, int enable, double* ms, uint64_t* launches) {
    return guarded([&] {
        require_device(ctx);
        join_slots(ctx);
        CK(cudaStreamSynchronize(ctx->stream));
        for (int k = 0; k < SST_KT_COUNT; ++k) {
            if (ms) ms[k] = ctx->kt_ms[k];
            if (launches) launches[k] = ctx->kt_n[k];
        }
        if (enable) {
            for (int k = 0; k < SST_KT_COUNT; ++k) {
                ctx->kt_ms[k] = 0.0;
                ctx->kt_n[k] = 0;
            }
        }
        ctx->ktime = enable != 0;
    });
}

int sst_gpu_read_stats(sst_gpu_ctx* ctx, sst_path_stats* stats) {
    return guarded([&] {
        require_device(ctx);
        collect_stats(ctx, stats);
    });
}

int sst_gpu_upload_models(sst_gpu_ctx* ctx, const sst_model_desc models[3]) {
    return guarded([&] {
        require_device(ctx);
        if (!models) throw InvalidArgument("null model descriptors");
        HostModel m[3];
        for (int k = 0; k < 3; ++k) {
            const sst_model_desc& d = models[k];
            m[k].kind = d.kind;
            m[k].p_in = d.p_in;
            m[k].p_out = d.p_out;
            m[k].depth = d.depth;
            m[k].width = d.width;
            m[k].latent = d.latent;
            m[k].sigma_ref = d.sigma_ref;
            m[k].n_ref = d.n_ref;
            if (!d.layers || d.n_layers == 0) throw InvalidArgument("model has no layers");
            for (uint32_t i = 0; i < d.n_layers; ++i) {
                const sst_layer_desc& l = d.layers[i];
                if (!l.weights || !l.bias || !l.out_dim || !l.in_dim) throw InvalidArgument("empty layer");
                HostLayer hl;
                hl.out_dim = l.out_dim;
                hl.in_dim = l.in_dim;
                hl.w.assign(l.weights, l.weights + static_cast<size_t>(l.out_dim) * l.in_dim);
                hl.b.assign(l.bias, l.bias + l.out_dim);
                m[k].layers.push_back(std::move(hl));
            }
        }
        set_models(ctx, m);
        ensure_constants(ctx);
    });
}

int sst_gpu_load_models_dir(sst_gpu_ctx* ctx, const char* dir) {
    return guarded([&] {
        require_device(ctx);
        if (!dir) throw InvalidArgument("null directory");
        const std::string d(dir);
        HostModel m[3] = {load_ssnn(d + "/lengthgen.ssnn"), load_ssnn(d + "/pathgen.ssnn"),
                          load_ssnn(d + "/eventgen.ssnn")};
        set_models(ctx, m);
        ensure_constants(ctx);
    });
}

int sst_gpu_sphere_step_batch(sst_gpu_ctx* ctx, uint64_t n, const sst_step_in* in, int with_event_default,
                              sst_step_out* out, int ptr_kind, sst_decode_counters* counters) {
    return guarded([&] {
        require_device(ctx);
        if (!in || !out) throw InvalidArgument("null batch descriptors");
        if (ptr_kind != SST_PTR_HOST && ptr_kind != SST_PTR_DEVICE) throw InvalidArgument("bad ptr_kind");
        const ConstLock lk = ensure_constants(ctx);
        if (n == 0) return;
        if (ptr_kind == SST_PTR_HOST) {
            for (uint64_t i = 0; i < n; ++i) {
                if (!(in->sigma_t[i] >= 0.0 && in->r_sphere[i] >= 0.0)) throw DomainError("rescale_sigma: negative input");
                if (!(in->r_sphere[i] > 0.0)) throw DomainError("to_world: r_sphere must be > 0");
            }
        }
        ctx->error.reserve(8 + 3 * sizeof(unsigned long long));
        int* derr = ctx->error.as<int>();
        unsigned long long* dcnt = reinterpret_cast<unsigned long long*>(ctx->error.as<char>() + 8);
        CK(cudaMemsetAsync(ctx->error.p, 0, 8 + 3 * sizeof(unsigned long long), ctx->stream));
        StepBatchArgs a{};
        a.n = n;
        a.with_event_default = with_event_default;
        a.error = derr;
        a.counters = dcnt;
        if (ptr_kind == SST_PTR_DEVICE) {
            a.sigma_t = in->sigma_t; a.g = in->g; a.phi = in->phi; a.w_in = in->w_in; a.center = in->center;
            a.r = in->r_sphere; a.with_event = in->with_event; a.rng_state = in->rng_state;
            a.absorbed = out->absorbed; a.n_events = out->n_events; a.exit_pos = out->exit_position;
            a.exit_dir = out->exit_direction; a.has_rep = out->has_representative; a.rep_pos = out->rep_position;
            a.rep_dir = out->rep_direction; a.lambda = out->lambda_weight;
            CK(ctx->precision == SST_PREC_F64 ? f64::launch_step_batch(a, ctx->stream)
                                              : f32::launch_step_batch(a, ctx->stream));
        } else {
            // staging: inputs 8+8+8+24+24+8+1+8 B, outputs 1+4+4*24+1+8 B per step, 16-B aligned segments
            const size_t in_b = n * 89 + 8 * 16, out_b = n * 110 + 8 * 16;
            ctx->step_in.reserve(in_b);
            ctx->step_out.reserve(out_b);
            char* pi = ctx->step_in.as<char>();
            char* po = ctx->step_out.as<char>();
            auto h2d = [&](const void* src, size_t bytes) {
                char* dst = pi;
                CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
                pi += (bytes + 15) / 16 * 16;
                return dst;
            };
            auto dal = [&](size_t bytes) {
                char* dst = po;
                po += (bytes + 15) / 16 * 16;
                return dst;
            };
            a.sigma_t = reinterpret_cast<const double*>(h2d(in->sigma_t, 8 * n));
            a.g = reinterpret_cast<const double*>(h2d(in->g, 8 * n));
            a.phi = reinterpret_cast<const double*>(h2d(in->phi, 8 * n));
            a.w_in = reinterpret_cast<const double*>(h2d(in->w_in, 24 * n));
            a.center = reinterpret_cast<const double*>(h2d(in->center, 24 * n));
            a.r = reinterpret_cast<const double*>(h2d(in->r_sphere, 8 * n));
            a.with_event = in->with_event ? reinterpret_cast<const uint8_t*>(h2d(in->with_event, n)) : nullptr;
            a.rng_state = reinterpret_cast<uint64_t*>(h2d(in->rng_state, 8 * n));
            a.absorbed = reinterpret_cast<uint8_t*>(dal(n));
            a.n_events = reinterpret_cast<uint32_t*>(dal(4 * n));
            a.exit_pos = reinterpret_cast<double*>(dal(24 * n));
            a.exit_dir = reinterpret_cast<double*>(dal(24 * n));
            a.has_rep = reinterpret_cast<uint8_t*>(dal(n));
            a.rep_pos = reinterpret_cast<double*>(dal(24 * n));
            a.rep_dir = reinterpret_cast<double*>(dal(24 * n));
            a.lambda = reinterpret_cast<double*>(dal(8 * n));
            CK(ctx->precision == SST_PREC_F64 ? f64::launch_step_batch(a, ctx->stream) : f32::launch_step_batch(a, ctx->stream));
            auto d2h = [&](void* dst, const void* src, size_t bytes) {
                CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
            };
            d2h(in->rng_state, a.rng_state, 8 * n);
            d2h(out->absorbed, a.absorbed, n);
            d2h(out->n_events, a.n_events, 4 * n);
            d2h(out->exit_position, a.exit_pos, 24 * n);
            d2h(out->exit_direction, a.exit_dir, 24 * n);
            d2h(out->has_representative, a.has_rep, n);
            d2h(out->rep_position, a.rep_pos, 24 * n);
            d2h(out->rep_direction, a.rep_dir, 24 * n);
            d2h(out->lambda_weight, a.lambda, 8 * n);
        }
        int herr = 0;
        unsigned long long hc[3];
        CK(cudaMemcpyAsync(&herr, derr, sizeof herr, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(hc, dcnt, sizeof hc, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        if (counters) {
            counters->length += hc[0];
            counters->path += hc[1];
            counters->event += hc[2];
        }
        if (herr) throw RuntimeError("decoder produced non-finite output twice");
    });
}

int sst_gpu_upload_scene(sst_gpu_ctx* ctx, const sst_scene_desc* scene) {
    return guarded([&] {
        require_device(ctx);
        // in-flight asynchronous renders read the scene buffers: drain them first
        join_slots(ctx);
        CK(cudaStreamSynchronize(ctx->stream));
        upload_scene(ctx, scene);
    });
}

int sst_gpu_scene_info(sst_gpu_ctx* ctx, uint64_t* h2d_bytes, uint32_t* n_nodes, uint32_t* n_triangles) {
    return guarded([&] {
        if (!ctx || !ctx->scene) throw InvalidArgument("no scene uploaded");
        if (h2d_bytes) *h2d_bytes = ctx->scene_bytes;
        if (n_nodes) *n_nodes = ctx->n_nodes;
        if (n_triangles) *n_triangles = ctx->n_tris;
    });
}

int sst_gpu_get_sdf(sst_gpu_ctx* ctx, uint32_t obj, double origin[3], double* voxel, uint32_t dims[3],
                    float* values) {
    return guarded([&] {
        if (!ctx || !ctx->scene) throw InvalidArgument("no scene uploaded");
        if (obj >= ctx->objects.size()) throw InvalidArgument("object index out of range");
        const ObjectHost& o = ctx->objects[obj];
        for (int a = 0; a < 3; ++a) {
            if (origin) origin[a] = o.sdf_origin[a];
            if (dims) dims[a] = o.dims[a];
        }
        if (voxel) *voxel = o.sdf_voxel;
        if (values) std::memcpy(values, o.sdf.data(), o.sdf.size() * sizeof(float));
    });
}

int sst_gpu_render(sst_gpu_ctx* ctx, int integrator, int nee, uint32_t spp_total, uint32_t sample_begin,
                   uint32_t sample_end, uint64_t seed, double* film_sum, double* film_sumsq, int ptr_kind,
                   sst_path_stats* stats) {
    return guarded([&] {
        require_device(ctx);
        check_render_ready(ctx, integrator);
        if (spp_total == 0) throw InvalidArgument("spp must be >= 1");
        if (sample_begin >= sample_end || sample_end > spp_total) throw InvalidArgument("bad sample range");
        if (!film_sum || !film_sumsq) throw InvalidArgument("null film buffers");
        if (ptr_kind != SST_PTR_HOST && ptr_kind != SST_PTR_DEVICE) throw InvalidArgument("bad ptr_kind");
        if (ctx->precision == SST_PREC_F64)
            render_impl<double>(ctx, integrator, nee, spp_total, sample_begin, sample_end, seed, film_sum,
                                film_sumsq, ptr_kind, stats);
        else
            render_impl<float>(ctx, integrator, nee, spp_total, sample_begin, sample_end, seed, film_sum,
                               film_sumsq, ptr_kind, stats);
    });
}

int sst_gpu_generate_dataset(sst_gpu_ctx* ctx, uint64_t n, double s_lo, double s_hi, double g_lo, double g_hi,
                             int phi_kind, double phi_a, double phi_b, uint64_t seed, uint64_t first,
                             sst_training_sample* out, int ptr_kind, sst_dataset_stats* stats) {
    static_assert(sizeof(sst_training_sample) == sizeof(TrainingSampleDev), "sample layout");
    return guarded([&] {
        require_device(ctx);
        // generate_dataset argument checks (dataset.cpp:44-48)
        if (n == 0) throw InvalidArgument("generate_dataset: n_samples must be > 0");
        if (!(s_lo >= 0.0 && s_hi >= s_lo)) throw InvalidArgument("generate_dataset: invalid sigma_t range");
        if (!(g_lo >= -1.0 && g_hi <= 1.0 && g_hi >= g_lo)) throw InvalidArgument("generate_dataset: invalid g range");
        if (phi_kind < 0 || phi_kind > 2) throw InvalidArgument("unknown PhiSampler kind");
        if (!out) throw InvalidArgument("null output buffer");
        if (ptr_kind != SST_PTR_HOST && ptr_kind != SST_PTR_DEVICE) throw InvalidArgument("bad ptr_kind");
        ensure_pipeline(ctx);
        join_slots(ctx);
        const uint64_t chunk = ptr_kind == SST_PTR_DEVICE ? n : std::min<uint64_t>(n, 1ull << 24);
        ScopedBuf dout, dmisc;
        if (ptr_kind == SST_PTR_HOST) dout.reserve(chunk * sizeof(TrainingSampleDev));
        dmisc.reserve(8 + 8 + 4 * 8);
        unsigned long long* work = dmisc.as<unsigned long long>();
        unsigned long long* st = work + 1;
        int* err = reinterpret_cast<int*>(st + 3);
        CK(cudaMemsetAsync(dmisc.p, 0, 8 + 8 + 4 * 8, ctx->stream));
        if (!ctx->ev0) {
            CK(cudaEventCreate(&ctx->ev0));
            CK(cudaEventCreate(&ctx->ev1));
        }
        CK(cudaEventRecord(ctx->ev0, ctx->stream));
        for (uint64_t b = 0; b < n; b += chunk) {
            const uint64_t m = std::min(chunk, n - b);
            DatasetArgs a{};
            a.n = m;
            a.first = first + b;
            a.s_lo = s_lo;
            a.s_hi = s_hi;
            a.g_lo = g_lo;
            a.g_hi = g_hi;
            a.phi_kind = phi_kind;
            a.phi_a = phi_a;
            a.phi_b = phi_b;
            a.seed = seed;
            a.out = ptr_kind == SST_PTR_DEVICE ? reinterpret_cast<TrainingSampleDev*>(out) + b
                                               : dout.as<TrainingSampleDev>();
            a.work = work;
            a.stats = st;
            a.error = err;
            CK(cudaMemsetAsync(work, 0, 8, ctx->stream));
            CK(ctx->precision == SST_PREC_F64 ? f64::launch_dataset(a, ctx->stream) : f32::launch_dataset(a, ctx->stream));
            if (ptr_kind == SST_PTR_HOST)
                CK(cudaMemcpyAsync(out + b, dout.p, m * sizeof(TrainingSampleDev), cudaMemcpyDeviceToHost, ctx->stream));
        }
        CK(cudaEventRecord(ctx->ev1, ctx->stream));
        unsigned long long hs[3];
        int herr = 0;
        CK(cudaMemcpyAsync(hs, st, sizeof hs, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(&herr, err, sizeof herr, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        if (herr) throw RuntimeError("walk_sphere: event cap exceeded");
        if (stats) {
            stats->walks += n;
            stats->events += hs[0];
            stats->replay_events += hs[1];
            stats->max_events = std::max<uint64_t>(stats->max_events, hs[2]);
            stats->device_ms += ms;
        }
    });
}

int sst_gpu_verify_culling(sst_gpu_ctx* ctx, uint64_t n, uint64_t seed, sst_cull_report* out) {
    return guarded([&] {
        require_device(ctx);
        if (!ctx->scene) throw InvalidArgument("no scene uploaded (sst_gpu_upload_scene)");
        if (!out) throw InvalidArgument("null output pointer");
        *out = sst_cull_report{};
        drain_jobs(ctx);
        if (ctx->precision == SST_PREC_F64) verify_culling_impl<double>(ctx, n, seed, out);
        else verify_culling_impl<float>(ctx, n, seed, out);
    });
}

int sst_gpu_nee_identity(sst_gpu_ctx* ctx, uint64_t walks, uint32_t resamples, double sigma_t, double g,
                         double phi, const double light_pos[3], uint64_t seed, sst_nee_identity_report* out) {
    return guarded([&] {
        require_device(ctx);
        if (!out || !light_pos) throw InvalidArgument("null argument");
        if (!(sigma_t > 0.0) || !(g > -1.0 && g < 1.0) || !(phi >= 0.0 && phi <= 1.0) || resamples == 0)
            throw DomainError("nee_identity: sigma_t > 0, g in (-1, 1), phi in [0, 1], resamples >= 1");
        if (light_pos[0] * light_pos[0] + light_pos[1] * light_pos[1] + light_pos[2] * light_pos[2] <= 1.0)
            throw InvalidArgument("nee_identity: the light must lie outside the unit sphere");
        ScopedBuf buf;
        buf.reserve(3 * sizeof(double) + 3 * sizeof(unsigned long long));
        CK(cudaMemsetAsync(buf.p, 0, 3 * sizeof(double) + 3 * sizeof(unsigned long long), ctx->stream));
        NeeIdentityArgs a{};
        a.walks = walks;
        a.resamples = resamples;
        a.sigma_t = sigma_t;
        a.g = g;
        a.phi = phi;
        for (int k = 0; k < 3; ++k) a.light[k] = light_pos[k];
        a.seed = seed;
        a.sums = buf.as<double>();
        a.counts = reinterpret_cast<unsigned long long*>(buf.as<char>() + 3 * sizeof(double));
        CK(ctx->precision == SST_PREC_F64 ? f64::launch_nee_identity(a, ctx->stream)
                                          : f32::launch_nee_identity(a, ctx->stream));
        double h[3];
        unsigned long long c[3];
        CK(cudaMemcpyAsync(h, a.sums, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaMemcpyAsync(c, a.counts, sizeof c, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        out->walks = c[0];
        out->events = c[1];
        out->resamples = c[2];
        const double w = c[0] ? static_cast<double>(c[0]) : 1.0;
        out->full_mean = h[0] / w;
        out->single_mean = h[1] / w;
        out->diff_stderr = std::sqrt(h[2] / w) / std::sqrt(w);
    });
}

int sst_gpu_trace_paths(sst_gpu_ctx* ctx, int integrator, int nee, uint64_t seed, uint64_t n,
                        const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel, double* radiance,
                        uint32_t* segments, sst_path_stats* stats) {
    return sst_gpu_trace_paths_ex(ctx, integrator, nee, seed, n, pixel, sample, channel, radiance, segments, nullptr,
                                  stats);
}

int sst_gpu_trace_paths_ex(sst_gpu_ctx* ctx, int integrator, int nee, uint64_t seed, uint64_t n,
                           const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel, double* radiance,
                           uint32_t* segments, double* exit_state, sst_path_stats* stats) {
    return guarded([&] {
        require_device(ctx);
        check_render_ready(ctx, integrator);
        if (n == 0) return;
        if (!pixel || !sample || !channel || !radiance) throw InvalidArgument("null path key buffers");
        if (ctx->precision == SST_PREC_F64)
            trace_paths_impl<double>(ctx, integrator, nee, seed, n, pixel, sample, channel, radiance, segments,
                                     exit_state, stats);
        else
            trace_paths_impl<float>(ctx, integrator, nee, seed, n, pixel, sample, channel, radiance, segments,
                                    exit_state, stats);
    });
}

// ---------------------------------------------------------------- host utilities
namespace {
void export_mesh(const HostMesh& m, double** pos, uint32_t* nv, uint32_t** tris, uint32_t* nt) {
    if (!pos || !nv || !tris || !nt) throw InvalidArgument("null output pointer");
    *pos = static_cast<double*>(std::malloc(m.pos.size() * 3 * sizeof(double)));
    *tris = static_cast<uint32_t*>(std::malloc(m.tri.size() * 3 * sizeof(uint32_t)));
    if (!*pos || !*tris) throw std::bad_alloc();
    for (size_t i = 0; i < m.pos.size(); ++i)
        for (int a = 0; a < 3; ++a) (*pos)[3 * i + a] = m.pos[i][a];
    for (size_t i = 0; i < m.tri.size(); ++i)
        for (int a = 0; a < 3; ++a) (*tris)[3 * i + a] = m.tri[i][a];
    *nv = static_cast<uint32_t>(m.pos.size());
    *nt = static_cast<uint32_t>(m.tri.size());
}
}  // namespace

int sst_mesh_icosphere(int subdivisions, double radius, double** positions, uint32_t* n_vertices,
                       uint32_t** triangles, uint32_t* n_triangles) {
    return guarded([&] { export_mesh(make_icosphere(subdivisions, radius), positions, n_vertices, triangles, n_triangles); });
}

int sst_mesh_bumpy_sphere(int subdivisions, double radius, double amplitude, double frequency, double** positions,
                          uint32_t* n_vertices, uint32_t** triangles, uint32_t* n_triangles) {
    return guarded([&] {
        export_mesh(make_bumpy_sphere(subdivisions, radius, amplitude, frequency), positions, n_vertices, triangles,
                    n_triangles);
    });
}

int sst_mesh_load_obj(const char* path, double scale, double** positions, uint32_t* n_vertices,
                      uint32_t** triangles, uint32_t* n_triangles, uint64_t* dropped) {
    return guarded([&] {
        if (!path) throw InvalidArgument("null path");
        const HostMesh m = load_obj(path, scale);
        export_mesh(m, positions, n_vertices, triangles, n_triangles);
        if (dropped) *dropped = m.dropped;
    });
}

void sst_mesh_free(double* positions, uint32_t* triangles) {
    std::free(positions);
    std::free(triangles);
}

int sst_sdf_save(const char* path, const double origin[3], double voxel, const uint32_t dims[3], const float* values,
                 uint64_t fp) {
    return guarded([&] {
        if (!path || !origin || !dims || !values) throw InvalidArgument("null argument");
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        if (!f) throw RuntimeError(std::string("cannot open for writing: ") + path);
        auto put = [&](const void* p, size_t n) { f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); };
        const uint32_t version = 1;
        put("SSDF", 4);
        put(&version, 4);
        put(&fp, 8);
        put(dims, 12);
        const float o[4] = {static_cast<float>(origin[0]), static_cast<float>(origin[1]), static_cast<float>(origin[2]),
                            static_cast<float>(voxel)};
        put(o, 16);
        put(values, static_cast<size_t>(dims[0]) * dims[1] * dims[2] * sizeof(float));
        f.close();
        if (!f) throw RuntimeError("write failure on close");
    });
}

int sst_sdf_load(const char* path, double origin[3], double* voxel, uint32_t dims[3], float** values, uint64_t* fp) {
    return guarded([&] {
        if (!path || !origin || !voxel || !dims || !values) throw InvalidArgument("null argument");
        std::ifstream f(path, std::ios::binary);
        if (!f) throw RuntimeError(std::string("cannot open for reading: ") + path);
        const std::string what = std::string("sdf ") + path;
        char magic[4];
        f.read(magic, 4);
        if (!f || std::memcmp(magic, "SSDF", 4) != 0) throw RuntimeError(what + ": bad magic bytes");
        uint32_t version = 0;
        f.read(reinterpret_cast<char*>(&version), 4);
        if (version != 1) throw RuntimeError(what + ": unsupported version");
        uint64_t fpv = 0;
        f.read(reinterpret_cast<char*>(&fpv), 8);
        f.read(reinterpret_cast<char*>(dims), 12);
        float o[4];
        f.read(reinterpret_cast<char*>(o), 16);
        const size_t n = static_cast<size_t>(dims[0]) * dims[1] * dims[2];
        if (!f || n == 0 || n > (1ull << 32)) throw RuntimeError(what + ": implausible dims");
        float* v = static_cast<float*>(std::malloc(n * sizeof(float)));
        if (!v) throw std::bad_alloc();
        f.read(reinterpret_cast<char*>(v), static_cast<std::streamsize>(n * sizeof(float)));
        if (!f) {
            std::free(v);
            throw RuntimeError(what + ": truncated or corrupt file");
        }
        for (int a = 0; a < 3; ++a) origin[a] = o[a];
        *voxel = o[3];
        *values = v;
        if (fp) *fp = fpv;
    });
}

void sst_sdf_free(float* values) { std::free(values); }

int sst_dataset_save(const char* path, uint64_t count, float s_lo, float s_hi, float g_lo, float g_hi,
                     uint32_t phi_kind, float phi_a, float phi_b, uint64_t seed, const void* samples) {
    return guarded([&] {
        if (!path || (!samples && count)) throw InvalidArgument("null argument");
        std::ofstream f(path, std::ios::binary | std::ios::trunc);
        if (!f) throw RuntimeError(std::string("cannot open for writing: ") + path);
        auto put = [&](const void* p, size_t n) { f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); };
        const uint32_t version = 1;
        put("SSWK", 4);
        put(&version, 4);
        put(&count, 8);
        put(&s_lo, 4);
        put(&s_hi, 4);
        put(&g_lo, 4);
        put(&g_hi, 4);
        put(&phi_kind, 4);
        put(&phi_a, 4);
        put(&phi_b, 4);
        put(&seed, 8);
        put(samples, count * sizeof(TrainingSampleDev));  // records are the packed little-endian fields
        f.close();
        if (!f) throw RuntimeError("write failure on close");
    });
}

int sst_dataset_load(const char* path, sst_dataset_header* header, void* samples, uint64_t capacity) {
    return guarded([&] {
        if (!path || !header) throw InvalidArgument("null argument");
        std::ifstream f(path, std::ios::binary);
        if (!f) throw RuntimeError(std::string("cannot open for reading: ") + path);
        const std::string what = std::string("dataset ") + path;
        char magic[4];
        f.read(magic, 4);
        if (!f || std::memcmp(magic, "SSWK", 4) != 0) throw RuntimeError(what + ": bad magic bytes");
        auto get = [&](void* p, size_t n) { f.read(static_cast<char*>(p), static_cast<std::streamsize>(n)); };
        sst_dataset_header h{};
        get(&h.version, 4);
        if (!f) throw RuntimeError(what + ": truncated or corrupt file");
        if (h.version != 1) throw RuntimeError(what + ": unsupported version");
        get(&h.count, 8);
        get(&h.sigma_t_lo, 4);
        get(&h.sigma_t_hi, 4);
        get(&h.g_lo, 4);
        get(&h.g_hi, 4);
        get(&h.phi_kind, 4);
        get(&h.phi_a, 4);
        get(&h.phi_b, 4);
        get(&h.seed, 8);
        if (!f) throw RuntimeError(what + ": truncated or corrupt file");
        // the records must all be there (the reference reads them and checks the stream)
        const std::streamoff here = f.tellg();
        f.seekg(0, std::ios::end);
        const std::streamoff end = f.tellg();
        f.seekg(here);
        const uint64_t rec = sizeof(TrainingSampleDev);
        if (end < here || static_cast<uint64_t>(end - here) / rec < h.count)
            throw RuntimeError(what + ": truncated or corrupt file");
        *header = h;
        if (!samples) return;
        if (capacity < h.count) throw InvalidArgument("sample buffer smaller than the dataset");
        get(samples, h.count * rec);  // records are the packed little-endian fields
        if (!f) throw RuntimeError(what + ": truncated or corrupt file");
    });
}

int sst_dataset_export_csv(const char* path, uint64_t count, const void* samples) {
    return guarded([&] {
        if (!path || (!samples && count)) throw InvalidArgument("null argument");
        std::FILE* f = std::fopen(path, "w");
        if (!f) throw RuntimeError(std::string("cannot open for writing: ") + path);
        std::fputs("sigma_t,g,phi,n_events,cos_theta,alpha,beta,X0,X1,X2,W0,W1,W2\n", f);
        const auto* s = static_cast<const TrainingSampleDev*>(samples);
        for (uint64_t i = 0; i < count; ++i) {
            const TrainingSampleDev& r = s[i];
            std::fprintf(f, "%.9g,%.9g,%.9g,%u,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g,%.9g\n", r.sigma_t, r.g,
                         r.phi, r.n_events, r.cos_theta, r.alpha, r.beta, r.rep_position[0], r.rep_position[1],
                         r.rep_position[2], r.rep_direction[0], r.rep_direction[1], r.rep_direction[2]);
        }
        if (std::fclose(f) != 0) throw RuntimeError(std::string("write failure: ") + path);
    });
}

int sst_image_save_pfm(const char* path, uint32_t w, uint32_t h, const float* rgb) {
    return guarded([&] {
        if (!path || !rgb) throw InvalidArgument("null argument");
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) throw RuntimeError(std::string("cannot open for writing: ") + path);
        out << "PF\n" << w << " " << h << "\n-1.0\n";
        for (uint32_t y = h; y-- > 0;)
            out.write(reinterpret_cast<const char*>(rgb + static_cast<size_t>(y) * w * 3),
                      static_cast<std::streamsize>(w) * 3 * sizeof(float));
        if (!out) throw RuntimeError(std::string("write failure: ") + path);
    });
}

int sst_image_save_pfm_gray(const char* path, uint32_t w, uint32_t h, const float* v) {
    return guarded([&] {
        if (!path || !v) throw InvalidArgument("null argument");
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) throw RuntimeError(std::string("cannot open for writing: ") + path);
        out << "Pf\n" << w << " " << h << "\n-1.0\n";
        for (uint32_t y = h; y-- > 0;)
            out.write(reinterpret_cast<const char*>(v + static_cast<size_t>(y) * w),
                      static_cast<std::streamsize>(w) * sizeof(float));
        if (!out) throw RuntimeError(std::string("write failure: ") + path);
    });
}

int sst_image_load_pfm(const char* path, uint32_t* width, uint32_t* height, float* rgb,
                       uint64_t capacity) {
    return guarded([&] {
        if (!path || !width || !height) throw InvalidArgument("null argument");
        std::ifstream in(path, std::ios::binary);
        if (!in) throw RuntimeError(std::string("cannot open: ") + path);
        std::string tag;
        uint32_t w = 0, h = 0;
        double scale = 0.0;
        in >> tag;
        if (tag != "PF") throw RuntimeError(std::string("not a color PFM file: ") + path);
        in >> w >> h >> scale;
        in.get();
        if (scale >= 0.0) throw RuntimeError(std::string("big-endian PFM unsupported: ") + path);
        *width = w;
        *height = h;
        const uint64_t n = static_cast<uint64_t>(w) * h * 3;
        if (!rgb) return;  // size query
        if (capacity < n) throw InvalidArgument("rgb buffer too small");
        for (uint32_t y = h; y-- > 0;)
            in.read(reinterpret_cast<char*>(rgb + static_cast<size_t>(y) * w * 3),
                    static_cast<std::streamsize>(w) * 3 * sizeof(float));
        if (!in) throw RuntimeError(std::string("truncated PFM: ") + path);
    });
}

// 8-bit sRGB truecolor PNG, one IDAT at zlib level 9, filter 0 (image.cpp:75-138).
// The file is assembled in one host buffer and written with a single call.
int sst_image_save_png(const char* path, uint32_t w, uint32_t h, const float* rgb) {
    return guarded([&] {
        if (!path || !rgb) throw InvalidArgument("null argument");
        auto srgb8 = [](float linear) -> uint8_t {
            double v = std::fmin(1.0, std::fmax(0.0, static_cast<double>(linear)));
            v = v <= 0.0031308 ? 12.92 * v : 1.055 * std::pow(v, 1.0 / 2.4) - 0.055;
            return static_cast<uint8_t>(std::lround(v * 255.0));
        };
        const size_t stride = static_cast<size_t>(w) * 3 + 1;
        std::vector<uint8_t> scan(stride * h);
        for (uint32_t y = 0; y < h; ++y) {
            uint8_t* row = scan.data() + y * stride;
            row[0] = 0;
            const float* src = rgb + static_cast<size_t>(y) * w * 3;
            for (size_t i = 0; i < static_cast<size_t>(w) * 3; ++i) row[1 + i] = srgb8(src[i]);
        }
        uLongf zlen = compressBound(static_cast<uLong>(scan.size()));
        std::vector<uint8_t> z(zlen);
        if (compress2(z.data(), &zlen, scan.data(), static_cast<uLong>(scan.size()), 9) != Z_OK)
            throw RuntimeError(std::string("PNG deflate failure: ") + path);

        std::vector<uint8_t> file{0x89, 'P', 'N', 'G', '\r', '\n', 0x1A, '\n'};
        auto be32 = [&file](uint32_t v) {
            for (int s = 24; s >= 0; s -= 8) file.push_back(static_cast<uint8_t>(v >> s));
        };
        auto chunk = [&](const char* type, const uint8_t* data, size_t len) {
            be32(static_cast<uint32_t>(len));
            const size_t at = file.size();
            file.insert(file.end(), type, type + 4);
            if (len) file.insert(file.end(), data, data + len);
            be32(static_cast<uint32_t>(crc32(0L, file.data() + at, static_cast<uInt>(len + 4))));
        };
        uint8_t ihdr[13] = {};
        for (int i = 0; i < 4; ++i) {
            ihdr[i] = static_cast<uint8_t>(w >> (24 - 8 * i));
            ihdr[4 + i] = static_cast<uint8_t>(h >> (24 - 8 * i));
        }
        ihdr[8] = 8;  // bit depth
        ihdr[9] = 2;  // truecolor
        chunk("IHDR", ihdr, sizeof ihdr);
        chunk("IDAT", z.data(), zlen);
        chunk("IEND", nullptr, 0);

        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) throw RuntimeError(std::string("cannot open for writing: ") + path);
        out.write(reinterpret_cast<const char*>(file.data()), static_cast<std::streamsize>(file.size()));
        if (!out) throw RuntimeError(std::string("write failure: ") + path);
    });
}

}  // extern "C"

// ------------------------------------------------------------------ CVAE training (§8f #3)
void sst_train_config_default(sst_train_config* c) {
    if (!c) return;
    *c = sst_train_config{};
    c->lr = 1e-3;
    c->batch_size = 512;
    c->epochs = 100;
    c->weight_decay = 1e-4;
    c->seed = 1;
    c->validation_fraction = 0.05;
    c->depth = c->width = c->latent = -1;
}

namespace {

const char* kind_name(int kind) {  // model_kind_name (cvae.cpp:35-42)
    static const char* names[3] = {"lengthgen", "pathgen", "eventgen"};
    return names[kind];
}

// Fisher-Yates with RandomStream draws, exactly as train_model (cvae.cpp:261-266, 284-286).
void shuffle_in_place(std::vector<uint32_t>& v, HostStream& rng) {
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[static_cast<size_t>(rng.uniform() * i)]);
}

// Trace / planar-buffer layout and the phase-2 ownership plan for one spec (train.h).
void plan_training(TrainArgs& a, const CvaeSpecH& s, uint32_t batch, int cluster) {
    const MlpShape sh[2] = {encoder_shape(s), decoder_shape(s)};
    a.p_in = static_cast<int>(s.p_in);
    a.p_out = static_cast<int>(s.p_out);
    a.latent = static_cast<int>(s.latent);
    int off = 0, poff = 0;
    size_t goff = 0;
    for (int m = 0; m < 2; ++m) {
        TrainNetK& N = a.net[m];
        N.n_layers = static_cast<int>(sh[m].in.size());
        for (int l = 0; l < N.n_layers; ++l) {
            N.in[l] = static_cast<int>(sh[m].in[l]);
            N.out[l] = static_cast<int>(sh[m].out[l]);
            N.woff[l] = poff;
            poff += N.in[l] * N.out[l] + N.out[l];
            N.xo[l] = off;
            off += N.in[l];
            N.po[l] = off;
            off += N.out[l];
            N.dlo[l] = off;
            off += N.out[l];
            // planar regions start 16-byte aligned (TMA bulk copies, train.cu)
            N.gx[l] = goff;
            goff += (static_cast<size_t>(batch) * N.in[l] + 1) & ~size_t(1);
            N.gd[l] = goff;
            goff += (static_cast<size_t>(batch) * N.out[l] + 1) & ~size_t(1);
        }
    }
    a.din_o = off;
    off += a.net[1].in[0];
    a.eps_o = off;
    off += a.latent;
    a.term_o = off;  // per-component KL / log-likelihood terms
    off += a.latent + a.p_out;
    a.loss_o = off;
    off += 1;
    a.ts = off | 1;  // odd row stride: conflict-free 64-bit smem accesses across samples
    a.gloss = goff;
    a.n_params = poff;
    a.n_params_pad = (poff + 1) & ~1;
    // shared memory: parameters + max(chunk trace rows, phase-2 staging) + chunk ids
    const size_t budget = 200 * 1024;
    const size_t fixed = static_cast<size_t>(a.n_params_pad) * 8;
    const uint32_t S = (batch + cluster - 1) / cluster;
    int max_row = 0;
    for (int m = 0; m < 2; ++m)
        for (int l = 0; l < a.net[m].n_layers; ++l) max_row = std::max(max_row, a.net[m].in[l] + a.net[m].out[l] + 1);
    const size_t avail = (budget - fixed) / 8 - 64;  // doubles, minus the ids slack
    a.chunk = static_cast<int>(std::min<size_t>(std::min<size_t>(S, 64), avail / a.ts));
    if (a.chunk < 1) throw InvalidArgument("GPU training: network too large for shared memory");
    a.stage_cap = static_cast<int>(
        std::min<size_t>(avail, static_cast<size_t>(std::min<uint32_t>(batch, 1024) + 2) * max_row + 6));
    if (a.stage_cap < 2 * max_row + 6) throw InvalidArgument("GPU training: network too large for shared memory");
    const size_t region = std::max<size_t>(static_cast<size_t>(a.chunk) * a.ts, a.stage_cap);
    a.smem_bytes = fixed + region * 8 + static_cast<size_t>(a.chunk) * 4 + 16;
    // phase-2 units: every layer gets >= 1 CTA; spare CTAs split the largest layers by rows.
    struct Lay { int m, l, parts; double size; };
    std::vector<Lay> lays;
    for (int m = 0; m < 2; ++m)
        for (int l = 0; l < a.net[m].n_layers; ++l) {
            const int need = (a.net[m].out[l] * (a.net[m].in[l] + 1) + kTrainThreads * kTrainMaxQ - 1) /
                             (kTrainThreads * kTrainMaxQ);
            lays.push_back({m, l, need, static_cast<double>(a.net[m].out[l]) * (a.net[m].in[l] + 1)});
        }
    int used = 0;
    for (auto& L : lays) used += L.parts;
    if (used > cluster) throw InvalidArgument("GPU training: too many layers for one cluster (depth too large)");
    while (used < cluster) {
        Lay* best = nullptr;
        for (auto& L : lays)
            if (L.parts < a.net[L.m].out[L.l] && (!best || L.size / L.parts > best->size / best->parts)) best = &L;
        if (!best) break;
        ++best->parts;
        ++used;
    }
    a.n_units = 0;
    for (auto& L : lays) {
        const int out = a.net[L.m].out[L.l];
        for (int p = 0; p < L.parts; ++p) {
            a.unit_model[a.n_units] = L.m;
            a.unit_layer[a.n_units] = L.l;
            a.unit_r0[a.n_units] = out * p / L.parts;
            a.unit_r1[a.n_units] = out * (p + 1) / L.parts;
            ++a.n_units;
        }
    }
}

}  // namespace

namespace {

// One model being trained (one kind, one cluster, one stream).
struct KindRun {
    int kind = 0;
    CvaeSpecH spec;
    std::vector<double> enc, dec, params;
    TrainArgs a{};
    int cluster = 16;
    cudaStream_t st = nullptr;
    ScopedBuf dx, dc, dpar, dm, dv, dt, dbc, dtrace, dbl, dvl;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, done[2] = {nullptr, nullptr};
    std::vector<double> bl, vl;
    unsigned long long t_final = 0;
    ~KindRun() {
        for (cudaEvent_t e : {ev0, ev1, done[0], done[1]})
            if (e) cudaEventDestroy(e);
    }
};

void validate_train_config(const sst_train_config* cfg) {  // TrainConfig::validate (cvae.cpp:214-222)
    if (!cfg) throw InvalidArgument("null TrainConfig");
    if (!(cfg->lr > 0.0)) throw InvalidArgument("TrainConfig: lr must be > 0");
    if (cfg->batch_size == 0) throw InvalidArgument("TrainConfig: batch_size must be > 0");
    if (cfg->epochs == 0) throw InvalidArgument("TrainConfig: epochs must be > 0");
    if (!(cfg->weight_decay >= 0.0)) throw InvalidArgument("TrainConfig: negative weight decay");
    if (!(cfg->validation_fraction >= 0.0 && cfg->validation_fraction < 1.0))
        throw InvalidArgument("TrainConfig: validation fraction out of range");
}

CvaeSpecH train_spec(int kind, const sst_train_config* cfg) {
    CvaeSpecH spec = production_spec(kind);
    if (cfg->depth > 0) spec.depth = static_cast<uint32_t>(cfg->depth);
    if (cfg->width > 0) spec.width = static_cast<uint32_t>(cfg->width);
    if (cfg->latent > 0) spec.latent = static_cast<uint32_t>(cfg->latent);
    validate_spec(spec);
    if (spec.depth + 1 > static_cast<uint32_t>(kTrainMaxLayers) || spec.width > static_cast<uint32_t>(kTrainMaxWidth) ||
        spec.latent > static_cast<uint32_t>(kTrainMaxLatent))
        throw InvalidArgument("GPU training supports depth <= 4, width <= 32, latent <= 16");
    return spec;
}

// train_model (cvae.cpp:234-347) for nk kinds over the same dataset and config. The
// validation split and the per-epoch shuffles depend only on (seed, epoch), so all
// kinds share them; each kind trains on its own stream and cluster, concurrently.
void train_impl(sst_gpu_ctx* ctx, const int* kinds, int nk, const sst_training_sample* samples, uint64_t n,
                int ptr_kind, uint64_t dataset_seed, const sst_train_config* cfg, sst_epoch_stats* const* epochs_out,
                const char* const* ssnn_paths, int include_encoder, double* const* params_out, int install,
                sst_train_stats* const* stats_out) {
    validate_train_config(cfg);
    if (n == 0 || !samples) throw InvalidArgument("train_model: empty dataset");
    if (ptr_kind != SST_PTR_HOST && ptr_kind != SST_PTR_DEVICE) throw InvalidArgument("bad ptr_kind");
    if (n > 0xFFFFFFFFull) throw InvalidArgument("train_model: more than 2^32 samples");
    std::vector<std::unique_ptr<KindRun>> runs;
    for (int k = 0; k < nk; ++k) {
        if (kinds[k] < 0 || kinds[k] > 2) throw InvalidArgument("unknown model kind");
        auto r = std::make_unique<KindRun>();
        r->kind = kinds[k];
        r->spec = train_spec(r->kind, cfg);
        make_cvae_params(r->kind, r->spec, cfg->seed, r->enc, r->dec);
        runs.push_back(std::move(r));
    }
    // seed-fixed validation split (cvae.cpp:259-270)
    std::vector<uint32_t> order(n);
    std::iota(order.begin(), order.end(), 0u);
    {
        HostStream split(cfg->seed, 0x05 /* kTrainSplit */);
        shuffle_in_place(order, split);
    }
    const auto n_val = static_cast<size_t>(cfg->validation_fraction * static_cast<double>(n));
    std::vector<uint32_t> val_idx(order.begin(), order.begin() + n_val);
    std::vector<uint32_t> train_idx(order.begin() + n_val, order.end());
    if (train_idx.empty()) throw InvalidArgument("train_model: no training samples left");
    const uint32_t B = cfg->batch_size;
    const uint32_t n_train = static_cast<uint32_t>(train_idx.size());
    const uint32_t nb = (n_train + B - 1) / B;
    const uint32_t E = cfg->epochs;
    const double beta1 = 0.9, beta2 = 0.999, adam_eps = 1e-8;  // AdamWConfig (mlp.hpp:95-101)
    // AdamW bias corrections 1 - beta^t (adamw_step, mlp.cpp:217-218) with the host's pow
    const uint64_t t_max = static_cast<uint64_t>(E) * nb;
    std::vector<double> bc(2 * (t_max + 1));
    for (uint64_t t = 0; t <= t_max; ++t) {
        bc[2 * t] = 1.0 - std::pow(beta1, static_cast<double>(t));
        bc[2 * t + 1] = 1.0 - std::pow(beta2, static_cast<double>(t));
    }

    ensure_pipeline(ctx);
    join_slots(ctx);
    cudaStream_t main = ctx->stream;
    ScopedBuf dsamp, dval, dord[2];
    const void* sp = samples;
    if (ptr_kind == SST_PTR_HOST) {
        dsamp.reserve(n * sizeof(TrainingSampleDev));
        CK(cudaMemcpyAsync(dsamp.p, samples, n * sizeof(TrainingSampleDev), cudaMemcpyHostToDevice, main));
        sp = dsamp.p;
    }
    dval.reserve(std::max<size_t>(n_val, 1) * 4);
    if (n_val) CK(cudaMemcpyAsync(dval.p, val_idx.data(), n_val * 4, cudaMemcpyHostToDevice, main));
    for (auto& o : dord) o.reserve(static_cast<size_t>(n_train) * 4);
    cudaEvent_t ev_ready = nullptr, ev_order[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
    uint32_t* pin[2] = {nullptr, nullptr};
    struct Cleanup {
        cudaEvent_t* evs[3];
        uint32_t** pin;
        ~Cleanup() {
            for (int i = 0; i < 2; ++i) {
                if (evs[2][i]) cudaEventSynchronize(evs[2][i]);
                if (pin[i]) cudaFreeHost(pin[i]);
            }
            for (cudaEvent_t* e : {evs[0], evs[1], evs[1] + 1, evs[2], evs[2] + 1})
                if (*e) cudaEventDestroy(*e);
        }
    } cleanup{{&ev_ready, ev_order, copied}, pin};
    CK(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
        CK(cudaEventCreateWithFlags(&ev_order[i], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&copied[i], cudaEventDisableTiming));
        CK(cudaHostAlloc(reinterpret_cast<void**>(&pin[i]), static_cast<size_t>(n_train) * 4, cudaHostAllocDefault));
    }
    CK(cudaEventRecord(ev_ready, main));

    for (int k = 0; k < nk; ++k) {
        KindRun& r = *runs[k];
        r.st = k == 0 ? main : ctx->slots[k - 1].s;
        CK(cudaEventCreate(&r.ev0));
        CK(cudaEventCreate(&r.ev1));
        for (auto& d : r.done) CK(cudaEventCreateWithFlags(&d, cudaEventDisableTiming));
        plan_training(r.a, r.spec, B, 16);
        r.cluster = train_cluster_size(r.a.smem_bytes);
        if (r.cluster == 0) throw CudaFailure("GPU training: no thread-block cluster fits this device");
        if (r.cluster != 16) plan_training(r.a, r.spec, B, r.cluster);
        CK(cudaStreamWaitEvent(r.st, ev_ready, 0));
        r.dx.reserve(n * r.spec.p_out * sizeof(double));
        r.dc.reserve(n * r.spec.p_in * sizeof(double));
        TrainPrepArgs pa{};
        pa.samples = sp;
        pa.n = n;
        pa.kind = r.kind;
        pa.log1p_sigma_ref = std::log1p(200.0);  // NormConstants defaults (cvae.hpp:43-46)
        pa.log_n_ref = std::log(1e4);
        pa.x = r.dx.as<double>();
        pa.cnd = r.dc.as<double>();
        CK(launch_train_prep(pa, r.st));
        r.params = r.enc;
        r.params.insert(r.params.end(), r.dec.begin(), r.dec.end());
        const size_t np = r.params.size();
        r.dpar.reserve(np * 8);
        r.dm.reserve(np * 8);
        r.dv.reserve(np * 8);
        r.dt.reserve(8);
        CK(cudaMemcpyAsync(r.dpar.p, r.params.data(), np * 8, cudaMemcpyHostToDevice, r.st));
        CK(cudaMemsetAsync(r.dm.p, 0, np * 8, r.st));
        CK(cudaMemsetAsync(r.dv.p, 0, np * 8, r.st));
        CK(cudaMemsetAsync(r.dt.p, 0, 8, r.st));
        r.dbc.reserve(bc.size() * 8);
        CK(cudaMemcpyAsync(r.dbc.p, bc.data(), bc.size() * 8, cudaMemcpyHostToDevice, r.st));
        r.dtrace.reserve((r.a.gloss + B + 16) * 8);  // + slack: bulk copies round up to 16 bytes
        r.dbl.reserve(static_cast<size_t>(E) * nb * 8);
        r.dvl.reserve(std::max<size_t>(static_cast<size_t>(E) * n_val, 1) * 8);
        TrainArgs& a = r.a;
        a.x = r.dx.as<double>();
        a.cnd = r.dc.as<double>();
        a.batch = B;
        a.n_batches = nb;
        a.seed = cfg->seed;
        a.params = r.dpar.as<double>();
        a.adam_m = r.dm.as<double>();
        a.adam_v = r.dv.as<double>();
        a.t_io = r.dt.as<unsigned long long>();
        a.bc = r.dbc.as<double>();
        a.lr = cfg->lr;
        a.wd = cfg->weight_decay;
        a.beta1 = beta1;
        a.beta2 = beta2;
        a.eps = adam_eps;
        a.gtrace = r.dtrace.as<double>();
        CK(cudaEventRecord(r.ev0, r.st));
    }

    // Epoch loop: the host shuffles epoch e+1 while the device trains epoch e; the
    // order buffers alternate so a copy never overwrites an order still being read.
    for (uint32_t e = 0; e < E; ++e) {
        const int slot = static_cast<int>(e & 1);
        HostStream sh(cfg->seed, 0x03 /* kTrainShuffle */, e);
        shuffle_in_place(train_idx, sh);
        CK(cudaEventSynchronize(copied[slot]));
        std::memcpy(pin[slot], train_idx.data(), static_cast<size_t>(n_train) * 4);
        if (e >= 2)
            for (auto& rp : runs) CK(cudaStreamWaitEvent(main, rp->done[slot], 0));
        CK(cudaMemcpyAsync(dord[slot].p, pin[slot], static_cast<size_t>(n_train) * 4, cudaMemcpyHostToDevice, main));
        CK(cudaEventRecord(copied[slot], main));
        CK(cudaEventRecord(ev_order[slot], main));
        for (auto& rp : runs) {
            KindRun& r = *rp;
            if (r.st != main) CK(cudaStreamWaitEvent(r.st, ev_order[slot], 0));
            TrainArgs ta = r.a;
            ta.order = dord[slot].as<uint32_t>();
            ta.n_order = n_train;
            ta.epoch = e;
            ta.batch_loss = r.dbl.as<double>() + static_cast<size_t>(e) * nb;
            CK(launch_train_epoch(ta, r.cluster, r.st));
            if (n_val) {
                TrainArgs va = r.a;
                va.order = dval.as<uint32_t>();
                va.n_order = static_cast<uint32_t>(n_val);
                va.epoch = e;
                va.batch_loss = r.dvl.as<double>() + static_cast<size_t>(e) * n_val;
                CK(launch_train_eval(va, r.st));
            }
            CK(cudaEventRecord(r.done[slot], r.st));
        }
    }
    for (auto& rp : runs) {
        KindRun& r = *rp;
        CK(cudaEventRecord(r.ev1, r.st));
        r.bl.resize(static_cast<size_t>(E) * nb);
        r.vl.resize(static_cast<size_t>(E) * n_val);
        CK(cudaMemcpyAsync(r.bl.data(), r.dbl.p, r.bl.size() * 8, cudaMemcpyDeviceToHost, r.st));
        if (n_val) CK(cudaMemcpyAsync(r.vl.data(), r.dvl.p, r.vl.size() * 8, cudaMemcpyDeviceToHost, r.st));
        CK(cudaMemcpyAsync(r.params.data(), r.dpar.p, r.params.size() * 8, cudaMemcpyDeviceToHost, r.st));
        CK(cudaMemcpyAsync(&r.t_final, r.dt.p, 8, cudaMemcpyDeviceToHost, r.st));
    }
    for (auto& rp : runs) CK(cudaStreamSynchronize(rp->st));

    uint64_t fp = 0;
    bool have_fp = false;
    for (int k = 0; k < nk; ++k) {
        KindRun& r = *runs[k];
        // EpochStats (cvae.cpp:300-345): finite batches only; validation in val_idx order.
        uint64_t rejected = 0;
        for (uint32_t e = 0; e < E; ++e) {
            double epoch_loss = 0.0;
            size_t epoch_samples = 0, finite = 0;
            for (uint32_t b = 0; b < nb; ++b) {
                const double x = r.bl[static_cast<size_t>(e) * nb + b];
                if (!std::isfinite(x)) {
                    ++rejected;
                    continue;
                }
                ++finite;
                epoch_loss += x;
                epoch_samples += std::min<size_t>(B, n_train - static_cast<size_t>(b) * B);
            }
            if (finite == 0)
                throw RuntimeError(std::string("train_model(") + kind_name(r.kind) +
                                   "): diverged, every batch non-finite in epoch " + std::to_string(e));
            if (epochs_out && epochs_out[k]) {
                sst_epoch_stats& es = epochs_out[k][e];
                es.train_loss = epoch_loss / static_cast<double>(std::max<size_t>(1, epoch_samples));
                double v = 0.0;
                for (size_t i = 0; i < n_val; ++i) v += r.vl[static_cast<size_t>(e) * n_val + i];
                es.validation_loss = n_val ? v / static_cast<double>(n_val) : es.train_loss;
            }
        }
        for (double& v : r.params) v = static_cast<double>(static_cast<float>(v));  // quantize_f32
        if (params_out && params_out[k]) std::memcpy(params_out[k], r.params.data(), r.params.size() * 8);
        r.enc.assign(r.params.begin(), r.params.begin() + r.enc.size());
        r.dec.assign(r.params.begin() + r.enc.size(), r.params.end());
        const bool want_fp = (ssnn_paths && ssnn_paths[k]) || (stats_out && stats_out[k]);
        if (want_fp && !have_fp) {  // Dataset::fingerprint (dataset.cpp:32-38): version, count, seed, records
            std::vector<uint8_t> host_copy;
            const uint8_t* bytes = reinterpret_cast<const uint8_t*>(samples);
            if (ptr_kind == SST_PTR_DEVICE) {
                host_copy.resize(n * sizeof(TrainingSampleDev));
                CK(cudaMemcpy(host_copy.data(), samples, host_copy.size(), cudaMemcpyDeviceToHost));
                bytes = host_copy.data();
            }
            const uint32_t version = 1;
            const uint64_t count = n;
            fp = fnv(&version, sizeof version);
            fp = fnv(&count, sizeof count, fp);
            fp = fnv(&dataset_seed, sizeof dataset_seed, fp);
            fp = fnv(bytes, n * sizeof(TrainingSampleDev), fp);
            have_fp = true;
        }
        if (ssnn_paths && ssnn_paths[k])
            save_ssnn(ssnn_paths[k], r.kind, r.spec, 200.0, 1e4, fp, r.dec, include_encoder ? &r.enc : nullptr);
        if (stats_out && stats_out[k]) {
            sst_train_stats& st = *stats_out[k];
            float ms = 0.0f;
            CK(cudaEventElapsedTime(&ms, r.ev0, r.ev1));
            st.steps = r.t_final;
            st.rejected_batches = rejected;
            st.sample_passes = static_cast<uint64_t>(E) * n_train;
            st.encoder_params = static_cast<uint32_t>(r.enc.size());
            st.decoder_params = static_cast<uint32_t>(r.dec.size());
            st.dataset_fingerprint = fp;
            st.device_ms = ms;
        }
    }
    if (install) {
        for (auto& rp : runs) {
            ctx->host_models[rp->kind] = model_from_params(rp->kind, rp->spec, 200.0, 1e4, rp->dec);
            ctx->have_model[rp->kind] = true;
        }
        if (ctx->have_model[0] && ctx->have_model[1] && ctx->have_model[2]) {
            HostModel m[3] = {ctx->host_models[0], ctx->host_models[1], ctx->host_models[2]};
            set_models(ctx, m);
            ensure_constants(ctx);
        }
    }
}

}  // namespace

int sst_gpu_train_model(sst_gpu_ctx* ctx, int kind, const sst_training_sample* samples, uint64_t n, int ptr_kind,
                        uint64_t dataset_seed, const sst_train_config* cfg, sst_epoch_stats* epochs_out,
                        const char* ssnn_path, int include_encoder, double* params_out, int install,
                        sst_train_stats* stats) {
    return guarded([&] {
        require_device(ctx);
        sst_epoch_stats* eo[1] = {epochs_out};
        const char* paths[1] = {ssnn_path};
        double* po[1] = {params_out};
        sst_train_stats* so[1] = {stats};
        train_impl(ctx, &kind, 1, samples, n, ptr_kind, dataset_seed, cfg, eo, paths, include_encoder, po, install, so);
    });
}

int sst_gpu_train_models(sst_gpu_ctx* ctx, const sst_training_sample* samples, uint64_t n, int ptr_kind,
                         uint64_t dataset_seed, const sst_train_config* cfg, sst_epoch_stats* epochs_out,
                         const char* out_dir, int include_encoder, int install, sst_train_stats* stats) {
    return guarded([&] {
        require_device(ctx);
        const int kinds[3] = {0, 1, 2};
        const uint32_t E = cfg ? cfg->epochs : 0;
        sst_epoch_stats* eo[3] = {nullptr, nullptr, nullptr};
        sst_train_stats* so[3] = {nullptr, nullptr, nullptr};
        std::string names[3];
        const char* paths[3] = {nullptr, nullptr, nullptr};
        for (int k = 0; k < 3; ++k) {
            if (epochs_out) eo[k] = epochs_out + static_cast<size_t>(k) * E;
            if (stats) so[k] = stats + k;
            if (out_dir) {
                names[k] = std::string(out_dir) + "/" + kind_name(k) + ".ssnn";
                paths[k] = names[k].c_str();
            }
        }
        train_impl(ctx, kinds, 3, samples, n, ptr_kind, dataset_seed, cfg, eo, paths, include_encoder, nullptr,
                   install, so);
    });
}
