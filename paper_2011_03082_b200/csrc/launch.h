// launch.h -- host-side entry points of the two kernel translation units.
#pragma once

#include <cuda_runtime.h>

#include "types.cuh"

namespace sstg {

constexpr int kTraceBlock = 32;  // one warp per block: a long-path tail strands one warp, not a block

#define SST_DECLARE_LAUNCHERS(NS, REAL)                                                          \
    namespace NS {                                                                              \
    cudaError_t upload_constants(const double* weights1332, const double* norms6, cudaStream_t); \
    cudaError_t launch_step_batch(const StepBatchArgs& a, cudaStream_t s);                      \
    cudaError_t launch_trace(const TraceArgs<REAL>& a, bool st, bool explicit_keys,             \
                             cudaStream_t s);                                                   \
    cudaError_t launch_wf_init(const TraceArgs<REAL>& a, cudaStream_t s);                       \
    cudaError_t launch_wf_cam_filter(const TraceArgs<REAL>& a, bool explicit_keys, uint32_t n_keys, \
                                     uint32_t* list, uint32_t* count, cudaStream_t s);            \
    cudaError_t launch_wf_iteration(const TraceArgs<REAL>& a, bool st, bool explicit_keys,      \
                                    cudaStream_t s, cudaEvent_t* ev, cudaStream_t side,         \
                                    cudaEvent_t fork, cudaEvent_t join, uint32_t live_hint);    \
    cudaError_t launch_wf_finish(const TraceArgs<REAL>& a, bool st, bool explicit_keys,         \
                                 cudaStream_t s);                                               \
    cudaError_t launch_film(const REAL* radiance, uint64_t stride, uint32_t n_samples,          \
                            double* sum, double* sumsq, cudaStream_t s);                        \
    cudaError_t launch_dataset(const DatasetArgs& a, cudaStream_t s);                           \
    cudaError_t launch_verify_cull(const CullCheckArgs<REAL>& a, cudaStream_t s);               \
    cudaError_t launch_nee_identity(const NeeIdentityArgs& a, cudaStream_t s);                  \
    }

SST_DECLARE_LAUNCHERS(f32, float)
SST_DECLARE_LAUNCHERS(f64, double)
#undef SST_DECLARE_LAUNCHERS

// Exact FP64 SDF build (kernels_f64.cu): build_sdf semantics of sdf.cpp:20-58.
struct SdfBuildArgs {
    const double* tri_vertices;  // [9 * n_tris] (a, b, c) per triangle
    uint32_t n_tris;
    double origin[3];
    double voxel;
    uint32_t dims[3];
    double half_diagonal;
    double dirs[9];    // normalised inside-test directions (bvh.cpp:206-208)
    int watertight;    // parity vote if 1, generalized winding number if 0
    float* values;
};
cudaError_t launch_sdf_build(const SdfBuildArgs& a, cudaStream_t s);

// Skip-grid build (kernels_f64.cu): q = floor(max(0, d(center) - half_diag) / unit),
// d = exact unsigned point-triangle distance (FP64), saturated at 255.
struct SkipBuildArgs {
    const double* tri_vertices;  // [9 * n_tris]
    uint32_t n_tris;
    double origin[3];
    double voxel, half_diagonal, unit;
    uint32_t dims[3];
    uint8_t* values;
};
cudaError_t launch_skip_build(const SkipBuildArgs& a, cudaStream_t s);

// Light-space culling grid build (kernels_f64.cu). caps: per triangle kCapStride
// doubles: cone {axis xyz, half angle, cos, sin} (from the light) that contains it,
// then the three unit vertex directions (exact gnomonic test per cube face).
constexpr int kCapStride = 15;
struct LightGridArgs {
    const double* caps;
    uint32_t n_tris;
    uint32_t res;         // cells per cube face edge
    double eps;           // angular padding (rad)
    uint32_t* counts;     // pass 0: [6 res^2] list lengths
    const uint32_t* offsets;  // pass 1: [6 res^2 + 1]
    uint32_t* lists;      // pass 1
    int fill;
};
cudaError_t launch_light_grid(const LightGridArgs& a, cudaStream_t s);
// out[k] = tris[idx[k]]: FP32 triangle records in light-grid list order (kernels_f64.cu).
cudaError_t launch_gather_tris(const uint32_t* idx, const TriF* tris, uint64_t n, TriF* out, cudaStream_t s);
cudaError_t launch_grid_sigma(TriF* tris, uint64_t n, const ObjK<float>* objs, cudaStream_t s);

}  // namespace sstg
