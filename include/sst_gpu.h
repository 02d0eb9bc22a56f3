/*
 * sst_gpu.h -- C ABI of the B200 (sm_100a) sphere-tracing subsurface renderer.
 *
 * This is the drop-in boundary for the reference's hot path (reference =
 * /root/reference, "sstrace", C++20, namespace sst). The reference has no FFI
 * layer; its path sits behind plain C++ functions. Each entry point below
 * names the reference interface it replaces (file:line under
 * /root/reference/proj/core/). A header-only C++ mirror that rethrows the
 * reference's std:: exception types lives in include/sst_b200.hpp.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes, no exceptions cross the boundary.
 *  - Return codes mirror the reference's exception classes:
 *      SST_OK                 0
 *      SST_E_INVALID_ARGUMENT 1  std::invalid_argument (bad shapes/config)
 *      SST_E_RUNTIME          2  std::runtime_error (I/O, bad magic, wrong kind,
 *                                decoder non-finite twice: scatter.cpp:44-58)
 *      SST_E_DOMAIN           3  std::domain_error (out-of-range physics,
 *                                optics.cpp:16-25, scatter.cpp:34-38)
 *      SST_E_CUDA             4  CUDA failure / no device (there is NO CPU
 *                                fallback: the library fails loudly)
 *    The message of the last failure on the calling thread is returned by
 *    sst_gpu_last_error().
 *  - One context per device. Calls on one context are serialised on the
 *    context's CUDA stream. Host buffers are caller-owned and copied; device
 *    buffers passed with SST_PTR_DEVICE must live on the context's device.
 *  - Films are returned as SUMS (sum of radiance and of radiance^2 per pixel and
 *    channel) so that sample-slab shards add up across GPUs.
 */
#ifndef SST_GPU_H
#define SST_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SST_GPU_ABI_VERSION 4  /* 3: sst_scene_desc light_kind / light_direction; 4: sst_cull_report planes */

enum {
    SST_OK = 0,
    SST_E_INVALID_ARGUMENT = 1,
    SST_E_RUNTIME = 2,
    SST_E_DOMAIN = 3,
    SST_E_CUDA = 4
};

/* Arithmetic of the device path. F32 is the production path; F64 is the
 * parity mode (same kernels instantiated in double). */
enum { SST_PREC_F32 = 0, SST_PREC_F64 = 1 };

/* Integrators: brute-force delta tracking (reference mode)
 * and learned sphere tracing. */
enum { SST_INTEGRATOR_PT = 0, SST_INTEGRATOR_ST = 1 };

/* Where the pointers of a batch call live. */
enum { SST_PTR_HOST = 0, SST_PTR_DEVICE = 1 };

/* Reference model kinds (cvae.hpp:16-20, ModelKind). */
enum { SST_MODEL_LENGTH = 0, SST_MODEL_PATH = 1, SST_MODEL_EVENT = 2 };

/* Stream salts (rng.hpp:53-63, namespace stream_salt). */
#define SST_SALT_DATASET 0x01u
#define SST_SALT_RENDER_PIXEL 0x06u
#define SST_SALT_RENDER_CHANNEL 0x07u

typedef struct sst_gpu_ctx sst_gpu_ctx;

/* ------------------------------------------------------------------------ */
/* Context                                                                   */
/* ------------------------------------------------------------------------ */

int sst_gpu_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* sst_gpu_last_error(void);

/* Creates a context on `device` (CUDA ordinal). Fails with SST_E_CUDA when no
 * device is present -- there is no CPU fallback. */
int sst_gpu_create(int device, sst_gpu_ctx** out);
void sst_gpu_destroy(sst_gpu_ctx* ctx);
/* SST_PREC_F32 (default) or SST_PREC_F64. */
int sst_gpu_set_precision(sst_gpu_ctx* ctx, int precision);
int sst_gpu_get_device(const sst_gpu_ctx* ctx);
/* The context's cudaStream_t (as void*), for callers that enqueue their own
 * work (e.g. a torch/NCCL film reduce) behind ours. */
void* sst_gpu_stream(sst_gpu_ctx* ctx);
int sst_gpu_synchronize(sst_gpu_ctx* ctx);

/* ------------------------------------------------------------------------ */
/* CVAE-weight interface: replaces ScatterModels / CvaeModel / load_model     */
/* (scatter.hpp:28-39, scatter.cpp:22-32, cvae.hpp:52-60, cvae.cpp:379-425)   */
/* ------------------------------------------------------------------------ */

typedef struct {
    uint32_t out_dim;
    uint32_t in_dim;
    const float* weights; /* row-major [out_dim x in_dim] (mlp.hpp:18-23) */
    const float* bias;    /* [out_dim] */
} sst_layer_desc;

typedef struct {
    uint32_t kind; /* SST_MODEL_* ; checked like scatter.cpp:15-27 */
    uint32_t p_in, p_out, depth, width, latent; /* CvaeSpec (cvae.hpp:29-38) */
    double sigma_ref, n_ref;                    /* NormConstants (cvae.hpp:43-50) */
    uint32_t n_layers;
    const sst_layer_desc* layers; /* decoder only: input latent+p_in -> 2*p_out */
} sst_model_desc;

/* Uploads the three decoders (LengthGen, PathGen, EventGen), kind-checked.
 * Only the production architectures of Table 1 (CvaeSpec::production_default,
 * cvae.cpp:51-58) have compiled device evaluators; other shapes return
 * SST_E_INVALID_ARGUMENT. */
int sst_gpu_upload_models(sst_gpu_ctx* ctx, const sst_model_desc models[3]);
/* Parses dir/{lengthgen,pathgen,eventgen}.ssnn (SSNN v1, cvae.cpp:349-425) and
 * uploads them: the equivalent of ScatterModels::load_dir (scatter.cpp:29-32). */
int sst_gpu_load_models_dir(sst_gpu_ctx* ctx, const char* dir);

/* ------------------------------------------------------------------------ */
/* RandomStream helpers (rng.hpp:15-50). The stream state after construction */
/* is one u64; draw k is mix(state + k * 0x9E3779B97F4A7C15).                */
/* ------------------------------------------------------------------------ */

uint64_t sst_rng_init(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t s3);

/* ------------------------------------------------------------------------ */
/* Per-step operator: replaces sample_sphere_step (scatter.hpp:119-122,       */
/* scatter.cpp:152-177). n independent steps; vectors are xyz-interleaved.   */
/* rng_state[i] is the RandomStream state on entry and is advanced in place   */
/* by exactly the draws the reference consumes (7 / 24 / 46 per absorbed /   */
/* survived / survived+event outcome, plus retries).                          */
/* ------------------------------------------------------------------------ */

typedef struct {
    const double* sigma_t;   /* [n] world extinction */
    const double* g;         /* [n] */
    const double* phi;       /* [n] */
    const double* w_in;      /* [3n] unit incoming direction */
    const double* center;    /* [3n] */
    const double* r_sphere;  /* [n] */
    const uint8_t* with_event; /* [n] 0/1, or NULL = all with_event_default */
    uint64_t* rng_state;     /* [n] in/out */
} sst_step_in;

typedef struct {
    uint8_t* absorbed;       /* [n] */
    uint32_t* n_events;      /* [n] */
    double* exit_position;   /* [3n] */
    double* exit_direction;  /* [3n] */
    uint8_t* has_representative; /* [n] */
    double* rep_position;    /* [3n] */
    double* rep_direction;   /* [3n] */
    double* lambda_weight;   /* [n] */
} sst_step_out;

typedef struct {
    uint64_t length, path, event; /* DecodeCounters (scatter.hpp:18-25) */
} sst_decode_counters;

int sst_gpu_sphere_step_batch(sst_gpu_ctx* ctx, uint64_t n, const sst_step_in* in,
                              int with_event_default, sst_step_out* out, int ptr_kind,
                              sst_decode_counters* counters /* may be NULL; accumulated */);

/* ------------------------------------------------------------------------ */
/* Scene: mesh + medium + SDF per object, point light, camera, background.   */
/* SPEC.md:526-529 (Scene), mesh.hpp:15-30, sdf.hpp:19-33, optics.hpp:16-26. */
/* ------------------------------------------------------------------------ */

typedef struct {
    double sigma_t, g, phi; /* MediumParams; validated like optics.cpp:21-25 */
} sst_medium;

typedef struct {
    const double* positions;  /* [3 * n_vertices] */
    uint32_t n_vertices;
    const uint32_t* triangles; /* [3 * n_triangles], outward CCW winding */
    uint32_t n_triangles;
    sst_medium media[3];      /* per RGB channel */
    /* Conservative SDF grid of THIS object (SdfGrid, sdf.hpp:19-33):
     * values z-major (z*dy + y)*dx + x, negative inside, already reduced by
     * half the voxel diagonal. values == NULL asks the library to build it on
     * the GPU at `sdf_resolution` voxels along the largest axis (build_sdf,
     * sdf.cpp:20-58; bit-identical to the reference's FP64 build). */
    double sdf_origin[3];
    double sdf_voxel;
    uint32_t sdf_dims[3];
    const float* sdf_values;
    uint32_t sdf_resolution;
} sst_object_desc;

typedef struct {
    uint32_t n_objects;
    const sst_object_desc* objects;
    double light_position[3]; /* point light */
    double light_power[3];    /* Phi per channel; inverse-square falloff */
    double background[3];     /* radiance added when a path escapes */
    double cam_position[3];
    double cam_look_at[3];
    double cam_up[3];
    double cam_vfov_deg;
    uint32_t width, height;
    double r_min;             /* <= 0: max(2/sigma_t, 1.5 voxel) */
    uint32_t max_pt_events;   /* 0: 1e6 */
    uint32_t max_st_steps;    /* 0: 1e5 */
    /* Light model: 0 = point light at light_position, light_power =
     * Phi, inverse-square falloff; 1 = directional light: light_direction points TOWARD
     * the light (normalised here), light_power = irradiance E, no falloff, and the shadow
     * ray's optical depth is measured out to the last boundary exit. */
    uint32_t light_kind;
    double light_direction[3];
} sst_scene_desc;

/* Uploads the scene: builds the BVH on the host, builds missing SDFs on the
 * GPU, copies everything to device memory owned by the context. */
int sst_gpu_upload_scene(sst_gpu_ctx* ctx, const sst_scene_desc* scene);
/* Device footprint of the uploaded scene: bytes copied host->device by the last
 * sst_gpu_upload_scene (BVH nodes + triangles in both precisions, SDF grids,
 * medium tables), BVH node and triangle counts. */
int sst_gpu_scene_info(sst_gpu_ctx* ctx, uint64_t* h2d_bytes, uint32_t* n_nodes, uint32_t* n_triangles);
/* Copies back the SDF grid of object `obj` (values may be NULL to query the
 * dims/origin/voxel only). */
int sst_gpu_get_sdf(sst_gpu_ctx* ctx, uint32_t obj, double origin[3], double* voxel,
                    uint32_t dims[3], float* values);

/* PathStats plus bookkeeping. */
typedef struct {
    uint64_t paths;          /* traced (pixel, sample, channel) paths */
    uint64_t segments;       /* sphere_steps + pt_events */
    uint64_t sphere_steps;
    uint64_t pt_events;      /* delta-tracking collisions (PT, or ST fallback) */
    uint64_t decodes_length, decodes_path, decodes_event;
    uint64_t absorbed, escaped, capped, errors;
    uint64_t shadow_rays;
    /* work counters: nearest-hit traversals, BVH interior nodes visited, triangle
     * tests (nearest + shadow), live-lane loop iterations, warp loop iterations */
    uint64_t traversals, node_visits, triangle_tests, lane_iterations, warp_iterations;
    /* triangle tests of NEE shadow rays (part of triangle_tests); path-slot visits of
     * the wavefront logic pass */
    uint64_t shadow_triangle_tests, wavefront_slot_visits;
    double device_ms;        /* kernel time of the render call */
} sst_path_stats;

/* Renders samples [sample_begin, sample_end) of an spp_total frame and ADDS
 * into film_sum / film_sumsq ([3 * width * height], row 0 on top, RGB
 * interleaved; Image layout of image.hpp:13-29). Pointers are host or device
 * per ptr_kind (device: double, must be zeroed by the caller before the first
 * slab). RNG keys: camera jitter RandomStream(seed, kRenderPixel, pixel,
 * sample); path RandomStream(seed, kRenderChannel, pixel, 3*sample+channel).
 * Host pointers or a non-NULL stats make the call synchronous (stats accumulated,
 * including counters of earlier unread asynchronous calls). Device pointers with
 * stats == NULL return after enqueueing: consecutive calls pipeline on the
 * context's internal streams (long-path tails overlap the next slab); collect with
 * sst_gpu_read_stats, and only read the film after it or sst_gpu_synchronize. */
int sst_gpu_render(sst_gpu_ctx* ctx, int integrator, int nee, uint32_t spp_total,
                   uint32_t sample_begin, uint32_t sample_end, uint64_t seed, double* film_sum,
                   double* film_sumsq, int ptr_kind, sst_path_stats* stats);

/* Waits for all enqueued work, adds the counters accumulated since the last read
 * (and their device time) into *stats and resets them. */
int sst_gpu_read_stats(sst_gpu_ctx* ctx, sst_path_stats* stats);

/* Per-kernel device time (measurement aid for the roofline): with enable = 1 the
 * render / trace calls bracket every kernel launch with CUDA events on its own
 * stream and synchronise after each wavefront iteration (slower; for measurement
 * passes only); ms[k] / launches[k] accumulate per kernel kind k (SST_KT_*).
 * enable = 1 resets the accumulators, 0 stops; both first copy the current values
 * (after synchronising) into ms / launches when those are non-NULL. */
enum {
    SST_KT_WF_LOGIC = 0, SST_KT_WF_GEN = 1, SST_KT_WF_TRACE = 2, SST_KT_WF_SPHERE = 3,
    SST_KT_WF_SHADOW = 4, SST_KT_WF_RESET = 5, SST_KT_WF_TAIL = 6, SST_KT_MEGAKERNEL = 7,
    SST_KT_FILM = 8, SST_KT_COUNT = 9
};
int sst_gpu_kernel_timing(sst_gpu_ctx* ctx, int enable, double* ms, uint64_t* launches);

/* Per-path parity entry: traces n explicit (pixel, sample, channel) paths and
 * returns their radiance and segment counts (host pointers). */
int sst_gpu_trace_paths(sst_gpu_ctx* ctx, int integrator, int nee, uint64_t seed, uint64_t n,
                        const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                        double* radiance, uint32_t* segments, sst_path_stats* stats);
/* ... plus each path's exit state (exit_state: host double [6 n], may be NULL): the
 * position and direction when the path ended -- escape: the last boundary exit (or the
 * camera) and the escape direction; absorption or step cap: the collision point (a
 * sphere step's centre) and the incoming direction. The "per-path exit state" of the
 * parity bar; oracle/ref_shim.cpp ref_trace_paths_ex defines the same for the reference. */
int sst_gpu_trace_paths_ex(sst_gpu_ctx* ctx, int integrator, int nee, uint64_t seed, uint64_t n,
                           const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                           double* radiance, uint32_t* segments, double* exit_state, sst_path_stats* stats);

/* ------------------------------------------------------------------------ */
/* Verification hooks (csrc/verify.cuh): properties the fast paths rely on,    */
/* checked on the device against exact FP64 references.                       */
/* ------------------------------------------------------------------------ */

/* Conservativeness of the flight-culling rules (acceptance 8, extended
 * to every rule): n random in-medium free flights of the uploaded scene (half uniform
 * in an object's SDF box, half 1e-6..1e-1 below its surface; exponential lengths at
 * the medium's density) through the context precision's production predicates -- SDF
 * safe radius, skip-grid radius, convex / two-ball end-point containment -- and every
 * culled flight checked against all triangles in exact FP64 (no epsilon); every
 * queried radius against the exact point-mesh distance. Any violation is a bug. */
typedef struct {
    uint64_t flights;
    uint64_t culled_sdf, culled_skip, culled_endpoint_convex, culled_endpoint_twoball;
    uint64_t violations_sdf, violations_skip, violations_endpoint_convex, violations_endpoint_twoball;
    uint64_t radius_violations;      /* SDF safe radius > exact distance to the surface */
    uint64_t skip_radius_violations; /* skip-grid radius > exact distance */
    /* (v4) convex end point strictly inside the face planes of its SDF voxel */
    uint64_t culled_endpoint_planes, violations_endpoint_planes;
} sst_cull_report;
int sst_gpu_verify_culling(sst_gpu_ctx* ctx, uint64_t n, uint64_t seed, sst_cull_report* out);

/* NEE estimator identity (acceptance 7; single_sample_nee_weight,
 * SPEC.md:567-575) on brute-force unit-sphere walks (walk_sphere, sphere_walk.cpp:22-50)
 * at (sigma_t, g, phi): full per-event sum F = sum_k phi^k f(X_k) against the
 * single-representative estimate Lambda f(X_k*), k* ~ phi^k drawn by the dataset
 * generator's sample_representative (sphere_walk.cpp:75-102), averaged over `resamples`
 * draws per walk; f = point-light NEE term (light at light_pos, outside the sphere). */
typedef struct {
    uint64_t walks, events, resamples;
    double full_mean;      /* mean over walks of F */
    double single_mean;    /* mean over walks of the resampled single-representative estimate */
    double diff_stderr;    /* standard error of (single - full) per walk, over walks */
} sst_nee_identity_report;
int sst_gpu_nee_identity(sst_gpu_ctx* ctx, uint64_t walks, uint32_t resamples, double sigma_t, double g,
                         double phi, const double light_pos[3], uint64_t seed, sst_nee_identity_report* out);

/* ------------------------------------------------------------------------ */
/* Config 4: CVAE training-data generation, the device form of  */
/* generate_dataset (dataset.cpp:40-92) over walk_sphere / parameterize_exit /    */
/* sample_representative (sphere_walk.cpp:22-102). Sample i uses                 */
/* RandomStream(seed, kDataset, i) like the reference, so any index range can be */
/* generated on any GPU (sharding: disjoint [first_index, first_index + n)).      */
/* ------------------------------------------------------------------------ */

/* TrainingSample (dataset.hpp:17-27): 52 bytes, the SSWK record layout. */
typedef struct {
    float sigma_t, g, phi;
    uint32_t n_events;
    float cos_theta, alpha, beta;
    float rep_position[3];
    float rep_direction[3];
} sst_training_sample;

/* PhiSampler kinds (dataset.hpp:30-41). */
enum { SST_PHI_LOG_COMPLEMENT = 0, SST_PHI_FIXED = 1, SST_PHI_UNIFORM = 2 };

typedef struct {
    uint64_t walks;           /* samples generated */
    uint64_t events;          /* scattering events simulated (sum of N) */
    uint64_t replay_events;   /* events re-simulated to reach the representative */
    uint64_t max_events;      /* largest N */
    double device_ms;
} sst_dataset_stats;

/* Samples [first_index, first_index + n). Host or device `out` per ptr_kind.
 * Errors: SST_E_INVALID_ARGUMENT for the reference's range checks
 * (dataset.cpp:44-48); SST_E_RUNTIME when a walk exceeds 1e6 events. */
int sst_gpu_generate_dataset(sst_gpu_ctx* ctx, uint64_t n, double sigma_t_lo, double sigma_t_hi,
                             double g_lo, double g_hi, int phi_kind, double phi_a, double phi_b,
                             uint64_t seed, uint64_t first_index, sst_training_sample* out,
                             int ptr_kind, sst_dataset_stats* stats);

/* ------------------------------------------------------------------------ */
/* CVAE training: the device form of train_model            */
/* (cvae.cpp:234-347) -- minibatch AdamW on the ELBO (cvae.cpp:117-183,          */
/* mlp.cpp:100-228), FP64 like the reference. Same init (make_cvae, cvae.cpp:79-91),*/
/* validation split, per-epoch shuffle and per-sample latent noise streams       */
/* (RandomStream salts kTrainInit/Shuffle/Latent/Split, rng.hpp:55-58), the same   */
/* per-sample operation order and the same in-order batch gradient sums.         */
/* ------------------------------------------------------------------------ */

/* TrainConfig (cvae.hpp:101-114); depth/width/latent <= 0 keep the production  */
/* default of the model kind (CvaeSpec::production_default, cvae.cpp:51-57).     */
typedef struct {
    double lr;
    uint32_t batch_size;
    uint32_t epochs;
    double weight_decay;
    uint64_t seed;
    double validation_fraction;
    int32_t depth, width, latent;
} sst_train_config;

/* EpochStats (cvae.hpp:116-119). */
typedef struct {
    double train_loss;
    double validation_loss;
} sst_epoch_stats;

typedef struct {
    uint64_t steps;              /* AdamW steps taken (finite batches) */
    uint64_t rejected_batches;   /* batches skipped for a non-finite loss */
    uint64_t sample_passes;      /* training-sample forward+backward passes */
    uint32_t encoder_params, decoder_params;
    uint64_t dataset_fingerprint;  /* Dataset::fingerprint (dataset.cpp:32-38) */
    double device_ms;
} sst_train_stats;

/* The reference defaults (lr 1e-3, batch 512, 100 epochs, wd 1e-4, seed 1, 5% validation). */
void sst_train_config_default(sst_train_config* cfg);

/* train_model(kind, dataset, cfg) for kind 0 = LengthGen, 1 = PathGen, 2 = EventGen.
 * `samples` (host or device per ptr_kind) holds the n TrainingSample records of a
 * dataset whose header seed is `dataset_seed` (only used for the model's dataset
 * fingerprint). `epochs` (may be NULL) receives cfg->epochs EpochStats. When
 * `ssnn_path` is non-NULL the trained model is written with save_model
 * (cvae.cpp:349-377; encoder included iff include_encoder). `params_out` (may be
 * NULL) receives the f32-quantised encoder then decoder parameters as doubles in
 * flatten_parameters order (mlp.cpp:230-238). When `install` is non-zero the
 * trained decoder replaces the context's decoder of that kind (like
 * ScatterModels::load_dir on the saved files).
 * Errors mirror the reference: SST_E_INVALID_ARGUMENT for TrainConfig::validate /
 * CvaeSpec::validate / empty data / no training samples left, SST_E_RUNTIME when
 * every batch of an epoch is non-finite ("diverged") or the file cannot be
 * written; SST_E_INVALID_ARGUMENT also for specs beyond the device kernel's
 * limits (depth <= 4, width <= 32, latent <= 16). */
int sst_gpu_train_model(sst_gpu_ctx* ctx, int kind, const sst_training_sample* samples, uint64_t n,
                        int ptr_kind, uint64_t dataset_seed, const sst_train_config* cfg,
                        sst_epoch_stats* epochs, const char* ssnn_path, int include_encoder,
                        double* params_out, int install, sst_train_stats* stats);

/* The three decoders of a ScatterModels bundle (LengthGen, PathGen, EventGen) trained
 * CONCURRENTLY on one dataset and config (each kind on its own stream and cluster;
 * results identical to three sst_gpu_train_model calls). `epochs` (may be NULL) is
 * [3][cfg->epochs]; `stats` (may be NULL) is [3]. With out_dir non-NULL the models
 * are written as out_dir/{lengthgen,pathgen,eventgen}.ssnn (the layout
 * ScatterModels::load_dir reads, scatter.cpp:29-32); install != 0 makes them the
 * context's decoders. */
int sst_gpu_train_models(sst_gpu_ctx* ctx, const sst_training_sample* samples, uint64_t n, int ptr_kind,
                         uint64_t dataset_seed, const sst_train_config* cfg, sst_epoch_stats* epochs,
                         const char* out_dir, int include_encoder, int install, sst_train_stats* stats);

#ifdef __cplusplus
}
#endif

#endif /* SST_GPU_H */
