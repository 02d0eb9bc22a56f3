/*
 * oracle/sst_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (sstrace, /root/reference)
 * used as the parity checker for the CUDA path. Only tests/, bench.py's
 * cpu_baseline leg and __graft_entry__.smoke() may load liboracle.so.
 * Parity is pinned: tests/test_oracle_*.py check this restatement against
 * the reference library built from its own sources (oracle/_ref) and against
 * committed golden vectors generated from it (tests/golden/).
 */
#ifndef SST_ORACLE_H
#define SST_ORACLE_H

#include <stdint.h>

#include "sst_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

/* RandomStream (rng.hpp:15-50) */
typedef struct { uint64_t state; } so_rng;
uint64_t so_rng_init(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t s3);
uint64_t so_next_u64(so_rng* r);
double so_uniform(so_rng* r);
double so_normal(so_rng* r);
void so_rng_draws(uint64_t state, uint64_t n, uint64_t* u64, double* uni, double* nor);

/* optics (optics.cpp:27-75); rc: 0 ok, SST_E_DOMAIN on domain error */
int so_hg_eval(double g, double c, double* out);
int so_hg_sample_cos(double g, double u, double* out);
int so_hg_sample(double g, const double w[3], double u1, double u2, double out[3]);
int so_transmittance(double sigma_t, double d, double* out);
int so_sample_free_path(double sigma_t, double xi, double* out);
int so_absorption_prob(uint64_t n, double phi, double* out);
double so_representative_weight_sum(uint64_t n, double phi);
double so_softplus(double x);

/* models (cvae.cpp / mlp.cpp / scatter.cpp) */
typedef struct so_models so_models;
int so_models_load_dir(const char* dir, so_models** out);
void so_models_free(so_models* m);
void so_models_counters(const so_models* m, uint64_t out[3]);
int so_cvae_decode(const so_models* m, int kind, const double* z, const double* c, double* mu,
                   double* lv);
int so_to_world(double ct, double alpha, double beta, const double w_in[3], const double center[3],
                double r, double psi, double pos[3], double dir[3]);
/* Same structs as the C ABI; rng_state advanced in place. */
int so_sphere_step_batch(so_models* m, uint64_t n, const sst_step_in* in, int with_event_default,
                         sst_step_out* out);

/* geometry */
double so_query_safe_radius(const double origin[3], double voxel, const uint32_t dims[3],
                            const float* values, const double p[3]);
/* Brute-force conservative SDF build (sdf.cpp:20-58 semantics). Two-phase:
 * values == NULL only fills origin/voxel/dims. */
int so_build_sdf(const double* pos, uint32_t nv, const uint32_t* tris, uint32_t nt,
                 uint32_t resolution, double origin[3], double* voxel, uint32_t dims[3],
                 float* values);

/* scene + integrators */
typedef struct so_scene so_scene;
int so_scene_create(const sst_scene_desc* d, so_scene** out);
void so_scene_free(so_scene* s);
int so_bvh_intersect(const so_scene* s, const double o[3], const double d[3], double t_min,
                     double t_max, double* t, int64_t* tri);
int so_trace_paths(const so_scene* s, so_models* m, int integrator, int nee, uint64_t seed,
                   uint64_t n, const uint32_t* pixel, const uint32_t* sample,
                   const uint8_t* channel, double* radiance, uint32_t* segments,
                   sst_path_stats* stats);
/* so_trace_paths plus each path's exit state (double [6 n]: final position, direction). */
int so_trace_paths_ex(const so_scene* s, so_models* m, int integrator, int nee, uint64_t seed,
                      uint64_t n, const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                      double* radiance, uint32_t* segments, double* exit_state, sst_path_stats* stats);

/* Config 4: training-data generation (dataset.cpp:40-92 generate_dataset,
 * sphere_walk.cpp:22-102). Record layout = TrainingSample (dataset.hpp:17-27). */
typedef struct {
    float sigma_t, g, phi;
    uint32_t n_events;
    float cos_theta, alpha, beta;
    float rep_position[3];
    float rep_direction[3];
} so_sample;
int so_generate_dataset(uint64_t n, double s_lo, double s_hi, double g_lo, double g_hi, int phi_kind,
                        double phi_a, double phi_b, uint64_t seed, uint64_t first_index, so_sample* out);

/* CVAE training (train_model, cvae.cpp:234-347); params_out = f32-quantised encoder then decoder. */
int so_train_model(int kind, const so_sample* samples, uint64_t n, const sst_train_config* cfg,
                   sst_epoch_stats* epochs, double* params_out);
uint64_t so_dataset_fingerprint(const so_sample* s, uint64_t n, uint64_t seed);

const char* so_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
