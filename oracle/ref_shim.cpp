// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE (checker + CPU baseline), never shipped.
//
// An extern "C" shim over the reference library (compiled from
// /root/reference/proj/core/src by oracle/Makefile into oracle/_ref/), plus the
// integrator the reference declares but does not ship (proj/core/CMakeLists.txt:14,16
// list src/scene.cpp and src/render.cpp, which are missing). The integrator is
// restated from SPEC.md:540-566 and composed ONLY of reference functions:
//   Bvh::intersect / intersect_all (bvh.cpp:115-179), query_safe_radius (sdf.cpp:60-69),
//   sample_sphere_step (scatter.cpp:152-177), sample_free_path / hg_sample /
//   hg_eval / transmittance (optics.cpp:27-60), RandomStream (rng.hpp:15-50),
//   parallel_for (parallel.hpp:27-51).
// The exact loop semantics (draw order, NEE weighting, caps, RNG keys) are fixed in
// DESIGN.md "Integrator semantics" and are shared bit-for-bit with oracle/sst_oracle.c
// and the CUDA kernels.

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sst/bvh.hpp"
#include "sst/cvae.hpp"
#include "sst/dataset.hpp"
#include "sst/image.hpp"
#include "sst/mesh.hpp"
#include "sst/optics.hpp"
#include "sst/parallel.hpp"
#include "sst/rng.hpp"
#include "sst/scatter.hpp"
#include "sst/sdf.hpp"
#include "sst/sphere_walk.hpp"
#include "sst_gpu.h"

using namespace sst;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SST_E_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SST_E_DOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SST_E_RUNTIME;
    }
}

RandomStream make_stream(const uint64_t* key, uint64_t skip) {
    RandomStream r(key[0], key[1], key[2], key[3]);
    for (uint64_t i = 0; i < skip; ++i) r.next_u64();
    return r;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- RNG (rng.hpp)
void ref_rng_u64(const uint64_t key[4], uint64_t skip, uint64_t n, uint64_t* out) {
    RandomStream r = make_stream(key, skip);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_rng_uniform(const uint64_t key[4], uint64_t skip, uint64_t n, double* out) {
    RandomStream r = make_stream(key, skip);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
void ref_rng_normal(const uint64_t key[4], uint64_t skip, uint64_t n, double* out) {
    RandomStream r = make_stream(key, skip);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.normal();
}

// ---------------------------------------------------------------- optics (optics.cpp)
int ref_hg_eval(double g, double c, double* out) { return guarded([&] { *out = hg_eval(g, c); }); }
int ref_hg_sample_cos(double g, double u, double* out) {
    return guarded([&] { *out = hg_sample_cos(g, u); });
}
int ref_hg_sample(double g, const double w[3], double u1, double u2, double out[3]) {
    return guarded([&] {
        const Vec3 v = hg_sample(g, Vec3(w[0], w[1], w[2]), u1, u2);
        out[0] = v.x; out[1] = v.y; out[2] = v.z;
    });
}
int ref_transmittance(double s, double d, double* out) {
    return guarded([&] { *out = transmittance(s, d); });
}
int ref_sample_free_path(double s, double xi, double* out) {
    return guarded([&] { *out = sample_free_path(s, xi); });
}
int ref_absorption_prob(uint64_t n, double phi, double* out) {
    return guarded([&] { *out = absorption_prob(n, phi); });
}
int ref_representative_weight_sum(uint64_t n, double phi, double* out) {
    return guarded([&] { *out = representative_weight_sum(n, phi); });
}
double ref_softplus(double x) { return softplus(x); }
int ref_rescale_sigma(double s, double r, double* out) {
    return guarded([&] { *out = rescale_sigma(s, r); });
}
int ref_test_absorption(uint64_t n, double phi, double u) { return test_absorption(n, phi, u) ? 1 : 0; }

int ref_to_world(double cos_theta, double alpha, double beta, const double w_in[3],
                 const double center[3], double r, double psi, double pos[3], double dir[3]) {
    return guarded([&] {
        const WorldExit we = to_world(cos_theta, alpha, beta, Vec3(w_in[0], w_in[1], w_in[2]),
                                      Vec3(center[0], center[1], center[2]), r, psi);
        pos[0] = we.position.x; pos[1] = we.position.y; pos[2] = we.position.z;
        dir[0] = we.direction.x; dir[1] = we.direction.y; dir[2] = we.direction.z;
    });
}

// parameterize_exit on a synthetic record (sphere_walk.cpp:52-73).
void ref_parameterize_exit(const double w_in[3], const double exit_pos[3], const double exit_dir[3],
                           double out[3]) {
    WalkRecord rec;
    rec.events.push_back({Vec3(0, 0, 0), Vec3(w_in[0], w_in[1], w_in[2])});
    rec.exit_position = Vec3(exit_pos[0], exit_pos[1], exit_pos[2]);
    rec.exit_direction = Vec3(exit_dir[0], exit_dir[1], exit_dir[2]);
    rec.radius = 1.0;
    const ExitParams p = parameterize_exit(rec);
    out[0] = p.cos_theta; out[1] = p.alpha; out[2] = p.beta;
}

// ---------------------------------------------------------------- models (cvae.cpp / scatter.cpp)
void* ref_models_load(const char* dir) {
    ScatterModels* m = nullptr;
    const int rc = guarded([&] { m = new ScatterModels(ScatterModels::load_dir(dir)); });
    return rc == 0 ? m : nullptr;
}
void ref_models_free(void* h) { delete static_cast<ScatterModels*>(h); }
void ref_models_counters(void* h, uint64_t out[3]) {
    auto* m = static_cast<ScatterModels*>(h);
    out[0] = m->counters.length; out[1] = m->counters.path; out[2] = m->counters.event;
}
void ref_models_reset_counters(void* h) { static_cast<ScatterModels*>(h)->counters.reset(); }

// Decoder mean/log-var (cvae_decode, cvae.cpp:93-98) for one model kind.
int ref_cvae_decode(void* h, int kind, const double* z, const double* c, double* mu, double* lv) {
    return guarded([&] {
        auto* m = static_cast<ScatterModels*>(h);
        const CvaeModel& model = kind == 0 ? m->length : (kind == 1 ? m->path : m->event);
        const GaussianHead head = cvae_decode(model, std::span<const double>(z, model.spec.latent),
                                              std::span<const double>(c, model.spec.p_in));
        for (size_t i = 0; i < head.mu.size(); ++i) { mu[i] = head.mu[i]; lv[i] = head.log_var[i]; }
    });
}

// Batch of independent sample_sphere_step calls (scatter.cpp:152-177).
// keys: [4n] RandomStream ctor words; skip: draws consumed before the step.
// draws_used[i] = RNG draws consumed by the step.
int ref_sphere_step_batch(void* h, uint64_t n, const double* sigma_t, const double* g,
                          const double* phi, const double* w_in, const double* center,
                          const double* r, const uint8_t* with_event, const uint64_t* keys,
                          const uint64_t* skip, uint8_t* absorbed, uint32_t* n_events,
                          double* exit_pos, double* exit_dir, uint8_t* has_rep, double* rep_pos,
                          double* rep_dir, double* lambda, uint64_t* draws_used) {
    auto* m = static_cast<ScatterModels*>(h);
    return guarded([&] {
        for (uint64_t i = 0; i < n; ++i) {
            RandomStream rs = make_stream(keys + 4 * i, skip ? skip[i] : 0);
            // count draws through a probe copy: RandomStream is a value type.
            const SphereStepOutcome o = sample_sphere_step(
                *m, sigma_t[i], g[i], phi[i], Vec3(w_in[3 * i], w_in[3 * i + 1], w_in[3 * i + 2]),
                Vec3(center[3 * i], center[3 * i + 1], center[3 * i + 2]), r[i],
                with_event ? with_event[i] != 0 : true, rs);
            if (draws_used) {
                RandomStream probe = make_stream(keys + 4 * i, skip ? skip[i] : 0);
                const uint64_t after = rs.next_u64();
                uint64_t k = 0;
                while (probe.next_u64() != after && k < 100000) ++k;
                draws_used[i] = k;
            }
            absorbed[i] = o.absorbed;
            n_events[i] = o.n_events;
            const Vec3* v[4] = {&o.exit_position_world, &o.exit_direction_world,
                                &o.rep_position_world, &o.rep_direction_world};
            double* dst[4] = {exit_pos, exit_dir, rep_pos, rep_dir};
            for (int a = 0; a < 4; ++a) {
                dst[a][3 * i] = v[a]->x; dst[a][3 * i + 1] = v[a]->y; dst[a][3 * i + 2] = v[a]->z;
            }
            has_rep[i] = o.has_representative;
            lambda[i] = o.lambda_weight;
        }
    });
}

// Deterministic desk-scale weights: generate_dataset + train_model
// for the three kinds, saved as SSNN (with encoder) into outdir.
int ref_make_weights(const char* outdir, uint64_t n_samples, uint32_t epochs, uint64_t data_seed,
                     uint64_t train_seed, double* final_val_loss /* [3] */) {
    return guarded([&] {
        PhiSampler phi;  // LogComplement [-5, -0.5] (dataset.hpp:30-41)
        const Dataset ds = generate_dataset(n_samples, 0.0, 200.0, -1.0, 1.0, phi, data_seed);
        const ModelKind kinds[3] = {ModelKind::kLength, ModelKind::kPath, ModelKind::kEvent};
        for (int k = 0; k < 3; ++k) {
            TrainConfig cfg;
            cfg.epochs = epochs;
            cfg.seed = train_seed;
            const TrainResult res = train_model(kinds[k], ds, cfg);
            if (final_val_loss) final_val_loss[k] = res.epochs.back().validation_loss;
            save_model(std::string(outdir) + "/" + model_kind_name(kinds[k]) + ".ssnn", res.model,
                       true);
        }
    });
}

// generate_dataset (dataset.cpp:40-92) -> TrainingSample records (52 B each, dataset.hpp:17-27).
int ref_generate_dataset(uint64_t n, double s_lo, double s_hi, double g_lo, double g_hi, int phi_kind,
                         double phi_a, double phi_b, uint64_t seed, void* out) {
    return guarded([&] {
        PhiSampler ps;
        ps.kind = static_cast<PhiSampler::Kind>(phi_kind);
        ps.a = phi_a;
        ps.b = phi_b;
        const Dataset ds = generate_dataset(n, s_lo, s_hi, g_lo, g_hi, ps, seed);
        static_assert(sizeof(TrainingSample) == 52, "TrainingSample layout");
        std::memcpy(out, ds.samples.data(), n * sizeof(TrainingSample));
    });
}

// train_model (cvae.cpp:234-347) on n TrainingSample records; writes the SSNN file
// (save_model, cvae.cpp:349-377) when path != NULL, the per-epoch stats, and the
// f32-quantised encoder+decoder parameters in flatten_parameters order.
int ref_train_model(int kind, const void* samples, uint64_t n, uint64_t dataset_seed,
                    const sst_train_config* c, const char* path, int include_encoder,
                    sst_epoch_stats* epochs, double* params_out, uint64_t* fingerprint) {
    return guarded([&] {
        Dataset ds;
        ds.header.count = n;
        ds.header.seed = dataset_seed;
        ds.samples.resize(n);
        std::memcpy(ds.samples.data(), samples, n * sizeof(TrainingSample));
        TrainConfig cfg;
        cfg.lr = c->lr;
        cfg.batch_size = c->batch_size;
        cfg.epochs = c->epochs;
        cfg.weight_decay = c->weight_decay;
        cfg.seed = c->seed;
        cfg.validation_fraction = c->validation_fraction;
        cfg.depth = c->depth;
        cfg.width = c->width;
        cfg.latent = c->latent;
        const TrainResult res = train_model(static_cast<ModelKind>(kind), ds, cfg);
        if (epochs)
            for (size_t e = 0; e < res.epochs.size(); ++e)
                epochs[e] = {res.epochs[e].train_loss, res.epochs[e].validation_loss};
        if (params_out) {
            const auto a = flatten_parameters(res.model.encoder);
            const auto b = flatten_parameters(res.model.decoder);
            std::memcpy(params_out, a.data(), a.size() * sizeof(double));
            std::memcpy(params_out + a.size(), b.data(), b.size() * sizeof(double));
        }
        if (fingerprint) *fingerprint = res.model.dataset_fingerprint;
        if (path) save_model(path, res.model, include_encoder != 0);
    });
}

// save_dataset (dataset.cpp:94-119) of n records (for SSWK byte-compatibility tests).
int ref_save_dataset(const char* path, uint64_t n, double s_lo, double s_hi, double g_lo, double g_hi,
                     int phi_kind, double phi_a, double phi_b, uint64_t seed, const void* samples) {
    return guarded([&] {
        Dataset ds;
        ds.header.count = n;
        ds.header.sigma_t_lo = static_cast<float>(s_lo);
        ds.header.sigma_t_hi = static_cast<float>(s_hi);
        ds.header.g_lo = static_cast<float>(g_lo);
        ds.header.g_hi = static_cast<float>(g_hi);
        ds.header.phi.kind = static_cast<PhiSampler::Kind>(phi_kind);
        ds.header.phi.a = phi_a;
        ds.header.phi.b = phi_b;
        ds.header.seed = seed;
        ds.samples.resize(n);
        std::memcpy(ds.samples.data(), samples, n * sizeof(TrainingSample));
        save_dataset(path, ds);
    });
}

// load_dataset (dataset.cpp:121-151): hdr = {version, sigma_t_lo, sigma_t_hi, g_lo, g_hi,
// phi_kind, phi_a, phi_b}; the records are copied when samples != nullptr.
int ref_load_dataset(const char* path, double hdr[8], uint64_t* count, uint64_t* seed, void* samples,
                     uint64_t capacity) {
    return guarded([&] {
        const Dataset ds = load_dataset(path);
        const DatasetHeader& h = ds.header;
        const double v[8] = {double(h.version), h.sigma_t_lo, h.sigma_t_hi, h.g_lo, h.g_hi,
                             double(static_cast<uint32_t>(h.phi.kind)), h.phi.a, h.phi.b};
        std::memcpy(hdr, v, sizeof v);
        *count = h.count;
        *seed = h.seed;
        if (samples) {
            if (capacity < ds.samples.size()) throw std::invalid_argument("capacity");
            std::memcpy(samples, ds.samples.data(), ds.samples.size() * sizeof(TrainingSample));
        }
    });
}

// export_dataset_csv (dataset.cpp:153-164) of n records.
int ref_export_dataset_csv(const char* path, uint64_t n, const void* samples) {
    return guarded([&] {
        Dataset ds;
        ds.header.count = n;
        ds.samples.resize(n);
        std::memcpy(ds.samples.data(), samples, n * sizeof(TrainingSample));
        export_dataset_csv(path, ds);
    });
}

// save_png (image.cpp:101-138) for the PNG byte-compatibility test. (The reference's PFM
// writers/reader use iostream number formatting, which crashes when this library is
// dlopen'ed into Python next to the system libstdc++; the PFM tests check the format directly.)
int ref_save_png(const char* path, uint32_t w, uint32_t h, const float* rgb) {
    return guarded([&] {
        Image img(w, h);
        std::memcpy(img.pixels.data(), rgb, static_cast<size_t>(w) * h * 3 * sizeof(float));
        save_png(path, img);
    });
}
// Ground-truth unit-sphere walks (sphere_walk.cpp:22-50) -> (N, cos_theta, alpha, beta).
int ref_walk_stats(double sigma_t, double g, uint64_t seed, uint64_t n, uint32_t* n_events,
                   double* exit_params) {
    return guarded([&] {
        for (uint64_t i = 0; i < n; ++i) {
            RandomStream rng(seed, 0x08, i);
            const WalkRecord w = walk_unit_sphere(sigma_t, g, rng);
            const ExitParams p = parameterize_exit(w);
            n_events[i] = w.n_events();
            exit_params[3 * i] = p.cos_theta; exit_params[3 * i + 1] = p.alpha;
            exit_params[3 * i + 2] = p.beta;
        }
    });
}

// ---------------------------------------------------------------- meshes (mesh.cpp)
// Two-phase: call with positions == NULL to get the counts.
static void export_mesh(const TriangleMesh& m, double* pos, uint32_t* tris, uint32_t* nv, uint32_t* nt) {
    *nv = static_cast<uint32_t>(m.positions.size());
    *nt = static_cast<uint32_t>(m.faces.size());
    if (!pos) return;
    for (size_t i = 0; i < m.positions.size(); ++i) {
        pos[3 * i] = m.positions[i].x; pos[3 * i + 1] = m.positions[i].y; pos[3 * i + 2] = m.positions[i].z;
    }
    for (size_t i = 0; i < m.faces.size(); ++i)
        for (int k = 0; k < 3; ++k) tris[3 * i + k] = m.faces[i][k];
}
void ref_make_icosphere(int subdiv, double radius, double* pos, uint32_t* tris, uint32_t* nv,
                        uint32_t* nt) {
    export_mesh(make_icosphere(subdiv, radius), pos, tris, nv, nt);
}
void ref_make_bumpy_sphere(int subdiv, double radius, double amp, double freq, double* pos,
                           uint32_t* tris, uint32_t* nv, uint32_t* nt) {
    export_mesh(make_bumpy_sphere(subdiv, radius, amp, freq), pos, tris, nv, nt);
}

static TriangleMesh import_mesh(const double* pos, uint32_t nv, const uint32_t* tris, uint32_t nt) {
    TriangleMesh m;
    m.positions.resize(nv);
    for (uint32_t i = 0; i < nv; ++i) m.positions[i] = Vec3(pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]);
    m.faces.resize(nt);
    for (uint32_t i = 0; i < nt; ++i) m.faces[i] = {tris[3 * i], tris[3 * i + 1], tris[3 * i + 2]};
    m.compute_face_normals();
    return m;
}

// ---------------------------------------------------------------- BVH (bvh.cpp)
int ref_bvh_intersect(const double* pos, uint32_t nv, const uint32_t* tris, uint32_t nt, uint64_t n,
                      const double* orig, const double* dir, const double* tmax, double t_min,
                      double* t_out, int64_t* tri_out, uint32_t* n_all) {
    return guarded([&] {
        const TriangleMesh m = import_mesh(pos, nv, tris, nt);
        const Bvh bvh(m);
        std::vector<Hit> hits;
        for (uint64_t i = 0; i < n; ++i) {
            Ray ray{Vec3(orig[3 * i], orig[3 * i + 1], orig[3 * i + 2]),
                    Vec3(dir[3 * i], dir[3 * i + 1], dir[3 * i + 2]), tmax ? tmax[i] : 1e300};
            const auto h = bvh.intersect(ray, t_min);
            t_out[i] = h ? h->t : -1.0;
            tri_out[i] = h ? static_cast<int64_t>(h->triangle) : -1;
            if (n_all) {
                bvh.intersect_all(ray, hits, t_min);
                n_all[i] = static_cast<uint32_t>(hits.size());
            }
        }
    });
}

// ---------------------------------------------------------------- SDF (sdf.cpp)
// Two-phase: values == NULL returns dims/origin/voxel only.
int ref_build_sdf(const double* pos, uint32_t nv, const uint32_t* tris, uint32_t nt,
                  uint32_t resolution, double origin[3], double* voxel, uint32_t dims[3],
                  float* values) {
    return guarded([&] {
        const TriangleMesh m = import_mesh(pos, nv, tris, nt);
        const Bvh bvh(m);
        const SdfGrid g = build_sdf(m, bvh, resolution);
        origin[0] = g.origin.x; origin[1] = g.origin.y; origin[2] = g.origin.z;
        *voxel = g.voxel_size;
        for (int a = 0; a < 3; ++a) dims[a] = g.dims[a];
        if (values) std::memcpy(values, g.values.data(), g.values.size() * sizeof(float));
    });
}

double ref_query_safe_radius(const double origin[3], double voxel, const uint32_t dims[3],
                             const float* values, const double p[3]) {
    SdfGrid g;
    g.origin = Vec3(origin[0], origin[1], origin[2]);
    g.voxel_size = voxel;
    for (int a = 0; a < 3; ++a) g.dims[a] = dims[a];
    g.values.assign(values, values + static_cast<size_t>(dims[0]) * dims[1] * dims[2]);
    return query_safe_radius(g, Vec3(p[0], p[1], p[2]));
}

// ---------------------------------------------------------------- integrator
struct RefScene {
    TriangleMesh mesh;
    std::unique_ptr<Bvh> bvh;
    std::vector<uint32_t> tri_obj;
    std::vector<SdfGrid> sdf;
    std::vector<MediumParams> media;  // [obj*3 + channel]
    Vec3 light_pos;
    bool directional;
    Vec3 light_dir;
    double light_power[3];
    double background[3];
    Vec3 cam_pos, cam_fwd, cam_right, cam_up;
    double tan_half, aspect;
    uint32_t width, height;
    double r_min_override;
    uint32_t max_pt, max_st;
};

void* ref_scene_create(const sst_scene_desc* d) {
    RefScene* s = nullptr;
    const int rc = guarded([&] {
        auto sc = std::make_unique<RefScene>();
        for (uint32_t o = 0; o < d->n_objects; ++o) {
            const sst_object_desc& od = d->objects[o];
            const uint32_t base = static_cast<uint32_t>(sc->mesh.positions.size());
            for (uint32_t i = 0; i < od.n_vertices; ++i)
                sc->mesh.positions.push_back(
                    Vec3(od.positions[3 * i], od.positions[3 * i + 1], od.positions[3 * i + 2]));
            for (uint32_t i = 0; i < od.n_triangles; ++i) {
                sc->mesh.faces.push_back({base + od.triangles[3 * i], base + od.triangles[3 * i + 1],
                                          base + od.triangles[3 * i + 2]});
                sc->tri_obj.push_back(o);
            }
            for (int c = 0; c < 3; ++c) {
                MediumParams mp{od.media[c].sigma_t, od.media[c].g, od.media[c].phi};
                mp.validate();
                sc->media.push_back(mp);
            }
            SdfGrid g;
            if (od.sdf_values) {
                g.origin = Vec3(od.sdf_origin[0], od.sdf_origin[1], od.sdf_origin[2]);
                g.voxel_size = od.sdf_voxel;
                for (int a = 0; a < 3; ++a) g.dims[a] = od.sdf_dims[a];
                g.values.assign(od.sdf_values, od.sdf_values + static_cast<size_t>(g.dims[0]) *
                                                                   g.dims[1] * g.dims[2]);
            } else {
                const TriangleMesh single = import_mesh(od.positions, od.n_vertices, od.triangles,
                                                        od.n_triangles);
                const Bvh b(single);
                g = build_sdf(single, b, od.sdf_resolution ? od.sdf_resolution : 64);
            }
            sc->sdf.push_back(std::move(g));
        }
        sc->mesh.compute_face_normals();
        sc->bvh = std::make_unique<Bvh>(sc->mesh);
        sc->light_pos = Vec3(d->light_position[0], d->light_position[1], d->light_position[2]);
        sc->directional = d->light_kind == 1;
        if (sc->directional) {
            const Vec3 ld(d->light_direction[0], d->light_direction[1], d->light_direction[2]);
            sc->light_dir = ld / std::sqrt(dot(ld, ld));
        }
        for (int c = 0; c < 3; ++c) {
            sc->light_power[c] = d->light_power[c];
            sc->background[c] = d->background[c];
        }
        sc->cam_pos = Vec3(d->cam_position[0], d->cam_position[1], d->cam_position[2]);
        const Vec3 look(d->cam_look_at[0], d->cam_look_at[1], d->cam_look_at[2]);
        const Vec3 up(d->cam_up[0], d->cam_up[1], d->cam_up[2]);
        sc->cam_fwd = normalize(look - sc->cam_pos);
        sc->cam_right = normalize(cross(sc->cam_fwd, up));
        sc->cam_up = cross(sc->cam_right, sc->cam_fwd);
        sc->tan_half = std::tan(d->cam_vfov_deg * 3.14159265358979323846 / 360.0);
        sc->width = d->width;
        sc->height = d->height;
        sc->aspect = static_cast<double>(d->width) / static_cast<double>(d->height);
        sc->r_min_override = d->r_min;
        sc->max_pt = d->max_pt_events ? d->max_pt_events : 1000000u;
        sc->max_st = d->max_st_steps ? d->max_st_steps : 100000u;
        s = sc.release();
    });
    return rc == 0 ? s : nullptr;
}
void ref_scene_free(void* h) { delete static_cast<RefScene*>(h); }

struct PathResult {
    double radiance = 0.0;
    uint32_t segments = 0, sphere_steps = 0, pt_events = 0, shadow = 0;
    int end = 0;  // 0 escaped, 1 absorbed, 2 capped
    // exit state: position and direction when the path ends (escape: the last boundary
    // exit / camera and the escape direction; absorption or cap: the collision point and
    // the incoming direction)
    Vec3 x, w;
};

static double r_min_for(const RefScene& s, int obj, int c) {
    if (s.r_min_override > 0.0) return s.r_min_override;
    const double sig = s.media[obj * 3 + c].sigma_t;
    if (!(sig > 0.0)) return 1e300;
    return std::fmax(2.0 / sig, 1.5 * s.sdf[obj].voxel_size);
}

// NEE toward the point light from p (inside object obj) with incoming direction w:
// weight * Phi * hg(g, w.wl) * exp(-tau) / d^2, tau accumulated over the sorted
// hits of intersect_all on [p, x_L].
static double nee_term(const RefScene& s, int obj, int c, const Vec3& p, const Vec3& w,
                       double weight, std::vector<Hit>& hits) {
    // directional light: to the last boundary exit, irradiance, no 1/d^2
    const Vec3 to_l = s.directional ? s.light_dir : s.light_pos - p;
    const double d2 = s.directional ? 1.0 : dot(to_l, to_l);
    const double d = s.directional ? 1e30 : std::sqrt(d2);
    const Vec3 wl = s.directional ? s.light_dir : to_l / d;
    Ray ray{p, wl, d};
    s.bvh->intersect_all(ray, hits);
    double tau = 0.0, t_prev = 0.0;
    int cur = obj;
    for (const Hit& h : hits) {
        if (cur >= 0) tau += s.media[cur * 3 + c].sigma_t * (h.t - t_prev);
        const int j = static_cast<int>(s.tri_obj[h.triangle]);
        cur = (cur == j) ? -1 : j;
        t_prev = h.t;
    }
    if (cur >= 0) tau += s.media[cur * 3 + c].sigma_t * (d - t_prev);
    const double phase = hg_eval(s.media[obj * 3 + c].g, dot(w, wl));
    return weight * s.light_power[c] * phase * transmittance(1.0, tau) / d2;
}

static PathResult trace_one(const RefScene& s, const ScatterModels* models, int integrator, bool nee,
                            uint64_t seed, uint32_t pixel, uint32_t sample, int c) {
    PathResult res;
    // Camera ray (DESIGN.md "Integrator semantics" §camera).
    RandomStream cam(seed, stream_salt::kRenderPixel, pixel, sample);
    const double jx = cam.uniform();
    const double jy = cam.uniform();
    const uint32_t px = pixel % s.width, py = pixel / s.width;
    const double sx = (2.0 * (px + jx) / s.width - 1.0) * s.tan_half * s.aspect;
    const double sy = (1.0 - 2.0 * (py + jy) / s.height) * s.tan_half;
    Vec3 x = s.cam_pos;
    Vec3 w = normalize(s.cam_fwd + s.cam_right * sx + s.cam_up * sy);

    RandomStream rng(seed, stream_salt::kRenderChannel, pixel, 3ull * sample + c);
    std::vector<Hit> hits;
    const uint32_t cap = integrator == SST_INTEGRATOR_ST ? s.max_st : s.max_pt;

    for (;;) {  // outside all objects
        const auto entry = s.bvh->intersect(Ray{x, w, 1e300});
        if (!entry) {
            res.radiance += s.background[c];
            res.end = 0;
            res.x = x;
            res.w = w;
            return res;
        }
        const int obj = static_cast<int>(s.tri_obj[entry->triangle]);
        const MediumParams& m = s.media[obj * 3 + c];
        const double r_min = r_min_for(s, obj, c);
        x = x + w * entry->t;
        for (;;) {  // inside obj: free flight
            const double t_free = m.sigma_t > 0.0 ? sample_free_path(m.sigma_t, rng.uniform()) : 1e300;
            const auto exit = s.bvh->intersect(Ray{x, w, t_free});
            if (exit) {
                x = x + w * exit->t;
                break;  // left the medium (index-matched boundary)
            }
            x = x + w * t_free;  // collision
            if (res.segments >= cap) {
                res.radiance = 0.0;  // dropped
                res.end = 2;
                res.x = x;
                res.w = w;
                return res;
            }
            ++res.segments;
            double r = 0.0;
            if (integrator == SST_INTEGRATOR_ST) r = query_safe_radius(s.sdf[obj], x);
            if (integrator == SST_INTEGRATOR_ST && r > r_min) {
                ++res.sphere_steps;
                const SphereStepOutcome o =
                    sample_sphere_step(*models, m.sigma_t, m.g, m.phi, w, x, r, nee, rng);
                if (o.absorbed) {
                    res.end = 1;
                    res.x = x;
                    res.w = w;
                    return res;
                }
                if (nee) {
                    res.radiance += nee_term(s, obj, c, o.rep_position_world, o.rep_direction_world,
                                             o.lambda_weight, hits);
                    ++res.shadow;
                }
                x = o.exit_position_world;
                w = o.exit_direction_world;
            } else {
                ++res.pt_events;
                if (!(rng.uniform() < m.phi)) {  // Russian roulette by albedo
                    res.end = 1;
                    res.x = x;
                    res.w = w;
                    return res;
                }
                if (nee) {
                    res.radiance += nee_term(s, obj, c, x, w, 1.0, hits);
                    ++res.shadow;
                }
                const double u1 = rng.uniform();
                const double u2 = rng.uniform();
                w = hg_sample(m.g, w, u1, u2);
            }
        }
    }
}

// Traces n explicit paths (parallel_for over paths; SST_THREADS threads).
int ref_trace_paths_ex(void* scene, void* models, int integrator, int nee, uint64_t seed, uint64_t n,
                       const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                       double* radiance, uint32_t* segments, double* exit_state, sst_path_stats* stats);

int ref_trace_paths(void* scene, void* models, int integrator, int nee, uint64_t seed, uint64_t n,
                    const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                    double* radiance, uint32_t* segments, sst_path_stats* stats) {
    return ref_trace_paths_ex(scene, models, integrator, nee, seed, n, pixel, sample, channel, radiance, segments,
                              nullptr, stats);
}

// ... and each path's exit state (exit_state: double [6 n], position then direction).
int ref_trace_paths_ex(void* scene, void* models, int integrator, int nee, uint64_t seed, uint64_t n,
                       const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                       double* radiance, uint32_t* segments, double* exit_state, sst_path_stats* stats) {
    auto* s = static_cast<RefScene*>(scene);
    auto* m = static_cast<ScatterModels*>(models);
    if (integrator == SST_INTEGRATOR_ST && !m) {
        g_err = "sphere tracing requires models";
        return SST_E_INVALID_ARGUMENT;
    }
    std::atomic<uint64_t> steps{0}, events{0}, absorbed{0}, escaped{0}, capped{0}, shadow{0};
    std::atomic<int> failed{0};
    std::string fail_msg;
    parallel_for(n, [&](uint64_t i) {
        try {
            const PathResult r = trace_one(*s, m, integrator, nee != 0, seed, pixel[i], sample[i], channel[i]);
            radiance[i] = r.radiance;
            if (segments) segments[i] = r.segments;
            if (exit_state) {
                double* e = exit_state + 6 * i;
                e[0] = r.x.x;
                e[1] = r.x.y;
                e[2] = r.x.z;
                e[3] = r.w.x;
                e[4] = r.w.y;
                e[5] = r.w.z;
            }
            steps += r.sphere_steps;
            events += r.pt_events;
            shadow += r.shadow;
            if (r.end == 0) ++escaped;
            else if (r.end == 1) ++absorbed;
            else ++capped;
        } catch (const std::exception& e) {
            if (failed.fetch_add(1) == 0) fail_msg = e.what();
        }
    });
    if (failed) {
        g_err = fail_msg;
        return SST_E_RUNTIME;
    }
    if (stats) {
        stats->paths += n;
        stats->sphere_steps += steps;
        stats->pt_events += events;
        stats->segments += steps + events;
        stats->absorbed += absorbed;
        stats->escaped += escaped;
        stats->capped += capped;
        stats->shadow_rays += shadow;
    }
    return 0;
}

}  // extern "C"
