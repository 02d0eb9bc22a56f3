// sst_ref_adapter.hpp -- the drop-in seam between the reference's own C++ types
// (namespace sst, proj/core/include/sst/*.hpp) and the B200 library (sst_gpu.h).
//
// A caller of the reference keeps its scene, medium, CVAE-weight and film types and
// swaps the hot path:
//
//   reference (proj/core)                                   this adapter
//   -----------------------------------------------------   -----------------------------------------------
//   sst::ScatterModels::load_dir(dir)   (scatter.cpp:29-32)  load_models_dir(ctx, dir)
//   ScatterModels already in memory     (scatter.hpp:28-39)  upload_models(ctx, models)
//   sst::sample_sphere_step(models, ...,                     sample_sphere_step(ctx, models, ..., rng)
//       RandomStream& rng)              (scatter.cpp:152-177)    same arguments, same RNG advance,
//                                                              same DecodeCounters bookkeeping
//   TriangleMesh + MediumParams[3] + SdfGrid                 SceneBuilder::add_object(mesh, media, sdf)
//       (mesh.hpp:15-30, optics.hpp:16-26, sdf.hpp:19-33)
//   render(scene, integrator, spp, seed, nee) -> Image       render(ctx, integrator, spp, seed, nee)
//       (image.hpp:13-29)                       -> sst::Image
//   generate_dataset(n, ..., PhiSampler, seed)               generate_dataset(ctx, n, ..., phi, seed)
//       (dataset.cpp:40-92)                                      -> sst::Dataset
//
// Header-only; include it with the reference's include directory on the path
// (-I proj/core/include) and link libsst_gpu.so. Errors are the reference's std::
// exception types (sst_b200::check).
#pragma once

#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "sst/dataset.hpp"
#include "sst/image.hpp"
#include "sst/mesh.hpp"
#include "sst/optics.hpp"
#include "sst/rng.hpp"
#include "sst/scatter.hpp"
#include "sst/sdf.hpp"
#include "sst_b200.hpp"

namespace sst_b200 {
namespace ref {

// ---------------------------------------------------------------- RandomStream
// RandomStream (rng.hpp:15-50) is one u64 of state; the device library takes and
// returns exactly that state, so a caller's stream advances as under the reference.
static_assert(sizeof(sst::RandomStream) == sizeof(uint64_t) && std::is_trivially_copyable_v<sst::RandomStream>,
              "RandomStream is expected to hold one u64 of state (rng.hpp:49)");
inline uint64_t stream_state(const sst::RandomStream& r) {
    uint64_t s;
    std::memcpy(&s, &r, sizeof s);
    return s;
}
inline void set_stream_state(sst::RandomStream& r, uint64_t s) { std::memcpy(static_cast<void*>(&r), &s, sizeof s); }

inline sst::Vec3 v3(const Vec3& v) { return sst::Vec3(v.x, v.y, v.z); }
inline Vec3 v3(const sst::Vec3& v) { return Vec3{v.x, v.y, v.z}; }

// ---------------------------------------------------------------- CVAE weights
// ScatterModels::load_dir (scatter.cpp:29-32): the library parses the SSNN files.
inline void load_models_dir(Context& ctx, const std::string& dir) { ctx.load_models_dir(dir); }

// In-memory ScatterModels (e.g. straight out of train_model): the three decoders.
// Weights are f32-quantised doubles in the reference (mlp.hpp:14-17), so the float
// copies are exact.
inline void upload_models(Context& ctx, const sst::ScatterModels& m) {
    const sst::CvaeModel* models[3] = {&m.length, &m.path, &m.event};
    std::vector<std::vector<float>> store;
    std::vector<sst_layer_desc> layers[3];
    sst_model_desc desc[3];
    for (int k = 0; k < 3; ++k) {
        const sst::CvaeModel& cm = *models[k];
        for (const sst::DenseLayer& l : cm.decoder.layers) {
            store.emplace_back(l.weights.begin(), l.weights.end());
            const float* w = store.back().data();
            store.emplace_back(l.bias.begin(), l.bias.end());
            layers[k].push_back(sst_layer_desc{l.out_dim, l.in_dim, w, store.back().data()});
        }
        desc[k].kind = static_cast<uint32_t>(cm.kind);
        desc[k].p_in = cm.spec.p_in;
        desc[k].p_out = cm.spec.p_out;
        desc[k].depth = cm.spec.depth;
        desc[k].width = cm.spec.width;
        desc[k].latent = cm.spec.latent;
        desc[k].sigma_ref = cm.norms.sigma_ref;
        desc[k].n_ref = cm.norms.n_ref;
        desc[k].n_layers = static_cast<uint32_t>(layers[k].size());
        desc[k].layers = nullptr;
    }
    // pointers into `store` are stable only once every vector is in place
    size_t idx = 0;
    for (int k = 0; k < 3; ++k) {
        for (auto& l : layers[k]) {
            l.weights = store[idx++].data();
            l.bias = store[idx++].data();
        }
        desc[k].layers = layers[k].data();
    }
    check(sst_gpu_upload_models(ctx.handle(), desc));
}

// ---------------------------------------------------------------- per-step operator
struct StepArgs {
    double sigma_t_world, g, phi;
    sst::Vec3 w_in_world, center;
    double r_sphere;
    bool with_event;
};

// Batched sample_sphere_step (scatter.cpp:152-177) on the device. rngs[i] is the
// caller's RandomStream of step i and is advanced by the draws the reference
// consumes; models.counters gets the decode counts, like the reference's wrappers.
inline std::vector<sst::SphereStepOutcome> sample_sphere_steps(Context& ctx, const sst::ScatterModels& models,
                                                               const std::vector<StepArgs>& steps,
                                                               std::vector<sst::RandomStream>& rngs) {
    if (rngs.size() != steps.size()) throw std::invalid_argument("one RandomStream per step");
    std::vector<StepInput> in(steps.size());
    std::vector<uint64_t> state(steps.size());
    for (size_t i = 0; i < steps.size(); ++i) {
        const StepArgs& s = steps[i];
        in[i] = StepInput{s.sigma_t_world, s.g, s.phi, v3(s.w_in_world), v3(s.center), s.r_sphere, s.with_event};
        state[i] = stream_state(rngs[i]);
    }
    sst_decode_counters dc{};
    const std::vector<SphereStepOutcome> got = ctx.sample_sphere_steps(in, state, &dc);
    models.counters.length += dc.length;
    models.counters.path += dc.path;
    models.counters.event += dc.event;
    std::vector<sst::SphereStepOutcome> out(got.size());
    for (size_t i = 0; i < got.size(); ++i) {
        set_stream_state(rngs[i], state[i]);
        sst::SphereStepOutcome& o = out[i];
        o.absorbed = got[i].absorbed;
        o.n_events = got[i].n_events;
        o.exit_position_world = v3(got[i].exit_position_world);
        o.exit_direction_world = v3(got[i].exit_direction_world);
        o.has_representative = got[i].has_representative;
        o.rep_position_world = v3(got[i].rep_position_world);
        o.rep_direction_world = v3(got[i].rep_direction_world);
        o.lambda_weight = got[i].lambda_weight;
    }
    return out;
}

// The reference's signature (scatter.hpp:119-122) plus the device context.
inline sst::SphereStepOutcome sample_sphere_step(Context& ctx, const sst::ScatterModels& models,
                                                 double sigma_t_world, double g, double phi,
                                                 const sst::Vec3& w_in_world, const sst::Vec3& center,
                                                 double r_sphere, bool with_event, sst::RandomStream& rng) {
    std::vector<sst::RandomStream> r{rng};
    auto o = sample_sphere_steps(ctx, models, {StepArgs{sigma_t_world, g, phi, w_in_world, center, r_sphere,
                                                        with_event}}, r);
    rng = r[0];
    return o[0];
}

// ---------------------------------------------------------------- scene
// Flattened copies an sst_object_desc points into (kept alive by the SceneBuilder).
struct ObjectBuffers {
    std::vector<double> positions;
    std::vector<uint32_t> triangles;
    std::vector<float> sdf;
};

// TriangleMesh + per-channel MediumParams + optional SdfGrid -> sst_object_desc.
// sdf == nullptr asks the library to build it (build_sdf, sdf.cpp:20-58, at
// sdf_resolution; bit-identical to the reference's).
inline sst_object_desc to_desc(const sst::TriangleMesh& mesh, const sst::MediumParams (&media)[3],
                               const sst::SdfGrid* sdf, ObjectBuffers& keep, uint32_t sdf_resolution = 64) {
    for (const auto& m : media) m.validate();  // std::domain_error like the reference (optics.cpp:21-25)
    keep.positions.resize(3 * mesh.positions.size());
    for (size_t i = 0; i < mesh.positions.size(); ++i) {
        keep.positions[3 * i] = mesh.positions[i].x;
        keep.positions[3 * i + 1] = mesh.positions[i].y;
        keep.positions[3 * i + 2] = mesh.positions[i].z;
    }
    keep.triangles.resize(3 * mesh.faces.size());
    for (size_t f = 0; f < mesh.faces.size(); ++f)
        for (int c = 0; c < 3; ++c) keep.triangles[3 * f + c] = mesh.faces[f][c];
    sst_object_desc d{};
    d.positions = keep.positions.data();
    d.n_vertices = static_cast<uint32_t>(mesh.positions.size());
    d.triangles = keep.triangles.data();
    d.n_triangles = static_cast<uint32_t>(mesh.faces.size());
    for (int c = 0; c < 3; ++c) d.media[c] = sst_medium{media[c].sigma_t, media[c].g, media[c].phi};
    d.sdf_resolution = sdf_resolution;
    if (sdf) {
        keep.sdf = sdf->values;
        d.sdf_origin[0] = sdf->origin.x;
        d.sdf_origin[1] = sdf->origin.y;
        d.sdf_origin[2] = sdf->origin.z;
        d.sdf_voxel = sdf->voxel_size;
        for (int a = 0; a < 3; ++a) d.sdf_dims[a] = sdf->dims[a];
        d.sdf_values = keep.sdf.data();
    }
    return d;
}

// Scene from reference types: objects, light, camera, background.
class SceneBuilder {
  public:
    SceneBuilder() {
        d_.light_position[2] = 0.0;
        d_.light_power[0] = d_.light_power[1] = d_.light_power[2] = 1.0;
        d_.cam_position[2] = 3.0;
        d_.cam_up[1] = 1.0;
        d_.cam_vfov_deg = 40.0;
        d_.width = d_.height = 256;
        d_.light_direction[1] = 1.0;
    }
    SceneBuilder& add_object(const sst::TriangleMesh& mesh, const sst::MediumParams (&media)[3],
                             const sst::SdfGrid* sdf = nullptr, uint32_t sdf_resolution = 64) {
        bufs_.emplace_back();
        objs_.push_back(to_desc(mesh, media, sdf, bufs_.back(), sdf_resolution));
        return *this;
    }
    SceneBuilder& point_light(const sst::Vec3& p, const sst::Vec3& phi_rgb) {
        d_.light_kind = 0;
        set(d_.light_position, p);
        set(d_.light_power, phi_rgb);
        return *this;
    }
    SceneBuilder& directional_light(const sst::Vec3& toward_light, const sst::Vec3& e_rgb) {
        d_.light_kind = 1;
        set(d_.light_direction, toward_light);
        set(d_.light_power, e_rgb);
        return *this;
    }
    SceneBuilder& camera(const sst::Vec3& pos, const sst::Vec3& look_at, const sst::Vec3& up, double vfov_deg,
                         uint32_t width, uint32_t height) {
        set(d_.cam_position, pos);
        set(d_.cam_look_at, look_at);
        set(d_.cam_up, up);
        d_.cam_vfov_deg = vfov_deg;
        d_.width = width;
        d_.height = height;
        return *this;
    }
    SceneBuilder& background(const sst::Vec3& rgb) {
        set(d_.background, rgb);
        return *this;
    }
    SceneBuilder& r_min(double r) {
        d_.r_min = r;
        return *this;
    }
    // The descriptor; valid while this builder lives and is not modified.
    const sst_scene_desc& desc() {
        d_.n_objects = static_cast<uint32_t>(objs_.size());
        d_.objects = objs_.data();
        return d_;
    }

  private:
    static void set(double (&a)[3], const sst::Vec3& v) {
        a[0] = v.x;
        a[1] = v.y;
        a[2] = v.z;
    }
    sst_scene_desc d_{};
    std::vector<ObjectBuffers> bufs_;
    std::vector<sst_object_desc> objs_;
};

// ---------------------------------------------------------------- film
inline sst::Image to_ref_image(const Image& img) {
    sst::Image out(img.width, img.height);
    out.sample_count = img.sample_count;
    out.pixels = img.pixels;
    return out;
}
inline Image from_ref_image(const sst::Image& img) {
    Image out;
    out.width = img.width;
    out.height = img.height;
    out.sample_count = img.sample_count;
    out.pixels = img.pixels;
    return out;
}

// render(scene, integrator, spp, seed, nee) -> sst::Image of the scene
// last uploaded with ctx.upload_scene(builder.desc()).
inline sst::Image render(Context& ctx, int integrator, uint32_t spp, uint64_t seed, bool nee,
                         sst_path_stats* stats = nullptr) {
    return to_ref_image(ctx.render(integrator, spp, seed, nee, stats));
}

// ---------------------------------------------------------------- training data
static_assert(sizeof(sst::TrainingSample) == sizeof(sst_training_sample), "TrainingSample layout (dataset.hpp:17-27)");

// generate_dataset (dataset.cpp:40-92) on the device -> sst::Dataset (same header, same
// records: sample i uses RandomStream(seed, kDataset, i) as in the reference).
inline sst::Dataset generate_dataset(Context& ctx, uint64_t n, double s_lo, double s_hi, double g_lo, double g_hi,
                                     const sst::PhiSampler& phi, uint64_t seed, sst_dataset_stats* stats = nullptr) {
    const auto rec = ctx.generate_dataset(n, s_lo, s_hi, g_lo, g_hi, static_cast<int>(phi.kind), phi.a, phi.b,
                                          seed, stats);
    sst::Dataset ds;
    ds.header.count = n;
    ds.header.sigma_t_lo = static_cast<float>(s_lo);
    ds.header.sigma_t_hi = static_cast<float>(s_hi);
    ds.header.g_lo = static_cast<float>(g_lo);
    ds.header.g_hi = static_cast<float>(g_hi);
    ds.header.phi = phi;
    ds.header.seed = seed;
    ds.samples.resize(n);
    if (n) std::memcpy(static_cast<void*>(ds.samples.data()), rec.data(), n * sizeof(sst_training_sample));
    return ds;
}

}  // namespace ref
}  // namespace sst_b200
