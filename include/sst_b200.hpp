// sst_b200.hpp -- header-only C++ mirror of the reference's interfaces for the hot
// path, implemented over the C ABI (sst_gpu.h / libsst_gpu.so). A reference-side
// caller (namespace sst, /root/reference/proj/core) switches by replacing
//
//   sst::ScatterModels::load_dir(dir)                       (scatter.cpp:29-32)
//   sst::sample_sphere_step(models, s, g, phi, w, c, r, ev, rng)  (scatter.cpp:152-177)
//   render(scene, integrator, spp, seed, nee)                (missing in ref)
//
// with sst_b200::Context::load_models_dir / sample_sphere_step(s) / render. Errors are
// rethrown as the same std:: exception types the reference throws.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sst_gpu.h"
#include "sst_host.h"

namespace sst_b200 {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int rc) {
    if (rc == SST_OK) return;
    const std::string msg = sst_gpu_last_error();
    switch (rc) {
        case SST_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case SST_E_DOMAIN: throw std::domain_error(msg);
        case SST_E_CUDA: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

struct Vec3 {
    double x = 0, y = 0, z = 0;
};

// Mirrors sst::SphereStepOutcome (scatter.hpp:105-114).
struct SphereStepOutcome {
    bool absorbed = false;
    uint32_t n_events = 1;
    Vec3 exit_position_world, exit_direction_world;
    bool has_representative = false;
    Vec3 rep_position_world, rep_direction_world;
    double lambda_weight = 0.0;
};

struct StepInput {
    double sigma_t_world, g, phi;
    Vec3 w_in_world, center;
    double r_sphere;
    bool with_event;
};

// Linear-RGB float framebuffer, row 0 on top (sst::Image, image.hpp:13-29).
struct Image {
    uint32_t width = 0, height = 0, sample_count = 0;
    std::vector<float> pixels;
};

class Context {
  public:
    explicit Context(int device = 0, int precision = SST_PREC_F32) {
        check(sst_gpu_create(device, &ctx_));
        check(sst_gpu_set_precision(ctx_, precision));
    }
    ~Context() { sst_gpu_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;

    sst_gpu_ctx* handle() { return ctx_; }

    // ScatterModels::load_dir
    void load_models_dir(const std::string& dir) { check(sst_gpu_load_models_dir(ctx_, dir.c_str())); }

    // Batched sample_sphere_step; rng_states[i] is the RandomStream state
    // (sst_rng_init(seed, s1, s2, s3)) and is advanced like RandomStream&.
    std::vector<SphereStepOutcome> sample_sphere_steps(const std::vector<StepInput>& in,
                                                       std::vector<uint64_t>& rng_states,
                                                       sst_decode_counters* counters = nullptr) {
        const size_t n = in.size();
        if (rng_states.size() != n) throw std::invalid_argument("rng_states size mismatch");
        std::vector<double> sig(n), g(n), phi(n), w(3 * n), c(3 * n), r(n);
        std::vector<uint8_t> ev(n);
        for (size_t i = 0; i < n; ++i) {
            sig[i] = in[i].sigma_t_world;
            g[i] = in[i].g;
            phi[i] = in[i].phi;
            w[3 * i] = in[i].w_in_world.x; w[3 * i + 1] = in[i].w_in_world.y; w[3 * i + 2] = in[i].w_in_world.z;
            c[3 * i] = in[i].center.x; c[3 * i + 1] = in[i].center.y; c[3 * i + 2] = in[i].center.z;
            r[i] = in[i].r_sphere;
            ev[i] = in[i].with_event ? 1 : 0;
        }
        std::vector<uint8_t> absorbed(n), has_rep(n);
        std::vector<uint32_t> nev(n);
        std::vector<double> ep(3 * n), ed(3 * n), rp(3 * n), rd(3 * n), lam(n);
        sst_step_in si{sig.data(), g.data(), phi.data(), w.data(), c.data(), r.data(), ev.data(), rng_states.data()};
        sst_step_out so{absorbed.data(), nev.data(), ep.data(), ed.data(), has_rep.data(), rp.data(), rd.data(), lam.data()};
        check(sst_gpu_sphere_step_batch(ctx_, n, &si, 1, &so, SST_PTR_HOST, counters));
        std::vector<SphereStepOutcome> out(n);
        for (size_t i = 0; i < n; ++i) {
            out[i].absorbed = absorbed[i] != 0;
            out[i].n_events = nev[i];
            out[i].exit_position_world = {ep[3 * i], ep[3 * i + 1], ep[3 * i + 2]};
            out[i].exit_direction_world = {ed[3 * i], ed[3 * i + 1], ed[3 * i + 2]};
            out[i].has_representative = has_rep[i] != 0;
            out[i].rep_position_world = {rp[3 * i], rp[3 * i + 1], rp[3 * i + 2]};
            out[i].rep_direction_world = {rd[3 * i], rd[3 * i + 1], rd[3 * i + 2]};
            out[i].lambda_weight = lam[i];
        }
        return out;
    }

    // Single-step form with the reference's signature shape.
    SphereStepOutcome sample_sphere_step(double sigma_t_world, double g, double phi, const Vec3& w_in,
                                         const Vec3& center, double r_sphere, bool with_event,
                                         uint64_t& rng_state) {
        std::vector<uint64_t> s{rng_state};
        auto o = sample_sphere_steps({{sigma_t_world, g, phi, w_in, center, r_sphere, with_event}}, s);
        rng_state = s[0];
        return o[0];
    }

    void upload_scene(const sst_scene_desc& scene) {
        check(sst_gpu_upload_scene(ctx_, &scene));
        width_ = scene.width;
        height_ = scene.height;
    }

    // render(scene, integrator, spp, seed, nee) -> (Image, PathStats)
    Image render(int integrator, uint32_t spp, uint64_t seed, bool nee, sst_path_stats* stats = nullptr) {
        const size_t n = static_cast<size_t>(width_) * height_ * 3;
        std::vector<double> sum(n, 0.0), sq(n, 0.0);
        sst_path_stats local{};
        check(sst_gpu_render(ctx_, integrator, nee ? 1 : 0, spp, 0, spp, seed, sum.data(), sq.data(),
                             SST_PTR_HOST, stats ? stats : &local));
        Image img;
        img.width = width_;
        img.height = height_;
        img.sample_count = spp;
        img.pixels.resize(n);
        for (size_t i = 0; i < n; ++i) img.pixels[i] = static_cast<float>(sum[i] / spp);
        return img;
    }

    // generate_dataset(n, sigma_t range, g range, phi sampler, seed)  (dataset.cpp:40-92)
    std::vector<sst_training_sample> generate_dataset(uint64_t n, double s_lo, double s_hi, double g_lo, double g_hi,
                                                      int phi_kind, double phi_a, double phi_b, uint64_t seed,
                                                      sst_dataset_stats* stats = nullptr) {
        std::vector<sst_training_sample> out(n);
        check(sst_gpu_generate_dataset(ctx_, n, s_lo, s_hi, g_lo, g_hi, phi_kind, phi_a, phi_b, seed, 0, out.data(),
                                       SST_PTR_HOST, stats));
        return out;
    }

    // train_model(kind, dataset, cfg) + save_model(path, model, with_encoder)  (cvae.cpp:234-377)
    std::vector<sst_epoch_stats> train_model(int kind, const std::vector<sst_training_sample>& samples,
                                             uint64_t dataset_seed, const sst_train_config& cfg,
                                             const std::string& ssnn_path = "", bool include_encoder = true,
                                             bool install = false, sst_train_stats* stats = nullptr) {
        std::vector<sst_epoch_stats> epochs(cfg.epochs);
        check(sst_gpu_train_model(ctx_, kind, samples.data(), samples.size(), SST_PTR_HOST, dataset_seed, &cfg,
                                  epochs.data(), ssnn_path.empty() ? nullptr : ssnn_path.c_str(),
                                  include_encoder ? 1 : 0, nullptr, install ? 1 : 0, stats));
        return epochs;
    }

  private:
    sst_gpu_ctx* ctx_ = nullptr;
    uint32_t width_ = 0, height_ = 0;
};

}  // namespace sst_b200
