// ref_adapter_check.cpp -- TEST INFRASTRUCTURE (built by oracle/Makefile where the
// reference sources exist; runs from tests/test_ref_adapter.py).
//
// Compiles include/sst_ref_adapter.hpp against the reference's own headers
// (proj/core/include) and links the reference library (oracle/_ref/libsst_ref.so)
// next to libsst_gpu.so, then:
//   1. builds a scene from reference types (sst::make_icosphere, sst::MediumParams,
//      sst::build_sdf) and checks the descriptor the adapter produces;
//   2. with a device: runs the adapter's sample_sphere_step (FP32 and FP64) against
//      the reference's sst::sample_sphere_step on the same RandomStreams, uploads the
//      reference's in-memory ScatterModels, renders the scene into an sst::Image and
//      generates an sst::Dataset compared with the reference's generate_dataset.
// Prints one line per check; exit code 0 = every check passed ("no device" skips 2).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sst/bvh.hpp"
#include "sst/dataset.hpp"
#include "sst/mesh.hpp"
#include "sst/scatter.hpp"
#include "sst/sdf.hpp"
#include "sst_ref_adapter.hpp"

namespace {
int failures = 0;
void expect(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what);
    if (!ok) ++failures;
}
}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_adapter_check <models_dir>\n");
        return 2;
    }
    const std::string models_dir = argv[1];
    namespace ad = sst_b200::ref;

    // 1. scene from reference types
    const sst::TriangleMesh mesh = sst::make_icosphere(3, 1.0);
    const sst::Bvh bvh(mesh);
    const sst::SdfGrid sdf = sst::build_sdf(mesh, bvh, 24);
    const sst::MediumParams media[3] = {{10.0, 0.8, 0.99999}, {10.0, 0.8, 0.99995}, {10.0, 0.8, 0.975}};
    ad::SceneBuilder b;
    b.add_object(mesh, media, &sdf)
        .point_light(sst::Vec3(0, 2, 2), sst::Vec3(1, 1, 1))
        .camera(sst::Vec3(0, 0, 3), sst::Vec3(0, 0, 0), sst::Vec3(0, 1, 0), 40.0, 32, 32);
    const sst_scene_desc& d = b.desc();
    bool same = d.n_objects == 1 && d.objects[0].n_vertices == mesh.positions.size() &&
                d.objects[0].n_triangles == mesh.faces.size();
    for (size_t i = 0; same && i < mesh.positions.size(); ++i)
        same = d.objects[0].positions[3 * i] == mesh.positions[i].x &&
               d.objects[0].positions[3 * i + 1] == mesh.positions[i].y &&
               d.objects[0].positions[3 * i + 2] == mesh.positions[i].z;
    for (size_t f = 0; same && f < mesh.faces.size(); ++f)
        for (int c = 0; c < 3; ++c) same = same && d.objects[0].triangles[3 * f + c] == mesh.faces[f][c];
    expect(same, "to_desc: mesh positions and faces");
    bool sdf_same = d.objects[0].sdf_voxel == sdf.voxel_size && d.objects[0].sdf_origin[0] == sdf.origin.x;
    for (int a = 0; a < 3; ++a) sdf_same = sdf_same && d.objects[0].sdf_dims[a] == sdf.dims[a];
    sdf_same = sdf_same && std::memcmp(d.objects[0].sdf_values, sdf.values.data(), sdf.values.size() * 4) == 0;
    expect(sdf_same, "to_desc: SdfGrid origin/voxel/dims/values");
    expect(d.objects[0].media[2].phi == 0.975 && d.objects[0].media[0].sigma_t == 10.0, "to_desc: MediumParams");
    expect(d.light_kind == 0 && d.light_position[1] == 2.0 && d.width == 32 && d.cam_vfov_deg == 40.0,
           "SceneBuilder: light and camera");
    bool threw = false;
    try {
        const sst::MediumParams bad[3] = {{-1.0, 0.0, 1.0}, {1.0, 0.0, 1.0}, {1.0, 0.0, 1.0}};
        ad::ObjectBuffers keep;
        ad::to_desc(mesh, bad, nullptr, keep);
    } catch (const std::domain_error&) {
        threw = true;
    }
    expect(threw, "to_desc: invalid MediumParams -> std::domain_error (optics.cpp:21-25)");
    sst::Image ri(4, 3);
    ri.sample_count = 7;
    for (size_t i = 0; i < ri.pixels.size(); ++i) ri.pixels[i] = 0.25f * i;
    const sst::Image back = ad::to_ref_image(ad::from_ref_image(ri));
    expect(back.width == 4 && back.height == 3 && back.sample_count == 7 && back.pixels == ri.pixels,
           "Image <-> sst::Image");
    sst::RandomStream rs(5, 6, 7, 8);
    expect(ad::stream_state(rs) == sst_rng_init(5, 6, 7, 8), "RandomStream state == sst_rng_init");

    // 2. device checks
    int dev_count_ok = 1;
    try {
        sst_b200::Context probe(0);
    } catch (const sst_b200::CudaError& e) {
        std::printf("no device (%s): conversion checks only\n", e.what());
        dev_count_ok = 0;
    }
    if (dev_count_ok) {
        const sst::ScatterModels models = sst::ScatterModels::load_dir(models_dir);
        const int n = 4000;
        std::vector<ad::StepArgs> args;
        std::vector<sst::RandomStream> r_ref, r_dev;
        sst::RandomStream pick(99, 1, 2, 3);
        for (int i = 0; i < n; ++i) {
            sst::Vec3 w(pick.normal(), pick.normal(), pick.normal());
            w = w / std::sqrt(w.x * w.x + w.y * w.y + w.z * w.z);
            args.push_back({pick.uniform(1.0, 150.0), pick.uniform(-0.9, 0.9), 1.0 - std::pow(10.0, pick.uniform(-5.0, -1.0)),
                            w, sst::Vec3(pick.normal(), pick.normal(), pick.normal()), pick.uniform(0.05, 1.0),
                            pick.uniform() < 0.7});
            r_ref.emplace_back(31, 6, i, 0);
        }
        r_dev = r_ref;
        std::vector<sst::SphereStepOutcome> ref(n);
        models.counters.reset();
        for (int i = 0; i < n; ++i) {
            const auto& a = args[i];
            ref[i] = sst::sample_sphere_step(models, a.sigma_t_world, a.g, a.phi, a.w_in_world, a.center, a.r_sphere,
                                             a.with_event, r_ref[i]);
        }
        const uint64_t ref_decodes = models.counters.total();
        for (int prec : {SST_PREC_F64, SST_PREC_F32}) {
            sst_b200::Context ctx(0, prec);
            ad::upload_models(ctx, models);  // in-memory ScatterModels
            std::vector<sst::RandomStream> rd = r_dev;
            models.counters.reset();
            const auto got = ad::sample_sphere_steps(ctx, models, args, rd);
            int abs_same = 0, state_same = 0, pos_close = 0;
            for (int i = 0; i < n; ++i) {
                abs_same += got[i].absorbed == ref[i].absorbed && got[i].n_events == ref[i].n_events;
                state_same += ad::stream_state(rd[i]) == ad::stream_state(r_ref[i]);
                const sst::Vec3 dp = got[i].exit_position_world - ref[i].exit_position_world;
                const double e = std::sqrt(dp.x * dp.x + dp.y * dp.y + dp.z * dp.z);
                pos_close += ref[i].absorbed || e <= 1e-4 * (1.0 + std::sqrt(ref[i].exit_position_world.x *
                                                                              ref[i].exit_position_world.x));
            }
            char msg[256];
            const bool f64 = prec == SST_PREC_F64;
            std::snprintf(msg, sizeof msg, "%s sample_sphere_step vs sst::sample_sphere_step: outcome %d/%d, "
                          "RNG state %d/%d, exit position %d/%d", f64 ? "FP64" : "FP32", abs_same, n, state_same, n,
                          pos_close, n);
            expect(f64 ? (abs_same == n && state_same == n && pos_close == n)
                       : (abs_same >= 0.99 * n && state_same >= 0.99 * n && pos_close >= 0.99 * n), msg);
            if (f64) expect(models.counters.total() == ref_decodes, "DecodeCounters bookkeeping equals the reference's");
            if (!f64) {
                ctx.upload_scene(b.desc());
                sst_path_stats st{};
                const sst::Image img = ad::render(ctx, SST_INTEGRATOR_ST, 4, 1, true, &st);
                bool finite = img.width == 32 && img.height == 32 && img.sample_count == 4;
                double sum = 0;
                for (float v : img.pixels) {
                    finite = finite && std::isfinite(v);
                    sum += v;
                }
                expect(finite && sum > 0.0 && st.paths == 32u * 32u * 3u * 4u, "render -> sst::Image");
            } else {
                const sst::PhiSampler phi;
                const sst::Dataset ours = ad::generate_dataset(ctx, 300, 0.0, 80.0, -0.9, 0.9, phi, 17);
                const sst::Dataset theirs = sst::generate_dataset(300, 0.0, 80.0, -0.9, 0.9, phi, 17);
                const bool eq = ours.samples.size() == theirs.samples.size() &&
                                std::memcmp(static_cast<const void*>(ours.samples.data()), static_cast<const void*>(theirs.samples.data()),
                                            300 * sizeof(sst::TrainingSample)) == 0 &&
                                ours.fingerprint() == theirs.fingerprint();
                expect(eq, "FP64 generate_dataset -> sst::Dataset byte-identical (records + fingerprint)");
            }
        }
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "PASSED", failures);
    return failures ? 1 : 0;
}
