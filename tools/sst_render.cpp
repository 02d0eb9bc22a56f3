// sst_render -- C++ command-line driver over include/sst_b200.hpp (the reference's
// missing cmd_render, for the two built-in benchmark scenes).
//
//   sst_render --scene c1|c5 [--integrator st|pt] [--spp N] [--seed S] [--nee 0|1]
//              [--width W --height H] [--models DIR] [--out image.pfm|image.png] [--precision f32|f64]
//
// Exit codes: 0 ok, 1 usage, 2 data/model, 3 internal (incl. no GPU).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "sst_b200.hpp"

namespace {

struct Mesh {
    double* pos = nullptr;
    uint32_t* tri = nullptr;
    uint32_t nv = 0, nt = 0;
    ~Mesh() { sst_mesh_free(pos, tri); }
};

int usage() {
    std::fprintf(stderr,
                 "usage: sst_render --scene c1|c5 [--integrator st|pt] [--spp N] [--seed S] [--nee 0|1]\n"
                 "                  [--width W] [--height H] [--models DIR] [--out F.pfm|F.png] [--precision f32|f64]\n"
                 "                  [--dir-light X,Y,Z E]  (directional light toward X,Y,Z, irradiance E)\n");
    return 1;
}

}  // namespace

int main(int argc, char** argv) {
    std::string scene = "c1", integ = "st", models = "tests/golden/models", out, prec = "f32";
    uint32_t spp = 16, width = 0, height = 0;
    uint64_t seed = 1;
    int nee = 1;
    double dir_light[3] = {0.0, 0.0, 0.0}, dir_e = 0.0;
    bool directional = false;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> const char* { return i + 1 < argc ? argv[++i] : nullptr; };
        const char* v = nullptr;
        if (a == "--scene" && (v = next())) scene = v;
        else if (a == "--integrator" && (v = next())) integ = v;
        else if (a == "--spp" && (v = next())) spp = static_cast<uint32_t>(std::atoi(v));
        else if (a == "--seed" && (v = next())) seed = std::strtoull(v, nullptr, 10);
        else if (a == "--nee" && (v = next())) nee = std::atoi(v);
        else if (a == "--width" && (v = next())) width = static_cast<uint32_t>(std::atoi(v));
        else if (a == "--height" && (v = next())) height = static_cast<uint32_t>(std::atoi(v));
        else if (a == "--models" && (v = next())) models = v;
        else if (a == "--out" && (v = next())) out = v;
        else if (a == "--precision" && (v = next())) prec = v;
        else if (a == "--dir-light" && (v = next())) {
            const char* e = next();
            if (!e || std::sscanf(v, "%lf,%lf,%lf", &dir_light[0], &dir_light[1], &dir_light[2]) != 3) return usage();
            dir_e = std::atof(e);
            directional = true;
        }
        else return usage();
    }
    if ((scene != "c1" && scene != "c5") || (integ != "st" && integ != "pt") || spp == 0) return usage();
    try {
        Mesh m;
        sst_b200::check(sst_mesh_icosphere(3, 1.0, &m.pos, &m.nv, &m.tri, &m.nt));
        const int n_obj = scene == "c1" ? 1 : 4;
        const double sig[4] = {scene == "c1" ? 10.0 : 20.0, 40.0, 80.0, 160.0};
        const double phi[3] = {0.99999, 0.99995, 0.975};
        std::vector<std::vector<double>> pos(n_obj);
        std::vector<sst_object_desc> objs(n_obj);
        for (int o = 0; o < n_obj; ++o) {
            const double off = scene == "c1" ? 0.0 : -3.3 + 2.2 * o;
            pos[o].assign(m.pos, m.pos + 3 * m.nv);
            for (uint32_t k = 0; k < m.nv; ++k) pos[o][3 * k] += off;
            sst_object_desc& od = objs[o];
            std::memset(&od, 0, sizeof od);
            od.positions = pos[o].data();
            od.n_vertices = m.nv;
            od.triangles = m.tri;
            od.n_triangles = m.nt;
            for (int c = 0; c < 3; ++c) od.media[c] = {sig[o], 0.8, phi[c]};
            od.sdf_resolution = 64;
        }
        sst_scene_desc d;
        std::memset(&d, 0, sizeof d);
        d.n_objects = static_cast<uint32_t>(n_obj);
        d.objects = objs.data();
        const double lp[3] = {0.0, scene == "c1" ? 2.0 : 4.0, scene == "c1" ? 2.0 : 4.0};
        const double pw = scene == "c1" ? 1.0 : 20.0;
        for (int a = 0; a < 3; ++a) {
            d.light_position[a] = lp[a];
            d.light_power[a] = pw;
            d.cam_look_at[a] = 0.0;
        }
        if (directional) {
            d.light_kind = 1;
            for (int a = 0; a < 3; ++a) {
                d.light_direction[a] = dir_light[a];
                d.light_power[a] = dir_e;
            }
        }
        d.cam_position[2] = scene == "c1" ? 3.0 : 7.5;
        d.cam_up[1] = 1.0;
        d.cam_vfov_deg = 40.0;
        d.width = width ? width : (scene == "c1" ? 256 : 1920);
        d.height = height ? height : (scene == "c1" ? 256 : 1080);

        sst_b200::Context ctx(0, prec == "f64" ? SST_PREC_F64 : SST_PREC_F32);
        try {
            ctx.load_models_dir(models);
        } catch (const std::exception& e) {
            std::fprintf(stderr, "model error: %s\n", e.what());
            return 2;
        }
        ctx.upload_scene(d);
        sst_path_stats st{};
        const auto t0 = std::chrono::steady_clock::now();
        const sst_b200::Image img = ctx.render(integ == "st" ? SST_INTEGRATOR_ST : SST_INTEGRATOR_PT, spp, seed, nee != 0, &st);
        const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (!out.empty()) {
            const bool png = out.size() > 4 && out.compare(out.size() - 4, 4, ".png") == 0;
            sst_b200::check((png ? sst_image_save_png : sst_image_save_pfm)(out.c_str(), img.width, img.height,
                                                                          img.pixels.data()));
        }
        std::printf("{\"scene\": \"%s\", \"integrator\": \"%s\", \"spp\": %u, \"paths\": %llu, \"segments\": %llu, "
                    "\"sphere_steps\": %llu, \"pt_events\": %llu, \"device_ms\": %.3f, \"wall_s\": %.3f, "
                    "\"segments_per_s\": %.6g}\n",
                    scene.c_str(), integ.c_str(), spp, (unsigned long long)st.paths, (unsigned long long)st.segments,
                    (unsigned long long)st.sphere_steps, (unsigned long long)st.pt_events, st.device_ms, wall,
                    st.segments / (st.device_ms * 1e-3));
        return 0;
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 3;
    }
}
