// host.h -- internal C++ host-side helpers (model files, meshes, BVH build).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace sstg {

// Error classes mapped onto the C ABI codes (sst_gpu.h).
struct InvalidArgument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct DomainError : std::domain_error {
    using std::domain_error::domain_error;
};
struct RuntimeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct HostLayer {
    uint32_t out_dim = 0, in_dim = 0;
    std::vector<float> w, b;
};

// Decoder half of a CvaeModel (cvae.hpp:52-60).
struct HostModel {
    uint32_t kind = 0, p_in = 0, p_out = 0, depth = 0, width = 0, latent = 0;
    double sigma_ref = 200.0, n_ref = 1e4;
    std::vector<HostLayer> layers;
};

// load_model (cvae.cpp:379-425): SSNN v1; the encoder, if present, is skipped.
HostModel load_ssnn(const std::string& path);
// Validates kind tags (scatter.cpp:15-27) and the production shapes the device
// evaluator is compiled for, then packs W0,b0,W1,b1,W2,b2 per model (1332 values)
// plus per-model {log1p(sigma_ref), log(n_ref)}.
void pack_models(const HostModel (&m)[3], std::vector<double>& weights, double norms[6]);

struct HostMesh {
    std::vector<std::array<double, 3>> pos;
    std::vector<std::array<uint32_t, 3>> tri;
    uint64_t dropped = 0;
};
HostMesh make_icosphere(int subdivisions, double radius);
HostMesh make_bumpy_sphere(int subdivisions, double radius, double amplitude, double frequency);
HostMesh load_obj(const std::string& path, double scale);
bool is_watertight(const std::vector<std::array<uint32_t, 3>>& tri);
// Every vertex on one side of every face plane (closed convex polyhedron).
bool is_convex(const double* pos, uint32_t nv, const std::vector<std::array<uint32_t, 3>>& tri);

// Flattened BVH2 for the device (binned-SAH build, <= 4 triangles per leaf).
struct FlatBvh {
    std::vector<uint8_t> nodes_f32, tris_f32;  // NodeF[], TriF[]
    std::vector<uint8_t> nodes_f64, tris_f64;  // NodeD[], TriD[]
    uint32_t n_nodes = 0, n_tris = 0;
    std::vector<uint32_t> order;  // leaf position -> input triangle index
};
// tri_vertices: [n][3] corners; tri_obj: object id per triangle.
FlatBvh build_bvh(const std::vector<std::array<std::array<double, 3>, 3>>& tri_vertices,
                  const std::vector<uint32_t>& tri_obj);

}  // namespace sstg
