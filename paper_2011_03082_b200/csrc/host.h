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
    uint32_t max_depth = 0;       // interior levels on the deepest root-leaf path (stack bound)
    // Per object: the interior node whose subtree holds exactly that object's triangles,
    // when the objects' bounding boxes are pairwise disjoint (a ray inside object o then
    // meets o's surface before any other triangle); -1 = start at the root.
    std::vector<int32_t> obj_root;
    std::vector<uint32_t> order;  // leaf position -> input triangle index
};
// tri_vertices: [n][3] corners; tri_obj: object id per triangle.
FlatBvh build_bvh(const std::vector<std::array<std::array<double, 3>, 3>>& tri_vertices,
                  const std::vector<uint32_t>& tri_obj);

// ------------------------------------------------------------------ training (host side)
// RandomStream (rng.hpp:15-50) on the host: the split / shuffle / init streams.
struct HostStream {
    uint64_t s;
    HostStream(uint64_t seed, uint64_t s1 = 0, uint64_t s2 = 0, uint64_t s3 = 0);
    uint64_t next_u64();
    double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + uniform() * (hi - lo); }
};

// CvaeSpec (cvae.hpp:28-38).
struct CvaeSpecH {
    uint32_t p_in = 0, p_out = 0, depth = 2, width = 8, latent = 2;
};
CvaeSpecH production_spec(int kind);  // CvaeSpec::production_default (cvae.cpp:51-57)
void validate_spec(const CvaeSpecH& s);  // CvaeSpec::validate (cvae.cpp:60-65)

// Layer shapes of the encoder / decoder MLPs of a spec (make_gaussian_mlp, mlp.cpp:52-58).
struct MlpShape {
    std::vector<uint32_t> in, out;
    size_t params() const;
};
MlpShape encoder_shape(const CvaeSpecH& s);
MlpShape decoder_shape(const CvaeSpecH& s);

// make_cvae (cvae.cpp:79-91): Glorot-uniform weights from RandomStream(seed, kTrainInit,
// kind), encoder then decoder, log-variance head biases -2, quantised to f32.
void make_cvae_params(int kind, const CvaeSpecH& s, uint64_t seed, std::vector<double>& enc,
                      std::vector<double>& dec);

// save_model (cvae.cpp:349-377). enc may be null (no encoder section).
void save_ssnn(const std::string& path, int kind, const CvaeSpecH& s, double sigma_ref, double n_ref,
               uint64_t fingerprint, const std::vector<double>& dec, const std::vector<double>* enc);

// HostModel (decoder half) from flattened decoder parameters.
HostModel model_from_params(int kind, const CvaeSpecH& s, double sigma_ref, double n_ref,
                            const std::vector<double>& dec);

}  // namespace sstg
