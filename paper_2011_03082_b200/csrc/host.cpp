// host.cpp -- host-side pieces of the library: SSNN parsing, meshes, the BVH
// build for the device, SSDF / PFM files. No device work here.
#include "host.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <numeric>
#include <sstream>
#include <unordered_map>

#include "rng.cuh"
#include "types.cuh"

namespace sstg {

// ------------------------------------------------------------------ SSNN
namespace {
struct Reader {
    std::ifstream in;
    std::string what;
    explicit Reader(const std::string& path) : in(path, std::ios::binary), what("model " + path) {
        if (!in) throw RuntimeError("cannot open for reading: " + path);
    }
    template <class T>
    T get() {
        unsigned char b[sizeof(T)] = {};
        in.read(reinterpret_cast<char*>(b), sizeof(T));
        T v;
        std::memcpy(&v, b, sizeof(T));  // little-endian host (x86-64)
        return v;
    }
};
}  // namespace

HostModel load_ssnn(const std::string& path) {
    Reader r(path);
    char magic[4] = {};
    r.in.read(magic, 4);
    if (!r.in || std::memcmp(magic, "SSNN", 4) != 0) throw RuntimeError(r.what + ": bad magic bytes");
    const uint32_t version = r.get<uint32_t>();
    if (version != 1) throw RuntimeError(r.what + ": unsupported version " + std::to_string(version));
    HostModel m;
    m.kind = r.get<uint32_t>();
    const bool with_encoder = r.get<uint32_t>() != 0;
    (void)with_encoder;
    m.p_in = r.get<uint32_t>();
    m.p_out = r.get<uint32_t>();
    m.depth = r.get<uint32_t>();
    m.width = r.get<uint32_t>();
    m.latent = r.get<uint32_t>();
    m.sigma_ref = r.get<double>();
    m.n_ref = r.get<double>();
    (void)r.get<uint64_t>();  // dataset fingerprint
    const uint32_t n_layers = r.get<uint32_t>();
    if (!r.in || n_layers == 0 || n_layers > 64) throw RuntimeError(r.what + ": implausible layer count");
    m.layers.resize(n_layers);
    for (auto& l : m.layers) {
        l.out_dim = r.get<uint32_t>();
        l.in_dim = r.get<uint32_t>();
        if (!r.in || l.out_dim == 0 || l.in_dim == 0 || l.out_dim > 4096 || l.in_dim > 4096)
            throw RuntimeError(r.what + ": implausible layer shape");
        l.w.resize(static_cast<size_t>(l.out_dim) * l.in_dim);
        l.b.resize(l.out_dim);
        r.in.read(reinterpret_cast<char*>(l.w.data()), l.w.size() * sizeof(float));
        r.in.read(reinterpret_cast<char*>(l.b.data()), l.b.size() * sizeof(float));
    }
    if (!r.in) throw RuntimeError(r.what + ": truncated or corrupt file");
    if (m.layers.front().in_dim != m.latent + m.p_in || m.layers.back().out_dim != 2 * m.p_out)
        throw RuntimeError(r.what + ": decoder shape disagrees with header");
    return m;
}

void pack_models(const HostModel (&m)[3], std::vector<double>& weights, double norms[6]) {
    // production_default (cvae.cpp:51-58): {p_in, p_out, depth, width, latent}
    static const uint32_t spec[3][5] = {{2, 1, 2, 8, 2}, {3, 3, 2, 16, 5}, {7, 6, 2, 16, 5}};
    static const char* names[3] = {"lengthgen", "pathgen", "eventgen"};
    weights.clear();
    for (int k = 0; k < 3; ++k) {
        const HostModel& h = m[k];
        if (h.kind != static_cast<uint32_t>(k))
            throw RuntimeError("ScatterModels: model bundle has wrong kind tag");
        const uint32_t in = spec[k][4] + spec[k][0], w = spec[k][3], out = 2 * spec[k][1];
        const bool ok = h.p_in == spec[k][0] && h.p_out == spec[k][1] && h.latent == spec[k][4] &&
                        h.layers.size() == 3 && h.layers[0].in_dim == in && h.layers[0].out_dim == w &&
                        h.layers[1].in_dim == w && h.layers[1].out_dim == w &&
                        h.layers[2].in_dim == w && h.layers[2].out_dim == out;
        if (!ok)
            throw InvalidArgument(std::string(names[k]) +
                                  ": only the production architecture of Table 1 "
                                  "(CvaeSpec::production_default) has a compiled device evaluator");
        for (const auto& l : h.layers) {
            for (float v : l.w) weights.push_back(v);
            for (float v : l.b) weights.push_back(v);
        }
        if (!(h.sigma_ref > 0.0) || !(h.n_ref > 1.0)) throw RuntimeError(std::string(names[k]) + ": bad normalisation constants");
        norms[2 * k] = std::log1p(h.sigma_ref);
        norms[2 * k + 1] = std::log(h.n_ref);
    }
    if (weights.size() != 1332) throw InvalidArgument("decoder parameter count mismatch");
}

// ------------------------------------------------------------------ meshes
namespace {
using P3 = std::array<double, 3>;
P3 normalize3(P3 v) {
    const double len = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
    return {v[0] / len, v[1] / len, v[2] / len};
}
}  // namespace

// Subdivided icosahedron (same construction and vertex order as mesh.cpp:154-185).
HostMesh make_icosphere(int subdivisions, double radius) {
    if (subdivisions < 0 || subdivisions > 9) throw InvalidArgument("icosphere subdivisions out of range");
    const double t = (1.0 + std::sqrt(5.0)) / 2.0;
    std::vector<P3> v;
    const double raw[12][3] = {{-1, t, 0}, {1, t, 0}, {-1, -t, 0}, {1, -t, 0}, {0, -1, t}, {0, 1, t},
                               {0, -1, -t}, {0, 1, -t}, {t, 0, -1}, {t, 0, 1}, {-t, 0, -1}, {-t, 0, 1}};
    for (const auto& r : raw) v.push_back(normalize3({r[0], r[1], r[2]}));
    std::vector<std::array<uint32_t, 3>> f = {
        {0, 11, 5}, {0, 5, 1}, {0, 1, 7}, {0, 7, 10}, {0, 10, 11}, {1, 5, 9}, {5, 11, 4},
        {11, 10, 2}, {10, 7, 6}, {7, 1, 8}, {3, 9, 4}, {3, 4, 2}, {3, 2, 6}, {3, 6, 8},
        {3, 8, 9}, {4, 9, 5}, {2, 4, 11}, {6, 2, 10}, {8, 6, 7}, {9, 8, 1}};
    std::unordered_map<uint64_t, uint32_t> cache;
    auto mid = [&](uint32_t a, uint32_t b) {
        const uint64_t key = a < b ? (uint64_t(a) << 32 | b) : (uint64_t(b) << 32 | a);
        const auto it = cache.find(key);
        if (it != cache.end()) return it->second;
        const P3& p = v[a];
        const P3& q = v[b];
        v.push_back(normalize3({p[0] + q[0], p[1] + q[1], p[2] + q[2]}));
        const uint32_t idx = static_cast<uint32_t>(v.size() - 1);
        cache.emplace(key, idx);
        return idx;
    };
    for (int s = 0; s < subdivisions; ++s) {
        std::vector<std::array<uint32_t, 3>> next;
        next.reserve(f.size() * 4);
        for (const auto& x : f) {
            const uint32_t ab = mid(x[0], x[1]), bc = mid(x[1], x[2]), ca = mid(x[2], x[0]);
            next.push_back({x[0], ab, ca});
            next.push_back({x[1], bc, ab});
            next.push_back({x[2], ca, bc});
            next.push_back({ab, bc, ca});
        }
        f.swap(next);
    }
    HostMesh m;
    for (const auto& p : v) m.pos.push_back({p[0] * radius, p[1] * radius, p[2] * radius});
    m.tri = std::move(f);
    return m;
}

// Radially perturbed icosphere (mesh.cpp:187-197).
HostMesh make_bumpy_sphere(int subdivisions, double radius, double amplitude, double frequency) {
    HostMesh m = make_icosphere(subdivisions, 1.0);
    for (auto& p : m.pos) {
        const double bump = 1.0 + amplitude * std::sin(frequency * p[0]) * std::sin(frequency * p[1]) *
                                      std::cos(frequency * p[2]);
        const double s = radius * bump;
        p = {p[0] * s, p[1] * s, p[2] * s};
    }
    return m;
}

// OBJ reader (mesh.cpp:77-122 semantics).
HostMesh load_obj(const std::string& path, double scale) {
    std::ifstream in(path);
    if (!in) throw RuntimeError("cannot open mesh: " + path);
    HostMesh m;
    std::string line;
    size_t line_no = 0;
    auto bad = [&](const std::string& what) {
        return RuntimeError("OBJ parse error at line " + std::to_string(line_no) + ": " + what);
    };
    while (std::getline(in, line)) {
        ++line_no;
        std::istringstream ls(line);
        std::string tag;
        if (!(ls >> tag)) continue;
        if (tag == "v") {
            double x, y, z;
            if (!(ls >> x >> y >> z)) throw bad("bad vertex");
            m.pos.push_back({x * scale, y * scale, z * scale});
        } else if (tag == "f") {
            std::vector<uint32_t> idx;
            std::string tok;
            while (ls >> tok) {
                const std::string head = tok.substr(0, tok.find('/'));
                long i = 0;
                try {
                    i = std::stol(head);
                } catch (const std::exception&) {
                    throw bad("bad face index '" + tok + "'");
                }
                if (i < 0) i = static_cast<long>(m.pos.size()) + i + 1;
                if (i < 1 || static_cast<size_t>(i) > m.pos.size()) throw bad("face index out of range '" + tok + "'");
                idx.push_back(static_cast<uint32_t>(i - 1));
            }
            if (idx.size() < 3) throw bad("face needs at least 3 vertices");
            for (size_t k = 2; k < idx.size(); ++k) {
                const std::array<uint32_t, 3> t = {idx[0], idx[k - 1], idx[k]};
                bool degen = t[0] == t[1] || t[1] == t[2] || t[0] == t[2];
                if (!degen) {
                    const P3 &a = m.pos[t[0]], &b = m.pos[t[1]], &c = m.pos[t[2]];
                    const double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
                    const double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
                    const double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                                         e1[0] * e2[1] - e1[1] * e2[0]};
                    degen = !(n[0] * n[0] + n[1] * n[1] + n[2] * n[2] > 0.0);
                }
                if (degen) ++m.dropped;
                else m.tri.push_back(t);
            }
        }
    }
    if (m.pos.empty() || m.tri.empty()) throw RuntimeError("OBJ file has no usable geometry: " + path);
    if (!is_watertight(m.tri))
        std::fprintf(stderr, "warning: mesh %s is not watertight; inside tests fall back to winding numbers\n",
                     path.c_str());
    return m;
}

bool is_convex(const double* pos, uint32_t nv, const std::vector<std::array<uint32_t, 3>>& tri) {
    if (static_cast<double>(nv) * tri.size() > 4e8) return false;  // too big to check: assume not
    double scale = 0.0;
    for (uint32_t i = 0; i < 3 * nv; ++i) scale = std::fmax(scale, std::fabs(pos[i]));
    const double tol = 1e-9 * std::fmax(scale, 1.0);
    for (const auto& f : tri) {
        const double* a = pos + 3 * f[0];
        const double* b = pos + 3 * f[1];
        const double* c = pos + 3 * f[2];
        const double e1[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
        const double e2[3] = {c[0] - a[0], c[1] - a[1], c[2] - a[2]};
        double n[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
        const double l = std::sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        if (!(l > 0)) continue;
        for (int k = 0; k < 3; ++k) n[k] /= l;
        double lo = 0.0, hi = 0.0;
        for (uint32_t v = 0; v < nv; ++v) {
            const double* p = pos + 3 * v;
            const double d = n[0] * (p[0] - a[0]) + n[1] * (p[1] - a[1]) + n[2] * (p[2] - a[2]);
            lo = std::fmin(lo, d);
            hi = std::fmax(hi, d);
        }
        if (lo < -tol && hi > tol) return false;  // vertices on both sides of a face plane
    }
    return !tri.empty();
}

bool is_watertight(const std::vector<std::array<uint32_t, 3>>& tri) {
    std::unordered_map<uint64_t, int> edges;
    for (const auto& f : tri)
        for (int e = 0; e < 3; ++e) {
            uint32_t a = f[e], b = f[(e + 1) % 3];
            if (a > b) std::swap(a, b);
            edges[uint64_t(a) << 32 | b] += 1;
        }
    for (const auto& kv : edges)
        if (kv.second != 2) return false;
    return !tri.empty();
}

// ------------------------------------------------------------------ BVH build
namespace {

struct Box {
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    void grow(const double* p) {
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], p[a]);
            hi[a] = std::max(hi[a], p[a]);
        }
    }
    void grow(const Box& b) {
        for (int a = 0; a < 3; ++a) {
            lo[a] = std::min(lo[a], b.lo[a]);
            hi[a] = std::max(hi[a], b.hi[a]);
        }
    }
    double area() const {
        const double dx = hi[0] - lo[0], dy = hi[1] - lo[1], dz = hi[2] - lo[2];
        if (dx < 0) return 0.0;
        return 2.0 * (dx * dy + dy * dz + dz * dx);
    }
};

struct TmpNode {
    Box b0, b1;
    int32_t c0 = -1, c1 = -1;
};

struct Builder {
    const std::vector<std::array<std::array<double, 3>, 3>>& tv;
    std::vector<uint32_t> order;
    std::vector<std::array<double, 3>> cent;
    std::vector<Box> tbox;
    std::vector<TmpNode> nodes;

    explicit Builder(const std::vector<std::array<std::array<double, 3>, 3>>& t) : tv(t) {
        const size_t n = t.size();
        order.resize(n);
        std::iota(order.begin(), order.end(), 0u);
        cent.resize(n);
        tbox.resize(n);
        for (size_t i = 0; i < n; ++i) {
            for (int k = 0; k < 3; ++k) tbox[i].grow(t[i][k].data());
            for (int a = 0; a < 3; ++a) cent[i][a] = (t[i][0][a] + t[i][1][a] + t[i][2][a]) / 3.0;
        }
    }

    Box range_box(uint32_t b, uint32_t e) const {
        Box r;
        for (uint32_t i = b; i < e; ++i) r.grow(tbox[order[i]]);
        return r;
    }

    static int32_t leaf(uint32_t first, uint32_t count) {
        return ~static_cast<int32_t>((first << 3) | count);
    }

    uint32_t split(uint32_t b, uint32_t e) {
        constexpr int kBins = 16;
        Box cb;
        for (uint32_t i = b; i < e; ++i) cb.grow(cent[order[i]].data());
        double best_cost = 1e300;
        int best_axis = -1, best_bin = 0;
        for (int a = 0; a < 3; ++a) {
            const double ext = cb.hi[a] - cb.lo[a];
            if (!(ext > 0.0)) continue;
            Box bins[kBins];
            uint32_t cnt[kBins] = {};
            for (uint32_t i = b; i < e; ++i) {
                int k = static_cast<int>((cent[order[i]][a] - cb.lo[a]) / ext * kBins);
                k = std::min(kBins - 1, std::max(0, k));
                bins[k].grow(tbox[order[i]]);
                ++cnt[k];
            }
            Box left[kBins];
            uint32_t lc[kBins];
            Box acc;
            uint32_t c = 0;
            for (int k = 0; k < kBins; ++k) {
                acc.grow(bins[k]);
                c += cnt[k];
                left[k] = acc;
                lc[k] = c;
            }
            Box racc;
            uint32_t rc = 0;
            for (int k = kBins - 1; k >= 1; --k) {
                racc.grow(bins[k]);
                rc += cnt[k];
                if (lc[k - 1] == 0 || rc == 0) continue;
                const double cost = left[k - 1].area() * lc[k - 1] + racc.area() * rc;
                if (cost < best_cost) {
                    best_cost = cost;
                    best_axis = a;
                    best_bin = k;
                }
            }
        }
        uint32_t mid;
        if (best_axis < 0) {
            mid = b + (e - b) / 2;
        } else {
            const double ext = cb.hi[best_axis] - cb.lo[best_axis];
            auto it = std::partition(order.begin() + b, order.begin() + e, [&](uint32_t t) {
                int k = static_cast<int>((cent[t][best_axis] - cb.lo[best_axis]) / ext * kBins);
                k = std::min(kBins - 1, std::max(0, k));
                return k < best_bin;
            });
            mid = static_cast<uint32_t>(it - order.begin());
            if (mid == b || mid == e) mid = b + (e - b) / 2;
        }
        return mid;
    }

    int32_t build(uint32_t b, uint32_t e) {
        if (e - b <= 4) return leaf(b, e - b);
        const uint32_t idx = static_cast<uint32_t>(nodes.size());
        nodes.emplace_back();
        const uint32_t mid = split(b, e);
        const int32_t l = build(b, mid);
        const int32_t r = build(mid, e);
        nodes[idx].b0 = range_box(b, mid);
        nodes[idx].b1 = range_box(mid, e);
        nodes[idx].c0 = l;
        nodes[idx].c1 = r;
        return static_cast<int32_t>(idx);
    }
};

float down(double v) {
    float f = static_cast<float>(v);
    if (static_cast<double>(f) > v) f = std::nextafter(f, -INFINITY);
    return f - (std::fabs(f) * 2e-7f + 1e-7f);
}
float up(double v) {
    float f = static_cast<float>(v);
    if (static_cast<double>(f) < v) f = std::nextafter(f, INFINITY);
    return f + (std::fabs(f) * 2e-7f + 1e-7f);
}
double pad_lo(double v) { return v - (std::fabs(v) * 1e-12 + 1e-300); }
double pad_hi(double v) { return v + (std::fabs(v) * 1e-12 + 1e-300); }

}  // namespace

FlatBvh build_bvh(const std::vector<std::array<std::array<double, 3>, 3>>& tv,
                  const std::vector<uint32_t>& tri_obj) {
    if (tv.empty()) throw InvalidArgument("scene has no triangles");
    if (tv.size() >= (1u << 28)) throw InvalidArgument("too many triangles");
    Builder bld(tv);
    const uint32_t n = static_cast<uint32_t>(tv.size());
    if (n <= 4) {
        TmpNode root;
        root.b0 = bld.range_box(0, n);
        root.b1 = root.b0;
        root.c0 = Builder::leaf(0, n);
        root.c1 = Builder::leaf(0, 0);
        bld.nodes.push_back(root);
    } else {
        bld.build(0, n);
    }
    FlatBvh out;
    out.n_nodes = static_cast<uint32_t>(bld.nodes.size());
    {  // deepest root-to-leaf path (traversal stacks hold at most one entry per level)
        std::vector<uint32_t> depth(out.n_nodes, 1);
        for (uint32_t i = 0; i < out.n_nodes; ++i) {  // parents precede children
            for (int32_t c : {bld.nodes[i].c0, bld.nodes[i].c1})
                if (c >= 0) depth[c] = depth[i] + 1;
            out.max_depth = std::max(out.max_depth, depth[i]);
        }
    }
    out.n_tris = n;
    out.order = bld.order;
    // Object id of every child subtree (-1 when mixed): lets a traversal cull the
    // object a ray is leaving when that object is convex.
    auto code_obj = [&](int32_t code, const std::vector<int32_t>& node_obj) -> int32_t {
        if (code >= 0) return node_obj[code];
        const uint32_t leaf = static_cast<uint32_t>(~code);
        const uint32_t first = leaf >> 3, count = leaf & 7u;
        if (count == 0) return -1;
        const int32_t o = static_cast<int32_t>(tri_obj[bld.order[first]]);
        for (uint32_t k = first + 1; k < first + count; ++k)
            if (static_cast<int32_t>(tri_obj[bld.order[k]]) != o) return -1;
        return o;
    };
    std::vector<int32_t> node_obj(out.n_nodes, -1);
    for (int32_t i = static_cast<int32_t>(out.n_nodes) - 1; i >= 0; --i) {  // children have larger indices
        const int32_t a = code_obj(bld.nodes[i].c0, node_obj), b = code_obj(bld.nodes[i].c1, node_obj);
        node_obj[i] = (a == b) ? a : -1;
    }
    {  // per-object traversal roots (see host.h FlatBvh::obj_root)
        uint32_t n_obj = 0;
        for (uint32_t t : tri_obj) n_obj = std::max(n_obj, t + 1);
        std::vector<Box> ob(n_obj);
        for (size_t i = 0; i < tv.size(); ++i)
            for (int k = 0; k < 3; ++k) ob[tri_obj[i]].grow(tv[i][k].data());
        bool disjoint = true;
        for (uint32_t a = 0; a < n_obj && disjoint; ++a)
            for (uint32_t b = a + 1; b < n_obj && disjoint; ++b) {
                bool overlap = true;
                for (int k = 0; k < 3; ++k)
                    overlap &= ob[a].lo[k] <= ob[b].hi[k] && ob[b].lo[k] <= ob[a].hi[k];
                disjoint = !overlap;
            }
        out.obj_root.assign(n_obj, -1);
        if (disjoint && n_obj > 1) {
            std::vector<int32_t> parent(out.n_nodes, -1), count(n_obj, 0), cand(n_obj, -1);
            for (uint32_t i = 0; i < out.n_nodes; ++i)
                for (int32_t c : {bld.nodes[i].c0, bld.nodes[i].c1})
                    if (c >= 0) parent[c] = static_cast<int32_t>(i);
            for (uint32_t i = 0; i < out.n_nodes; ++i) {
                const int32_t o = node_obj[i];
                if (o >= 0 && (parent[i] < 0 || node_obj[parent[i]] < 0)) {
                    ++count[o];
                    cand[o] = static_cast<int32_t>(i);
                }
            }
            for (uint32_t o = 0; o < n_obj; ++o)
                if (count[o] == 1) out.obj_root[o] = cand[o];
        }
    }
    std::vector<NodeF> nf(out.n_nodes);
    std::vector<NodeD> nd(out.n_nodes);
    for (uint32_t i = 0; i < out.n_nodes; ++i) {
        const TmpNode& t = bld.nodes[i];
        nf[i].a = make_float4(down(t.b0.lo[0]), up(t.b0.hi[0]), down(t.b0.lo[1]), up(t.b0.hi[1]));
        nf[i].b = make_float4(down(t.b1.lo[0]), up(t.b1.hi[0]), down(t.b1.lo[1]), up(t.b1.hi[1]));
        nf[i].c = make_float4(down(t.b0.lo[2]), up(t.b0.hi[2]), down(t.b1.lo[2]), up(t.b1.hi[2]));
        const int32_t o0 = code_obj(t.c0, node_obj), o1 = code_obj(t.c1, node_obj);
        nf[i].d = make_int4(t.c0, t.c1, o0, o1);
        for (int a = 0; a < 3; ++a) {
            nd[i].lo0[a] = pad_lo(t.b0.lo[a]);
            nd[i].hi0[a] = pad_hi(t.b0.hi[a]);
            nd[i].lo1[a] = pad_lo(t.b1.lo[a]);
            nd[i].hi1[a] = pad_hi(t.b1.hi[a]);
        }
        nd[i].c0 = t.c0;
        nd[i].c1 = t.c1;
        nd[i].pad0 = o0;
        nd[i].pad1 = o1;
    }
    std::vector<TriF> tf(n);
    std::vector<TriD> td(n);
    for (uint32_t i = 0; i < n; ++i) {
        const auto& t = tv[bld.order[i]];
        const uint32_t obj = tri_obj[bld.order[i]];
        double e1[3], e2[3];
        for (int a = 0; a < 3; ++a) {
            e1[a] = t[1][a] - t[0][a];  // b - a, bvh.cpp:13
            e2[a] = t[2][a] - t[0][a];  // c - a
        }
        float objf, idf;
        std::memcpy(&objf, &obj, 4);
        std::memcpy(&idf, &i, 4);
        tf[i].v0o = make_float4(static_cast<float>(t[0][0]), static_cast<float>(t[0][1]),
                                static_cast<float>(t[0][2]), objf);
        tf[i].e1i = make_float4(static_cast<float>(e1[0]), static_cast<float>(e1[1]),
                                static_cast<float>(e1[2]), idf);
        tf[i].e2 = make_float4(static_cast<float>(e2[0]), static_cast<float>(e2[1]),
                               static_cast<float>(e2[2]), 0.0f);
        for (int a = 0; a < 3; ++a) {
            td[i].v0[a] = t[0][a];
            td[i].e1[a] = e1[a];
            td[i].e2[a] = e2[a];
        }
        td[i].obj = obj;
        td[i].id = i;
    }
    auto bytes = [](const auto& v) {
        std::vector<uint8_t> b(v.size() * sizeof(v[0]));
        std::memcpy(b.data(), v.data(), b.size());
        return b;
    };
    out.nodes_f32 = bytes(nf);
    out.nodes_f64 = bytes(nd);
    out.tris_f32 = bytes(tf);
    out.tris_f64 = bytes(td);
    return out;
}

// ------------------------------------------------------------------ training (host side)
HostStream::HostStream(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t s3) : s(rng_key(seed, s1, s2, s3)) {}

uint64_t HostStream::next_u64() {
    s += kGolden;
    return mix64(s);
}

CvaeSpecH production_spec(int kind) {
    CvaeSpecH s;
    switch (kind) {
        case 0: s = {2, 1, 2, 8, 2}; break;
        case 1: s = {3, 3, 2, 16, 5}; break;
        case 2: s = {7, 6, 2, 16, 5}; break;
        default: throw InvalidArgument("unknown model kind");
    }
    return s;
}

void validate_spec(const CvaeSpecH& s) {
    if (s.p_in == 0 || s.p_out == 0 || s.width == 0 || s.latent == 0)
        throw InvalidArgument("CvaeSpec: zero dimension");
    if ((s.p_in + s.latent) % 4 != 0)
        throw InvalidArgument("CvaeSpec: p_in + latent must be a multiple of four");
}

size_t MlpShape::params() const {
    size_t n = 0;
    for (size_t i = 0; i < in.size(); ++i) n += static_cast<size_t>(in[i]) * out[i] + out[i];
    return n;
}

static MlpShape mlp_shape(uint32_t input, uint32_t output, uint32_t depth, uint32_t width) {
    MlpShape m;
    uint32_t in = input;
    for (uint32_t d = 0; d <= depth; ++d) {
        const uint32_t out = d == depth ? output : width;
        m.in.push_back(in);
        m.out.push_back(out);
        in = out;
    }
    return m;
}

MlpShape encoder_shape(const CvaeSpecH& s) { return mlp_shape(s.p_out + s.p_in, 2 * s.latent, s.depth, s.width); }
MlpShape decoder_shape(const CvaeSpecH& s) { return mlp_shape(s.latent + s.p_in, 2 * s.p_out, s.depth, s.width); }

// make_mlp + make_gaussian_mlp (mlp.cpp:32-58), flattened (weights then bias per layer).
static std::vector<double> gaussian_mlp(const MlpShape& m, uint32_t p_out, HostStream& rng) {
    std::vector<double> flat;
    flat.reserve(m.params());
    for (size_t l = 0; l < m.in.size(); ++l) {
        const double bound = std::sqrt(6.0 / (static_cast<double>(m.in[l]) + m.out[l]));
        for (size_t i = 0; i < static_cast<size_t>(m.in[l]) * m.out[l]; ++i) flat.push_back(rng.uniform(-bound, bound));
        const bool head = l + 1 == m.in.size();
        for (uint32_t r = 0; r < m.out[l]; ++r) flat.push_back(head && r >= p_out ? -2.0 : 0.0);
    }
    for (double& v : flat) v = static_cast<double>(static_cast<float>(v));  // quantize_f32 (mlp.cpp:25-30)
    return flat;
}

void make_cvae_params(int kind, const CvaeSpecH& s, uint64_t seed, std::vector<double>& enc, std::vector<double>& dec) {
    validate_spec(s);
    HostStream rng(seed, 0x02 /* kTrainInit */, static_cast<uint64_t>(kind));
    enc = gaussian_mlp(encoder_shape(s), s.latent, rng);
    dec = gaussian_mlp(decoder_shape(s), s.p_out, rng);
}

namespace {
struct Writer {
    std::ofstream out;
    std::string path;
    explicit Writer(const std::string& p) : out(p, std::ios::binary | std::ios::trunc), path(p) {
        if (!out) throw RuntimeError("cannot open for writing: " + p);
    }
    template <class T>
    void put(T v) {  // little-endian host (x86-64 / aarch64)
        out.write(reinterpret_cast<const char*>(&v), sizeof v);
    }
};

void write_mlp(Writer& w, const MlpShape& m, const std::vector<double>& flat) {
    w.put<uint32_t>(static_cast<uint32_t>(m.in.size()));
    size_t off = 0;
    for (size_t l = 0; l < m.in.size(); ++l) {
        w.put<uint32_t>(m.out[l]);
        w.put<uint32_t>(m.in[l]);
        const size_t n = static_cast<size_t>(m.in[l]) * m.out[l] + m.out[l];
        for (size_t i = 0; i < n; ++i) w.put<float>(static_cast<float>(flat[off + i]));
        off += n;
    }
}
}  // namespace

void save_ssnn(const std::string& path, int kind, const CvaeSpecH& s, double sigma_ref, double n_ref,
               uint64_t fingerprint, const std::vector<double>& dec, const std::vector<double>* enc) {
    Writer w(path);
    w.out.write("SSNN", 4);
    w.put<uint32_t>(1);
    w.put<uint32_t>(static_cast<uint32_t>(kind));
    w.put<uint32_t>(enc ? 1u : 0u);
    w.put<uint32_t>(s.p_in);
    w.put<uint32_t>(s.p_out);
    w.put<uint32_t>(s.depth);
    w.put<uint32_t>(s.width);
    w.put<uint32_t>(s.latent);
    w.put<double>(sigma_ref);
    w.put<double>(n_ref);
    w.put<uint64_t>(fingerprint);
    write_mlp(w, decoder_shape(s), dec);
    if (enc) write_mlp(w, encoder_shape(s), *enc);
    w.out.close();
    if (!w.out) throw RuntimeError("write failure on close");
}

HostModel model_from_params(int kind, const CvaeSpecH& s, double sigma_ref, double n_ref,
                            const std::vector<double>& dec) {
    HostModel m;
    m.kind = static_cast<uint32_t>(kind);
    m.p_in = s.p_in;
    m.p_out = s.p_out;
    m.depth = s.depth;
    m.width = s.width;
    m.latent = s.latent;
    m.sigma_ref = sigma_ref;
    m.n_ref = n_ref;
    const MlpShape sh = decoder_shape(s);
    size_t off = 0;
    for (size_t l = 0; l < sh.in.size(); ++l) {
        HostLayer hl;
        hl.out_dim = sh.out[l];
        hl.in_dim = sh.in[l];
        const size_t nw = static_cast<size_t>(hl.out_dim) * hl.in_dim;
        for (size_t i = 0; i < nw; ++i) hl.w.push_back(static_cast<float>(dec[off + i]));
        for (size_t i = 0; i < hl.out_dim; ++i) hl.b.push_back(static_cast<float>(dec[off + nw + i]));
        off += nw + hl.out_dim;
        m.layers.push_back(std::move(hl));
    }
    return m;
}

}  // namespace sstg
