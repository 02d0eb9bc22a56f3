/*
 * oracle/sst_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker; never the
 * product path, never linked into libsst_gpu.so).
 *
 * Plain-C restatement of the reference's hot path. Every function cites the
 * reference file:line it restates (paths relative to /root/reference/proj/core/).
 * Floating-point expressions keep the reference's operation order and the file
 * is compiled with -ffp-contract=off, so results are bit-identical to the
 * reference build (pinned by tests/test_oracle_*.py and tests/golden/).
 * The integrator (absent from the reference: CMakeLists.txt:14,16) follows
 * SPEC.md:540-566 as fixed in DESIGN.md "Integrator semantics".
 */
#include "sst_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[1024];

static int fail(int rc, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return rc;
}

const char* so_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ vec3 (vec3.hpp) */
typedef struct { double x, y, z; } v3;
static v3 V(double x, double y, double z) { v3 r = {x, y, z}; return r; }
static v3 add(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 sub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 mul(v3 a, double s) { return V(a.x * s, a.y * s, a.z * s); }
static v3 dvs(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static double dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }          /* vec3.hpp:31 */
static v3 cross(v3 a, v3 b) {                                                          /* vec3.hpp:33-35 */
    return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static double length(v3 v) { return sqrt(dot(v, v)); }
static v3 normalize(v3 v) { double l = length(v); return V(v.x / l, v.y / l, v.z / l); } /* vec3.hpp:40-43 */
static v3 ld3(const double* p) { return V(p[0], p[1], p[2]); }
static void st3(double* p, v3 v) { p[0] = v.x; p[1] = v.y; p[2] = v.z; }
static double comp(v3 v, int a) { return a == 0 ? v.x : (a == 1 ? v.y : v.z); }

/* orthonormal_basis, vec3.hpp:53-59 */
static void onb(v3 n, v3* b1, v3* b2) {
    const double sign = copysign(1.0, n.z);
    const double a = -1.0 / (sign + n.z);
    const double b = n.x * n.y * a;
    *b1 = V(1.0 + sign * n.x * n.x * a, sign * b, -sign * n.x);
    *b2 = V(b, sign + n.y * n.y * a, -n.y);
}

/* Mat3 column-major, vec3.hpp:62-83 */
typedef struct { v3 c0, c1, c2; } m3;
static v3 mv(m3 m, v3 v) { return add(add(mul(m.c0, v.x), mul(m.c1, v.y)), mul(m.c2, v.z)); }
static m3 mm(m3 a, m3 b) { m3 r = {mv(a, b.c0), mv(a, b.c1), mv(a, b.c2)}; return r; }
static m3 frame_to(v3 w) { m3 r; onb(w, &r.c0, &r.c1); r.c2 = w; return r; }
static m3 rotation_z(double ang) {
    const double c = cos(ang), s = sin(ang);
    m3 r = {V(c, s, 0.0), V(-s, c, 0.0), V(0.0, 0.0, 1.0)};
    return r;
}

/* ------------------------------------------------------------------ RNG (rng.hpp:15-50) */
static uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
uint64_t so_rng_init(uint64_t seed, uint64_t s1, uint64_t s2, uint64_t s3) {
    uint64_t s = mix(seed);
    s = mix(s ^ (s1 + 0x9E3779B97F4A7C15ULL));
    s = mix(s ^ (s2 + 0xBF58476D1CE4E5B9ULL));
    s = mix(s ^ (s3 + 0x94D049BB133111EBULL));
    return s;
}
uint64_t so_next_u64(so_rng* r) {
    r->state += 0x9E3779B97F4A7C15ULL;
    return mix(r->state);
}
double so_uniform(so_rng* r) { return (double)(so_next_u64(r) >> 11) * 0x1.0p-53; }
double so_normal(so_rng* r) {
    const double u1 = 1.0 - so_uniform(r);
    const double u2 = so_uniform(r);
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}
void so_rng_draws(uint64_t state, uint64_t n, uint64_t* u64, double* uni, double* nor) {
    so_rng a = {state}, b = {state}, c = {state};
    for (uint64_t i = 0; i < n; ++i) {
        if (u64) u64[i] = so_next_u64(&a);
        if (uni) uni[i] = so_uniform(&b);
        if (nor) nor[i] = so_normal(&c);
    }
}

/* ------------------------------------------------------------------ optics (optics.cpp) */
#define kInv4Pi 0.07957747154594766788
#define kTwoPi 6.28318530717958647692
static int bad_g(double g) { return !(g > -1.0 && g < 1.0); }

int so_hg_eval(double g, double c, double* out) {                     /* optics.cpp:27-31 */
    if (bad_g(g)) return fail(SST_E_DOMAIN, "HG anisotropy g must lie in (-1, 1)");
    const double denom = 1.0 + g * g - 2.0 * g * c;
    *out = kInv4Pi * (1.0 - g * g) / (denom * sqrt(denom));
    return 0;
}
static double hg_cos(double g, double u) {                             /* optics.cpp:33-39 */
    if (fabs(g) < 1e-4) return 1.0 - 2.0 * u;
    const double s = (1.0 - g * g) / (1.0 + g - 2.0 * g * u);
    const double c = (1.0 + g * g - s * s) / (2.0 * g);
    return c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
}
int so_hg_sample_cos(double g, double u, double* out) {
    if (bad_g(g)) return fail(SST_E_DOMAIN, "HG anisotropy g must lie in (-1, 1)");
    *out = hg_cos(g, u);
    return 0;
}
static v3 hg_sample(double g, v3 w_in, double u1, double u2) {         /* optics.cpp:41-48 */
    const double ct = hg_cos(g, u1);
    const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    const double ph = kTwoPi * u2;
    v3 b1, b2;
    onb(w_in, &b1, &b2);
    return add(add(mul(b1, st * cos(ph)), mul(b2, st * sin(ph))), mul(w_in, ct));
}
int so_hg_sample(double g, const double w[3], double u1, double u2, double out[3]) {
    if (bad_g(g)) return fail(SST_E_DOMAIN, "HG anisotropy g must lie in (-1, 1)");
    st3(out, hg_sample(g, ld3(w), u1, u2));
    return 0;
}
int so_transmittance(double s, double d, double* out) {               /* optics.cpp:50-53 */
    if (!(d >= 0.0)) return fail(SST_E_DOMAIN, "transmittance distance must be >= 0");
    *out = exp(-s * d);
    return 0;
}
int so_sample_free_path(double s, double xi, double* out) {           /* optics.cpp:55-60 */
    if (!(s > 0.0)) return fail(SST_E_DOMAIN, "sample_free_path requires sigma_t > 0");
    if (!(xi >= 0.0 && xi < 1.0)) return fail(SST_E_DOMAIN, "free-path variate must lie in [0, 1)");
    *out = -log1p(-xi) / s;
    return 0;
}
static double absorption_prob(uint64_t n, double phi) {                /* optics.cpp:62-67 */
    if (n == 0 || phi >= 1.0) return 0.0;
    if (phi <= 0.0) return 1.0;
    return -expm1((double)n * log(phi));
}
int so_absorption_prob(uint64_t n, double phi, double* out) {
    if (!(phi >= 0.0 && phi <= 1.0)) return fail(SST_E_DOMAIN, "albedo phi must lie in [0, 1]");
    *out = absorption_prob(n, phi);
    return 0;
}
double so_representative_weight_sum(uint64_t n, double phi) {         /* optics.cpp:69-75 */
    if (n == 0 || phi <= 0.0) return 0.0;
    if (phi >= 1.0) return (double)n;
    const double phi_n = exp((double)n * log(phi));
    return phi * (1.0 - phi_n) / (1.0 - phi);
}
double so_softplus(double x) { return fmax(x, 0.0) + log1p(exp(-fabs(x))); } /* mlp.cpp:60-62 */

/* ------------------------------------------------------------------ models */
typedef struct { uint32_t out_dim, in_dim; double* w; double* b; } so_layer;
typedef struct {
    uint32_t kind, p_in, p_out, depth, width, latent;
    double sigma_ref, n_ref;
    uint32_t n_layers;
    so_layer layers[16];
} so_model;
struct so_models { so_model m[3]; uint64_t counters[3]; };

static int rd(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n; }

/* load_model, cvae.cpp:379-425 (SSNN v1; decoder kept, encoder skipped) */
static int load_model(const char* path, so_model* m) {
    FILE* f = fopen(path, "rb");
    char msg[512];
    if (!f) { snprintf(msg, sizeof msg, "cannot open for reading: %s", path); return fail(SST_E_RUNTIME, msg); }
    char magic[4];
    uint32_t h[8];
    uint64_t fp;
    int ok = rd(f, magic, 4) && memcmp(magic, "SSNN", 4) == 0;
    if (!ok) { fclose(f); snprintf(msg, sizeof msg, "model %s: bad magic bytes", path); return fail(SST_E_RUNTIME, msg); }
    ok = rd(f, h, sizeof h) && rd(f, &m->sigma_ref, 8) && rd(f, &m->n_ref, 8) && rd(f, &fp, 8);
    if (ok && h[0] != 1) { fclose(f); snprintf(msg, sizeof msg, "model %s: unsupported version %u", path, h[0]); return fail(SST_E_RUNTIME, msg); }
    m->kind = h[1]; m->p_in = h[3]; m->p_out = h[4]; m->depth = h[5]; m->width = h[6]; m->latent = h[7];
    uint32_t nl = 0;
    ok = ok && rd(f, &nl, 4) && nl > 0 && nl <= 16;
    m->n_layers = ok ? nl : 0;
    for (uint32_t i = 0; ok && i < nl; ++i) {
        so_layer* L = &m->layers[i];
        ok = rd(f, &L->out_dim, 4) && rd(f, &L->in_dim, 4) && L->out_dim && L->in_dim &&
             L->out_dim <= 4096 && L->in_dim <= 4096;
        if (!ok) break;
        const size_t nw = (size_t)L->out_dim * L->in_dim;
        float* tmp = (float*)malloc((nw + L->out_dim) * sizeof(float));
        ok = rd(f, tmp, (nw + L->out_dim) * sizeof(float));
        L->w = (double*)malloc(nw * sizeof(double));
        L->b = (double*)malloc(L->out_dim * sizeof(double));
        for (size_t k = 0; k < nw; ++k) L->w[k] = tmp[k];
        for (size_t k = 0; k < L->out_dim; ++k) L->b[k] = tmp[nw + k];
        free(tmp);
    }
    fclose(f);
    if (!ok) { snprintf(msg, sizeof msg, "model %s: truncated or corrupt file", path); return fail(SST_E_RUNTIME, msg); }
    if (m->layers[0].in_dim != m->latent + m->p_in || m->layers[nl - 1].out_dim != 2 * m->p_out) {
        snprintf(msg, sizeof msg, "model %s: decoder shape disagrees with header", path);
        return fail(SST_E_RUNTIME, msg);
    }
    return 0;
}

static void free_model(so_model* m) {
    for (uint32_t i = 0; i < m->n_layers; ++i) { free(m->layers[i].w); free(m->layers[i].b); }
    m->n_layers = 0;
}

void so_models_free(so_models* m) {
    if (!m) return;
    for (int k = 0; k < 3; ++k) free_model(&m->m[k]);
    free(m);
}

/* ScatterModels::load_dir + kind check, scatter.cpp:15-32 */
int so_models_load_dir(const char* dir, so_models** out) {
    static const char* names[3] = {"lengthgen", "pathgen", "eventgen"};
    so_models* ms = (so_models*)calloc(1, sizeof(so_models));
    for (int k = 0; k < 3; ++k) {
        char path[1024];
        snprintf(path, sizeof path, "%s/%s.ssnn", dir, names[k]);
        const int rc = load_model(path, &ms->m[k]);
        if (rc) { so_models_free(ms); return rc; }
        if (ms->m[k].kind != (uint32_t)k) {
            so_models_free(ms);
            return fail(SST_E_RUNTIME, "ScatterModels: model bundle has wrong kind tag");
        }
    }
    *out = ms;
    return 0;
}

void so_models_counters(const so_models* m, uint64_t out[3]) {
    for (int k = 0; k < 3; ++k) out[k] = m->counters[k];
}

/* mlp_forward (mlp.cpp:70-87) + cvae_decode log-var clamp (cvae.cpp:20-22,93-98) */
static void decode(const so_model* m, const double* in, double* mu, double* lv) {
    double a[4096], b[4096];
    memcpy(a, in, m->layers[0].in_dim * sizeof(double));
    double *cur = a, *nxt = b;
    for (uint32_t li = 0; li < m->n_layers; ++li) {
        const so_layer* L = &m->layers[li];
        for (uint32_t r = 0; r < L->out_dim; ++r) {
            double acc = L->b[r];
            const double* wr = L->w + (size_t)r * L->in_dim;
            for (uint32_t c = 0; c < L->in_dim; ++c) acc += wr[c] * cur[c];
            nxt[r] = (li + 1 == m->n_layers) ? acc : so_softplus(acc);
        }
        double* t = cur; cur = nxt; nxt = t;
    }
    for (uint32_t i = 0; i < m->p_out; ++i) {
        mu[i] = cur[i];
        lv[i] = fmin(10.0, fmax(-10.0, cur[m->p_out + i]));
    }
}

int so_cvae_decode(const so_models* ms, int kind, const double* z, const double* c, double* mu,
                   double* lv) {
    const so_model* m = &ms->m[kind];
    double in[64];
    for (uint32_t i = 0; i < m->latent; ++i) in[i] = z[i];
    for (uint32_t i = 0; i < m->p_in; ++i) in[m->latent + i] = c[i];
    decode(m, in, mu, lv);
    return 0;
}

/* NormConstants, cvae.cpp:67-77 */
static double norm_sigma(const so_model* m, double s) { return log1p(fmax(0.0, s)) / log1p(m->sigma_ref); }
static double norm_n(const so_model* m, double n) { return log(fmax(1.0, n)) / log(m->n_ref); }

/* decode_with_retry, scatter.cpp:44-58: z then eps draws, reparameterize
 * (mlp.cpp:204-212), retry once on non-finite output. */
static int decode_sample(so_models* ms, int kind, const double* c, so_rng* rng, double* out) {
    const so_model* m = &ms->m[kind];
    for (int attempt = 0; attempt < 2; ++attempt) {
        double in[64], eps[32], mu[32], lv[32];
        for (uint32_t i = 0; i < m->latent; ++i) in[i] = so_normal(rng);
        for (uint32_t i = 0; i < m->p_out; ++i) eps[i] = so_normal(rng);
        ms->counters[kind] += 1;
        for (uint32_t i = 0; i < m->p_in; ++i) in[m->latent + i] = c[i];
        decode(m, in, mu, lv);
        int finite = 1;
        for (uint32_t i = 0; i < m->p_out; ++i) {
            out[i] = mu[i] + exp(0.5 * lv[i]) * eps[i];
            finite = finite && isfinite(out[i]);
        }
        if (finite) return 0;
    }
    return fail(SST_E_RUNTIME, "decoder produced non-finite output twice");
}

typedef struct { m3 rot; v3 center; double radius; } frame_t;
static v3 point_to_world(const frame_t* f, v3 p) { return add(f->center, mul(mv(f->rot, p), f->radius)); }

/* to_world, scatter.cpp:102-129 (make_sphere_frame :93-100) */
static void to_world(double ct, double al, double be, v3 w_in, v3 center, double r, double psi,
                     v3* pos, v3* dir, frame_t* fr) {
    fr->rot = mm(frame_to(w_in), rotation_z(psi));
    fr->center = center;
    fr->radius = r;
    const double st = sqrt(fmax(0.0, 1.0 - ct * ct));
    const v3 e_n = V(st, 0.0, ct);
    *pos = point_to_world(fr, e_n);
    v3 e_b, b2;
    if (st < 1e-9) onb(e_n, &e_b, &b2);
    else e_b = normalize(cross(V(0.0, 0.0, 1.0), e_n));
    const v3 e_t = cross(e_b, e_n);
    const double nc = sqrt(fmax(0.0, 1.0 - al * al - be * be));
    const v3 d = normalize(add(add(mul(e_b, al), mul(e_t, be)), mul(e_n, nc)));
    *dir = mv(fr->rot, d);
}

int so_to_world(double ct, double al, double be, const double w_in[3], const double center[3],
                double r, double psi, double pos[3], double dir[3]) {
    if (!(r > 0.0)) return fail(SST_E_DOMAIN, "to_world: r_sphere must be > 0");
    v3 p, d;
    frame_t f;
    to_world(ct, al, be, ld3(w_in), ld3(center), r, psi, &p, &d, &f);
    st3(pos, p); st3(dir, d);
    return 0;
}

typedef struct {
    int absorbed;
    uint32_t n;
    v3 exit_pos, exit_dir;
    int has_rep;
    v3 rep_pos, rep_dir;
    double lambda;
} step_out;

/* sample_sphere_step, scatter.cpp:152-177 (+ sample_num_events :62-70,
 * test_absorption :72-74, sample_exit :76-91, sample_event :131-150) */
static int sphere_step(so_models* ms, double sigma_t, double g, double phi, v3 w_in, v3 center,
                       double r, int with_event, so_rng* rng, step_out* o) {
    memset(o, 0, sizeof *o);
    o->n = 1;
    if (!(sigma_t >= 0.0 && r >= 0.0)) return fail(SST_E_DOMAIN, "rescale_sigma: negative input");
    const double ss = sigma_t * r;
    double out[8];
    /* LengthGen */
    double cl[2] = {norm_sigma(&ms->m[0], ss), g};
    int rc = decode_sample(ms, 0, cl, rng, out);
    if (rc) return rc;
    const double nn = exp(out[0] * log(ms->m[0].n_ref));
    o->n = !(nn < 4e9) ? 4000000000u : (uint32_t)fmax(1.0, round(nn));
    const double u = so_uniform(rng);
    if (u < absorption_prob(o->n, phi)) { o->absorbed = 1; return 0; }
    /* PathGen */
    double cp[3] = {norm_sigma(&ms->m[1], ss), g, norm_n(&ms->m[1], (double)o->n)};
    rc = decode_sample(ms, 1, cp, rng, out);
    if (rc) return rc;
    const double ct = fmin(1.0, fmax(-1.0, out[0]));
    double al = out[1], be = out[2];
    const double r2 = al * al + be * be;
    if (r2 > 1.0) { const double inv = 1.0 / sqrt(r2); al *= inv; be *= inv; }
    const double psi = kTwoPi * so_uniform(rng);
    if (!(r > 0.0)) return fail(SST_E_DOMAIN, "to_world: r_sphere must be > 0");
    frame_t fr;
    to_world(ct, al, be, w_in, center, r, psi, &o->exit_pos, &o->exit_dir, &fr);
    if (with_event) {
        double ce[7] = {norm_sigma(&ms->m[2], ss), g, phi, ct, al, be, norm_n(&ms->m[2], (double)o->n)};
        rc = decode_sample(ms, 2, ce, rng, out);
        if (rc) return rc;
        v3 X = V(out[0], out[1], out[2]);
        const double lx = length(X);
        if (lx >= 1.0) X = mul(X, 0.999 / lx);
        v3 W = V(out[3], out[4], out[5]);
        const double lw = length(W);
        W = lw > 0.0 ? dvs(W, lw) : V(0.0, 0.0, 1.0);
        o->has_rep = 1;
        o->rep_pos = point_to_world(&fr, X);
        o->rep_dir = mv(fr.rot, W);
        o->lambda = so_representative_weight_sum(o->n, phi);
    }
    return 0;
}

int so_sphere_step_batch(so_models* ms, uint64_t n, const sst_step_in* in, int with_event_default,
                         sst_step_out* out) {
    for (uint64_t i = 0; i < n; ++i) {
        so_rng rng = {in->rng_state[i]};
        step_out o;
        const int we = in->with_event ? in->with_event[i] != 0 : with_event_default != 0;
        const int rc = sphere_step(ms, in->sigma_t[i], in->g[i], in->phi[i], ld3(in->w_in + 3 * i),
                                   ld3(in->center + 3 * i), in->r_sphere[i], we, &rng, &o);
        if (rc) return rc;
        in->rng_state[i] = rng.state;
        out->absorbed[i] = (uint8_t)o.absorbed;
        out->n_events[i] = o.n;
        st3(out->exit_position + 3 * i, o.exit_pos);
        st3(out->exit_direction + 3 * i, o.exit_dir);
        out->has_representative[i] = (uint8_t)o.has_rep;
        st3(out->rep_position + 3 * i, o.rep_pos);
        st3(out->rep_direction + 3 * i, o.rep_dir);
        out->lambda_weight[i] = o.lambda;
    }
    return 0;
}

/* ------------------------------------------------------------------ SDF (sdf.cpp) */
double so_query_safe_radius(const double origin[3], double voxel, const uint32_t dims[3],
                            const float* values, const double p[3]) {   /* sdf.cpp:60-69 */
    const double rx = (p[0] - origin[0]) / voxel;
    const double ry = (p[1] - origin[1]) / voxel;
    const double rz = (p[2] - origin[2]) / voxel;
    if (rx < 0.0 || ry < 0.0 || rz < 0.0) return 0.0;
    const uint32_t x = (uint32_t)rx, y = (uint32_t)ry, z = (uint32_t)rz;
    if (x >= dims[0] || y >= dims[1] || z >= dims[2]) return 0.0;
    const float v = values[((size_t)z * dims[1] + y) * dims[0] + x];
    return v < 0.0f ? -(double)v : 0.0;
}

/* Moller-Trumbore, bvh.cpp:11-27 (same operation order) */
static int ray_tri(v3 o, v3 d, double t_max, v3 a, v3 b, v3 c, double t_min, double* t_out) {
    const v3 e1 = sub(b, a), e2 = sub(c, a);
    const v3 pvec = cross(d, e2);
    const double det = dot(e1, pvec);
    if (fabs(det) < 1e-14) return 0;
    const double inv_det = 1.0 / det;
    const v3 tvec = sub(o, a);
    const double u = dot(tvec, pvec) * inv_det;
    if (u < 0.0 || u > 1.0) return 0;
    const v3 qvec = cross(tvec, e1);
    const double v = dot(d, qvec) * inv_det;
    if (v < 0.0 || u + v > 1.0) return 0;
    const double t = dot(e2, qvec) * inv_det;
    if (t <= t_min || t >= t_max) return 0;
    *t_out = t;
    return 1;
}

/* point_triangle_distance_squared, mesh.cpp:199-233 */
static double pt_tri_d2(v3 p, v3 a, v3 b, v3 c) {
    const v3 ab = sub(b, a), ac = sub(c, a), ap = sub(p, a);
    const double d1 = dot(ab, ap), d2 = dot(ac, ap);
    if (d1 <= 0.0 && d2 <= 0.0) { v3 q = sub(p, a); return dot(q, q); }
    const v3 bp = sub(p, b);
    const double d3 = dot(ab, bp), d4 = dot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) { v3 q = sub(p, b); return dot(q, q); }
    const double vc = d1 * d4 - d3 * d2;
    if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double v = d1 / (d1 - d3);
        v3 q = sub(p, add(a, mul(ab, v)));
        return dot(q, q);
    }
    const v3 cp = sub(p, c);
    const double d5 = dot(ab, cp), d6 = dot(ac, cp);
    if (d6 >= 0.0 && d5 <= d6) { v3 q = sub(p, c); return dot(q, q); }
    const double vb = d5 * d2 - d1 * d6;
    if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        const double w = d2 / (d2 - d6);
        v3 q = sub(p, add(a, mul(ac, w)));
        return dot(q, q);
    }
    const double va = d3 * d6 - d5 * d4;
    if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
        const double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
        v3 q = sub(p, add(b, mul(sub(c, b), w)));
        return dot(q, q);
    }
    const double denom = 1.0 / (va + vb + vc);
    const double v = vb * denom, w = vc * denom;
    v3 q = sub(p, add(add(a, mul(ab, v)), mul(ac, w)));
    return dot(q, q);
}

/* build_sdf, sdf.cpp:20-58, brute force over triangles (the BVH only prunes;
 * min distance and hit parity are structure-independent). Watertight meshes
 * assumed (parity inside test, bvh.cpp:204-217). */
int so_build_sdf(const double* pos, uint32_t nv, const uint32_t* tris, uint32_t nt,
                 uint32_t resolution, double origin[3], double* voxel, uint32_t dims[3],
                 float* values) {
    if (resolution < 8) return fail(SST_E_INVALID_ARGUMENT, "build_sdf: resolution must be >= 8");
    v3 lo = V(1e300, 1e300, 1e300), hi = V(-1e300, -1e300, -1e300);
    for (uint32_t i = 0; i < nv; ++i) {
        lo = V(fmin(lo.x, pos[3 * i]), fmin(lo.y, pos[3 * i + 1]), fmin(lo.z, pos[3 * i + 2]));
        hi = V(fmax(hi.x, pos[3 * i]), fmax(hi.y, pos[3 * i + 1]), fmax(hi.z, pos[3 * i + 2]));
    }
    const v3 ext = sub(hi, lo);
    const double me = fmax(ext.x, fmax(ext.y, ext.z));
    if (!(me > 0.0)) return fail(SST_E_INVALID_ARGUMENT, "build_sdf: empty mesh bounds");
    const double vs = me / resolution;
    const v3 org = sub(lo, V(vs, vs, vs));
    for (int a = 0; a < 3; ++a) dims[a] = (uint32_t)ceil(comp(ext, a) / vs - 1e-9) + 2;
    st3(origin, org);
    *voxel = vs;
    if (!values) return 0;
    const double half_diag = 0.5 * sqrt(3.0) * vs;
    const v3 dirs[3] = {normalize(V(0.5380, 0.1123, 0.8354)), normalize(V(-0.8312, 0.3052, 0.4643)),
                        normalize(V(0.1710, -0.9364, 0.3063))};
    for (uint32_t z = 0; z < dims[2]; ++z)
        for (uint32_t y = 0; y < dims[1]; ++y)
            for (uint32_t x = 0; x < dims[0]; ++x) {
                const v3 c = add(org, V((x + 0.5) * vs, (y + 0.5) * vs, (z + 0.5) * vs));
                double best = 1e300;
                int votes = 0;
                for (int k = 0; k < 3; ++k) {
                    uint32_t hits = 0;
                    for (uint32_t t = 0; t < nt; ++t) {
                        const v3 A = ld3(pos + 3 * tris[3 * t]), B = ld3(pos + 3 * tris[3 * t + 1]),
                                 Cc = ld3(pos + 3 * tris[3 * t + 2]);
                        if (k == 0) best = fmin(best, pt_tri_d2(c, A, B, Cc));
                        double th;
                        hits += (uint32_t)ray_tri(c, dirs[k], 1e300, A, B, Cc, 1e-9, &th);
                    }
                    if (hits % 2 == 1) ++votes;
                }
                const double d = sqrt(best);
                const double cons = fmax(0.0, d - half_diag);
                values[((size_t)z * dims[1] + y) * dims[0] + x] = (float)(votes >= 2 ? -cons : cons);
            }
    return 0;
}

/* ------------------------------------------------------------------ BVH (bvh.cpp:43-179) */
typedef struct { v3 lo, hi; uint32_t left, first, count; } node_t;

struct so_scene {
    uint32_t nt;
    v3* tv;          /* [3*nt] triangle vertices */
    uint32_t* tobj;  /* [nt] */
    uint32_t* order;
    v3* cent;
    node_t* nodes;
    uint32_t n_nodes;
    uint32_t n_obj;
    sst_medium* media; /* [obj*3+c] */
    double (*sdf_o)[3];
    double* sdf_v;
    uint32_t (*sdf_d)[3];
    float** sdf_vals;
    v3 light; double power[3], bg[3];
    int directional; v3 ldir;
    v3 cam, fwd, right, up;
    double tan_half, aspect;
    uint32_t w, h;
    double r_min;
    uint32_t max_pt, max_st;
};

static uint32_t build(so_scene* s, uint32_t begin, uint32_t end) {
    const uint32_t ni = s->n_nodes++;
    v3 lo = V(1e300, 1e300, 1e300), hi = V(-1e300, -1e300, -1e300), clo = lo, chi = hi;
    for (uint32_t i = begin; i < end; ++i) {
        const uint32_t t = s->order[i];
        for (int k = 0; k < 3; ++k) {
            const v3 p = s->tv[3 * t + k];
            lo = V(fmin(lo.x, p.x), fmin(lo.y, p.y), fmin(lo.z, p.z));
            hi = V(fmax(hi.x, p.x), fmax(hi.y, p.y), fmax(hi.z, p.z));
        }
        const v3 c = s->cent[t];
        clo = V(fmin(clo.x, c.x), fmin(clo.y, c.y), fmin(clo.z, c.z));
        chi = V(fmax(chi.x, c.x), fmax(chi.y, c.y), fmax(chi.z, c.z));
    }
    s->nodes[ni].lo = lo;
    s->nodes[ni].hi = hi;
    const uint32_t count = end - begin;
    if (count <= 4) { s->nodes[ni].first = begin; s->nodes[ni].count = count; return ni; }
    const v3 e = sub(chi, clo);
    int axis = 0;
    if (e.y > e.x) axis = 1;
    if (e.z > comp(e, axis)) axis = 2;
    const double split = 0.5 * (comp(clo, axis) + comp(chi, axis));
    uint32_t i = begin, j = end;
    while (i < j) {
        if (comp(s->cent[s->order[i]], axis) < split) ++i;
        else { --j; const uint32_t t = s->order[i]; s->order[i] = s->order[j]; s->order[j] = t; }
    }
    uint32_t mid = i;
    if (mid == begin || mid == end) mid = begin + count / 2;
    const uint32_t l = build(s, begin, mid);
    const uint32_t r = build(s, mid, end);
    s->nodes[ni].left = l;
    s->nodes[ni].first = r;
    s->nodes[ni].count = 0;
    return ni;
}

static int slab_hit(const node_t* n, v3 o, v3 d, double t_min, double t_best) {   /* bvh.cpp:88-101 */
    double t0 = t_min, t1 = t_best;
    for (int a = 0; a < 3; ++a) {
        const double inv = 1.0 / comp(d, a);
        double nr = (comp(n->lo, a) - comp(o, a)) * inv;
        double fr = (comp(n->hi, a) - comp(o, a)) * inv;
        if (nr > fr) { const double t = nr; nr = fr; fr = t; }
        t0 = fmax(t0, nr);
        t1 = fmin(t1, fr);
        if (t0 > t1) return 0;
    }
    return 1;
}

/* Bvh::intersect, bvh.cpp:115-148 */
static int intersect(const so_scene* s, v3 o, v3 d, double t_min, double t_max, double* t_hit,
                     uint32_t* tri_hit) {
    double t_best = t_max;
    int found = 0;
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const node_t* n = &s->nodes[stack[--sp]];
        if (!slab_hit(n, o, d, t_min, t_best)) continue;
        if (n->count > 0) {
            for (uint32_t i = n->first; i < n->first + n->count; ++i) {
                const uint32_t t = s->order[i];
                double th;
                if (ray_tri(o, d, t_best, s->tv[3 * t], s->tv[3 * t + 1], s->tv[3 * t + 2], t_min, &th)) {
                    t_best = th;
                    *tri_hit = t;
                    found = 1;
                }
            }
        } else {
            stack[sp++] = n->left;
            stack[sp++] = n->first;
        }
    }
    *t_hit = t_best;
    return found;
}

int so_bvh_intersect(const so_scene* s, const double o[3], const double d[3], double t_min,
                     double t_max, double* t, int64_t* tri) {
    uint32_t th = 0;
    const int f = intersect(s, ld3(o), ld3(d), t_min, t_max, t, &th);
    *tri = f ? (int64_t)th : -1;
    if (!f) *t = -1.0;
    return f;
}

typedef struct { double t; uint32_t tri; } hit_t;
static int cmp_hit(const void* a, const void* b) {
    const double x = ((const hit_t*)a)->t, y = ((const hit_t*)b)->t;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Bvh::intersect_all, bvh.cpp:150-179 (sorted by t) */
static uint32_t intersect_all(const so_scene* s, v3 o, v3 d, double t_min, double t_max, hit_t* hits,
                              uint32_t cap) {
    uint32_t nh = 0;
    uint32_t stack[64];
    int sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
        const node_t* n = &s->nodes[stack[--sp]];
        if (!slab_hit(n, o, d, t_min, t_max)) continue;
        if (n->count > 0) {
            for (uint32_t i = n->first; i < n->first + n->count; ++i) {
                const uint32_t t = s->order[i];
                double th;
                if (ray_tri(o, d, t_max, s->tv[3 * t], s->tv[3 * t + 1], s->tv[3 * t + 2], t_min, &th) &&
                    nh < cap) {
                    hits[nh].t = th;
                    hits[nh].tri = t;
                    ++nh;
                }
            }
        } else {
            stack[sp++] = n->left;
            stack[sp++] = n->first;
        }
    }
    qsort(hits, nh, sizeof(hit_t), cmp_hit);
    return nh;
}

void so_scene_free(so_scene* s) {
    if (!s) return;
    free(s->tv); free(s->tobj); free(s->order); free(s->cent); free(s->nodes); free(s->media);
    free(s->sdf_o); free(s->sdf_v); free(s->sdf_d);
    if (s->sdf_vals) for (uint32_t o = 0; o < s->n_obj; ++o) free(s->sdf_vals[o]);
    free(s->sdf_vals);
    free(s);
}

static int valid_medium(const sst_medium* m) {                         /* optics.cpp:21-25 */
    return m->sigma_t >= 0.0 && m->g > -1.0 && m->g < 1.0 && m->phi >= 0.0 && m->phi <= 1.0;
}

int so_scene_create(const sst_scene_desc* d, so_scene** out) {
    if (!d || d->n_objects == 0) return fail(SST_E_INVALID_ARGUMENT, "scene has no objects");
    if (d->width == 0 || d->height == 0) return fail(SST_E_INVALID_ARGUMENT, "camera resolution must be >= 1x1");
    so_scene* s = (so_scene*)calloc(1, sizeof(so_scene));
    uint32_t nt = 0;
    for (uint32_t o = 0; o < d->n_objects; ++o) nt += d->objects[o].n_triangles;
    s->nt = nt;
    s->n_obj = d->n_objects;
    s->tv = (v3*)malloc(sizeof(v3) * 3 * nt);
    s->tobj = (uint32_t*)malloc(sizeof(uint32_t) * nt);
    s->order = (uint32_t*)malloc(sizeof(uint32_t) * nt);
    s->cent = (v3*)malloc(sizeof(v3) * nt);
    s->nodes = (node_t*)calloc(2 * nt + 1, sizeof(node_t));
    s->media = (sst_medium*)malloc(sizeof(sst_medium) * 3 * d->n_objects);
    s->sdf_o = malloc(sizeof(double[3]) * d->n_objects);
    s->sdf_v = (double*)malloc(sizeof(double) * d->n_objects);
    s->sdf_d = malloc(sizeof(uint32_t[3]) * d->n_objects);
    s->sdf_vals = (float**)calloc(d->n_objects, sizeof(float*));
    uint32_t k = 0;
    for (uint32_t o = 0; o < d->n_objects; ++o) {
        const sst_object_desc* od = &d->objects[o];
        for (uint32_t i = 0; i < od->n_triangles; ++i, ++k) {
            for (int c = 0; c < 3; ++c) {
                const uint32_t vi = od->triangles[3 * i + c];
                if (vi >= od->n_vertices) { so_scene_free(s); return fail(SST_E_INVALID_ARGUMENT, "triangle index out of range"); }
                s->tv[3 * k + c] = ld3(od->positions + 3 * vi);
            }
            s->tobj[k] = o;
            s->order[k] = k;
            s->cent[k] = dvs(add(add(s->tv[3 * k], s->tv[3 * k + 1]), s->tv[3 * k + 2]), 3.0);
        }
        for (int c = 0; c < 3; ++c) {
            if (!valid_medium(&od->media[c])) { so_scene_free(s); return fail(SST_E_DOMAIN, "invalid medium parameters"); }
            s->media[3 * o + c] = od->media[c];
        }
        if (od->sdf_values) {
            for (int a = 0; a < 3; ++a) { s->sdf_o[o][a] = od->sdf_origin[a]; s->sdf_d[o][a] = od->sdf_dims[a]; }
            s->sdf_v[o] = od->sdf_voxel;
            const size_t nvox = (size_t)od->sdf_dims[0] * od->sdf_dims[1] * od->sdf_dims[2];
            s->sdf_vals[o] = (float*)malloc(nvox * sizeof(float));
            memcpy(s->sdf_vals[o], od->sdf_values, nvox * sizeof(float));
        } else {
            const uint32_t res = od->sdf_resolution ? od->sdf_resolution : 64;
            int rc = so_build_sdf(od->positions, od->n_vertices, od->triangles, od->n_triangles, res,
                                  s->sdf_o[o], &s->sdf_v[o], s->sdf_d[o], NULL);
            if (rc) { so_scene_free(s); return rc; }
            const size_t nvox = (size_t)s->sdf_d[o][0] * s->sdf_d[o][1] * s->sdf_d[o][2];
            s->sdf_vals[o] = (float*)malloc(nvox * sizeof(float));
            so_build_sdf(od->positions, od->n_vertices, od->triangles, od->n_triangles, res, s->sdf_o[o],
                         &s->sdf_v[o], s->sdf_d[o], s->sdf_vals[o]);
        }
    }
    build(s, 0, nt);
    s->light = ld3(d->light_position);
    s->directional = d->light_kind == 1;
    s->ldir = s->directional ? normalize(ld3(d->light_direction)) : ld3(d->light_position);
    for (int c = 0; c < 3; ++c) { s->power[c] = d->light_power[c]; s->bg[c] = d->background[c]; }
    s->cam = ld3(d->cam_position);
    const v3 look = ld3(d->cam_look_at), up = ld3(d->cam_up);
    s->fwd = normalize(sub(look, s->cam));
    s->right = normalize(cross(s->fwd, up));
    s->up = cross(s->right, s->fwd);
    s->tan_half = tan(d->cam_vfov_deg * 3.14159265358979323846 / 360.0);
    s->w = d->width;
    s->h = d->height;
    s->aspect = (double)d->width / (double)d->height;
    s->r_min = d->r_min;
    s->max_pt = d->max_pt_events ? d->max_pt_events : 1000000u;
    s->max_st = d->max_st_steps ? d->max_st_steps : 100000u;
    *out = s;
    return 0;
}

/* ------------------------------------------------------------------ integrator */
static double r_min_for(const so_scene* s, uint32_t obj, int c) {
    if (s->r_min > 0.0) return s->r_min;
    const double sig = s->media[3 * obj + c].sigma_t;
    if (!(sig > 0.0)) return 1e300;
    return fmax(2.0 / sig, 1.5 * s->sdf_v[obj]);
}

/* NEE toward the point light */
static double nee_term(const so_scene* s, uint32_t obj, int c, v3 p, v3 w, double weight) {
    /* directional: d_t out to the last boundary exit, irradiance, no falloff */
    const v3 to_l = s->directional ? s->ldir : sub(s->light, p);
    const double d2 = s->directional ? 1.0 : dot(to_l, to_l);
    const double d = s->directional ? 1e30 : sqrt(d2);
    const v3 wl = s->directional ? s->ldir : dvs(to_l, d);
    hit_t hits[256];
    const uint32_t nh = intersect_all(s, p, wl, 1e-9, d, hits, 256);
    double tau = 0.0, t_prev = 0.0;
    int cur = (int)obj;
    for (uint32_t i = 0; i < nh; ++i) {
        if (cur >= 0) tau += s->media[3 * cur + c].sigma_t * (hits[i].t - t_prev);
        const int j = (int)s->tobj[hits[i].tri];
        cur = (cur == j) ? -1 : j;
        t_prev = hits[i].t;
    }
    if (cur >= 0) tau += s->media[3 * cur + c].sigma_t * (d - t_prev);
    double phase;
    so_hg_eval(s->media[3 * obj + c].g, dot(w, wl), &phase);
    return weight * s->power[c] * phase * exp(-1.0 * tau) / d2;
}

typedef struct { double L; uint32_t seg, steps, events, shadow; int end; int err; v3 x, w; } path_res;
/* exit state: the path's position and direction when it ends (escape: the last boundary
 * exit / camera and the escape direction; absorption or cap: the collision point and
 * the incoming direction) */
#define SO_END(code) do { r->x = x; r->w = w; r->end = (code); return; } while (0)

static void trace_one(const so_scene* s, so_models* ms, int integ, int nee, uint64_t seed,
                      uint32_t pixel, uint32_t sample, int c, path_res* r) {
    memset(r, 0, sizeof *r);
    so_rng cam = {so_rng_init(seed, SST_SALT_RENDER_PIXEL, pixel, sample)};
    const double jx = so_uniform(&cam);
    const double jy = so_uniform(&cam);
    const uint32_t px = pixel % s->w, py = pixel / s->w;
    const double sx = (2.0 * (px + jx) / s->w - 1.0) * s->tan_half * s->aspect;
    const double sy = (1.0 - 2.0 * (py + jy) / s->h) * s->tan_half;
    v3 x = s->cam;
    v3 w = normalize(add(add(s->fwd, mul(s->right, sx)), mul(s->up, sy)));
    so_rng rng = {so_rng_init(seed, SST_SALT_RENDER_CHANNEL, pixel, 3ull * sample + (uint64_t)c)};
    const uint32_t cap = integ == SST_INTEGRATOR_ST ? s->max_st : s->max_pt;
    for (;;) {
        double t;
        uint32_t tri;
        if (!intersect(s, x, w, 1e-9, 1e300, &t, &tri)) { r->L += s->bg[c]; SO_END(0); }
        const uint32_t obj = s->tobj[tri];
        const sst_medium m = s->media[3 * obj + c];
        const double rmin = r_min_for(s, obj, c);
        x = add(x, mul(w, t));
        for (;;) {
            const double t_free = m.sigma_t > 0.0 ? -log1p(-so_uniform(&rng)) / m.sigma_t : 1e300;
            const int hit_ = intersect(s, x, w, 1e-9, t_free, &t, &tri);
            if (getenv("SO_TRACE_DEBUG"))
                fprintf(stderr, "[orc] seg=%u obj=%u x=(%.17g,%.17g,%.17g) w=(%.17g,%.17g,%.17g) tfree=%.17g hit=%d thit=%.17g\n",
                        r->seg, obj, x.x, x.y, x.z, w.x, w.y, w.z, t_free, hit_, hit_ ? t : 0.0);
            if (hit_) { x = add(x, mul(w, t)); break; }
            x = add(x, mul(w, t_free));
            if (r->seg >= cap) { r->L = 0.0; SO_END(2); }
            ++r->seg;
            double rad = 0.0;
            if (integ == SST_INTEGRATOR_ST) {
                const double xp[3] = {x.x, x.y, x.z};
                rad = so_query_safe_radius(s->sdf_o[obj], s->sdf_v[obj], s->sdf_d[obj], s->sdf_vals[obj], xp);
                if (getenv("SO_TRACE_DEBUG")) fprintf(stderr, "[orc]   collide r=%.17g r_min=%.17g\n", rad, rmin);
            }
            if (integ == SST_INTEGRATOR_ST && rad > rmin) {
                ++r->steps;
                step_out o;
                if (sphere_step(ms, m.sigma_t, m.g, m.phi, w, x, rad, nee, &rng, &o)) { r->err = 1; r->L = 0.0; r->x = x; r->w = w; return; }
                if (o.absorbed) SO_END(1);
                if (nee) { r->L += nee_term(s, obj, c, o.rep_pos, o.rep_dir, o.lambda); ++r->shadow; }
                x = o.exit_pos;
                w = o.exit_dir;
            } else {
                ++r->events;
                if (!(so_uniform(&rng) < m.phi)) SO_END(1);
                if (nee) { r->L += nee_term(s, obj, c, x, w, 1.0); ++r->shadow; }
                const double u1 = so_uniform(&rng);
                const double u2 = so_uniform(&rng);
                w = hg_sample(m.g, w, u1, u2);
            }
        }
    }
}

int so_trace_paths(const so_scene* s, so_models* m, int integ, int nee, uint64_t seed, uint64_t n,
                   const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                   double* radiance, uint32_t* segments, sst_path_stats* st) {
    return so_trace_paths_ex(s, m, integ, nee, seed, n, pixel, sample, channel, radiance, segments, NULL, st);
}

int so_trace_paths_ex(const so_scene* s, so_models* m, int integ, int nee, uint64_t seed, uint64_t n,
                      const uint32_t* pixel, const uint32_t* sample, const uint8_t* channel,
                      double* radiance, uint32_t* segments, double* exit_state, sst_path_stats* st) {
    if (integ == SST_INTEGRATOR_ST && !m) return fail(SST_E_INVALID_ARGUMENT, "sphere tracing requires models");
    int err = 0;
    for (uint64_t i = 0; i < n; ++i) {
        path_res r;
        trace_one(s, m, integ, nee, seed, pixel[i], sample[i], channel[i], &r);
        radiance[i] = r.L;
        if (segments) segments[i] = r.seg;
        if (exit_state) {
            double* e = exit_state + 6 * i;
            e[0] = r.x.x; e[1] = r.x.y; e[2] = r.x.z;
            e[3] = r.w.x; e[4] = r.w.y; e[5] = r.w.z;
        }
        if (st) {
            st->paths += 1;
            st->segments += r.seg;
            st->sphere_steps += r.steps;
            st->pt_events += r.events;
            st->shadow_rays += r.shadow;
            st->escaped += r.end == 0 && !r.err;
            st->absorbed += r.end == 1;
            st->capped += r.end == 2;
            st->errors += (uint64_t)r.err;
        }
        err |= r.err;
    }
    if (m && st) {
        st->decodes_length = m->counters[0];
        st->decodes_path = m->counters[1];
        st->decodes_event = m->counters[2];
    }
    return err ? fail(SST_E_RUNTIME, "decoder produced non-finite output twice") : 0;
}

/* ------------------------------------------------------------------ config 4: dataset */
#ifndef SO_HG_ARG_ORDER_RTL
#define SO_HG_ARG_ORDER_RTL 1 /* g++ x86-64 evaluates hg_sample(g, w, rng.uniform(), rng.uniform())
                                 right to left: u2 is drawn first (pinned by the golden vectors) */
#endif

/* sphere_exit_t, sphere_walk.cpp:14-18 */
static double sphere_exit_t(v3 pos, v3 dir, double radius) {
    const double b = dot(pos, dir);
    const double c = dot(pos, pos) - radius * radius;
    return -b + sqrt(fmax(0.0, b * b - c));
}

typedef struct { v3 p, w; } walk_ev;

/* walk_sphere (sphere_walk.cpp:22-50) with radius 1; events grow in *ev. Returns n or 0 on cap. */
static uint64_t walk_unit(double sigma_t, double g, so_rng* rng, walk_ev** ev, uint64_t* cap,
                          v3* exit_pos, v3* exit_dir) {
    uint64_t n = 0;
    (*ev)[n].p = V(0.0, 0.0, 0.0);
    (*ev)[n].w = V(0.0, 0.0, 1.0);
    ++n;
    const int vacuum = sigma_t <= 1e-6;
    v3 pos = V(0.0, 0.0, 0.0), incoming = V(0.0, 0.0, 1.0);
    for (;;) {
        double u1, u2;
#if SO_HG_ARG_ORDER_RTL
        u2 = so_uniform(rng);
        u1 = so_uniform(rng);
#else
        u1 = so_uniform(rng);
        u2 = so_uniform(rng);
#endif
        const v3 dir = hg_sample(g, incoming, u1, u2);
        const double step = vacuum ? 2.0 : -log1p(-so_uniform(rng)) / sigma_t;
        const double t_exit = sphere_exit_t(pos, dir, 1.0);
        if (vacuum || step >= t_exit) {
            *exit_pos = add(pos, mul(dir, t_exit));
            *exit_dir = dir;
            return n;
        }
        pos = add(pos, mul(dir, step));
        if (n == *cap) {
            *cap *= 2;
            *ev = (walk_ev*)realloc(*ev, *cap * sizeof(walk_ev));
        }
        (*ev)[n].p = pos;
        (*ev)[n].w = dir;
        ++n;
        incoming = dir;
        if (n > 1000000) return 0;
    }
}

int so_generate_dataset(uint64_t n, double s_lo, double s_hi, double g_lo, double g_hi, int phi_kind,
                        double phi_a, double phi_b, uint64_t seed, uint64_t first, so_sample* out) {
    if (n == 0) return fail(SST_E_INVALID_ARGUMENT, "generate_dataset: n_samples must be > 0");
    if (!(s_lo >= 0.0 && s_hi >= s_lo)) return fail(SST_E_INVALID_ARGUMENT, "generate_dataset: invalid sigma_t range");
    if (!(g_lo >= -1.0 && g_hi <= 1.0 && g_hi >= g_lo)) return fail(SST_E_INVALID_ARGUMENT, "generate_dataset: invalid g range");
    uint64_t cap = 4096;
    walk_ev* ev = (walk_ev*)malloc(cap * sizeof(walk_ev));
    for (uint64_t j = 0; j < n; ++j) {
        const uint64_t i = first + j;
        so_rng rng = {so_rng_init(seed, SST_SALT_DATASET, i, 0)};          /* dataset.cpp:59 */
        const double sigma_t = s_lo + so_uniform(&rng) * (s_hi - s_lo);
        double g = g_lo + so_uniform(&rng) * (g_hi - g_lo);
        g = fmin(1.0 - 1e-6, fmax(-(1.0 - 1e-6), g));
        double phi;                                                        /* PhiSampler::sample */
        if (phi_kind == 0) phi = 1.0 - pow(10.0, phi_a + so_uniform(&rng) * (phi_b - phi_a));
        else if (phi_kind == 1) phi = phi_a;
        else phi = phi_a + so_uniform(&rng) * (phi_b - phi_a);
        v3 xe, we;
        const uint64_t ne = walk_unit(sigma_t, g, &rng, &ev, &cap, &xe, &we);
        if (ne == 0) { free(ev); return fail(SST_E_RUNTIME, "walk_sphere: event cap exceeded"); }
        /* parameterize_exit, sphere_walk.cpp:52-73 (w_in = (0,0,1), radius 1) */
        const v3 w_in = V(0.0, 0.0, 1.0);
        const v3 x_hat = dvs(xe, 1.0);
        const double ct = dot(w_in, x_hat);
        v3 e_b, b2;
        if (fabs(ct) > 1.0 - 1e-9) onb(x_hat, &e_b, &b2);
        else e_b = normalize(cross(w_in, x_hat));
        const v3 e_t = cross(e_b, x_hat);
        /* sample_representative, sphere_walk.cpp:75-102 */
        uint64_t k = 1;
        if (phi <= 0.0) {
            k = 1;
        } else if (phi >= 1.0) {
            uint64_t t = (uint64_t)(so_uniform(&rng) * (double)ne);
            k = 1 + (ne - 1 < t ? ne - 1 : t);
        } else {
            const double u = so_uniform(&rng);
            const double phi_n = exp((double)ne * log(phi));
            const double target = 1.0 - u * (1.0 - phi_n);
            k = (uint64_t)ceil(log(target) / log(phi));
            k = k < 1 ? 1 : (k > ne ? ne : k);
        }
        /* rotate by -psi_exit (dataset.cpp:71-74) */
        const double psi = atan2(xe.y, xe.x);
        const m3 undo = rotation_z(-psi);
        const v3 xs = mv(undo, ev[k - 1].p), ws = mv(undo, ev[k - 1].w);
        so_sample* o = out + j;
        o->sigma_t = (float)sigma_t;
        o->g = (float)g;
        o->phi = (float)phi;
        o->n_events = (uint32_t)ne;
        o->cos_theta = (float)ct;
        o->alpha = (float)dot(we, e_b);
        o->beta = (float)dot(we, e_t);
        o->rep_position[0] = (float)xs.x; o->rep_position[1] = (float)xs.y; o->rep_position[2] = (float)xs.z;
        o->rep_direction[0] = (float)ws.x; o->rep_direction[1] = (float)ws.y; o->rep_direction[2] = (float)ws.z;
    }
    free(ev);
    return 0;
}

/* ------------------------------------------------------------------ CVAE training
 * train_model (cvae.cpp:234-347) restated in plain C: make_cvae (cvae.cpp:79-91) with
 * make_mlp / make_gaussian_mlp (mlp.cpp:32-58), the ELBO forward / backward
 * (elbo_forward + cvae_elbo_loss_grad, cvae.cpp:117-183) over mlp_forward_trace /
 * mlp_backward (mlp.cpp:100-183), gaussian_kl / gaussian_loglik / reparameterize
 * (mlp.cpp:185-212) and adamw_step (mlp.cpp:214-228). Parameters are kept flat in
 * flatten_parameters order (per layer: weights row-major [out][in], then bias). */
#define SO_TMAX 64 /* widest layer this restatement handles */
typedef struct {
    uint32_t n;
    uint32_t in[8], out[8];
    size_t woff[8];
    size_t count;
} so_mlp;

static void so_mlp_shape(so_mlp* m, uint32_t input, uint32_t output, uint32_t depth, uint32_t width) {
    uint32_t in = input;
    size_t off = 0;
    m->n = depth + 1;
    for (uint32_t d = 0; d <= depth; ++d) {
        const uint32_t out = d == depth ? output : width;
        m->in[d] = in;
        m->out[d] = out;
        m->woff[d] = off;
        off += (size_t)in * out + out;
        in = out;
    }
    m->count = off;
}

/* make_gaussian_mlp: Glorot-uniform weights, zero bias, log-variance head bias -2 (mlp.hpp:43-44). */
static void so_mlp_init(const so_mlp* m, double* p, uint32_t p_out, so_rng* rng) {
    for (uint32_t l = 0; l < m->n; ++l) {
        const double bound = sqrt(6.0 / ((double)m->in[l] + m->out[l]));
        double* w = p + m->woff[l];
        for (size_t i = 0; i < (size_t)m->in[l] * m->out[l]; ++i) {
            const double u = so_uniform(rng);
            w[i] = -bound + u * (bound - -bound);
        }
        double* b = w + (size_t)m->in[l] * m->out[l];
        for (uint32_t r = 0; r < m->out[l]; ++r) b[r] = (l + 1 == m->n && r >= p_out) ? -2.0 : 0.0;
    }
    for (size_t i = 0; i < m->count; ++i) p[i] = (double)(float)p[i]; /* quantize_f32, mlp.cpp:25-30 */
}

static double so_softplus_derivative(double x) { /* mlp.cpp:64-68 */
    if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
    const double e = exp(x);
    return e / (1.0 + e);
}

/* mlp_forward_trace: xs[l] = input of layer l (xs[n] = output), pre[l] = pre-activations. */
static void so_mlp_fwd(const so_mlp* m, const double* p, double xs[][SO_TMAX], double pre[][SO_TMAX]) {
    for (uint32_t l = 0; l < m->n; ++l) {
        const double* w = p + m->woff[l];
        const double* b = w + (size_t)m->in[l] * m->out[l];
        for (uint32_t r = 0; r < m->out[l]; ++r) {
            double acc = b[r];
            for (uint32_t c = 0; c < m->in[l]; ++c) acc += w[(size_t)r * m->in[l] + c] * xs[l][c];
            pre[l][r] = acc;
            xs[l + 1][r] = (l + 1 == m->n) ? acc : so_softplus(acc);
        }
    }
}

/* mlp_backward: accumulates into g (flat, same layout as p); input_grad may be NULL. */
static void so_mlp_bwd(const so_mlp* m, const double* p, double xs[][SO_TMAX], double pre[][SO_TMAX],
                       const double* upstream, double* g, double* input_grad) {
    double delta[SO_TMAX], prev[SO_TMAX];
    memcpy(delta, upstream, m->out[m->n - 1] * sizeof(double));
    for (uint32_t li = m->n; li-- > 0;) {
        const uint32_t in = m->in[li], out = m->out[li];
        const double* w = p + m->woff[li];
        double* gw = g + m->woff[li];
        double* gb = gw + (size_t)in * out;
        if (li + 1 != m->n)
            for (uint32_t r = 0; r < out; ++r) delta[r] *= so_softplus_derivative(pre[li][r]);
        for (uint32_t r = 0; r < out; ++r) {
            gb[r] += delta[r];
            for (uint32_t c = 0; c < in; ++c) gw[(size_t)r * in + c] += delta[r] * xs[li][c];
        }
        if (li > 0 || input_grad) {
            for (uint32_t c = 0; c < in; ++c) prev[c] = 0.0;
            for (uint32_t r = 0; r < out; ++r)
                for (uint32_t c = 0; c < in; ++c) prev[c] += w[(size_t)r * in + c] * delta[r];
            memcpy(delta, prev, in * sizeof(double));
        }
    }
    if (input_grad) memcpy(input_grad, delta, m->in[0] * sizeof(double));
}

static double so_clamp_lv(double lv) { return fmin(10.0, fmax(-10.0, lv)); } /* cvae.cpp:22 */

typedef struct {
    uint32_t p_in, p_out, depth, width, latent;
} so_spec;

/* One ELBO evaluation (cvae_elbo_loss / cvae_elbo_loss_grad). */
static double so_elbo(const so_spec* s, const so_mlp* me, const so_mlp* md, const double* pe, const double* pd,
                      const double* x, const double* c, const double* eps, double* ge, double* gd) {
    double xe[8][SO_TMAX], pre_e[8][SO_TMAX], xd[8][SO_TMAX], pre_d[8][SO_TMAX];
    const uint32_t L = s->latent, P = s->p_out;
    for (uint32_t i = 0; i < P; ++i) xe[0][i] = x[i];
    for (uint32_t i = 0; i < s->p_in; ++i) xe[0][P + i] = c[i];
    so_mlp_fwd(me, pe, xe, pre_e);
    const double* oe = xe[me->n];
    double mu_e[SO_TMAX], lv_e[SO_TMAX];
    for (uint32_t i = 0; i < L; ++i) {
        mu_e[i] = oe[i];
        lv_e[i] = so_clamp_lv(oe[L + i]);
        xd[0][i] = mu_e[i] + exp(0.5 * lv_e[i]) * eps[i]; /* reparameterize, mlp.cpp:204-212 */
    }
    for (uint32_t i = 0; i < s->p_in; ++i) xd[0][L + i] = c[i];
    so_mlp_fwd(md, pd, xd, pre_d);
    const double* od = xd[md->n];
    double kl = 0.0, ll = 0.0;
    for (uint32_t i = 0; i < L; ++i) kl += mu_e[i] * mu_e[i] + exp(lv_e[i]) - 1.0 - lv_e[i];
    kl = 0.5 * kl;
    for (uint32_t i = 0; i < P; ++i) {
        const double lv = so_clamp_lv(od[P + i]);
        const double d = x[i] - od[i];
        ll += -0.91893853320467274178 - 0.5 * lv - d * d / (2.0 * exp(lv));
    }
    const double loss = kl - ll;
    if (!ge) return loss;
    double up_d[2 * SO_TMAX], din[SO_TMAX], up_e[2 * SO_TMAX];
    for (uint32_t i = 0; i < P; ++i) {
        const double lv = so_clamp_lv(od[P + i]);
        const double inv_var = exp(-lv);
        const double d = x[i] - od[i];
        up_d[i] = -d * inv_var;
        up_d[P + i] = fabs(lv) >= 10.0 ? 0.0 : 0.5 - 0.5 * d * d * inv_var;
    }
    so_mlp_bwd(md, pd, xd, pre_d, up_d, gd, din);
    for (uint32_t i = 0; i < L; ++i) {
        const double dz = din[i];
        up_e[i] = mu_e[i] + dz;
        const double dlv_kl = 0.5 * (exp(lv_e[i]) - 1.0);
        const double dlv_rep = dz * 0.5 * exp(0.5 * lv_e[i]) * eps[i];
        up_e[L + i] = fabs(lv_e[i]) >= 10.0 ? 0.0 : dlv_kl + dlv_rep;
    }
    so_mlp_bwd(me, pe, xe, pre_e, up_e, ge, NULL);
    return loss;
}

static void so_adamw(double* p, double* m, double* v, const double* g, size_t n, uint64_t t, double lr, double wd) {
    const double b1 = 0.9, b2 = 0.999, eps = 1e-8; /* AdamWConfig, mlp.hpp:95-101 */
    const double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
    for (size_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        const double mh = m[i] / bc1, vh = v[i] / bc2;
        p[i] -= lr * (mh / (sqrt(vh) + eps) + wd * p[i]);
    }
}

static void so_shuffle(uint32_t* v, size_t n, so_rng* rng) {
    for (size_t i = n; i > 1; --i) {
        const size_t j = (size_t)(so_uniform(rng) * (double)i);
        const uint32_t t = v[i - 1];
        v[i - 1] = v[j];
        v[j] = t;
    }
}

uint64_t so_dataset_fingerprint(const so_sample* s, uint64_t n, uint64_t seed) { /* dataset.cpp:32-38 */
    uint64_t h = 0xCBF29CE484222325ULL;
    const uint32_t version = 1;
    const unsigned char* parts[4] = {(const unsigned char*)&version, (const unsigned char*)&n,
                                     (const unsigned char*)&seed, (const unsigned char*)s};
    const size_t lens[4] = {4, 8, 8, (size_t)n * sizeof(so_sample)};
    for (int k = 0; k < 4; ++k)
        for (size_t i = 0; i < lens[k]; ++i) {
            h ^= parts[k][i];
            h *= 0x100000001B3ULL;
        }
    return h;
}

int so_train_model(int kind, const so_sample* samples, uint64_t n, const sst_train_config* cfg,
                   sst_epoch_stats* epochs, double* params_out) {
    if (!(cfg->lr > 0.0)) return fail(SST_E_INVALID_ARGUMENT, "TrainConfig: lr must be > 0");
    if (cfg->batch_size == 0) return fail(SST_E_INVALID_ARGUMENT, "TrainConfig: batch_size must be > 0");
    if (cfg->epochs == 0) return fail(SST_E_INVALID_ARGUMENT, "TrainConfig: epochs must be > 0");
    if (!(cfg->weight_decay >= 0.0)) return fail(SST_E_INVALID_ARGUMENT, "TrainConfig: negative weight decay");
    if (!(cfg->validation_fraction >= 0.0 && cfg->validation_fraction < 1.0))
        return fail(SST_E_INVALID_ARGUMENT, "TrainConfig: validation fraction out of range");
    if (n == 0) return fail(SST_E_INVALID_ARGUMENT, "train_model: empty dataset");
    static const so_spec defaults[3] = {{2, 1, 2, 8, 2}, {3, 3, 2, 16, 5}, {7, 6, 2, 16, 5}}; /* cvae.cpp:51-57 */
    if (kind < 0 || kind > 2) return fail(SST_E_INVALID_ARGUMENT, "unknown model kind");
    so_spec s = defaults[kind];
    if (cfg->depth > 0) s.depth = (uint32_t)cfg->depth;
    if (cfg->width > 0) s.width = (uint32_t)cfg->width;
    if (cfg->latent > 0) s.latent = (uint32_t)cfg->latent;
    if ((s.p_in + s.latent) % 4 != 0)
        return fail(SST_E_INVALID_ARGUMENT, "CvaeSpec: p_in + latent must be a multiple of four");
    if (s.depth > 6 || s.width > SO_TMAX || 2 * s.latent > SO_TMAX)
        return fail(SST_E_INVALID_ARGUMENT, "oracle: spec too large");
    so_mlp me, md;
    so_mlp_shape(&me, s.p_out + s.p_in, 2 * s.latent, s.depth, s.width);
    so_mlp_shape(&md, s.latent + s.p_in, 2 * s.p_out, s.depth, s.width);
    const size_t ne = me.count, nd = md.count;
    double* buf = (double*)calloc(5 * (ne + nd), sizeof(double));
    double *pe = buf, *pd = pe + ne, *ge = pd + nd, *gd = ge + ne, *me_ = gd + nd, *md_ = me_ + ne,
           *ve = md_ + nd, *vd = ve + ne;
    so_rng init = {so_rng_init(cfg->seed, 0x02, (uint64_t)kind, 0)}; /* kTrainInit */
    so_mlp_init(&me, pe, s.latent, &init);
    so_mlp_init(&md, pd, s.p_out, &init);
    /* targets / conditions (cvae.cpp:185-212), NormConstants sigma_ref 200, n_ref 1e4 */
    const uint32_t P = s.p_out, C = s.p_in;
    double* X = (double*)malloc((size_t)n * (P + C) * sizeof(double));
    double* Cn = X + (size_t)n * P;
    for (uint64_t i = 0; i < n; ++i) {
        const so_sample* t = samples + i;
        const double ns = log1p(fmax(0.0, (double)t->sigma_t)) / log1p(200.0);
        const double nn = log(fmax(1.0, (double)t->n_events)) / log(1e4);
        double* x = X + i * P;
        double* c = Cn + i * C;
        if (kind == 0) {
            x[0] = nn; c[0] = ns; c[1] = t->g;
        } else if (kind == 1) {
            x[0] = t->cos_theta; x[1] = t->alpha; x[2] = t->beta;
            c[0] = ns; c[1] = t->g; c[2] = nn;
        } else {
            for (int k = 0; k < 3; ++k) { x[k] = t->rep_position[k]; x[3 + k] = t->rep_direction[k]; }
            c[0] = ns; c[1] = t->g; c[2] = t->phi; c[3] = t->cos_theta; c[4] = t->alpha; c[5] = t->beta; c[6] = nn;
        }
    }
    uint32_t* order = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; ++i) order[i] = (uint32_t)i;
    so_rng split = {so_rng_init(cfg->seed, 0x05, 0, 0)}; /* kTrainSplit */
    so_shuffle(order, n, &split);
    const size_t n_val = (size_t)(cfg->validation_fraction * (double)n);
    uint32_t* val = order;
    uint32_t* tr = order + n_val;
    const size_t n_tr = n - n_val;
    int rc = 0;
    if (n_tr == 0) {
        rc = fail(SST_E_INVALID_ARGUMENT, "train_model: no training samples left");
        goto done;
    }
    uint64_t t = 0;
    double eps[SO_TMAX];
    for (uint32_t e = 0; e < cfg->epochs; ++e) {
        so_rng sh = {so_rng_init(cfg->seed, 0x03, e, 0)}; /* kTrainShuffle */
        so_shuffle(tr, n_tr, &sh);
        double epoch_loss = 0.0;
        size_t epoch_samples = 0, finite = 0;
        for (size_t start = 0; start < n_tr; start += cfg->batch_size) {
            const size_t end = start + cfg->batch_size < n_tr ? start + cfg->batch_size : n_tr;
            memset(ge, 0, (ne + nd) * sizeof(double));
            double bl = 0.0;
            for (size_t b = start; b < end; ++b) {
                const uint32_t i = tr[b];
                so_rng er = {so_rng_init(cfg->seed, 0x04, e, i)}; /* kTrainLatent */
                for (uint32_t k = 0; k < s.latent; ++k) eps[k] = so_normal(&er);
                bl += so_elbo(&s, &me, &md, pe, pd, X + (size_t)i * P, Cn + (size_t)i * C, eps, ge, gd);
            }
            const double inv = 1.0 / (double)(end - start);
            if (!isfinite(bl)) continue;
            ++finite;
            epoch_loss += bl;
            epoch_samples += end - start;
            for (size_t k = 0; k < ne + nd; ++k) ge[k] *= inv;
            ++t;
            so_adamw(pe, me_, ve, ge, ne, t, cfg->lr, cfg->weight_decay);
            so_adamw(pd, md_, vd, gd, nd, t, cfg->lr, cfg->weight_decay);
        }
        if (finite == 0) {
            rc = fail(SST_E_RUNTIME, "train_model: diverged, every batch non-finite");
            goto done;
        }
        const double train_loss = epoch_loss / (double)(epoch_samples ? epoch_samples : 1);
        double vl = 0.0;
        for (size_t k = 0; k < n_val; ++k) {
            so_rng er = {so_rng_init(cfg->seed, 0x04, e, val[k])};
            for (uint32_t j = 0; j < s.latent; ++j) eps[j] = so_normal(&er);
            vl += so_elbo(&s, &me, &md, pe, pd, X + (size_t)val[k] * P, Cn + (size_t)val[k] * C, eps, NULL, NULL);
        }
        if (epochs) {
            epochs[e].train_loss = train_loss;
            epochs[e].validation_loss = n_val ? vl / (double)n_val : train_loss;
        }
    }
    if (params_out)
        for (size_t k = 0; k < ne + nd; ++k) params_out[k] = (double)(float)pe[k]; /* pe, pd contiguous */
done:
    free(order);
    free(X);
    free(buf);
    return rc;
}
