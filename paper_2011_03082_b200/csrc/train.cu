// train.cu -- CVAE training kernels, FP64, compiled with -fmad=false.
// See train.h for the epoch structure. Reference: train_model (cvae.cpp:234-347),
// elbo_forward / cvae_elbo_loss_grad (cvae.cpp:117-183), mlp_forward_trace /
// mlp_backward / gaussian_kl / gaussian_loglik / reparameterize / adamw_step
// (mlp.cpp:100-228), softplus / softplus_derivative (mlp.cpp:60-68).
#include <cooperative_groups.h>
#include <cstdio>

#include "rng.cuh"
#include "train.h"
#include "types.cuh"

namespace cg = cooperative_groups;

#ifdef SST_TRAIN_PROFILE  // debug builds: per-phase clock accumulation, printed by CTA 0
__device__ unsigned long long g_prof[32];
#define PROF_MARK(i)                                                         \
    do {                                                                     \
        if (threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) {      \
            const long long now = clock64();                                 \
            g_prof[i] += now - prof_last;                                    \
            prof_last = now;                                                 \
        }                                                                    \
    } while (0)
#else
#define PROF_MARK(i) \
    do {             \
    } while (0)
#endif

namespace sstg {
namespace {

constexpr double kHalfLog2Pi = 0.91893853320467274178;  // mlp.cpp:12
constexpr double kLogVarClamp = 10.0;                   // cvae.cpp:20
constexpr uint64_t kSaltTrainLatent = 0x04;             // rng.hpp:57

// softplus (mlp.cpp:60-62) and softplus_derivative (mlp.cpp:64-68) from ONE exp(-|x|):
// softplus_derivative evaluates exp(-x)
// for x >= 0 and exp(x) for x < 0 -- both are exp(-|x|), so sharing the value is
// bit-identical to calling the two reference functions separately.
__device__ __forceinline__ double softplus_and_derivative(double x, double* deriv) {
    const double e = exp(-fabs(x));
    *deriv = x >= 0.0 ? 1.0 / (1.0 + e) : e / (1.0 + e);
    return fmax(x, 0.0) + log1p(e);
}
__device__ __forceinline__ double clamp_lv(double lv) {  // cvae.cpp:22
    return fmin(kLogVarClamp, fmax(-kLogVarClamp, lv));
}
__device__ __forceinline__ bool lv_clamped(double lv) { return fabs(lv) >= kLogVarClamp; }  // cvae.cpp:23

// mlp_forward_trace (mlp.cpp:100-121) of layer l for ns trace rows; one thread per
// (sample, output). acc = b[r]; acc += W[r][c] * X[c] in c order.
__device__ void fwd_layer(const TrainNetK& N, int l, const double* P, double* tr, int ts, int ns) {
    const int in = N.in[l], out = N.out[l];
    const bool hidden = l + 1 < N.n_layers;
    const double* W = P + N.woff[l];
    const double* bias = W + in * out;
    for (int it = threadIdx.x; it < ns * out; it += blockDim.x) {
        const int r = it / ns, s = it - r * ns;
        double* t = tr + s * ts;
        const double* xi = t + N.xo[l];
        const double* wr = W + r * in;
        double acc = bias[r];
        for (int c = 0; c < in; ++c) acc += wr[c] * xi[c];
        if (hidden) {  // hidden layers keep softplus'(pre) (all backward needs) instead of pre
            double deriv;
            t[N.xo[l + 1] + r] = softplus_and_derivative(acc, &deriv);
            t[N.po[l] + r] = deriv;
        } else {
            t[N.po[l] + r] = acc;
        }
    }
    __syncthreads();
}

// mlp_backward (mlp.cpp:147-183) delta propagation out of layer l: delta_prev[c] =
// sum_r W[r][c] * D_l[r] (r order), times softplus'(pre_{l-1}[c]) when layer l-1 is
// hidden (the multiply mlp_backward applies at the top of the next iteration), or
// into the input gradient `din` for l == 0.
__device__ void bwd_layer(const TrainNetK& N, int l, const double* P, double* tr, int ts, int ns, int din_o) {
    const int in = N.in[l], out = N.out[l];
    const double* W = P + N.woff[l];
    for (int it = threadIdx.x; it < ns * in; it += blockDim.x) {
        const int c = it / ns, s = it - c * ns;
        double* t = tr + s * ts;
        const double* d = t + N.dlo[l];
        double acc = 0.0;
        for (int r = 0; r < out; ++r) acc += W[r * in + c] * d[r];
        if (l > 0)
            t[N.dlo[l - 1] + c] = acc * t[N.po[l - 1] + c];  // * softplus'(pre_{l-1})
        else
            t[din_o + c] = acc;
    }
    __syncthreads();
}

// elbo_forward (+ cvae_elbo_loss_grad's backward when `backward`) for ns samples
// whose dataset indices are ids[0..ns) (cvae.cpp:117-183).
__device__ void elbo_chunk(const TrainArgs& a, const double* P, double* tr, const uint32_t* ids, int ns,
                           bool backward, long long& prof_last) {
    const TrainNetK& E = a.net[0];
    const TrainNetK& D = a.net[1];
    const int ts = a.ts, lat = a.latent, pin = a.p_in, pout = a.p_out;
    const int le = E.n_layers - 1, ld = D.n_layers - 1;
    // encoder input concat(x, c)
    const int ne = pout + pin;
    for (int it = threadIdx.x; it < ns * ne; it += blockDim.x) {
        const int s = it / ne, k = it - s * ne;
        const uint64_t id = ids[s];
        tr[s * ts + E.xo[0] + k] = k < pout ? __ldg(a.x + id * pout + k) : __ldg(a.cnd + id * pin + (k - pout));
    }
    __syncthreads();
    PROF_MARK(0);
    for (int l = 0; l <= le; ++l) fwd_layer(E, l, P, tr, ts, ns);
    PROF_MARK(1);
    // z = mu_e + exp(lv_e / 2) * eps (reparameterize, mlp.cpp:204-212); decoder input concat(z, c).
    // One thread per (sample, latent j): normal j of RandomStream(seed, kTrainLatent, epoch, i)
    // uses draws 2j+1, 2j+2, i.e. the counter state key + 2j * golden.
    const int nz = lat + pin;
    for (int it = threadIdx.x; it < ns * nz; it += blockDim.x) {
        const int j = it / ns, s = it - j * ns;
        double* t = tr + s * ts;
        const uint64_t id = ids[s];
        if (j < lat) {
            Rng rng{rng_key(a.seed, kSaltTrainLatent, a.epoch, id) + 2ull * j * kGolden};
            const double e = rng.normal<double>();
            const double* he = t + E.po[le];
            t[a.eps_o + j] = e;
            const double lv = clamp_lv(he[lat + j]);
            t[D.xo[0] + j] = he[j] + exp(0.5 * lv) * e;
        } else {
            t[D.xo[0] + j] = __ldg(a.cnd + id * pin + (j - lat));
        }
    }
    __syncthreads();
    PROF_MARK(2);
    for (int l = 0; l <= ld; ++l) fwd_layer(D, l, P, tr, ts, ns);
    PROF_MARK(3);
    // loss = gaussian_kl(mu_e, lv_e) - gaussian_loglik(x, mu_d, lv_d) (mlp.cpp:185-202);
    // decoder upstream d(-loglik)/d(mu_d, lv_d) (cvae.cpp:126-133). Terms in parallel per
    // (sample, component), then the in-order sums per sample.
    const int nk = lat + pout;
    for (int it = threadIdx.x; it < ns * nk; it += blockDim.x) {
        const int j = it / ns, s = it - j * ns;
        double* t = tr + s * ts;
        if (j < lat) {
            const double* he = t + E.po[le];
            const double mu = he[j], lv = clamp_lv(he[lat + j]);
            t[a.term_o + j] = mu * mu + exp(lv) - 1.0 - lv;
        } else {
            const int i = j - lat;
            const double* hd = t + D.po[ld];
            const double lv = clamp_lv(hd[pout + i]);
            const double d = __ldg(a.x + static_cast<uint64_t>(ids[s]) * pout + i) - hd[i];
            t[a.term_o + j] = -kHalfLog2Pi - 0.5 * lv - d * d / (2.0 * exp(lv));
            if (backward) {
                double* up = t + D.dlo[ld];
                const double inv_var = exp(-lv);
                up[i] = -d * inv_var;
                up[pout + i] = lv_clamped(lv) ? 0.0 : 0.5 - 0.5 * d * d * inv_var;
            }
        }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < ns; s += blockDim.x) {
        double* t = tr + s * ts;
        double kl = 0.0;
        for (int j = 0; j < lat; ++j) kl += t[a.term_o + j];
        kl = 0.5 * kl;
        double ll = 0.0;
        for (int i = 0; i < pout; ++i) ll += t[a.term_o + lat + i];
        t[a.loss_o] = kl - ll;
    }
    __syncthreads();
    PROF_MARK(4);
    if (!backward) return;
    for (int l = ld; l >= 0; --l) bwd_layer(D, l, P, tr, ts, ns, a.din_o);
    PROF_MARK(5);
    // encoder upstream through z = mu_e + exp(lv_e/2) eps plus the KL term (cvae.cpp:138-146)
    for (int it = threadIdx.x; it < ns * lat; it += blockDim.x) {
        const int i = it / ns, s = it - i * ns;
        double* t = tr + s * ts;
        const double* he = t + E.po[le];
        double* up = t + E.dlo[le];
        const double dz = t[a.din_o + i];
        const double lv = clamp_lv(he[lat + i]);
        up[i] = he[i] + dz;
        const double dlv_kl = 0.5 * (exp(lv) - 1.0);
        const double dlv_rep = dz * 0.5 * exp(0.5 * lv) * t[a.eps_o + i];
        up[lat + i] = lv_clamped(lv) ? 0.0 : dlv_kl + dlv_rep;
    }
    __syncthreads();
    PROF_MARK(6);
    for (int l = le; l >= 1; --l) bwd_layer(E, l, P, tr, ts, ns, a.din_o);
    PROF_MARK(7);
}

// ---- TMA bulk copies (cp.async.bulk) global -> shared with mbarrier completion
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(m)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
        ::"r"(smem_u32(m)), "r"(parity) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.global;\n fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t pad2(uint32_t n) { return (n + 1) & ~1u; }

struct Smem {
    double* P;     // parameters
    double* tr;    // phase-1 trace rows / phase-2 staging (union)
    uint32_t* ids;
};

__device__ Smem carve(const TrainArgs& a, double* base) {
    Smem m;
    m.P = base;
    m.tr = base + a.n_params_pad;
    const int region = max(a.chunk * a.ts, a.stage_cap);
    m.ids = reinterpret_cast<uint32_t*>(m.tr + region);
    return m;
}

__global__ void __launch_bounds__(kTrainThreads, 1) k_train_epoch(const __grid_constant__ TrainArgs a) {
    extern __shared__ __align__(16) double smem[];
    __shared__ double s_bl;
    __shared__ unsigned long long s_t;
    __shared__ __align__(8) uint64_t s_mbar;
    __shared__ double sm_one[1];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = static_cast<int>(cl.block_rank());
    const int C = static_cast<int>(cl.num_blocks());
    const int tid = threadIdx.x, nt = blockDim.x;
    const Smem sm = carve(a, smem);
    for (int i = tid; i < a.n_params; i += nt) sm.P[i] = a.params[i];
    if (tid == 0) {
        s_t = *a.t_io;
        sm_one[0] = 1.0;
        mbar_init(&s_mbar, 1);
    }
    uint32_t parity = 0;
    __syncthreads();
    cl.sync();  // every CTA's parameter copy is loaded before any DSMEM broadcast

    const uint32_t S = (a.batch + C - 1) / C;
    long long prof_last = clock64();
    for (uint32_t bi = 0; bi < a.n_batches; ++bi) {
        PROF_MARK(15);
        const uint32_t start = bi * a.batch;
        const uint32_t bcur = min(a.batch, a.n_order - start);
        // ---------------- phase 1: per-sample ELBO forward + backward for this CTA's slice
        const uint32_t lo = min(bcur, rank * S), hi = min(bcur, rank * S + S);
        for (uint32_t c0 = lo; c0 < hi; c0 += a.chunk) {
            const int ns = static_cast<int>(min(static_cast<uint32_t>(a.chunk), hi - c0));
            for (int s = tid; s < ns; s += nt) sm.ids[s] = __ldg(a.order + start + c0 + s);
            __syncthreads();
            elbo_chunk(a, sm.P, sm.tr, sm.ids, ns, true, prof_last);
            for (int m = 0; m < 2; ++m) {
                const TrainNetK& N = a.net[m];
                for (int l = 0; l < N.n_layers; ++l) {
                    const int in = N.in[l], out = N.out[l];
                    double* gx = a.gtrace + N.gx[l] + static_cast<size_t>(c0) * in;
                    double* gd = a.gtrace + N.gd[l] + static_cast<size_t>(c0) * out;
                    for (int it = tid; it < ns * in; it += nt) {
                        const int s = it / in, k = it - s * in;
                        __stcg(gx + it, sm.tr[s * a.ts + N.xo[l] + k]);
                    }
                    for (int it = tid; it < ns * out; it += nt) {
                        const int s = it / out, k = it - s * out;
                        __stcg(gd + it, sm.tr[s * a.ts + N.dlo[l] + k]);
                    }
                }
            }
            for (int s = tid; s < ns; s += nt) __stcg(a.gtrace + a.gloss + c0 + s, sm.tr[s * a.ts + a.loss_o]);
            __syncthreads();
            PROF_MARK(8);
        }
        fence_proxy_async();  // phase-1 generic stores -> phase-2 TMA reads (other CTAs)
        cl.sync();
        PROF_MARK(9);
        // ---------------- phase 2: in-order batch sums + AdamW for this CTA's parameter rows
        if (rank < a.n_units) {
            const TrainNetK& N = a.net[a.unit_model[rank]];
            const int l = a.unit_layer[rank], r0 = a.unit_r0[rank], r1 = a.unit_r1[rank];
            const int in = N.in[l], out = N.out[l];
            const int count = (r1 - r0) * (in + 1);
            double acc[kTrainMaxQ];
#pragma unroll
            for (int j = 0; j < kTrainMaxQ; ++j) acc[j] = 0.0;
            double bl = 0.0;
            const int row = in + out + 1;
            const uint32_t bs_max = static_cast<uint32_t>((a.stage_cap - 6) / row) & ~1u;
            for (uint32_t b0 = 0; b0 < bcur; b0 += bs_max) {
                const int bs = static_cast<int>(min(bs_max, bcur - b0));
                const uint32_t nx = pad2(bs * in), nd = pad2(bs * out), nl = pad2(bs);
                double* SX = sm.tr;
                double* SD = SX + nx;
                double* SL = SD + nd;
                if (tid == 0) {  // X_l, D_l, losses of samples [b0, b0 + bs): three bulk copies
                    fence_proxy_async();
                    mbar_expect_tx(&s_mbar, (nx + nd + nl) * 8u);
                    bulk_g2s(SX, a.gtrace + N.gx[l] + static_cast<size_t>(b0) * in, nx * 8u, &s_mbar);
                    bulk_g2s(SD, a.gtrace + N.gd[l] + static_cast<size_t>(b0) * out, nd * 8u, &s_mbar);
                    bulk_g2s(SL, a.gtrace + a.gloss + b0, nl * 8u, &s_mbar);
                }
                mbar_wait(&s_mbar, parity);
                parity ^= 1u;
                PROF_MARK(10);
#pragma unroll
                for (int j = 0; j < kTrainMaxQ; ++j) {
                    const int q = tid + j * nt;
                    if (q < count) {
                        const int r = r0 + q / (in + 1), c = q % (in + 1);
                        double g = acc[j];
                        // bias column: X = 1.0 (D * 1.0 == D exactly), no divergent second loop
                        const double* xp = c < in ? SX + c : sm_one;
                        const int xs = c < in ? in : 0;
                        const double* dp = SD + r;
#pragma unroll 8
                        for (int b = 0; b < bs; ++b) g += dp[b * out] * xp[b * xs];
                        acc[j] = g;
                    }
                }
                if (tid == nt - 1) {
                    double x = bl;
#pragma unroll 8
                    for (int b = 0; b < bs; ++b) x += SL[b];
                    bl = x;
                }
                __syncthreads();
            }
            if (tid == nt - 1) s_bl = bl;
            __syncthreads();
            PROF_MARK(11);
            const double batch_loss = s_bl;
            if (isfinite(batch_loss)) {  // train_model: a non-finite batch is skipped (cvae.cpp:305)
                const unsigned long long t = s_t + 1;
                const double bc1 = a.bc[2 * t], bc2 = a.bc[2 * t + 1];
                const double inv = 1.0 / static_cast<double>(bcur);
#pragma unroll
                for (int j = 0; j < kTrainMaxQ; ++j) {
                    const int q = tid + j * nt;
                    if (q < count) {
                        const int r = r0 + q / (in + 1), c = q % (in + 1);
                        const int idx = c < in ? N.woff[l] + r * in + c : N.woff[l] + out * in + r;
                        const double g = acc[j] * inv;  // MlpGradients::scale (mlp.cpp:139-145)
                        // adamw_step (mlp.cpp:214-228)
                        double m = a.adam_m[idx], v = a.adam_v[idx];
                        m = a.beta1 * m + (1.0 - a.beta1) * g;
                        v = a.beta2 * v + (1.0 - a.beta2) * g * g;
                        const double m_hat = m / bc1;
                        const double v_hat = v / bc2;
                        const double p = sm.P[idx];
                        const double pn = p - a.lr * (m_hat / (sqrt(v_hat) + a.eps) + a.wd * p);
                        a.adam_m[idx] = m;
                        a.adam_v[idx] = v;
                        a.params[idx] = pn;
                        for (int k = 0; k < C; ++k) *cl.map_shared_rank(sm.P + idx, k) = pn;
                    }
                }
                __syncthreads();
                if (tid == 0) s_t = t;
            }
            if (rank == 0 && tid == 0) a.batch_loss[bi] = batch_loss;
            PROF_MARK(12);
        }
        cl.sync();
        PROF_MARK(13);
    }
    if (rank == 0 && tid == 0) *a.t_io = s_t;
#ifdef SST_TRAIN_PROFILE
    if (rank == 0 && tid == 0) {
        printf("train-prof batches %u:", a.n_batches);
        for (int i = 0; i < 16; ++i) printf(" [%d]%.0f", i, static_cast<double>(g_prof[i]) / a.n_batches);
        printf("\n");
        for (int i = 0; i < 16; ++i) g_prof[i] = 0;
    }
#endif
}

__global__ void __launch_bounds__(kTrainThreads) k_train_eval(const __grid_constant__ TrainArgs a) {
    extern __shared__ __align__(16) double smem[];
    const Smem sm = carve(a, smem);
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int i = tid; i < a.n_params; i += nt) sm.P[i] = __ldg(a.params + i);
    for (uint32_t c0 = blockIdx.x * a.chunk; c0 < a.n_order; c0 += gridDim.x * a.chunk) {
        const int ns = static_cast<int>(min(static_cast<uint32_t>(a.chunk), a.n_order - c0));
        __syncthreads();
        for (int s = tid; s < ns; s += nt) sm.ids[s] = __ldg(a.order + c0 + s);
        __syncthreads();
        long long prof_last = 0;
        elbo_chunk(a, sm.P, sm.tr, sm.ids, ns, false, prof_last);
        for (int s = tid; s < ns; s += nt) a.batch_loss[c0 + s] = sm.tr[s * a.ts + a.loss_o];
    }
}

// target_for_sample / condition_for_sample (cvae.cpp:185-212) with NormConstants
// (cvae.cpp:67-73): sigma -> log1p(max(0, s)) / log1p(sigma_ref), n -> log(max(1, n)) / log(n_ref).
__global__ void k_train_prep(const TrainPrepArgs a) {
    const uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
    if (i >= a.n) return;
    const TrainingSampleDev s = static_cast<const TrainingSampleDev*>(a.samples)[i];
    const double ns = log1p(fmax(0.0, static_cast<double>(s.sigma_t))) / a.log1p_sigma_ref;
    const double nn = log(fmax(1.0, static_cast<double>(s.n_events))) / a.log_n_ref;
    const double g = s.g;
    if (a.kind == 0) {
        a.x[i] = nn;
        a.cnd[2 * i] = ns;
        a.cnd[2 * i + 1] = g;
    } else if (a.kind == 1) {
        a.x[3 * i] = s.cos_theta;
        a.x[3 * i + 1] = s.alpha;
        a.x[3 * i + 2] = s.beta;
        a.cnd[3 * i] = ns;
        a.cnd[3 * i + 1] = g;
        a.cnd[3 * i + 2] = nn;
    } else {
        for (int k = 0; k < 3; ++k) {
            a.x[6 * i + k] = s.rep_position[k];
            a.x[6 * i + 3 + k] = s.rep_direction[k];
        }
        double* c = a.cnd + 7 * i;
        c[0] = ns;
        c[1] = g;
        c[2] = s.phi;
        c[3] = s.cos_theta;
        c[4] = s.alpha;
        c[5] = s.beta;
        c[6] = nn;
    }
}

}  // namespace

cudaError_t launch_train_prep(const TrainPrepArgs& a, cudaStream_t s) {
    if (a.n == 0) return cudaSuccess;
    k_train_prep<<<static_cast<unsigned>((a.n + 255) / 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

int train_cluster_size(size_t smem_bytes) {
    cudaFuncSetAttribute(k_train_epoch, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes));
    cudaFuncSetAttribute(k_train_epoch, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {16, 8}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c);
        cfg.blockDim = dim3(kTrainThreads);
        cfg.dynamicSmemBytes = smem_bytes;
        cudaLaunchAttribute attr;
        attr.id = cudaLaunchAttributeClusterDimension;
        attr.val.clusterDim.x = c;
        attr.val.clusterDim.y = 1;
        attr.val.clusterDim.z = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_train_epoch, &cfg) == cudaSuccess && n > 0) return c;
        cudaGetLastError();
    }
    return 0;
}

cudaError_t launch_train_epoch(const TrainArgs& a, int cluster, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(k_train_epoch, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(a.smem_bytes));
    if (e != cudaSuccess) return e;
    if (cluster > 8) {
        e = cudaFuncSetAttribute(k_train_epoch, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(kTrainThreads);
    cfg.dynamicSmemBytes = a.smem_bytes;
    cfg.stream = s;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cluster;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_train_epoch, a);
}

cudaError_t launch_train_eval(const TrainArgs& a, cudaStream_t s) {
    if (a.n_order == 0) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_train_eval, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(a.smem_bytes));
    if (e != cudaSuccess) return e;
    const unsigned blocks = min(static_cast<unsigned>((a.n_order + a.chunk - 1) / a.chunk), 148u * 4u);
    k_train_eval<<<blocks, kTrainThreads, a.smem_bytes, s>>>(a);
    return cudaGetLastError();
}

}  // namespace sstg
