// train.h -- CVAE training on the GPU: the device form of
// train_model (cvae.cpp:234-347). Shared by train.cu (kernels) and api.cu (host
// orchestration).
//
// Structure of one epoch (one launch of k_train_epoch, one thread-block cluster):
//   for each minibatch of the epoch's shuffled order:
//     phase 1  every CTA of the cluster runs the ELBO forward + backward
//              (elbo_forward / cvae_elbo_loss_grad, cvae.cpp:117-183) for its slice of
//              the batch in shared memory, then writes the per-sample layer inputs X_l,
//              deltas D_l and losses to batch-planar global buffers (L2-resident);
//     cluster barrier (release/acquire);
//     phase 2  CTA k owns a block of parameter rows of one layer ("unit"): it stages
//              X_l and D_l of the whole batch into shared memory and sums
//              dW[r][c] = sum_b D_l[b][r] * X_l[b][c] (bias: sum_b D_l[b][r]) in batch
//              order -- the reference's per-sample accumulation order
//              (mlp_backward, mlp.cpp:160-166) -- then scales by 1/B and applies
//              AdamW (adamw_step, mlp.cpp:214-228) and broadcasts the new values into
//              every CTA's shared-memory parameter copy over DSMEM;
//     cluster barrier.
// Everything is FP64 and compiled with -fmad=false: the same operation order as the
// reference, up to CUDA-libm vs glibc last-ulp differences in exp / log1p / log / cos.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace sstg {

constexpr int kTrainMaxLayers = 5;   // depth <= 4
constexpr int kTrainMaxWidth = 32;
constexpr int kTrainMaxLatent = 16;
constexpr int kTrainThreads = 512;
constexpr int kTrainMaxUnits = 16;   // cluster size upper bound
constexpr int kTrainMaxQ = 4;        // parameters per thread in phase 2

struct TrainNetK {
    int n_layers;
    int in[kTrainMaxLayers], out[kTrainMaxLayers];
    int woff[kTrainMaxLayers];   // offset of W_l in the parameter array (b_l follows W_l)
    int xo[kTrainMaxLayers];     // smem trace offsets (doubles, per sample row): X_l
    int po[kTrainMaxLayers];     //   pre-activations of layer l (head: the output)
    int dlo[kTrainMaxLayers];    //   deltas of layer l (after the softplus derivative)
    size_t gx[kTrainMaxLayers];  // global planar regions: X_l as [batch][in]
    size_t gd[kTrainMaxLayers];  //                         D_l as [batch][out]
};

struct TrainArgs {
    TrainNetK net[2];  // 0 = encoder (input [x, c]), 1 = decoder (input [z, c])
    int p_in, p_out, latent;
    int n_params;      // encoder then decoder, flatten_parameters order
    int n_params_pad;  // rounded up to an even count (16-byte smem alignment)
    int ts;            // doubles per smem trace row
    int din_o, eps_o, term_o, loss_o;
    int chunk;         // samples per smem chunk in phase 1
    int stage_cap;     // doubles of smem for phase-2 staging
    size_t smem_bytes;

    const double* x;        // [n][p_out] targets (target_for_sample, cvae.cpp:201-212)
    const double* cnd;      // [n][p_in]  conditions (condition_for_sample, cvae.cpp:185-199)
    const uint32_t* order;  // train: this epoch's shuffled train_idx; eval: val_idx
    uint32_t n_order;
    uint32_t batch, n_batches;
    uint64_t seed;
    uint32_t epoch;

    double* params;  // [n_params] master copy (in/out)
    double* adam_m;  // [n_params]
    double* adam_v;  // [n_params]
    unsigned long long* t_io;  // AdamW step counter (shared by both states)
    const double* bc;          // [2 * (t_max + 1)]: 1 - beta1^t, 1 - beta2^t (host pow)
    double lr, wd, beta1, beta2, eps;

    double* gtrace;        // planar X_l / D_l regions + losses
    size_t gloss;          // offset of the [batch] loss region
    double* batch_loss;    // [n_batches] this epoch's batch losses (train) / [n] (eval)

    int n_units;
    int unit_model[kTrainMaxUnits], unit_layer[kTrainMaxUnits];
    int unit_r0[kTrainMaxUnits], unit_r1[kTrainMaxUnits];
};

// Per-sample targets and conditions in FP64 from TrainingSample records.
struct TrainPrepArgs {
    const void* samples;  // TrainingSampleDev[n] (52-byte records)
    uint64_t n;
    int kind;
    double log1p_sigma_ref, log_n_ref;  // host glibc values of the NormConstants denominators
    double* x;
    double* cnd;
};

cudaError_t launch_train_prep(const TrainPrepArgs& a, cudaStream_t s);
// One epoch of minibatch AdamW on one cluster of `cluster` CTAs.
cudaError_t launch_train_epoch(const TrainArgs& a, int cluster, cudaStream_t s);
// Validation losses (cvae_elbo_loss, cvae.cpp:113-116) for a.order[0..n_order) into a.batch_loss.
cudaError_t launch_train_eval(const TrainArgs& a, cudaStream_t s);
// Largest usable cluster size (16 if the non-portable size is available, else 8) for smem bytes.
int train_cluster_size(size_t smem_bytes);

}  // namespace sstg
