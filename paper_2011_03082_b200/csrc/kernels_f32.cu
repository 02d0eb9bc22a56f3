// kernels_f32.cu -- production FP32 instantiation of every device kernel.
#include <cstdint>

#define SST_REAL float
#define SST_NS f32

// Decoder weights and normalisation constants of this precision (decoder.cuh, step.cuh).
__constant__ float c_weights[1332];
__constant__ float c_norm[6];
// The same weights in the decoders' row-pair layout (decoder.cuh layer_pairs, FFMA2).
__constant__ float2 c_wpair[666];
#define SST_DECODER_PAIRS 1

#include "kernels_impl.cuh"
