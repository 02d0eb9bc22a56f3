// peak.cu -- FP32 FMA throughput microbenchmark (the roofline denominator for the
// FP32-pipe-bound render kernel; MEASURED_PEAKS.json only carries HBM and bf16 GEMM).
// Built as a separate library (libsst_peak.so) used by bench.py only.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kChains = 8;
constexpr int kIters = 8192;

__global__ void __launch_bounds__(256) k_ffma(float* out, float a, float b) {
    float acc[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = threadIdx.x * 1e-3f + i;
#pragma unroll 4
    for (int it = 0; it < kIters; ++it) {
#pragma unroll
        for (int i = 0; i < kChains; ++i) acc[i] = fmaf(acc[i], a, b);
    }
    float s = 0.0f;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s += acc[i];
    if (s == 12345.678f) out[threadIdx.x] = s;  // keeps the chains alive
}

}  // namespace

extern "C" double sst_peak_ffma_tflops(int device, int repeats) {
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    float* out = nullptr;
    cudaMalloc(&out, 1024 * sizeof(float));
    const int grid = sms * 8, block = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_ffma<<<grid, block>>>(out, 0.9999f, 1e-4f);  // warm-up
    cudaDeviceSynchronize();
    double best = 0.0;
    for (int r = 0; r < repeats; ++r) {
        cudaEventRecord(e0);
        k_ffma<<<grid, block>>>(out, 0.9999f, 1e-4f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * kChains * static_cast<double>(kIters) * grid * block;
        const double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
