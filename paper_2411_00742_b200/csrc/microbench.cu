// =====================================================================================
//  microbench.cu — roofline denominators measured on the box by bench.py (not part of
//  the product path): FP64 FMA throughput of the SIMT pipes (no FP64 figure exists in
//  MEASURED_PEAKS.json), measured with CUDA events.
// =====================================================================================
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int CHAINS = 16;

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
    double x[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-9 + c;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;   // keep the chains alive
}

}  // namespace

extern "C" {

// Returns achieved FP64 TFLOP/s (FMA = 2 flops) of a saturating DFMA kernel, best of `reps`.
double pbe_mb_dfma_tflops(int device, int reps) {
    if (cudaSetDevice(device) != cudaSuccess) return -1.0;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return -1.0;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    k_dfma<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);   // warm-up
    double best = 0.0;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        const double flops = 2.0 * CHAINS * (double)iters * blocks * threads;
        const double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
    }
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

}  // extern "C"
