// probe.cu -- measured roofline denominators for the FP64 material kernel.
//
// MEASURED_PEAKS.json has no FP64 figure, so bench.py measures the
// sustained DFMA throughput of the box it runs on with this kernel: eight
// independent FMA chains per thread, one full wave of resident CTAs per SM.
#include "common.cuh"

namespace {
__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1e-3 * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;  // keep the chains live
}
}  // namespace

// Sustained fp64 FMA throughput in TFLOP/s (2 flops per DFMA), best of `reps`.
extern "C" int am_probe_fp64_tflops(int reps, double* tflops) {
    double* d;
    AM_CUDA(cudaMalloc(&d, sizeof(double)));
    int dev, sms;
    AM_CUDA(cudaGetDevice(&dev));
    AM_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int blocks = sms * 8, threads = 256, iters = 8192;
    cudaEvent_t e0, e1;
    AM_CUDA(cudaEventCreate(&e0));
    AM_CUDA(cudaEventCreate(&e1));
    k_dfma<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);  // warm-up
    double best = 0.0;
    for (int r = 0; r < (reps > 0 ? reps : 1); ++r) {
        AM_CUDA(cudaEventRecord(e0));
        k_dfma<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
        AM_CUDA(cudaEventRecord(e1));
        AM_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        AM_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        const double flops = 2.0 * 8.0 * iters * double(blocks) * threads;
        const double tf = flops / (ms * 1e-3) / 1e12;
        best = tf > best ? tf : best;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(d);
    *tflops = best;
    return AM_OK;
}
