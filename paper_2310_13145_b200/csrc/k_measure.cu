// k_measure.cu -- the FP64 (non-tensor) pipe peak of this GPU, measured:
// the denominator of the branch kernels' roofline.  A DFMA chain microbenchmark: every thread
// runs 8 independent fma chains (enough independent work per warp to cover the DFMA latency),
// grid = 8 blocks of 256 threads per SM, timed with CUDA events; flops = 2 per DFMA.
#include <cuda_runtime.h>
#include <stdint.h>

#include "ucac.h"

namespace {

__global__ void __launch_bounds__(256) k_dfma_chain(int iters, double b, double c, double *sink) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
    double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == 123.456) sink[blockIdx.x] = s;   // never true; keeps the chains live
}

}  // namespace

extern "C" ucac_status ucac_measure_fp64_peak(int32_t iters, double *tflops, double *ms_out) {
    if (iters <= 0 || !tflops) return UCAC_EINVAL;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return UCAC_ECUDA;
    double *sink = nullptr;
    if (cudaMalloc(&sink, sizeof(double) * sms * 8) != cudaSuccess) return UCAC_ENOMEM;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 8, block = 256;
    k_dfma_chain<<<grid, block>>>(iters / 8 + 1, 0.999999, 1e-7, sink);   // warm-up (clocks up)
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k_dfma_chain<<<grid, block>>>(iters, 0.999999, 1e-7, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    if (err != cudaSuccess) return UCAC_ECUDA;
    const double flops = 2.0 * 8.0 * 8.0 * (double)iters * grid * block;
    *tflops = flops / (best * 1e-3) / 1e12;
    if (ms_out) *ms_out = best;
    return UCAC_OK;
}
