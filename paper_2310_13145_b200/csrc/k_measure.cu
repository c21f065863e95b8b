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

// Dependent-chain latencies (cycles per link), one warp, clock64 around each chain: the numbers
// behind DESIGN.md 11's argument on splitting one small solve over several lanes.
constexpr int LAT_N = 512;
__global__ void k_latency(double b, double c, double *out) {
    double a = threadIdx.x * 1e-12 + 1.0;
    long long t0, t1;
    const int lane = threadIdx.x & 31;
    // [0] DFMA
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < LAT_N; i++) a = fma(a, b, c);
    t1 = clock64();
    const double r0 = (double)(t1 - t0) / LAT_N;
    // [1] DADD
    double s = a;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < LAT_N; i++) s = s + c;
    t1 = clock64();
    const double r1 = (double)(t1 - t0) / LAT_N;
    // [2] one butterfly step of a warp reduction on doubles: v += shfl_xor(v, 1)
    double v = s;
    t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < LAT_N; i++) v = v + __shfl_xor_sync(0xffffffffu, v, 1);
    t1 = clock64();
    const double r2 = (double)(t1 - t0) / LAT_N;
    // [3] the branch kernels' reciprocal (MUFU.RCP64H + two Newton steps)
    double q = v * 1e-300 + 1.5;
    t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < LAT_N / 8; i++) {
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(q));
        double e = fma(-q, r, 1.0);
        r = fma(r, e, r);
        e = fma(-q, r, 1.0);
        q = fma(r, e, r) + 1.0;
    }
    t1 = clock64();
    const double r3 = (double)(t1 - t0) / (LAT_N / 8);
    // [4] IEEE sqrt
    double w = q;
    t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < LAT_N / 8; i++) w = sqrt(w) + 1.0;
    t1 = clock64();
    const double r4 = (double)(t1 - t0) / (LAT_N / 8);
    if (lane == 0) {
        out[0] = r0; out[1] = r1; out[2] = r2; out[3] = r3; out[4] = r4;
        out[5] = a + s + v + q + w;   // keeps every chain live
    }
}

}  // namespace

/* dependent-chain latencies in cycles: [0] DFMA, [1] DADD, [2] double shuffle + add (one
 * warp-reduction step), [3] the reciprocal of k_branch.cu (rcp.approx + 2 Newton steps), [4] IEEE sqrt */
extern "C" ucac_status ucac_measure_latencies(double *cycles5) {
    if (!cycles5) return UCAC_EINVAL;
    double *buf = nullptr;
    if (cudaMalloc(&buf, 6 * sizeof(double)) != cudaSuccess) return UCAC_ENOMEM;
    k_latency<<<1, 32>>>(0.999999, 1e-7, buf);   // warm-up
    k_latency<<<1, 32>>>(0.999999, 1e-7, buf);
    double h[6];
    cudaError_t e = cudaMemcpy(h, buf, sizeof h, cudaMemcpyDeviceToHost);
    cudaFree(buf);
    if (e != cudaSuccess) return UCAC_ECUDA;
    for (int k = 0; k < 5; k++) cycles5[k] = h[k];
    return UCAC_OK;
}

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
