// fp64_peak.cu -- measured FP64 (DFMA) peak of this B200, the denominator of
// k_project's FP64-pipe roofline ("FP64 pipe utilisation
// against a DFMA peak measured on the box").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
//   tools/fp64_peak  -> one JSON line
//
// Every thread runs 16 independent DFMA chains (enough ILP to cover the
// pipe latency); the grid is 148 SMs x 8 CTAs x 256 threads.  A DFMA is 2
// flops.  Best of 10 launches, CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CH = 16;

__global__ void __launch_bounds__(256) k_dfma(double* out, int iters, double a, double b) {
    double x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = threadIdx.x * 1e-3 + c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == 12345.678) out[0] = s;  // keep the chains alive
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
    float best = 1e30f;
    for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double dfma = (double)blocks * threads * iters * CH;
    const double tflops = 2.0 * dfma / (best * 1e-3) / 1e12;
    const double per_sm_clk = dfma / (best * 1e-3) / sms / (clk * 1e3);
    printf("{\"fp64_dfma_tflops\": %.3f, \"dfma_per_sm_per_clk_at_attr_clock\": %.2f, "
           "\"sms\": %d, \"attr_clock_mhz\": %.0f, \"ms\": %.4f, \"how\": \"%d CTAs x %d threads x "
           "%d iters x %d independent DFMA chains, best of 10, CUDA events\"}\n",
           tflops, per_sm_clk, sms, clk / 1e3, best, blocks, threads, iters, CH);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
