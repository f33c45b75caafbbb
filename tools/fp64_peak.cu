// FP64 (DFMA) peak microbenchmark for the SURVEY.md 8(d) FP64 roofline:
// every thread runs 8 independent FMA chains (enough ILP to cover the DFMA
// latency), grid = SMs x 4 blocks of 256 threads. Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
    if (s == 12345.678) out[0] = s; // keeps the chains live
}

int main() {
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    double* out;
    cudaMalloc(&out, sizeof(double));
    const int threads = 256, blocks = sms * 4, iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int w = 0; w < 3; ++w) k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) k_dfma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 2.0 * 8.0 * iters * double(threads) * blocks * reps;
    const double tf = flop / (ms * 1e-3) / 1e12;
    printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, \"dfma_per_clk_per_sm\": %.1f, "
           "\"kernel\": \"8 independent DFMA chains/thread, %d x %d threads, %d iterations x %d launches\", "
           "\"error\": \"%s\"}\n",
           tf, sms, clk / 1000, tf * 1e12 / 2.0 / sms / (clk * 1e3), blocks, threads, iters, reps,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
