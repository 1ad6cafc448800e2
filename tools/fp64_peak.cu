// Measured fp64 FMA pipe throughput of this GPU (the ALU roofline of the fp64 stencil variants):
// every thread runs 8 independent DFMA chains; 4 x SMs CTAs of 256 threads; best of 5 runs.
// Prints DFMA lane-ops per second, per SM per clock (at the SM clock the caller passes) and
// TFLOP/s (2 flops per FMA).
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = fma(x[k], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 12345.678) out[0] = s;    // keeps the chains live
}

int main(int argc, char **argv)
{
    const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    double *out;
    cudaMalloc(&out, 8);
    const int blocks = 4 * p.multiProcessorCount, threads = 256, iters = 1 << 14;
    k_dfma<<<blocks, threads>>>(out, 16, 0.999, 1e-3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k_dfma<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = (double)blocks * threads * iters * 8;   // DFMA lane-ops
    const double rate = ops / (best * 1e-3);
    printf("{\"dfma_lane_ops_per_s\": %.4e, \"per_sm_per_clk\": %.2f, \"fp64_tflops\": %.2f, \"sms\": %d, "
           "\"sm_mhz_assumed\": %.0f, \"ms\": %.4f}\n",
           rate, rate / p.multiProcessorCount / (mhz * 1e6), 2.0 * rate / 1e12, p.multiProcessorCount, mhz, best);
    return 0;
}
