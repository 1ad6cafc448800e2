// Micro-benchmarks that size the on-chip (resident) PCG design on the B200:
//  1. grid barrier + fixed-order reduction of one partial per CTA (1 CTA per SM)
//  2. L2 re-read bandwidth of a per-CTA slice of an L2-resident buffer
//  3. fp64 FMA issue rate per SM
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/mb_resident.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_barrier(unsigned long long *ctr, double *part, int iters, double *out)
{
    const int tid = threadIdx.x, P = gridDim.x;
    double acc = 1.0 + blockIdx.x;
    __shared__ double sh;
    for (int it = 0; it < iters; it++) {
        if (tid == 0) {
            part[(it & 1) * 1024 + blockIdx.x] = acc;
            __threadfence();
            atomicAdd(ctr, 1ull);
            const unsigned long long target = (unsigned long long)(it + 1) * P;
            while (ld_acq(ctr) < target) { }
        }
        __syncthreads();
        if (tid < 32) {
            double s = 0.0;
            for (int b = tid; b < P; b += 32) s += __ldcg(part + (it & 1) * 1024 + b);
            for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
            if (tid == 0) sh = s;
        }
        __syncthreads();
        acc = sh * 1e-3;
    }
    if (tid == 0 && blockIdx.x == 0) out[0] = acc;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_l2read(const double2 *buf, long long n2, int passes, double *out)
{
    const long long per = n2 / gridDim.x;
    const double2 *p = buf + per * blockIdx.x;
    double acc = 0.0;
    for (int it = 0; it < passes; it++) {
        for (long long i = threadIdx.x; i < per; i += NT * 4) {
            double2 v[4];
#pragma unroll
            for (int k = 0; k < 4; k++) v[k] = (i + k * NT < per) ? __ldcg(p + i + k * NT) : make_double2(0, 0);
#pragma unroll
            for (int k = 0; k < 4; k++) acc += v[k].x + v[k].y;
        }
    }
    if (acc == 12345.0) out[0] = acc;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_l2rmw(double2 *buf, long long n2, int passes, double a)
{
    const long long per = n2 / gridDim.x;
    double2 *p = buf + per * blockIdx.x;
    for (int it = 0; it < passes; it++) {
        for (long long i = threadIdx.x; i < per; i += NT * 4) {
            double2 v[4];
#pragma unroll
            for (int k = 0; k < 4; k++) v[k] = (i + k * NT < per) ? __ldcg(p + i + k * NT) : make_double2(0, 0);
#pragma unroll
            for (int k = 0; k < 4; k++) if (i + k * NT < per) { v[k].x += a; v[k].y += a; __stcg(p + i + k * NT, v[k]); }
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) k_dfma(int iters, double *out)
{
    double a[8];
#pragma unroll
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x * 1e-3 + k;
    const double m = 0.999999, c = 1e-7;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = fma(a[k], m, c);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += a[k];
    if (s == 1.2345) out[0] = s;
}

int main()
{
    int dev = 0, nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    unsigned long long *ctr;
    double *part, *out;
    CK(cudaMalloc(&ctr, 8));
    CK(cudaMalloc(&part, 2048 * 8));
    CK(cudaMalloc(&out, 8));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms;
    for (int P : {nsm, 144}) {
        const int iters = 20000;
        CK(cudaMemset(ctr, 0, 8));
        k_barrier<416><<<P, 416>>>(ctr, part, 100, out);
        CK(cudaDeviceSynchronize());
        CK(cudaMemset(ctr, 0, 8));
        cudaEventRecord(e0);
        k_barrier<416><<<P, 416>>>(ctr, part, iters, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("barrier+reduce P=%d: %.3f us per barrier\n", P, ms * 1e3 / iters);
    }
    for (double mb : {8.0, 16.0, 24.0, 32.0, 48.0, 64.0}) {
        const long long n2 = (long long)(mb * 1e6 / 16) / nsm * nsm;
        double2 *buf;
        CK(cudaMalloc(&buf, n2 * 16));
        CK(cudaMemset(buf, 0, n2 * 16));
        const int passes = 50;
        k_l2read<416><<<nsm, 416>>>(buf, n2, 2, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_l2read<416><<<nsm, 416>>>(buf, n2, passes, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("L2 re-read %5.1f MB: %.2f us/pass = %.2f TB/s\n", mb, ms * 1e3 / passes, n2 * 16.0 * passes / (ms * 1e-3) / 1e12);
        cudaEventRecord(e0);
        k_l2rmw<416><<<nsm, 416>>>(buf, n2, passes, 1.0);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        printf("L2 RMW     %5.1f MB: %.2f us/pass = %.2f TB/s (read+write)\n", mb, ms * 1e3 / passes, 2 * n2 * 16.0 * passes / (ms * 1e-3) / 1e12);
        cudaFree(buf);
    }
    {
        const int iters = 20000;
        k_dfma<416><<<nsm, 416>>>(100, out);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        k_dfma<416><<<nsm, 416>>>(iters, out);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        const double fmas = (double)nsm * 416 * iters * 8;
        printf("DFMA: %.2f T FMA/s = %.1f FMA/clk/SM at 1.965 GHz\n", fmas / (ms * 1e-3) / 1e12,
               fmas / (ms * 1e-3) / nsm / 1.965e9);
    }
    return 0;
}
