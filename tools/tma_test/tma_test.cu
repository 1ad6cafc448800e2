// Minimal TMA probe: which box coordinates work (negative / out-of-range / alignment).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_param(const __grid_constant__ CUtensorMap map, double *out, int *flag, int bw, int bh, int x0, int y0, int z0)
{
    extern __shared__ __align__(128) unsigned char sm[];
    double *buf = (double *)sm;
    __shared__ __align__(8) uint64_t bar;
    for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) buf[i] = -7.0;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(bw * bh * 8) : "memory");
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                     ::"r"(s32(buf)), "l"((uint64_t)&map), "r"(x0), "r"(y0), "r"(z0), "r"(s32(&bar)) : "memory");
    }
    unsigned ok = 0;
    for (long it = 0; it < 20000000 && !ok; it++)
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(s32(&bar)) : "memory");
    if (threadIdx.x == 0) *flag = ok;
    __syncthreads();
    for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char **argv)
{
    int bw = atoi(argv[1]), bh = atoi(argv[2]), x0 = atoi(argv[3]), y0 = atoi(argv[4]), z0 = atoi(argv[5]);
    void *fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    EncodeTiled_t enc = (EncodeTiled_t)fn;
    const int nx = 40, ny = 40, nz = 40;
    std::vector<double> h(nx * ny * nz);
    for (size_t i = 0; i < h.size(); i++) h[i] = (double)i + 1;
    double *d, *out; int *flag; cudaMalloc(&d, h.size() * 8); cudaMalloc(&out, 1 << 20); cudaMalloc(&flag, 4);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[3] = {nx, ny, nz}, strides[2] = {nx * 8, nx * ny * 8};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k_param<<<1, 128, 32768>>>(map, out, flag, bw, bh, x0, y0, z0);
    cudaError_t le = cudaGetLastError();
    cudaError_t e = cudaDeviceSynchronize();
    int fl = -1;
    std::vector<double> o(bw * bh, -1);
    if (e == cudaSuccess) { cudaMemcpy(&fl, flag, 4, cudaMemcpyDeviceToHost); cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost); }
    // check
    int bad = 0;
    for (int j = 0; j < bh && e == cudaSuccess; j++)
        for (int i = 0; i < bw; i++) {
            int x = x0 + i, y = y0 + j, z = z0;
            double ex = (x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nz) ? h[(z * ny + y) * nx + x] : 0.0;
            if (o[j * bw + i] != ex) bad++;
        }
    printf("box %dx%d at (%d,%d,%d): encode=%d launch=%s sync=%s tx_done=%d mismatches=%d o0=%g\n", bw, bh, x0, y0, z0, (int)r,
           cudaGetErrorString(le), cudaGetErrorString(e), fl, bad, o[0]);
    return 0;
}
