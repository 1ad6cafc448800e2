// hf_ablate.cuh -- NEXT row f4: the paper's two earlier interpretations of the assembly operator,
// rebuilt for sm_100a so that the comparison of §5.1 (Fig. 5, Table 1) can be rerun
// against the production stencil (Implementation 3 analogue, hf_kernels.cuh).
//
// Both variants compute exactly the apply of Eq. (1): y = c * sum_e A_e^T (aK k_e K_ref +
// aM c_e M_ref) A_e u + b with dense 8 x 8 voxel matrices (the Q1 tensor product, or the sum of the
// six P1 tets of f1), so they are checked against the same oracle as the stencil.  fp64 only,
// single-context grids only (no slabs); Dirichlet rows are not special-cased (as hf_apply).
//
// Implementation 1, "flexible DbD" (Eq. (3)): a preprocessing kernel stores every
// scaled element matrix A_e in global memory in element order ("Every elemental
// assembly matrix is stored in global memory"); pass 1 runs one thread per element-DoF pair:
// the element's 8 threads stage its 8 corner values in shared memory ("loads vertex data
// to local memory"), each computes one row dot product and stores it as its contribution to the
// global vertex in "vertex order" (slot j of node i = the element of which i is local corner j);
// pass 2 sums the 8 contributions of every vertex ("reads these 24 consecutive
// contribution and sums them") and fuses y = c (.) + b.
//
// Implementation 2, "single pass FG DbD" (Eq. (4)): one thread per output node gathers
// all 8 adjacent elements (27 input values, 8 (k, c) pairs) and loops over the 8 element-DoF
// contributions; the reference matrices sit in constant (kernel parameter) memory; a
// work group stages the 3 x 3 strips of u around its x-row segment ("3 x 3 rectangular blocks, as
// long as possible") and the 4 element rows of (k, c) in shared memory.
#pragma once
#include "hf_kernels.cuh"

namespace hf {

constexpr int DBD_W = 128;     // Impl 2: output nodes per CTA (one x-row segment)

// Impl 1 preprocessing: row j of A_e for thread (e, j); rows of one element are contiguous, so a
// warp writes 4 elements x 512 B contiguously.
__global__ void __launch_bounds__(256) k_ebe_store(Geom g, const void *kcp, Dense dn, double *A, long long nrows,
                                                   unsigned long long *launches)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0 && launches) atomicAdd(launches, 1ull);
    if (t >= nrows) return;
    const long long e = t >> 3;
    const int j = (int)(t & 7);
    const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
    const double2 kc = load_kc<double>(g, reinterpret_cast<const double2 *>(kcp), ex, ey, ez - g.zg0);
    double2 *row = reinterpret_cast<double2 *>(A + t * 8);
#pragma unroll
    for (int l = 0; l < 8; l += 2) {
        double2 v;
        v.x = kc.x * dn.K[j * 8 + l] + kc.y * dn.M[j * 8 + l];
        v.y = kc.x * dn.K[j * 8 + l + 1] + kc.y * dn.M[j * 8 + l + 1];
        row[l / 2] = v;
    }
}

// Impl 1 pass 1: contrib[8 i + j] = (A_e u_e)_j for the element e of which node i is corner j.
__global__ void __launch_bounds__(256) k_ebe_pass1(Geom g, const double *u, const double *A, double *contrib,
                                                   long long nelem, unsigned long long *launches)
{
    __shared__ double ue[32][8];
    const int el = threadIdx.x >> 3, j = threadIdx.x & 7;
    const long long e = (long long)blockIdx.x * 32 + el;
    if (blockIdx.x == 0 && threadIdx.x == 0 && launches) atomicAdd(launches, 1ull);
    const bool valid = e < nelem;
    long long nj = 0;
    if (valid) {
        const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
        nj = (long long)(ez + (j >> 2) - g.zg0) * g.plane + (long long)(ey + ((j >> 1) & 1)) * g.pitch + ex + (j & 1);
        ue[el][j] = u[nj];
    }
    __syncwarp();      // an element's 8 threads are in one warp
    if (!valid) return;
    const double2 *row = reinterpret_cast<const double2 *>(A + e * 64 + j * 8);
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < 8; l += 2) {
        const double2 a = row[l / 2];
        acc = fma(a.x, ue[el][l], acc);
        acc = fma(a.y, ue[el][l + 1], acc);
    }
    contrib[nj * 8 + j] = acc;
}

// Impl 1 pass 2: y_i = c * sum_j contrib[8 i + j] (existing elements only, fixed j order) + b_i.
__global__ void __launch_bounds__(256) k_ebe_pass2(Geom g, int nz, const double *contrib, double cc, const double *b,
                                                   double *y, long long nslots, unsigned long long *launches)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= nslots) return;
    const int x = (int)(i % g.pitch), yy = (int)((i / g.pitch) % g.ny1), z = (int)(i / g.plane) + g.zg0;
    if (x >= g.nx1) return;
    const double2 *cp = reinterpret_cast<const double2 *>(contrib + i * 8);
    double acc = 0.0;
#pragma unroll
    for (int h = 0; h < 4; h++) {
        const double2 v = cp[h];
#pragma unroll
        for (int q = 0; q < 2; q++) {
            const int j = 2 * h + q;
            const int ex = x - (j & 1), ey = yy - ((j >> 1) & 1), ez = z - (j >> 2);
            if (ex >= 0 && ey >= 0 && ez >= 0 && ex < g.nx && ey < g.ny && ez < nz) acc += q ? v.y : v.x;
        }
    }
    y[i] = cc * acc + (b ? b[i] : 0.0);
}

// Impl 2: one thread per output node (x0 + tid, yy, z); u strips (yy-1..yy+1, z-1..z+1) of
// DBD_W + 2 nodes and (k, c) rows (ey = yy-1, yy; ez = z-1, z) of DBD_W + 1 elements in smem.
__global__ void __launch_bounds__(DBD_W) k_dbd(Geom g, int nz, const double *u, const void *kcp, Dense dn, double cc,
                                               const double *b, double *y, unsigned long long *launches)
{
    __shared__ double us[9][DBD_W + 2];
    __shared__ double2 ks[4][DBD_W + 1];
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * DBD_W, yy = blockIdx.y, zl = blockIdx.z;
    const int z = zl + g.zg0;
    if ((blockIdx.x | blockIdx.y | blockIdx.z) == 0 && tid == 0 && launches) atomicAdd(launches, 1ull);
    const double2 *kc = reinterpret_cast<const double2 *>(kcp);
    for (int s = tid; s < 9 * (DBD_W + 2); s += DBD_W) {
        const int r = s / (DBD_W + 2), xi = s % (DBD_W + 2);
        const int xx = x0 - 1 + xi, ny = yy - 1 + r % 3, nzg = z - 1 + r / 3;
        double v = 0.0;
        if (xx >= 0 && xx < g.nx1 && ny >= 0 && ny < g.ny1 && nzg >= 0 && nzg < g.nz1g)
            v = u[(long long)(nzg - g.zg0) * g.plane + (long long)ny * g.pitch + xx];
        us[r][xi] = v;
    }
    for (int s = tid; s < 4 * (DBD_W + 1); s += DBD_W) {
        const int r = s / (DBD_W + 1), xi = s % (DBD_W + 1);
        const int ex = x0 - 1 + xi, ey = yy - 1 + (r & 1), ez = z - 1 + (r >> 1);
        double2 v = make_double2(0.0, 0.0);
        if (ez >= 0 && ez < nz) v = load_kc<double>(g, kc, ex, ey, ez - g.zg0);
        ks[r][xi] = v;
    }
    __syncthreads();
    const int x = x0 + tid;
    if (x >= g.nx1) return;
    double un[27];                            // the 27 input values of this work item
#pragma unroll
    for (int r = 0; r < 9; r++)
#pragma unroll
        for (int dx = 0; dx < 3; dx++) un[r * 3 + dx] = us[r][tid + dx];
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 8; j++) {            // node = local corner j of element (x-bx, yy-by, z-bz)
        const int bx = j & 1, by = (j >> 1) & 1, bz = j >> 2;
        const double2 k2 = ks[(1 - by) + 2 * (1 - bz)][tid + 1 - bx];
        double sk = 0.0, sm = 0.0;
#pragma unroll
        for (int l = 0; l < 8; l++) {
            const int lx = l & 1, ly = (l >> 1) & 1, lz = l >> 2;
            const double ul = un[((1 + ly - by) + 3 * (1 + lz - bz)) * 3 + 1 + lx - bx];
            sk = fma(dn.K[j * 8 + l], ul, sk);
            sm = fma(dn.M[j * 8 + l], ul, sm);
        }
        acc = fma(k2.x, sk, fma(k2.y, sm, acc));
    }
    const long long i = (long long)zl * g.plane + (long long)yy * g.pitch + x;
    y[i] = cc * acc + (b ? b[i] : 0.0);
}

}  // namespace hf
