// Resident PCG: one time step's whole solve (Alg. 1, readings R3-R6) in ONE cooperative
// launch whose CTAs keep the PCG vectors on chip.
//
// Why: at C3 (1M DoF) a PCG iteration of the streaming kernels moves ~112 MB through HBM/L2 and
// costs ~24 us.  The 148 SMs hold 148 x 227 KB = 33.6 MB of shared memory: enough for d (with a
// one-node halo), r, q/s and the material ids of a 1M-node grid.  Per iteration only the Jacobi
// inverse diagonal (8 B/node, L2-resident), the x update (a fire-and-forget red.add per node into
// the L2-resident output vector) and the s values on brick faces cross the L2.  What is left is
// the fp64 stencil arithmetic and two grid barriers per iteration carrying the Alg. 1 reductions
// (d^T q, then r^T s and r^T r).
//
// Partition: the node grid is cut into px x py x pz bricks, one per CTA (all co-resident:
// cooperative launch), each brick <= 31 x (NW - 1) x 16 nodes.  A CTA holds for its brick, in
// shared memory:
//   dS   d (or x0 / x for the residual kernels) on the brick + its one-node halo
//   rS   r on the owned nodes
//   qS   q = A d (kernel A), then s = P^-1 r (kernel B) on the owned nodes
//   ids  material id + 1 of every element touching an owned node
// x lives in the output vector U[(n+1) % 3] (global, L2-resident): x0 is stored there at the
// start, kernel B updates it by its owner thread (loads batched with the Jacobi loads).
// Stencil: the fp64 WHT sum factorisation of k_stencil (EL_Q1P arithmetic, bit-identical per
// node for the same input): lane = x column, warp = one element row, z marched in registers; the
// y seam between warps goes through shared memory (one __syncthreads per plane).
// Halo of d: d = s + beta d is applied on halo nodes too, from the neighbours' s (their brick-face
// values, stored to a global s vector before the barrier that ends kernel B) -- the consistency
// argument of the z-slabs: no extra synchronisation.
// Reductions: each CTA stores its partials and counts itself in with a release add; every CTA
// waits for the count and sums all partials in one fixed order, so every CTA takes the same loop
// decisions and results are deterministic run to run.
#pragma once

namespace hf {

constexpr int RES_NW = 13;                 // warps per CTA
constexpr int RES_R = 2;                   // element (and owned node) rows per warp
constexpr int RES_ROWS = RES_NW * RES_R;   // element rows per brick
constexpr int RES_NT = 32 * RES_NW;
constexpr int RES_PMAX = 160;              // CTAs (one per SM)
constexpr int RES_BZ_MAX = 16;             // planes per brick

struct ResSync {                           // zeroed before every launch (graph memset node)
    double part[2][RES_PMAX][4];
    unsigned long long ctr;                // arrivals: epoch k is complete at k P
};

struct ResArgs {
    Geom g;
    Lam lam;
    int px, py, pz;                        // bricks per axis; CTA b = ix + px (iy + py iz)
    int bxm, bym, bzm;                     // largest brick extents (shared-memory strides)
    const unsigned char *kid;              // material id + 1 per element, layer layout
    int kid_pitch;
    double pal[PAL_MAX][2];                // (k, c) of id m (entry 0 = (0, 0))
    int npal;
    const double *b, *invd;
    double *ring[3];                       // time-step ring (step n: u^n = U[n%3], x -> U[(n+1)%3])
    double *sg;                            // s exchange vector (node layout)
    double *dsave;                         // d across a residual replacement (node layout)
    CgState *st;
    ResSync *rs;
    int first;                             // run starts here: x0 = u^n at step 0
    unsigned long long *launches;
    unsigned long long *prof;              // NULL, or per-phase ns totals per CTA: prof[b * RES_PROF_N + k]
};
enum { RES_PROF_DUPD = 0, RES_PROF_STENCIL, RES_PROF_BARA, RES_PROF_B, RES_PROF_BARB, RES_PROF_INIT, RES_PROF_ITERS,
       RES_PROF_FENCE, RES_PROF_SPIN, RES_PROF_READ, RES_PROF_N };

struct ResSmem {                           // byte offsets of the dynamic shared-memory regions
    int XS, YS, ZS;                        // dS extents (x fastest)
    int XE, YE;                            // ids extents (x, y)
    size_t dS, rS, qS, palt, seam, red, ids, total;
};

__host__ __device__ inline ResSmem res_smem(int bxm, int bym, int bzm, int npal)
{
    ResSmem m;
    m.XS = bxm + 2; m.YS = bym + 2; m.ZS = bzm + 2;
    m.XE = bxm + 1; m.YE = bym + 1;
    size_t o = 0;
    auto al = [](size_t v) { return (v + 127) & ~(size_t)127; };   // 128-B aligned regions
    m.dS = o; o = al(o + (size_t)m.XS * m.YS * m.ZS * 8);
    m.rS = o; o = al(o + (size_t)bxm * bym * bzm * 8);
    m.qS = o; o = al(o + (size_t)bxm * bym * bzm * 8);
    m.palt = o; o = al(o + (size_t)npal * 64);
    m.seam = o; o = al(o + 2 * RES_NW * 32 * 8);
    m.red = o; o = al(o + (RES_NW + 1) * 4 * 8);
    m.ids = o; o += (size_t)m.XE * m.YE * (bzm + 1);
    m.total = (o + 127) & ~(size_t)127;
    return m;
}

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void red_add_f64(double *p, double v)
{
    asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Grid-wide sums of NV per-thread values (every thread of every CTA gets the same sums, in one
// fixed order: per warp xor tree, warps in order, CTAs b = lane, lane + 32, ... then a xor tree,
// lane 0's value).  Arrival: one release add per CTA on a counter after its partials; every CTA
// polls the counter (one thread, one word) until all P CTAs of this epoch arrived, then its warp 0
// reads the P partials.  A CTA that does not see every arrival within 20 s traps.
template <int NV>
__device__ __forceinline__ void res_allreduce(ResSync *rs, int P, int blk, unsigned long long epoch, double (&v)[NV],
                                              double *red, unsigned long long *pf = nullptr)
{
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int j = 0; j < NV; j++) {
        double x = v[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0) red[w * 4 + j] = x;
    }
    __syncthreads();
    if (w == 0) {
        if (lane == 0) {
            double s[4] = {0.0, 0.0, 0.0, 0.0};
            for (int k = 0; k < RES_NW; k++)
#pragma unroll
                for (int j = 0; j < NV; j++) s[j] += red[k * 4 + j];
            double *dst = rs->part[epoch & 1][blk];
#pragma unroll
            for (int j = 0; j < NV; j++) __stcg(dst + j, s[j]);
            const unsigned long long tf = pf ? globaltimer() : 0ull;
            __threadfence();
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&rs->ctr) : "memory");
            const unsigned long long target = epoch * (unsigned long long)P;
            const unsigned long long t0 = globaltimer();
            if (pf) pf[RES_PROF_FENCE] += t0 - tf;
            unsigned spins = 0;
            while (ld_acquire_gpu(&rs->ctr) < target) {
                if ((++spins & 255u) == 0 && globaltimer() - t0 > 20000000000ull) __trap();
            }
            if (pf) pf[RES_PROF_SPIN] += globaltimer() - t0;
        }
        __syncwarp();
        const unsigned long long tr = (pf && lane == 0) ? globaltimer() : 0ull;
        double s[NV];
#pragma unroll
        for (int j = 0; j < NV; j++) s[j] = 0.0;
        for (int b = lane; b < P; b += 32) {
            const double *src = rs->part[epoch & 1][b];
#pragma unroll
            for (int j = 0; j < NV; j++) s[j] += __ldcg(src + j);
        }
#pragma unroll
        for (int j = 0; j < NV; j++) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
        }
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < NV; j++) red[RES_NW * 4 + j] = s[j];
            if (pf) pf[RES_PROF_READ] += globaltimer() - tr;
        }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; j++) v[j] = red[RES_NW * 4 + j];
}

// What a thread knows about its place in the brick.
struct ResThr {
    const double *dS;
    const unsigned char *ids;
    const double *palt;          // [npal][8]
    double *seam;                // [2][NW][32]
    int XS, XY, XE, XYE;         // strides of dS and ids
    int lane, w;
    bool act;                    // this lane covers an element column of the brick (lane <= bx)
    int by, bz;
    unsigned own;                // bit e: owns node (lane, w R + e) of every plane
};

// The on-chip stencil: y = (aK K + aM M) v on the owned nodes of the brick, v = dS (the k_stencil
// EL_Q1P arithmetic with one element row per warp: x butterfly in registers + shuffle, the warp's
// element row, fused z butterfly with the material's (a, b) coefficients, the y seam through
// shared memory).  out(zi, y, centre) for this thread's owned node of plane Z0 + zi.
template <class Out>
__device__ __forceinline__ void res_stencil(const ResThr &t, Out &&out)
{
    constexpr int R = RES_R;
    double(*const seam)[RES_NW][32] = reinterpret_cast<double(*)[RES_NW][32]>(t.seam);
    const double(*const palt)[8] = reinterpret_cast<const double(*)[8]>(t.palt);
    const int lane = t.lane, w = t.w;
    double Fp[R][4], Cy[R][4], cen[R];
#pragma unroll
    for (int r = 0; r < R; r++) {
#pragma unroll
        for (int ch = 0; ch < 4; ch++) { Fp[r][ch] = 0.0; Cy[r][ch] = 0.0; }
        cen[r] = 0.0;
    }
    // node rows w R .. w R + R of the brick box (rows beyond by + 1 read as 0), element rows
    // w R .. w R + R - 1 (beyond by: material 0)
    bool rin[R + 1];
#pragma unroll
    for (int e = 0; e <= R; e++) rin[e] = t.act && w * R + e <= t.by + 1;
    const double *row = t.dS + w * R * t.XS + lane;
    const unsigned char *idr = t.ids + w * R * t.XE + lane;
#pragma unroll 1
    for (int it = 0; it <= t.bz + 1; ++it, row += t.XY) {
        double S[R + 1], D[R + 1], craw[R];
#pragma unroll
        for (int e = 0; e <= R; e++) {
            double v = 0.0, v1 = 0.0;
            if (rin[e]) { v = row[e * t.XS]; v1 = row[e * t.XS + 1]; }
            if (e < R) craw[e] = v;
            S[e] = v + v1;
            D[e] = v - v1;
        }
        if (it == 0) {
#pragma unroll
            for (int r = 0; r < R; r++) {
                Fp[r][0] = S[r] + S[r + 1];
                Fp[r][1] = S[r] - S[r + 1];
                Fp[r][2] = D[r] + D[r + 1];
                Fp[r][3] = D[r] - D[r + 1];
            }
        } else {
            // element layer it - 1: y butterfly, fused z butterfly + scaling
            double T[R][4];
#pragma unroll
            for (int r = 0; r < R; r++) {
                const int m = rin[r + 1] && w * R + r <= t.by ? idr[(it - 1) * t.XYE + r * t.XE] : 0;
                const double2 *pe = reinterpret_cast<const double2 *>(palt[m]);
                double Fc[4];
                Fc[0] = S[r] + S[r + 1];   // sx=0, sy=0
                Fc[1] = S[r] - S[r + 1];   // sx=0, sy=1
                Fc[2] = D[r] + D[r + 1];   // sx=1, sy=0
                Fc[3] = D[r] - D[r + 1];   // sx=1, sy=1
#pragma unroll
                for (int ch = 0; ch < 4; ch++) {
                    const double2 ab = pe[ch];
                    T[r][ch] = fma(ab.x, Fp[r][ch], fma(ab.y, Fc[ch], Cy[r][ch]));   // bottom plane it - 1
                    Cy[r][ch] = fma(ab.y, Fp[r][ch], ab.x * Fc[ch]);                // top plane it
                    Fp[r][ch] = Fc[ch];
                }
            }
            // backward y and x butterflies for node rows e = 0..R of plane it - 1
            double yv[R + 1];
#pragma unroll
            for (int e = 0; e <= R; e++) {
                double E0, E1;
                if (e == 0) { E0 = T[0][0] + T[0][1]; E1 = T[0][2] + T[0][3]; }
                else if (e == R) { E0 = T[R - 1][0] - T[R - 1][1]; E1 = T[R - 1][2] - T[R - 1][3]; }
                else {
                    E0 = (T[e][0] + T[e][1]) + (T[e - 1][0] - T[e - 1][1]);
                    E1 = (T[e][2] + T[e][3]) + (T[e - 1][2] - T[e - 1][3]);
                }
                const double left = __shfl_up_sync(0xffffffffu, E0 - E1, 1);
                yv[e] = (E0 + E1) + left;
            }
            seam[it & 1][w][lane] = yv[R];
            __syncthreads();
            if (it >= 2 && t.own) {          // node plane it - 1 = Z0 + (it - 2)
                if (w > 0) yv[0] += seam[it & 1][w - 1][lane];
#pragma unroll
                for (int e = 0; e < R; e++)
                    if ((t.own >> e) & 1u) out(it - 2, e, yv[e], cen[e]);
            }
        }
#pragma unroll
        for (int r = 0; r < R; r++) cen[r] = craw[r];
    }
}

__global__ void __launch_bounds__(RES_NT, 1) k_pcg_res(const __grid_constant__ ResArgs a)
{
    constexpr int NW = RES_NW;
    const Geom &g = a.g;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int blk = blockIdx.x, P = gridDim.x;
    if (blk == 0 && tid == 0 && a.launches) atomicAdd(a.launches, 1ull);

    // ---- state of this system (written by earlier kernels; the launch boundary orders them) ----
    CgState *const st = a.st;
    const CgHdr hd = load_hdr(st);
    if (hd.h0.x >= 0) return;                        // an earlier time step failed: nothing to do
    const int step = hd.h0.w, re = hd.h1.y, max_iter = hd.h2.y;
    const double rtol2 = st->rtol2;
    const int sidx = step % 3;
    const double *const un = a.ring[sidx];
    const double *const unm1 = a.ring[(sidx + 2) % 3];
    double *const xg = a.ring[(sidx + 1) % 3];
    const bool first = a.first && step == 0;

    // ---- this CTA's brick ---------------------------------------------------------------------
    const int ix = blk % a.px, iy = (blk / a.px) % a.py, iz = blk / (a.px * a.py);
    const int X0 = (int)((long long)ix * g.nx1 / a.px), X1 = (int)((long long)(ix + 1) * g.nx1 / a.px);
    const int Y0 = (int)((long long)iy * g.ny1 / a.py), Y1 = (int)((long long)(iy + 1) * g.ny1 / a.py);
    const int Z0 = (int)((long long)iz * g.nzl / a.pz), Z1 = (int)((long long)(iz + 1) * g.nzl / a.pz);
    const int bx = X1 - X0, by = Y1 - Y0, bz = Z1 - Z0;
    const ResSmem L = res_smem(a.bxm, a.bym, a.bzm, a.npal);
    extern __shared__ __align__(128) unsigned char smem[];
    double *const dS = reinterpret_cast<double *>(smem + L.dS);
    double *const rS = reinterpret_cast<double *>(smem + L.rS);
    double *const qS = reinterpret_cast<double *>(smem + L.qS);
    double(*const palt)[8] = reinterpret_cast<double(*)[8]>(smem + L.palt);
    double *const red = reinterpret_cast<double *>(smem + L.red);
    unsigned char *const ids = smem + L.ids;
    const int XS = L.XS, YS = L.YS, XY = L.XS * L.YS;

    // ---- per-CTA tables: the material coefficients of the fused z butterfly (as EL_Q1P), ids ----
    for (int i = tid; i < a.npal * 4; i += RES_NT) {
        const int m = i >> 2, ch = i & 3;
        const double kk = a.pal[m][0], cc = a.pal[m][1];
        palt[m][2 * ch] = fma(kk, a.lam.ka[ch], cc * a.lam.ma[ch]);
        palt[m][2 * ch + 1] = fma(kk, a.lam.kb[ch], cc * a.lam.mb[ch]);
    }
    const int XYE = L.XE * L.YE;
    for (int i = tid; i < XYE * (bz + 1); i += RES_NT) {
        const int lx = i % L.XE, ly = (i / L.XE) % L.YE, lz = i / XYE;
        const int ex = X0 - 1 + lx, ey = Y0 - 1 + ly, ez = Z0 - 1 + lz;
        unsigned char v = 0;
        if (lx <= bx && ly <= by && ex >= 0 && ex < g.nx && ey >= 0 && ey < g.ny && ez >= -1 && ez < g.nzl)
            v = a.kid[((long long)(ez + 1) * g.ny + ey) * a.kid_pitch + ex];
        ids[i] = v;
    }

    // ---- thread geometry: lane = x column X0 - 1 + lane, warp = node / element row Y0 - 1 + w ---
    ResThr T;
    T.dS = dS; T.ids = ids; T.palt = &palt[0][0]; T.seam = reinterpret_cast<double *>(smem + L.seam);
    T.XS = XS; T.XY = XY; T.XE = L.XE; T.XYE = XYE;
    T.lane = lane; T.w = w;
    constexpr int R = RES_R;
    T.act = lane <= bx;
    T.by = by;
    T.bz = bz;
    T.own = 0;
#pragma unroll
    for (int e = 0; e < R; e++)
        if (lane >= 1 && lane <= bx && w * R + e >= 1 && w * R + e <= by) T.own |= 1u << e;
    const int xi = X0 - 1 + lane;
    // owned node (row e) of plane zi (local plane zi + 1): shared index, global node index, dS cell
    auto oidx = [&](int zi, int e) -> int { return (zi * by + (w * R + e - 1)) * bx + (lane - 1); };
    auto nidx = [&](int zi, int e) -> long long {
        return (long long)(Z0 + zi) * g.plane + (long long)(Y0 - 1 + w * R + e) * g.pitch + xi;
    };
    auto cidx = [&](int zi, int e) -> int { return (zi + 1) * XY + (w * R + e) * XS + lane; };
    auto face = [&](int zi, int e) -> bool {
        return lane == 1 || lane == bx || w * R + e == 1 || w * R + e == by || zi == 0 || zi == bz - 1;
    };
    // the node of dS cell (lx, ly, lz) and whether it exists
    auto cell_node = [&](int lx, int ly, int lz, int &x, int &y, int &z) -> bool {
        x = X0 - 1 + lx; y = Y0 - 1 + ly; z = Z0 - 1 + lz;
        return lx <= bx + 1 && ly <= by + 1 && x >= 0 && x < g.nx1 && y >= 0 && y < g.ny1 && z >= 0 && z < g.nzl;
    };
    auto node_of = [&](int x, int y, int z) -> long long { return (long long)z * g.plane + (long long)y * g.pitch + x; };
    // f(c, lx, ly, lz) over every dS cell of planes 0..bz+1: warps over (z, y) rows, lanes over x
    auto for_cells = [&](auto &&f) {
        const int nrows = YS * (bz + 2);
        for (int row = w; row < nrows; row += NW) {
            const int ly = row % YS, lz = row / YS;
            for (int lx = lane; lx < XS; lx += 32) f(lz * XY + ly * XS + lx, lx, ly, lz);
        }
    };
    // the halo of the brick as rows: both z planes (rows ly = 0..by+1, positions lx), per inner
    // plane the two y rows (positions lx), then per inner plane the two x columns (positions ly)
    const int nhrow = 2 * (by + 2) + 4 * bz;
    auto halo_row = [&](int rI, int pos, int &lx, int &ly, int &lz) -> bool {
        if (rI < 2 * (by + 2)) {
            lz = rI < by + 2 ? 0 : bz + 1;
            ly = rI < by + 2 ? rI : rI - (by + 2);
            lx = pos;
            return pos <= bx + 1;
        }
        rI -= 2 * (by + 2);
        if (rI < 2 * bz) {
            lz = 1 + (rI >> 1);
            ly = (rI & 1) ? by + 1 : 0;
            lx = pos;
            return pos <= bx + 1;
        }
        rI -= 2 * bz;
        lz = 1 + (rI >> 1);
        lx = (rI & 1) ? bx + 1 : 0;
        ly = 1 + pos;
        return pos < by;
    };
    unsigned long long tp = 0;                 // CTA 0 thread 0: phase timer (a.prof)
    const bool prof = a.prof && tid == 0;
    unsigned long long *const pf = a.prof ? a.prof + blk * RES_PROF_N : nullptr;
    auto tick = [&](int k) {
        if (prof) { const unsigned long long t = globaltimer(); pf[k] += t - tp; tp = t; }
    };
    if (prof) tp = globaltimer();

    // ---- fill dS from a global node vector (the residual kernels' input x0 or x; Dirichlet nodes
    //      enter the constrained operator as 0, R3); store_x: x0 -> xg on the owned nodes -------
    auto fill_x = [&](auto &&val, bool store_x) {
        for_cells([&](int c, int lx, int ly, int lz) {
            int x, y, z;
            double v = 0.0;
            if (cell_node(lx, ly, lz, x, y, z)) {
                const long long n = node_of(x, y, z);
                v = val(n);
                if (store_x && lx >= 1 && lx <= bx && ly >= 1 && ly <= by && lz >= 1 && lz <= bz) __stcg(xg + n, v);
                double gv;
                if (is_dirichlet(g, x, y, z, gv)) v = 0.0;
            }
            dS[c] = v;
        });
        __syncthreads();
    };

    // residual kernel body: r = b - A v (identity rows on Dirichlet nodes), s = P^-1 r -> rS, qS
    // and the faces of sg; partials r^T s, r^T r, b_F^T b_F
    double acc[3];
    auto residual = [&]() {
        acc[0] = acc[1] = acc[2] = 0.0;
        res_stencil(T, [&](int zi, int e, double y, double) {
            const long long n = nidx(zi, e);
            double gv;
            const bool isd = is_dirichlet(g, xi, Y0 - 1 + w * R + e, Z0 + zi, gv);
            const double bv = __ldcg(a.b + n);
            const double r = isd ? 0.0 : bv - y;
            const double sv = r * __ldg(a.invd + n);
            const int o = oidx(zi, e);
            rS[o] = r;
            qS[o] = sv;
            if (face(zi, e)) __stcg(a.sg + n, sv);
            acc[0] = fma(r, sv, acc[0]);
            acc[1] = fma(r, r, acc[1]);
            if (!isd) acc[2] = fma(bv, bv, acc[2]);
        });
    };

    // ---- init (Alg. 1 lines 2-4): x0 = 2 u^n - u^(n-1) (u^n at step 0 of a run), r = b - A x0 ----
    fill_x([&](long long n) { return first ? __ldcg(un + n) : 2.0 * __ldcg(un + n) - __ldcg(unm1 + n); }, true);
    residual();
    unsigned long long epoch = 1;
    double s3[3] = {acc[0], acc[1], acc[2]};
    res_allreduce<3>(a.rs, P, blk, epoch++, s3, red);
    tick(RES_PROF_INIT);
    double delta = s3[0], rr = s3[1];
    const double bb = s3[2], thresh = rtol2 * bb;
    int status = ST_OK, zero_x = 0, iters = 0;
    double alpha = 0.0, dq = 0.0, beta = 0.0;
    for (int i = 0;; i++) {
        // ---- iteration start: stop test (R4), beta (R5) -------------------------------------
        if (!isfinite(delta) || !isfinite(rr) || !isfinite(bb)) { status = ST_BREAKDOWN; iters = i; break; }
        if (i == 0 && bb == 0.0) { zero_x = 1; iters = 0; break; }     // b_F = 0 -> x_F = 0
        const bool need = rr > thresh;
        if (!need || i >= max_iter) { if (need) status = ST_NOCONV; iters = i; break; }
        // ---- d = s + beta d on the halo (the neighbours' s): halo rows over warps, positions
        //      along a row over lanes, KR rows' loads in flight per lane -----------------------
        {
            constexpr int KR = 4;
            for (int r0 = w; r0 < nhrow; r0 += KR * NW) {
                double sv[KR][2];
                int cc[KR][2];
#pragma unroll
                for (int k = 0; k < KR; k++)
#pragma unroll
                    for (int q = 0; q < 2; q++) {
                        int lx, ly, lz, x, y, z;
                        cc[k][q] = -1;
                        sv[k][q] = 0.0;
                        const int rI = r0 + k * NW;
                        if (rI < nhrow && (q == 0 || bx + 2 > 32) && halo_row(rI, lane + 32 * q, lx, ly, lz) &&
                            cell_node(lx, ly, lz, x, y, z)) {
                            cc[k][q] = lz * XY + ly * XS + lx;
                            sv[k][q] = __ldcg(a.sg + node_of(x, y, z));
                        }
                    }
#pragma unroll
                for (int k = 0; k < KR; k++)
#pragma unroll
                    for (int q = 0; q < 2; q++)
                        if (cc[k][q] >= 0) dS[cc[k][q]] = i == 0 ? sv[k][q] : fma(beta, dS[cc[k][q]], sv[k][q]);
            }
        }
        // ... and on the owned nodes (s from qS, by their owner threads)
#pragma unroll
        for (int e = 0; e < R; e++) {
            if (!((T.own >> e) & 1u)) continue;
#pragma unroll 4
            for (int zi = 0; zi < bz; zi++) {
                const int c = cidx(zi, e);
                const double sv = qS[oidx(zi, e)];
                dS[c] = i == 0 ? sv : fma(beta, dS[c], sv);
            }
        }
        __syncthreads();
        tick(RES_PROF_DUPD);
        // ---- kernel A: q = A d, d^T q (Alg. 1 lines 6-7) -------------------------------------
        double a1[1] = {0.0};
        res_stencil(T, [&](int zi, int e, double y, double d) {
            double gv;
            const double q = is_dirichlet(g, xi, Y0 - 1 + w * R + e, Z0 + zi, gv) ? d : y;   // identity rows (R3)
            qS[oidx(zi, e)] = q;
            a1[0] = fma(d, q, a1[0]);
        });
        tick(RES_PROF_STENCIL);
        res_allreduce<1>(a.rs, P, blk, epoch++, a1, red, prof ? pf : nullptr);
        tick(RES_PROF_BARA);
        dq = a1[0];
        if (!(dq > 0.0) || !isfinite(dq) || !isfinite(delta)) { status = ST_BREAKDOWN; iters = i; break; }
        alpha = delta / dq;                              // line 8
        const bool replace = i > 0 && re > 0 && (i % re) == 0;    // line 10 (R6)
        // ---- kernel B: x += alpha d; r -= alpha q; s = P^-1 r (lines 9, 13, 15) ----------------
        double b2[2] = {0.0, 0.0};
        {
            constexpr int ZB = 4;                        // planes per batch of loads in flight
            for (int z0 = 0; z0 < bz; z0 += ZB) {
                double iv[ZB][R], xv[ZB][R];
#pragma unroll
                for (int k = 0; k < ZB; k++)
#pragma unroll
                    for (int e = 0; e < R; e++) {
                        const bool ok = z0 + k < bz && ((T.own >> e) & 1u);
                        iv[k][e] = (ok && !replace) ? __ldg(a.invd + nidx(z0 + k, e)) : 0.0;
                        xv[k][e] = ok ? __ldcg(xg + nidx(z0 + k, e)) : 0.0;
                    }
#pragma unroll
                for (int k = 0; k < ZB; k++) {
                    const int zi = z0 + k;
                    if (zi >= bz) break;
#pragma unroll
                    for (int e = 0; e < R; e++) {
                        if (!((T.own >> e) & 1u)) continue;
                        const int o = oidx(zi, e);
                        __stcg(xg + nidx(zi, e), fma(alpha, dS[cidx(zi, e)], xv[k][e]));
                        if (!replace) {
                            const double r = fma(-alpha, qS[o], rS[o]);
                            const double sv = r * iv[k][e];
                            rS[o] = r;
                            qS[o] = sv;
                            if (face(zi, e)) __stcg(a.sg + nidx(zi, e), sv);
                            b2[0] = fma(r, sv, b2[0]);
                            b2[1] = fma(r, r, b2[1]);
                        }
                    }
                }
            }
        }
        tick(RES_PROF_B);
        if (replace) {
            // r = b - A x (line 11): d of the owned nodes to global, every CTA's x (red.add) and d
            // visible after a barrier, then x (+ halo) as the stencil input, and d back
            for (int e = 0; e < R; e++)
                if ((T.own >> e) & 1u)
                    for (int zi = 0; zi < bz; zi++) __stcg(a.dsave + nidx(zi, e), dS[cidx(zi, e)]);
            __threadfence();
            double z1[1] = {0.0};
            res_allreduce<1>(a.rs, P, blk, epoch++, z1, red);
            fill_x([&](long long n) { return __ldcg(xg + n); }, false);
            residual();
            b2[0] = acc[0];
            b2[1] = acc[1];
            for_cells([&](int c, int lx, int ly, int lz) {
                int x, y, z;
                dS[c] = cell_node(lx, ly, lz, x, y, z) ? __ldcg(a.dsave + node_of(x, y, z)) : 0.0;
            });
        }
        res_allreduce<2>(a.rs, P, blk, epoch++, b2, red, prof ? pf : nullptr);
        // lines 16-17: delta_(i+1) = r^T s, beta = delta_(i+1) / delta_i (R5)
        beta = b2[0] / delta;
        delta = b2[0];
        rr = b2[1];
        iters = i + 1;
        tick(RES_PROF_BARB);
    }
    if (prof) pf[RES_PROF_ITERS] += iters;

    // ---- this solve's scalars (x is already in U[(n+1) % 3]) --------------------------------
    if (blk == 0 && tid == 0) {
        st->active = 0;
        st->status = status;
        st->zero_x = zero_x;
        st->iter = iters;
        st->b_iter = iters;
        st->rr = rr;
        st->bb = bb;
        st->thresh = thresh;
        st->delta[iters & 1] = delta;
        st->alpha = alpha;
        st->dq = dq;
    }
}

}  // namespace hf
