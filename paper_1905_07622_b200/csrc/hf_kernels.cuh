// hf_kernels.cuh -- sm_100a kernels of libheatfem (the hot path of arXiv 1905.07622).
//
// Citations: P:n = PAPER.md line n.  Rn = reading n in DESIGN.md.
//
// The operator apply (Eq. (1)) uses the element matrices in their Walsh-Hadamard
// eigenbasis: for a trilinear voxel every K_ref and M_ref is a tensor product of the 1D
// matrices (1/h)[[1,-1],[-1,1]] and (h/6)[[2,1],[1,2]], both diagonalised by H = [[1,1],[1,-1]]:
//      A_e = (1/8) H3 diag(aK k_e lamK + aM c_e lamM) H3,   H3 = H (x) H (x) H.
// H3 is applied by sum factorisation ACROSS elements: the x butterfly of an edge and the y
// butterfly of a face are computed once and shared by all elements touching them; the z
// butterfly and the diagonal scaling of an element collapse to 4 FMA-pairs per face channel:
//      T_bottom += a Fp + b Fc,   carry_top = b Fp + a Fc,   a = t0 + t1,  b = t0 - t1.
// About 50 fp64 operations per node.
//
// Data movement (the B200 part): a CTA owns a 31 x (NW*R - 1) tile of node columns and
// marches in z through a chunk of node planes.  Each node plane of the tile (34 x (NW*R+1)
// nodes of every input vector) and the element layer below it ((k, c) of 32 x NW*R elements)
// arrive by TMA (cp.async.bulk.tensor) into an NS-stage shared-memory ring guarded by
// mbarriers, NS-1 planes ahead of the compute.  Out-of-range coordinates are zero-filled by
// the TMA unit, so the domain boundary, the halo and phantom elements need no code.  Lane l
// of warp w holds node column X0-1+l and node rows Y0-1+w*R+r (r = 0..R); x neighbours are
// read from shared memory, outputs of the x butterfly move by warp shuffle, the y seam between
// warps through shared memory, and the z neighbours stay in registers.  No atomics on data:
// each output node is written by exactly one thread; reductions are fixed-order.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace hf {

#ifndef HF_SMEM_ROUND
#define HF_SMEM_ROUND(x) (((x) + 1023) & ~(size_t)1023)
#endif

constexpr int NPART = 4;      // partial sums per block
constexpr int TILE_X = 31;    // owned node columns per CTA
constexpr int BOXW = 34;      // fp64 node columns in a TMA box (even start <= X0-1, covers X0+31)
constexpr int NMAPS = 6;      // node tensor maps: ring U[0..2], d[0..1], s

enum { LD_RAW = 0, LD_GT = 1, LD_CGD = 2, LD_X0 = 3, LD_CG1 = 4, LD_CG1W = 5 };
enum { EP_APPLY = 0, EP_CGA = 1, EP_RESID = 2, EP_RESID_INIT = 3, EP_CG1 = 4, EP_CG1W = 5 };
enum { ST_OK = 0, ST_NOCONV = -3, ST_BREAKDOWN = -4 };
enum { ROT_NONE = 0, ROT_RHS = 1, ROT_INIT = 2, ROT_X = 3 };
enum { MAP_U0 = 0, MAP_D0 = 3, MAP_S = 5 };

// PCG state of one system (Alg. 1 scalars, device resident; the paper keeps them in device
// buffers too: delta/alpha/beta kernels P:507-573).  Every field is written by one block of one
// kernel and read only by LATER kernels (kernel boundaries order them), never by the kernel that
// writes it: delta is double-buffered by iteration parity for that reason.
// Several independent systems stacked along z in one context (batched forward simulations,
// a13) have one CgState each, st[0..nsys-1].  The LOOP fields (b_iter, step, a_iter,
// replace_every, replace, npart_b, npart_a, max_iter) are shared and live in st[0]: every active
// system is at the same PCG iteration of the same time step, so one loop counter serves all.
// The SYSTEM fields (first_failed, active, status, zero_x, iter, statistics, rtol2, delta,
// thresh, bb, rr, alpha, dq) are per system: each system has its own scalars and stop test.
// npart_a / npart_b count partial sums per system (the blocks of system j are contiguous).
struct CgState {
    // header: read by every PCG kernel at its start as 16-byte loads issued together (one L2
    // round trip instead of a chain of dependent scalar loads)
    int first_failed;       // first failing step, -1 if none
    int active;             // 1 while iterating                          (init 1; A, B: 0 to stop)
    int b_iter;             // completed iterations                       (init: 0, B: i + 1)
    int step;               // time-step counter (step-end kernel)
    int a_iter;             // i of the running iteration                 (A)
    int replace_every;      // option
    int replace;            // iteration a_iter replaces the residual     (B)
    int npart_b;            // partial-sum count of the last init / B / RESID
    int npart_a;            // partial-sum count of the last A
    int max_iter;           // option
    int status, zero_x;     // ST_*, b_F == 0                             (A, B)
    int iter;               // iterations of the finished solve           (A or B when stopping)
    int total_iters, max_iters_step, steps_done;
    double rtol2;           // option
    double delta[2];        // delta_i = r_i^T s_i in slot i & 1          (written by A_i)
    double thresh, bb, rr;  // rtol^2 ||b_F||^2, ||b_F||^2, last r^T r      (A)
    double alpha, dq;       // last alpha, d^T q                          (B)
    double alf[2];          // single-reduction PCG: alpha_i in slot i & 1 (CG1 kernel i)
};
static_assert(offsetof(CgState, a_iter) == 16 && offsetof(CgState, npart_a) == 32, "CgState header layout");

// the header words of a state (3 x 16 B, one round trip)
struct CgHdr {
    int4 h0, h1, h2;        // (first_failed, active, b_iter, step), (a_iter, replace_every, replace, npart_b),
                            // (npart_a, max_iter, status, zero_x)
};
// Through the read-only (L1) path: every warp of the grid reads these 48 bytes, and L2-only loads
// (__ldcg) made them an L2 hot spot (C3 kernel A +1.7 us); the kernel boundary makes the
// previous kernel's writes visible, and no block of this kernel reads a header word that a block
// of the same kernel writes.
__device__ __forceinline__ CgHdr load_hdr(const CgState *st)
{
    const int4 *p = reinterpret_cast<const int4 *>(st);
    return {__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}

struct Geom {
    int nx1, ny1, nzl;      // nodes in x, y; local node planes
    int zg0, nz1g;          // global index of local plane 0; global node planes
    int pitch;              // node row pitch (nx1 rounded up to 16 B: TMA strides)
    long long plane;        // pitch * ny1
    int nx, ny;             // elements in x, y
    int kpitch;             // (k, c) pairs per coefficient row (nx, or nx rounded up to even in fp32)
    unsigned dbits;         // Dirichlet face bits (R3)
    int zper;               // global node planes per stacked system (= nz1g for one system)
    double gval[6];
};

// Per face channel ch = 2 sx + sy (element wave numbers s0 = sx + 2 sy, s1 = s0 + 4):
// a = k (lk[s0] + lk[s1]) + c (lm[s0] + lm[s1]),  b = k (lk[s0] - lk[s1]) + c (lm[s0] - lm[s1]),
// lm[s] = aM lamM[s] / 8, lk[s] = aK lamK[s] / 8.
struct Lam {
    double ka[4], ma[4], kb[4], mb[4];
};
struct LamF {               // the same constants for the fp32 storage variant (NEXT row f3)
    float ka[4], ma[4], kb[4], mb[4];
};

// Dense voxel matrices (element variant EL_DENSE: the paper's 6-tet split, NEXT row f1):
// y_e = (k_e Ks + c_e Ms) u_e with Ks = aK K_ref, Ms = aM M_ref (8 x 8, local l = bx+2by+4bz).
struct Dense {
    double K[64], M[64];
};
struct DenseF {
    float K[64], M[64];
};

// storage / arithmetic type of the node vectors and (k, c) pairs: double (default) or float
// (NEXT row f3).  Reductions, PCG scalars and the CG state stay fp64 in both.
template <class Real> struct Vec2;
template <> struct Vec2<double> { using type = double2; };
template <> struct Vec2<float> { using type = float2; };

// element variants: Q1 hexahedra; the 6-tet split with one (k, c) per voxel (dense 8x8 voxel
// matrices); the 6-tet split with per-tet coefficients averaged from vertex values;
// Q1 hexahedra with coefficients given by material id (hf_set_material_ids, fp64 only): the
// stencil streams one uint8 id per element instead of a 16-B (k, c) pair and looks the
// element's z-butterfly coefficients up in a per-CTA shared-memory table
enum { EL_Q1 = 0, EL_DENSE = 1, EL_TETV = 2, EL_Q1P = 3 };
// z-plane loop of the Q1 kernels unrolled by 2: the loop-carried face transforms and centre values alternate
// between two register sets instead of being copied every plane (8.6 % of kernel A's executed
// instructions were such moves); C3 22.84 vs 23.19 us per PCG iteration (R = 2 tiles only, see PU)
#ifndef HF_PLANE_UNROLL
#define HF_PLANE_UNROLL 2
#endif
constexpr int kPlaneUnroll = HF_PLANE_UNROLL;   // unroll of the stencil's z-plane loop
constexpr int PAL_MAX = 64;        // material table entries; entry 0 = (0, 0) (outside the domain)
constexpr int PAL_BW = 48;         // ids per TMA box row: 16-aligned origin <= X0-1, covers X0+30

// Kuhn tets of a voxel (local node l = bx + 2 by + 4 bz): tet t follows 0 -> e_a -> e_a+e_b -> 7
// for the t-th axis order (x,y,z), (x,z,y), (y,x,z), (y,z,x), (z,x,y), (z,y,x)
__host__ __device__ constexpr int tet_loc(int t, int v)
{
    return v == 0 ? 0 : v == 3 ? 7
         : (t == 0 ? (v == 1 ? 1 : 3) : t == 1 ? (v == 1 ? 1 : 5) : t == 2 ? (v == 1 ? 2 : 3)
          : t == 3 ? (v == 1 ? 2 : 6) : t == 4 ? (v == 1 ? 4 : 5) : (v == 1 ? 4 : 6));
}

// EL_TETV constants: aK-scaled tet stiffness matrices in tet_loc order and the mass scale
// m = aM V_tet / 20 (M_ij = m (1 + delta_ij) for every tet)
struct TetV {
    double K[6][16];
    double m;
};
struct TetVF {
    float K[6][16];
    float m;
};

// ---- multi-GPU z-slabs over peer memory (the paper's dual-GPU split) ----
// Every rank owns a mailbox in its device memory; peers write into it over NVLink (CUDA IPC
// mappings across processes, plain pointers within one).  A kernel that produces PCG partial sums
// (init, A, B, residual replacement) publishes them itself: each block counts itself done, the
// last block sums the kernel's per-block partials in a fixed order, stores the NPART sums into
// slot (seq & 1) of EVERY rank's mailbox and then releases its flag there (= seq).  The kernels
// that produce s = P^{-1} r also store the first / last owned plane of s straight into the
// lower / upper neighbour's ghost-plane buffer.  A consumer kernel waits (one thread per CTA,
// acquire at system scope) until every rank's flag reached its own seq, then adds the ranks'
// sums in rank order -- bitwise the same on every rank, so every rank takes the same loop
// decisions.  No host call, no NCCL: the whole slab solve runs in the step graph.
constexpr int HF_MAX_RANKS = 8;

struct MailHdr {                      // head of a mailbox (device memory of its owner)
    double sums[2][HF_MAX_RANKS][NPART];      // slot, source rank
    unsigned long long flags[HF_MAX_RANKS];   // latest seq published by each rank
    unsigned long long xflags[HF_MAX_RANKS];  // latest one-off exchange sequence of each rank
    unsigned long long seq, xseq;             // this rank's counters (local use)
    unsigned int done, xdone;                 // blocks of the running producer that finished
};

struct PeerSync {                     // device copy per slab context
    int nranks, rank;
    MailHdr *mine;                    // this rank's mailbox
    MailHdr *peer[HF_MAX_RANKS];      // every rank's mailbox (peer[rank] == mine)
    void *gdst_lo, *gdst_hi;          // neighbour's ghost buffer for my first / last owned plane
    void *xdst_lo, *xdst_hi;          // neighbour's one-off exchange buffers (2 parity slots each)
    const void *xsrc_lo, *xsrc_hi;    // my one-off exchange buffers (written by the neighbours)
    long long lo0, hi0;               // slot offsets of my first / last owned plane
    long long plane;                  // slots per plane
    long long xslot;                  // slots per parity slot of an exchange buffer
};

struct Sync {               // per-system reduction plumbing
    CgState *st;
    const double *pin;      // partial sums of the previous kernel (NPART per block)
    int pin_n;              // their count; -1: taken from the state (npart_a / npart_b); > 0: fixed
                            // (every producer of pin writes exactly pin_n entries, see pout_pad)
    int pout_pad;           // > nblocks: block 0 zero-fills partial entries [nblocks, pout_pad) so
                            // that a consumer can always sum pout_pad entries (adding 0 is exact)
    double *pout;           // this kernel's partial sums (NPART per block)
    unsigned long long *launches;
    cudaGraphConditionalHandle h_while, h_if;
    int use_handles;        // set the WHILE handle (graph driver)
    int use_if;             // set the IF handle (only where the body has an IF node)
    int nsys;               // systems stacked along z (>= 1); st points at st[0..nsys-1]
    const PeerSync *peer;   // slab over peer memory: sums come from / go to the mailboxes
};

struct Maps {               // TMA descriptors (host copy; kernels read a device-memory copy)
    CUtensorMap node[NMAPS];
    CUtensorMap kc;         // fp64 view (2 nx, ny, nzl + 1) of the (k, c) pairs, layer L at z = L + 1
    CUtensorMap kcn;        // EL_TETV: per-node (k, c) pairs, view (2 nx1, ny1, nzl), node layout
    CUtensorMap ghost;      // slab over peer memory: s ghost planes (lo, hi) written by the neighbours
};
constexpr int MAP_KC = NMAPS;       // index of the kc map in a device Maps array
constexpr int MAP_KCN = NMAPS + 1;  // index of the per-node pair map
constexpr int MAP_GHOST = NMAPS + 2;   // index of the ghost-plane map

struct BArgs {
    double *x;
    const double *q, *invd;
    double *dbuf[2];        // d = dbuf[(iter & 1) ^ 1] (written by kernel A of this iteration)
    double *r, *s;
    long long n, own0, own1;
    long long sysn;         // node slots per stacked system (= n for one system)
    double *rot[3];         // if rot[0]: x = rot[(step + 1) % 3]
    Sync sy;
};

// Single-reduction PCG (Chronopoulos-Gear form of Alg. 1): one
// stencil kernel per iteration.  Kernel i (iteration parity par = i & 1, fixed per graph node)
// streams r_i, w_i = A u_i, s_{i-1} = A p_{i-1} and P^{-1} (TMA maps 0..3) and forms, on every
// node of its box, s_i = w_i + beta_i s_{i-1}, r_{i+1} = r_i - alpha_i s_i, u_{i+1} = P^{-1} r_{i+1};
// on its owned nodes it also writes s_i, r_{i+1}, p_i = u_i + beta_i p_{i-1}, x_{i+1} = x_i +
// alpha_i p_i; the stencil gives w_{i+1} = A u_{i+1}.  Partials: (r u, r r, b b (forwarded), w u).
// r, w, s are ping-pong buffers (read at halo nodes by other CTAs); p, x are pointwise.
struct CgOne {
    double *rout, *sout, *wout;   // r_{i+1}, s_i, w_{i+1} (slot par ^ 1; EP_CG1W: wout = w slot of its r)
    double *p;                    // p (in place)
    double *x;                    // the iterate; NULL: the time-step ring slot U[(step + 1) % 3]
    int par;                      // parity of the iteration (kernel i reads counter slot par)
};

struct StencilArgs {
    Geom g;
    Lam lam;
    double *out0;                 // q (CG A), r (residual), y (apply)
    double *out_s;                // s = P^{-1} r (residual kernels)
    const double *bvec, *invd;
    double *ring[3];              // time-step ring U (centre stores of the guess)
    double *dbuf[2];              // PCG direction ping-pong (centre stores of d_new)
    double *xout;                 // centre store of x0 when not rotating
    double c, s;
    int z_out0, z_out1, zchunk;   // output planes (local) and planes per CTA
    int zper_out;                 // output planes per stacked system (= z_out1 - z_out0 for one)
    int gz_lo, gz_hi;             // LD_CGD over peer memory: local planes whose s comes from the ghost map
    int zs0, zs1;                 // planes whose centre values are stored
    int dmode;                    // EP_APPLY: 0 none, 1 identity rows, 2 set g on D rows
    int first;                    // LD_X0: step 0 of the run (guess = u^0)
    int rot_role;                 // ROT_*: map slots resolved from st->step
    Sync sy;
    const CUtensorMap *tm;        // device copy of this launch's Maps (written once, never modified)
    int tm_fence;                 // 1: acquire the descriptors (their addresses may have been reused)
    LamF lamf;                    // fp32 variant: lam in float
    Dense dn;                     // EL_DENSE only
    DenseF dnf;                   // EL_DENSE, fp32 variant
    TetV tv;                      // EL_TETV only
    TetVF tvf;                    // EL_TETV, fp32 variant
    double pal[PAL_MAX][2];       // EL_Q1P: (k, c) of material id m (entry 0 = (0, 0))
    int npal;                     // EL_Q1P: table entries in use (materials + 1)
    BArgs fb;                     // FL_FUSEB: kernel B's arguments
    unsigned long long *gbar;     // FL_FUSEB: grid-barrier counter (monotonic)
    CgOne c1;                     // EP_CG1 / EP_CG1W: the single-reduction PCG's vectors
};
// Node-vector pointers of StencilArgs / BArgs / StepArgs are declared double* but address
// vectors of the context's storage type; kernels instantiated for Real = float reinterpret them.

__device__ __forceinline__ bool is_dirichlet(const Geom &g, int x, int y, int zl, double &val)
{
    const unsigned b = g.dbits;
    if (!b) return false;
    const int zg = zl + g.zg0;
    if ((b & 1u) && x == 0) { val = g.gval[0]; return true; }
    if ((b & 2u) && x == g.nx1 - 1) { val = g.gval[1]; return true; }
    if ((b & 4u) && y == 0) { val = g.gval[2]; return true; }
    if ((b & 8u) && y == g.ny1 - 1) { val = g.gval[3]; return true; }
    if (b & 48u) {                       // z faces of the system the plane belongs to
        const int zs = g.zper == g.nz1g ? zg : zg % g.zper;
        if ((b & 16u) && zs == 0) { val = g.gval[4]; return true; }
        if ((b & 32u) && zs == g.zper - 1) { val = g.gval[5]; return true; }
    }
    return false;
}

// ---- TMA / mbarrier primitives (PTX) --------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

#ifndef HF_WAIT_MODE
#define HF_WAIT_MODE 0
#endif
#ifndef HF_WAIT_HINT_NS
#define HF_WAIT_HINT_NS 100
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity)
{
#if HF_WAIT_MODE == 1
    // non-blocking probe in a spin loop (no suspension of the waiting warp)
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#elif HF_WAIT_MODE == 2
    // potentially blocking probe with a short suspend-time hint (ns)
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(HF_WAIT_HINT_NS)
        : "memory");
#else
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

#ifdef HF_DEBUG_WAIT
// debug builds: a wait that does not complete within ~2^24 polls records who waited (into mapped
// host memory, readable after the context dies) and traps instead of hanging
__device__ unsigned long long *g_dbg;   // [0..9] stuck wait, [10..15] heartbeats
__device__ __noinline__ void mbar_wait_dbg(uint64_t *bar, unsigned parity, int tag, int it)
{
    for (long long n = 0;; n++) {
        uint32_t ok;
        asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
                     "selp.u32 %0, 1, 0, P1;\n\t}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (ok) return;
        if (n == (1ll << 20)) {
            unsigned long long *d = g_dbg;
            if (d && atomicAdd(d, 1ull) == 0) {
                d[1] = tag; d[2] = it; d[3] = parity; d[4] = blockIdx.x; d[5] = blockIdx.y; d[6] = blockIdx.z;
                d[7] = threadIdx.x + 32 * threadIdx.y; d[8] = smem_u32(bar);
                uint64_t st;
                asm volatile("ld.shared.b64 %0, [%1];" : "=l"(st) : "r"(smem_u32(bar)));
                d[9] = st;
                __threadfence_system();
            }
            __trap();
        }
    }
}
#endif

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int x, int y, int z, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// a tensor map in global memory may have been rewritten since an SM cached it (address reuse)
__device__ __forceinline__ void tensormap_acquire(const CUtensorMap *m)
{
    asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"((uint64_t)m) : "memory");
}

__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// programmatic dependent launch (graph edges of type Programmatic, hf_ctx::pdl): wait for the
// previous kernel's completion and memory; allow the next kernel's CTAs to start launching.
// Both are no-ops for kernels launched without a programmatic dependency.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void prefetch_map(const CUtensorMap *m)
{
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)m) : "memory");
}

// ---- deterministic block reduction + last-block finalisation -----------------------------

template <int NT>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NPART], double *partials, int blk)
{
    __shared__ double red[NT / 32][NPART];
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int j = 0; j < NPART; j++) {
        double v = acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[wid][j] = v;
    }
    __syncthreads();
    if (tid < NPART) {
        double v = 0.0;
        for (int w = 0; w < NT / 32; w++) v += red[w][tid];
        partials[(long long)blk * NPART + tid] = v;
    }
}

// Grid-wide sums of the PREVIOUS kernel's per-block partials, computed redundantly by every
// block in one fixed order (deterministic, no atomics, no fences: the kernel boundary orders
// the producer's writes before these reads).  All threads return the same sums.
// The first round of the partial-sum loads (KU blocks per thread, all issued before any add):
// a kernel whose partial count is fixed (Sync::pin_n > 0) issues them right after
// griddepcontrol.wait, in parallel with its state header (prev_finish adds them later).
#ifndef HF_RP_KU
#define HF_RP_KU 4
#endif
struct PrevPre {
    double2 v[HF_RP_KU][2];
};

template <int NT, bool CG = false>
__device__ __forceinline__ void prev_load(const double *part, int n, int b0, PrevPre &pre)
{
    constexpr int KU = HF_RP_KU;
    static_assert(NPART == 4, "partials are read as 2 x double2");
#pragma unroll
    for (int k = 0; k < KU; k++) {
        const int b = b0 + k * NT;
        if (b < n) {
            const double2 *q = reinterpret_cast<const double2 *>(part + (long long)b * NPART);
            // CG: partials written by other CTAs of the SAME kernel (fused A+B, after the grid
            // barrier): through L2, never the non-coherent read-only path
            pre.v[k][0] = CG ? __ldcg(q) : __ldg(q);
            pre.v[k][1] = CG ? __ldcg(q + 1) : __ldg(q + 1);
        } else {
            pre.v[k][0] = make_double2(0.0, 0.0);
            pre.v[k][1] = make_double2(0.0, 0.0);
        }
    }
}

// Grid-wide sums of the PREVIOUS kernel's per-block partials, computed redundantly by every
// block in one fixed order (deterministic, no atomics, no fences: the kernel boundary orders
// the producer's writes before these reads).  All threads return the same sums.  pre: the first
// round's loads (prev_load at b0 = tid).
template <int NT, bool CG = false>
__device__ __forceinline__ void prev_finish(const PrevPre &pre0, const double *part, int n, double (&sums)[NPART])
{
    __shared__ double redp[NT / 32][NPART];
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    double acc[NPART];
#pragma unroll
    for (int j = 0; j < NPART; j++) acc[j] = 0.0;
    // KU blocks per thread per round with every load issued before the first add (one L2 round
    // trip for n <= KU * NT); the per-thread order stays b = tid, tid + NT, ... (fixed).  Every
    // block of the grid reads the same partials: through the read-only (L1) path, not L2-only
    // (-0.6 us per C3 iteration); they are written by the previous kernel only.
    constexpr int KU = HF_RP_KU;
    PrevPre pre = pre0;
    for (int b0 = tid; b0 < n; b0 += KU * NT) {
        if (b0 != tid) prev_load<NT, CG>(part, n, b0, pre);
#pragma unroll
        for (int k = 0; k < KU; k++) {
            if (b0 + k * NT < n) {
                acc[0] += pre.v[k][0].x;
                acc[1] += pre.v[k][0].y;
                acc[2] += pre.v[k][1].x;
                acc[3] += pre.v[k][1].y;
            }
        }
    }
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int j = 0; j < NPART; j++) {
        double v = acc[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) redp[wid][j] = v;
    }
    __syncthreads();
    if constexpr (NT / 32 * NPART == 32) {
        // every warp adds the warps' values in one xor butterfly over lanes l = NPART w + j (fp
        // addition commutes, so every lane, warp and block gets the same bits)
        double v = redp[lane / NPART][lane % NPART];
#pragma unroll
        for (int o = NPART; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
#pragma unroll
        for (int j = 0; j < NPART; j++) sums[j] = __shfl_sync(0xffffffffu, v, j);
    } else {
#pragma unroll
        for (int j = 0; j < NPART; j++) {
            double v = 0.0;
            for (int w = 0; w < NT / 32; w++) v += redp[w][j];
            sums[j] = v;
        }
    }
}

template <int NT, bool CG = false>
__device__ __forceinline__ void reduce_prev(const double *part, int n, double (&sums)[NPART])
{
    PrevPre pre;
    prev_load<NT, CG>(part, n, threadIdx.x + threadIdx.y * blockDim.x, pre);
    prev_finish<NT, CG>(pre, part, n, sums);
}

// zero-fill of the partial entries [nblk, sy.pout_pad) by block 0 (fixed consumer counts)
template <int NT>
__device__ __forceinline__ void pad_partials(const Sync &sy, int nblk, int blk, int tid)
{
    if (blk != 0 || sy.pout_pad <= nblk) return;
    for (int i = nblk * NPART + tid; i < sy.pout_pad * NPART; i += NT) sy.pout[i] = 0.0;
}

// sums of system sj's partials (the previous kernel's blocks of system sj are contiguous)
template <int NT>
__device__ __forceinline__ void prev_sums(const Sync &sy, int n_state, double (&sums)[NPART], int sj = 0)
{
    const int n = sy.pin_n >= 0 ? sy.pin_n : n_state;
    reduce_prev<NT>(sy.pin + (long long)sj * n * NPART, n, sums);
}

// ---- peer-memory protocol (see PeerSync) -------------------------------------------------

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// thread-level wait until flags[q] >= k for every rank q in [0, n) (mask: ranks to wait for);
// a peer that does not arrive within 30 s traps (a dead rank never hangs the GPU)
__device__ __forceinline__ void peer_spin(const unsigned long long *flags, unsigned mask, unsigned long long k)
{
    const unsigned long long t0 = globaltimer();
    for (int q = 0; mask >> q; q++) {
        if (!((mask >> q) & 1u)) continue;
        while (ld_acquire_sys(flags + q) < k) {
            __nanosleep(64);
            if (globaltimer() - t0 > 30000000000ull) __trap();
        }
    }
}

// sums of the latest published sequence over every rank, in rank order (consumer side)
template <int NT>
__device__ __forceinline__ void peer_sums(const PeerSync *pp, double (&sums)[NPART])
{
    __shared__ double ps_sh[NPART];
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    if (tid == 0) {
        const unsigned long long k = __ldcg(&pp->mine->seq);
        peer_spin(pp->mine->flags, (1u << pp->nranks) - 1u, k);
        double acc[NPART] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < pp->nranks; q++)
            for (int j = 0; j < NPART; j++) acc[j] += __ldcg(&pp->mine->sums[k & 1][q][j]);
        for (int j = 0; j < NPART; j++) ps_sh[j] = acc[j];
        asm volatile("fence.proxy.async.global;" ::: "memory");   // TMA reads of peer-written ghosts
    }
    __syncthreads();
    for (int j = 0; j < NPART; j++) sums[j] = ps_sh[j];
}

// producer side: after every block stored its partials (and ghost planes), the last block of
// the kernel publishes the fixed-order sums to every rank
template <int NT>
__device__ void peer_publish(const PeerSync *pp, const double *part, int nblk, bool remote)
{
    __shared__ int last_sh;
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    // order this thread's stores before the block's arrival: remote ghost stores (peer memory)
    // at system scope, the block's partials (tid < NPART, local memory) at GPU scope; the other
    // threads stored nothing the consumers read
    if (remote) __threadfence_system();
    else if (tid < NPART) __threadfence();
    __syncthreads();
    if (tid == 0) last_sh = atomicAdd(&pp->mine->done, 1u) == (unsigned)nblk - 1u;
    __syncthreads();
    if (!last_sh) return;
    __threadfence();
    double s[NPART];
    reduce_prev<NT, true>(part, nblk, s);
    if (tid == 0) {
        MailHdr *m = pp->mine;
        const unsigned long long k = m->seq + 1;
        m->seq = k;
        m->done = 0u;
        for (int q = 0; q < pp->nranks; q++)
            for (int j = 0; j < NPART; j++) pp->peer[q]->sums[k & 1][pp->rank][j] = s[j];
        // each release store orders this thread's sum stores (and, cumulatively, the blocks'
        // ghost stores fenced before their arrival) before the flag
        for (int q = 0; q < pp->nranks; q++) st_release_sys(&pp->peer[q]->flags[pp->rank], k);
    }
}

// my first / last owned plane of s, stored into the neighbours' ghost buffers (slot index i)
template <class Real>
__device__ __forceinline__ bool peer_ghost(const PeerSync *pp, long long i, Real v)
{
    bool st = false;
    if (pp->gdst_lo && i >= pp->lo0 && i < pp->lo0 + pp->plane) { reinterpret_cast<Real *>(pp->gdst_lo)[i - pp->lo0] = v; st = true; }
    if (pp->gdst_hi && i >= pp->hi0 && i < pp->hi0 + pp->plane) { reinterpret_cast<Real *>(pp->gdst_hi)[i - pp->hi0] = v; st = true; }
    return st;
}

// one-off exchange of a vector's ghost planes (state vectors at the start of a solve): send my
// boundary planes into the neighbours' exchange buffers, then receive theirs into my ghosts
template <class Real>
__global__ void k_xsend(const PeerSync *pp, const void *vp, unsigned long long *launches)
{
    const Real *v = reinterpret_cast<const Real *>(vp);
    const int tid = threadIdx.x;
    if (blockIdx.x == 0 && tid == 0 && launches) atomicAdd(launches, 1ull);
    const unsigned long long k = __ldcg(&pp->mine->xseq) + 1;   // this exchange's sequence
    const long long par = (long long)(k & 1) * pp->xslot;
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < pp->plane; i += (long long)gridDim.x * blockDim.x) {
        if (pp->xdst_lo) reinterpret_cast<Real *>(pp->xdst_lo)[par + i] = v[pp->lo0 + i];
        if (pp->xdst_hi) reinterpret_cast<Real *>(pp->xdst_hi)[par + i] = v[pp->hi0 + i];
    }
    __shared__ int last_sh;
    __threadfence_system();
    __syncthreads();
    if (tid == 0) last_sh = atomicAdd(&pp->mine->xdone, 1u) == gridDim.x - 1u;
    __syncthreads();
    if (!last_sh || tid != 0) return;
    MailHdr *m = pp->mine;
    m->xseq = k;
    m->xdone = 0u;
    __threadfence_system();
    if (pp->rank > 0) st_release_sys(&pp->peer[pp->rank - 1]->xflags[pp->rank], k);
    if (pp->rank + 1 < pp->nranks) st_release_sys(&pp->peer[pp->rank + 1]->xflags[pp->rank], k);
}

template <class Real>
__global__ void k_xrecv(const PeerSync *pp, void *vp, long long ghost_lo, long long ghost_hi, unsigned long long *launches)
{
    Real *v = reinterpret_cast<Real *>(vp);
    const int tid = threadIdx.x;
    if (blockIdx.x == 0 && tid == 0 && launches) atomicAdd(launches, 1ull);
    const unsigned long long k = __ldcg(&pp->mine->xseq);
    if (tid == 0) {
        unsigned mask = 0;
        if (pp->rank > 0) mask |= 1u << (pp->rank - 1);
        if (pp->rank + 1 < pp->nranks) mask |= 1u << (pp->rank + 1);
        peer_spin(pp->mine->xflags, mask, k);
    }
    __syncthreads();
    const long long par = (long long)(k & 1) * pp->xslot;
    const Real *lo = reinterpret_cast<const Real *>(pp->xsrc_lo), *hi = reinterpret_cast<const Real *>(pp->xsrc_hi);
    for (long long i = (long long)blockIdx.x * blockDim.x + tid; i < pp->plane; i += (long long)gridDim.x * blockDim.x) {
        if (ghost_lo >= 0) v[ghost_lo + i] = __ldcg(lo + par + i);
        if (ghost_hi >= 0) v[ghost_hi + i] = __ldcg(hi + par + i);
    }
}

// ---- scalar logic of Alg. 1 ------------------------------------------------------------

__device__ __forceinline__ void set_while(const Sync &sy, int v)
{
    if (sy.use_handles) cudaGraphSetConditional(sy.h_while, (unsigned)v);
}
__device__ __forceinline__ void set_if(const Sync &sy, int v)
{
    if (sy.use_handles && sy.use_if) cudaGraphSetConditional(sy.h_if, (unsigned)v);
}

// Start of iteration i (kernel A), from the sums of the init / B / RESID kernel before it:
// i = 0: delta_0 = r^T s, ||r||^2, ||b_F||^2 (Alg. 1 lines 2-4, reading R4);
// i > 0: delta_i, beta_i = delta_i / delta_{i-1} (lines 16-17, reading R5), stop test.
struct IterStart {
    bool go;
    double beta, delta, rr, thresh, bb;
    int status, zero_x;
};

// st: the system's state (delta, bb, thresh, rtol2); max_iter: the loop option
__device__ __forceinline__ IterStart iter_start(const CgState *st, int i, const double *s, int max_iter)
{
    IterStart r;
    r.delta = s[0];
    r.rr = s[1];
    r.status = ST_OK;
    r.zero_x = 0;
    r.beta = 0.0;
    if (i == 0) {
        r.bb = s[2];
        r.thresh = st->rtol2 * s[2];
    } else {
        r.bb = st->bb;
        r.thresh = st->thresh;
        r.beta = s[0] / st->delta[(i - 1) & 1];
    }
    if (!isfinite(s[0]) || !isfinite(s[1]) || !isfinite(r.bb)) { r.status = ST_BREAKDOWN; r.go = false; return r; }
    if (i == 0 && r.bb == 0.0) { r.zero_x = 1; r.go = false; return r; }   // b_F = 0 -> x_F = 0
    const bool need = r.rr > r.thresh;                                      // R4: ||r|| > tol ||b||
    r.go = need && i < max_iter;
    if (need && i >= max_iter) r.status = ST_NOCONV;
    return r;
}

// Start of iteration i of the single-reduction PCG (EP_CG1) from the previous kernel's sums
// s = (gamma_i = r_i^T u_i, r_i^T r_i, ||b_F||^2 (i = 0 only), delta_i = w_i^T u_i):
//   beta_0 = 0, alpha_0 = gamma_0 / delta_0;
//   beta_i = gamma_i / gamma_{i-1},  alpha_i = gamma_i / (delta_i - beta_i gamma_i / alpha_{i-1})
// (Chronopoulos & Gear; in exact arithmetic the alpha_i, beta_i of Alg. 1 lines 8 and 17, since
// delta_i - beta_i gamma_i / alpha_{i-1} = d_i^T A d_i).  The stop test is Alg. 1's (R4).
struct IterStart1 {
    bool go;
    double alpha, beta, gamma, rr, thresh, bb;
    int status, zero_x;
};

__device__ __forceinline__ IterStart1 iter_start_cg1(const CgState *st, int i, const double *s, int max_iter)
{
    IterStart1 r;
    r.gamma = s[0];
    r.rr = s[1];
    r.status = ST_OK;
    r.zero_x = 0;
    r.beta = 0.0;
    r.alpha = 0.0;
    double den = s[3];
    if (i == 0) {
        r.bb = s[2];
        r.thresh = st->rtol2 * s[2];
    } else {
        r.bb = st->bb;
        r.thresh = st->thresh;
        r.beta = s[0] / st->delta[(i - 1) & 1];
        den = s[3] - r.beta * s[0] / st->alf[(i - 1) & 1];
    }
    if (!isfinite(s[0]) || !isfinite(s[1]) || !isfinite(s[3]) || !isfinite(r.bb)) {
        r.status = ST_BREAKDOWN;
        r.go = false;
        return r;
    }
    if (i == 0 && r.bb == 0.0) { r.zero_x = 1; r.go = false; return r; }   // b_F = 0 -> x_F = 0
    const bool need = r.rr > r.thresh;                                      // R4: ||r|| > tol ||b||
    r.go = need && i < max_iter;
    if (need && i >= max_iter) r.status = ST_NOCONV;
    if (r.go) {
        r.alpha = r.gamma / den;
        if (!(den > 0.0) || !isfinite(r.alpha)) { r.status = ST_BREAKDOWN; r.go = false; }   // d^T A d <= 0
    }
    return r;
}

// ---- the stencil kernel (operator apply with fused prologue/epilogue) ---------------------

template <int R, int NW, int LD, class Real = double, int EL = EL_Q1>
struct StencilShape {
    static constexpr int ES = (int)sizeof(Real);
    static constexpr int H = NW * R + 1;                                     // node rows per box
    static constexpr int NA = LD == LD_RAW ? 1 : (LD == LD_GT ? 0 : (LD == LD_CG1 ? 4 : 2));   // node arrays per plane
    // box widths: the x origin must be 16-B aligned, so it starts up to 16/ES - 1 columns early
    static constexpr int BW = ES == 8 ? BOXW : 36;                           // node columns per box
    static constexpr int KW = ES == 8 ? 64 : 68;                             // kc values per box row
    static constexpr int AL = 128 / ES;                                      // elements per 128 B
    static constexpr int NODE_BOX = H * BW;                                  // elements per node box
    static constexpr int NODE_DBL = (NODE_BOX + AL - 1) / AL * AL;           // 128-B aligned slot
    // per-element (k, c) box: NW R element rows x KW; EL_TETV: per-node pairs, H rows x 2 BW;
    // EL_Q1P: NW R rows of PAL_BW uint8 material ids
    static constexpr int KC_BYTES = EL == EL_TETV ? H * 2 * BW * ES : (EL == EL_Q1P ? NW * R * PAL_BW : NW * R * KW * ES);
    static constexpr int KC_DBL = (KC_BYTES + ES - 1) / ES;
    static constexpr int STAGE_DBL = (NA * NODE_DBL + KC_DBL + AL - 1) / AL * AL;
    static constexpr unsigned STAGE_BYTES = NA * NODE_BOX * (unsigned)ES + KC_BYTES;   // TMA bytes
    static constexpr int PAL_BYTES = EL == EL_Q1P ? PAL_MAX * 8 * 8 : 0;    // (a, b) x 4 channels per material
    static constexpr int UB_BYTES = LD == LD_CG1 ? NODE_DBL * ES : 0;       // LD_CG1: the u plane (one node box)
    // rounded to 1 KB so that CTAs of different variants sharing an SM get aligned windows
    static size_t smem_bytes(int ns)
    {
        return HF_SMEM_ROUND((size_t)ns * STAGE_DBL * ES + 16 * ns + 2 * NW * 32 * ES + PAL_BYTES + UB_BYTES);
    }
};

// compile-time variant flags of the stencil kernel
enum {
    FL_MASK = 1,   // Dirichlet nodes enter the stencil as 0 (constrained operator P_F A P_F)
    FL_DIR = 2,    // Dirichlet rows in the epilogue (identity rows / r_D = 0 / set g)
    FL_HB = 4,     // EP_APPLY: y = c A u + s b (else y = c A u)
    FL_DSET = 8,   // EP_APPLY with FL_DIR: y_D = g (else y_D = u_D, identity rows)
    FL_FUSEB = 16, // EP_CGA: kernel B's work follows in the same launch after a grid barrier
    FL_PEER = 32,  // slab over peer memory: sums / ghost planes through the mailboxes (a.sy.peer)
};

// ---- PCG kernel B: x += alpha d; r -= alpha q; s = P^{-1} r; r^T s, r^T r ---------------
// (Alg. 1 lines 9, 13, 15, 16; the paper's knl_6, knl_7, knl_8, knl_9A-C, knl_10.)
// x is updated on every local node (ghost planes included, so slab ghosts stay consistent);
// r, s and the dot products only on owned nodes [own0, own1).  On a replacement iteration
// (i > 0, i mod replace_every == 0, Alg. 1 line 10) only x is updated: the residual kernel
// (EP_RESID) follows.  Also run inside kernel A's launch (FL_FUSEB) after a grid barrier.

// Kernel B's work of iteration `it` for one system (node slots [base, base + a.sysn)) on its
// blocks blk of nblk: alpha = delta / d^T q (Alg. 1 line 8); x += alpha d; r -= alpha q;
// s = P^{-1} r; partials r^T s, r^T r (lines 9-16), stored at partial slot pblk.  sst: the
// system's state; one_sys: the context has one system (its kernels drive the loop handles
// directly); glob: also do the loop duties (fused A+B launch, one system).
// FUSED: d and q were written by other CTAs of the same launch before a grid barrier, so they
// are read through L2 (ld.cg), never through the non-coherent read-only path.
template <int NT, class Real, bool FUSED, bool PEER = false>
__device__ __forceinline__ void cg_b_work(const BArgs &a, CgState *sst, bool one_sys, long long base, int blk,
                                          int nblk, int pblk, int tid, int it, int re, int step, double delta,
                                          double dq, bool glob)
{
    if (!(dq > 0.0) || !isfinite(dq) || !isfinite(delta)) {           // breakdown
        if (blk == 0 && tid == 0) {
            sst->status = ST_BREAKDOWN;
            sst->active = 0;
            sst->iter = it;
            if (one_sys) {
                set_while(a.sy, 0);
                set_if(a.sy, 0);
            }
        }
        return;
    }
    const double alpha = delta / dq;
    const Real alr = (Real)alpha;
    using V2 = typename Vec2<Real>::type;
    const Real *const qv_ = reinterpret_cast<const Real *>(a.q);
    const Real *const iv_ = reinterpret_cast<const Real *>(a.invd);
    Real *const rv_ = reinterpret_cast<Real *>(a.r);
    Real *const sv_ = reinterpret_cast<Real *>(a.s);
    const bool replace = it > 0 && re > 0 && (it % re) == 0;           // Alg. 1 line 10 (R6)
    const Real *dvec = reinterpret_cast<const Real *>(a.dbuf[(it & 1) ^ 1]);
    Real *xvec = reinterpret_cast<Real *>(a.rot[0] ? a.rot[(step + 1) % 3] : a.x);
    double acc[NPART] = {0.0, 0.0, 0.0, 0.0};
    bool remote = false;                     // this thread stored into a neighbour's memory
    const long long end = base + a.sysn;
    // BP aligned pairs per thread per sweep (slot counts are even: even row pitch), loads issued
    // up front; a pair never straddles the owned range (planes hold an even number of slots)
#ifndef HF_B_BP
#define HF_B_BP 2
#endif
    constexpr int BP = HF_B_BP;
    const long long sweep = (long long)nblk * NT * BP * 2;
    for (long long i0 = base + ((long long)blk * NT * BP + tid) * 2; i0 < end; i0 += sweep) {
        V2 xv[BP], dv[BP], rv[BP], qv[BP], iv[BP];
        bool in[BP], own[BP];
#pragma unroll
        for (int k = 0; k < BP; k++) {
            const long long i = i0 + (long long)k * NT * 2;
            in[k] = i < end;
            own[k] = in[k] && !replace && i >= a.own0 && i < a.own1;
            if (in[k]) {
                xv[k] = *reinterpret_cast<const V2 *>(xvec + i);
                dv[k] = FUSED ? __ldcg(reinterpret_cast<const V2 *>(dvec + i)) : *reinterpret_cast<const V2 *>(dvec + i);
            }
            if (own[k]) {
                rv[k] = *reinterpret_cast<const V2 *>(rv_ + i);
                qv[k] = FUSED ? __ldcg(reinterpret_cast<const V2 *>(qv_ + i)) : __ldg(reinterpret_cast<const V2 *>(qv_ + i));
                iv[k] = __ldg(reinterpret_cast<const V2 *>(iv_ + i));
            }
        }
#pragma unroll
        for (int k = 0; k < BP; k++) {
            const long long i = i0 + (long long)k * NT * 2;
            if (in[k]) {                        // x += alpha d  (line 9)
                xv[k].x = fma(alr, dv[k].x, xv[k].x);
                xv[k].y = fma(alr, dv[k].y, xv[k].y);
                *reinterpret_cast<V2 *>(xvec + i) = xv[k];
            }
            if (own[k]) {                       // r -= alpha q; s = P^{-1} r (lines 13, 15)
                rv[k].x = fma(-alr, qv[k].x, rv[k].x);
                rv[k].y = fma(-alr, qv[k].y, rv[k].y);
                V2 sv;
                sv.x = rv[k].x * iv[k].x;
                sv.y = rv[k].y * iv[k].y;
                acc[0] = fma((double)rv[k].x, (double)sv.x, acc[0]);
                acc[0] = fma((double)rv[k].y, (double)sv.y, acc[0]);
                acc[1] = fma((double)rv[k].x, (double)rv[k].x, acc[1]);
                acc[1] = fma((double)rv[k].y, (double)rv[k].y, acc[1]);
                *reinterpret_cast<V2 *>(rv_ + i) = rv[k];
                *reinterpret_cast<V2 *>(sv_ + i) = sv;
                if (PEER) {
                    remote |= peer_ghost<Real>(a.sy.peer, i, sv.x);
                    remote |= peer_ghost<Real>(a.sy.peer, i + 1, sv.y);
                }
            }
        }
    }
    pdl_trigger();
    if (!replace) {
        block_reduce_store<NT>(acc, a.sy.pout, pblk);
        pad_partials<NT>(a.sy, nblk, pblk, tid);
    }
    if (PEER && !replace) peer_publish<NT>(a.sy.peer, a.sy.pout, nblk, remote);
    if (blk == 0 && tid == 0) {
        sst->alpha = alpha;
        sst->dq = dq;
        if (glob) {
            CgState *st0 = a.sy.st;
            st0->b_iter = it + 1;
            st0->replace = replace;
            if (!replace) st0->npart_b = nblk;
            set_if(a.sy, replace ? 1 : 0);
        }
    }
}

template <int NT, class Real, bool PEER>
__global__ void __launch_bounds__(NT) k_cg_b(const BArgs a)
{
    const int tid = threadIdx.x;
    const int nsys = a.sy.nsys > 0 ? a.sy.nsys : 1;
    const int bps = (int)gridDim.x / nsys;                // blocks per system (contiguous)
    const int sj = (int)blockIdx.x / bps, blk = (int)blockIdx.x - sj * bps;
    if (blockIdx.x == 0 && tid == 0 && a.sy.launches) atomicAdd(a.sy.launches, 1ull);
    pdl_wait();
    // a fixed partial count (one system, no peer transport): kernel A's partials are requested
    // before the state header
    const bool pre_ok = !PEER && nsys == 1 && a.sy.pin_n > 0;
    PrevPre pre;
    if (pre_ok) prev_load<NT>(a.sy.pin, a.sy.pin_n, tid, pre);
    CgState *st0 = a.sy.st, *sst = st0 + sj;
    const CgHdr hd = load_hdr(st0);
    const CgHdr hs = sj ? load_hdr(sst) : hd;
    const int it = hd.h1.x, re = hd.h1.y, step = hd.h0.w;
    if (blockIdx.x == 0) {
        // loop duties (shared by the systems): leave the loop when no system iterates any more,
        // else advance the iteration and arm the replacement IF node (Alg. 1 line 10, R6)
        bool mine = tid == 0 && hd.h0.x < 0 && hd.h0.y;
        for (int j = 1 + tid; j < nsys; j += NT) mine |= st0[j].first_failed < 0 && st0[j].active;
        const bool any = nsys == 1 ? (hd.h0.x < 0 && hd.h0.y) : __syncthreads_or(mine);
        if (tid == 0 && !any) {
            set_while(a.sy, 0);
            set_if(a.sy, 0);
        } else if (tid == 0) {
            const bool replace = it > 0 && re > 0 && (it % re) == 0;
            st0->b_iter = it + 1;
            st0->replace = replace;
            if (!replace) st0->npart_b = bps;
            set_if(a.sy, replace ? 1 : 0);
        }
    }
    if (hs.h0.x >= 0 || !hs.h0.y) return;          // this system failed earlier / has converged
    // alpha_i = delta_i / (d_i^T q_i)  (Alg. 1 line 8) from kernel A's partials of this system
    double ps[NPART];
    if (PEER) peer_sums<NT>(a.sy.peer, ps);
    else {
        const int n = pre_ok ? a.sy.pin_n : (a.sy.pin_n >= 0 ? a.sy.pin_n : hd.h2.x);
        const double *pin = a.sy.pin + (long long)sj * n * NPART;
        if (!pre_ok) prev_load<NT>(pin, n, tid, pre);
        prev_finish<NT>(pre, pin, n, ps);
    }
    cg_b_work<NT, Real, false, PEER>(a, sst, nsys == 1, (long long)sj * a.sysn, blk, bps, (int)blockIdx.x, tid, it, re,
                               step, sst->delta[it & 1], ps[0], false);
}

// Grid-wide barrier of a launch whose CTAs are all co-resident (checked on the host with the
// occupancy API before a fused launch is used).  The counter only grows: a launch of nblk CTAs
// waits for the next multiple of nblk.  A wait that does not complete traps (no silent hang).
__device__ __forceinline__ void grid_barrier(unsigned long long *ctr, unsigned nblk, int tid)
{
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned long long old = atomicAdd(ctr, 1ull);
        const unsigned long long target = (old / nblk + 1) * nblk;
        unsigned long long v;
        long long spins = 0;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if (++spins > (1ll << 26)) __trap();
        } while (v < target);
    }
    __syncthreads();
}

#ifdef HF_TRACE
// debug builds (-DHF_TRACE): %globaltimer stamps of thread 0 of every kernel-A block
__device__ unsigned long long g_trace[4096][8];
__device__ __forceinline__ unsigned long long gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define HF_TR(k) do { if (EP == EP_CGA && tid == 0 && blk < 4096) g_trace[blk][k] = gtime(); } while (0)
#else
#define HF_TR(k) do { } while (0)
#endif

// (the single-reduction PCG kernel at R = 2 is held to 128 registers: two CTAs per SM; a
// minimum of 0 leaves the other kernels to the same register heuristic as no minimum, which an
// explicit 1 does not: it raised the apply from 72 to 104 registers)
template <int R, int NW, int NS, int LD, int EP, int FL, int EL, class Real>
__global__ void __launch_bounds__(32 * NW, (EP == EP_CG1 && R == 2) ? 2 : 0)
k_stencil(const __grid_constant__ StencilArgs a)
{
    using SH = StencilShape<R, NW, LD, Real, EL>;
    constexpr int KMAP = EL == EL_TETV ? MAP_KCN : MAP_KC;
    using V2 = typename Vec2<Real>::type;
    constexpr int ES = (int)sizeof(Real);
    constexpr int NT = 32 * NW;
    constexpr int NA = SH::NA;
    constexpr bool MASK = (FL & FL_MASK) != 0, DIR = (FL & FL_DIR) != 0;
    constexpr bool HB = (FL & FL_HB) != 0, DSET = (FL & FL_DSET) != 0;
    const Geom &g = a.g;
    Real *const out0 = reinterpret_cast<Real *>(a.out0);
    Real *const out_s = reinterpret_cast<Real *>(a.out_s);
    const Real *const bvec = reinterpret_cast<const Real *>(a.bvec);
    const Real *const invdv = reinterpret_cast<const Real *>(a.invd);
    // operator constants in the storage precision (compile-time selected)
    auto LKA = [&](int ch) -> Real { if constexpr (ES == 8) return a.lam.ka[ch]; else return a.lamf.ka[ch]; };
    auto LMA = [&](int ch) -> Real { if constexpr (ES == 8) return a.lam.ma[ch]; else return a.lamf.ma[ch]; };
    auto LKB = [&](int ch) -> Real { if constexpr (ES == 8) return a.lam.kb[ch]; else return a.lamf.kb[ch]; };
    auto LMB = [&](int ch) -> Real { if constexpr (ES == 8) return a.lam.mb[ch]; else return a.lamf.mb[ch]; };
    auto DK = [&](int i) -> Real { if constexpr (ES == 8) return a.dn.K[i]; else return a.dnf.K[i]; };
    auto DM = [&](int i) -> Real { if constexpr (ES == 8) return a.dn.M[i]; else return a.dnf.M[i]; };
    auto TK = [&](int t, int i) -> Real { if constexpr (ES == 8) return a.tv.K[t][i]; else return a.tvf.K[t][i]; };
    auto TMS = [&]() -> Real { if constexpr (ES == 8) return a.tv.m; else return a.tvf.m; };
    const int lane = threadIdx.x, w = threadIdx.y;
    const int tid = lane + 32 * w;
    const int blk = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblocks = gridDim.x * gridDim.y * gridDim.z;
    // stacked systems (a13): blockIdx.z = system * chunks-per-system + chunk, so the blocks of
    // system sj are contiguous (its partial sums too) and each z-chunk stays inside its system
    const int nsys = a.sy.nsys > 0 ? a.sy.nsys : 1;
    const int nchs = (int)gridDim.z / nsys;
    const int sj = (int)blockIdx.z / nchs;
    const int bps = nblocks / nsys;                        // blocks (partials) per system
    const bool sys_lead = blk == sj * bps && tid == 0;     // writes the system's scalars
    const bool glob_lead = blk == 0 && tid == 0;           // writes the shared loop fields
    if (blk == 0 && tid == 0 && a.sy.launches) atomicAdd(a.sy.launches, 1ull);
    // warm the SM's descriptor cache for every map this launch may use (which node maps it
    // uses depends on the state header, read next): one prefetch per lane of warp 0
    // (only descriptors that exist: kcn for EL_TETV, the ghost map on the peer transport)
    constexpr bool PEER = (FL & FL_PEER) != 0;
    if (w == 0 && (lane < NMAPS + 1 || (lane == MAP_KCN && EL == EL_TETV) || (lane == MAP_GHOST && PEER)))
        prefetch_map(a.tm + lane);
    HF_TR(0);
#ifdef HF_TRACE
    if (EP == EP_CGA && tid == 0 && blk < 4096) {
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        g_trace[blk][7] = sm;
    }
#endif

    extern __shared__ __align__(128) double smem_d[];
    Real *stage = reinterpret_cast<Real *>(smem_d);
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage + NS * SH::STAGE_DBL);
    if constexpr (EP == EP_CGA || EP == EP_CG1) {
        // independent of the previous kernel: may overlap its tail under a programmatic edge
        if (tid == 0) {
            for (int i = 0; i < NS; i++) mbar_init(&bars[i], 1);
            fence_mbar_init();
        }
        pdl_wait();
    }
    // kernel A with a fixed partial count (one system, no peer transport): the previous kernel's
    // partials are requested before the state header
    const bool pre_ok = EP == EP_CGA && !PEER && nsys == 1 && a.sy.pin_n > 0;
    PrevPre pre;
    if (pre_ok) prev_load<NT>(a.sy.pin, a.sy.pin_n, tid, pre);

    // ---- state checks and per-launch resolution of buffers ---------------------------------
    double beta = 0.0, delta_i = 0.0;
    int re_ = 0, step_ = 0;                                  // FL_FUSEB: header values for B
    int map0 = MAP_U0, map1 = MAP_U0 + 2, first = a.first;
    int it_i = 0;                                            // PCG iteration (kernel A)
    Real *cstore = reinterpret_cast<Real *>((EP == EP_CGA) ? a.dbuf[1] : a.xout);   // centre-value store target
    int npart_b = 0, max_iter = 0;
    CgState *const sst = a.sy.st ? a.sy.st + sj : nullptr;   // this block's system
    if (a.sy.st) {
        const CgHdr hd = load_hdr(a.sy.st);
        const CgHdr hs = sj ? load_hdr(sst) : hd;
        const int first_failed = hs.h0.x, active = hs.h0.y, b_iter = hd.h0.z, step = hd.h0.w;
        npart_b = hd.h1.w;
        max_iter = hd.h2.y;
        re_ = hd.h1.y;
        step_ = hd.h0.w;
        if (EP == EP_CG1) it_i = a.c1.par ? hd.h1.x : b_iter;   // iteration counter slot of this parity
        if (glob_lead) {
            // shared loop fields, written before any early exit (no block of this kernel reads them)
            CgState *st0 = a.sy.st;
            if (EP == EP_CGA) { st0->npart_a = bps; st0->a_iter = b_iter; }
            else if (EP == EP_RESID_INIT) { st0->npart_b = bps; st0->b_iter = 0; st0->replace = 0; }
            else if (EP == EP_RESID && hd.h1.z) st0->npart_b = bps;
        }
        if (first_failed >= 0) {                 // an earlier time step of this system failed
            if ((EP == EP_CGA || EP == EP_CG1) && nsys == 1 && sys_lead) { set_while(a.sy, 0); set_if(a.sy, 0); }
            return;
        }
        if (EP == EP_CGA || EP == EP_RESID || EP == EP_CG1 || EP == EP_CG1W) {
            if (!active) return;                 // converged / stopped: nothing to do
            if (EP == EP_RESID && !hd.h1.z) return;
        }
        if (LD == LD_CGD) {
            // d_i = s_i + beta_i d_{i-1};  d_{i-1} = dbuf[i & 1], d_i = dbuf[(i & 1) ^ 1]
            it_i = b_iter;
            const int par = it_i & 1;
            map0 = MAP_S;
            map1 = MAP_D0 + par;
            cstore = reinterpret_cast<Real *>(a.dbuf[par ^ 1]);
        }
        if (a.rot_role != ROT_NONE) {
            // time-step ring: step n reads U[n%3] (u^n), U[(n+2)%3] (u^{n-1}), writes U[(n+1)%3]
            const int s = step % 3;
            if (a.rot_role == ROT_RHS) map0 = MAP_U0 + s;
            else if (a.rot_role == ROT_INIT) {
                map0 = MAP_U0 + s;
                map1 = MAP_U0 + (s + 2) % 3;
                cstore = reinterpret_cast<Real *>(a.ring[(s + 1) % 3]);
                first = a.first && step == 0;
            } else map0 = MAP_U0 + (s + 1) % 3;
        }
    }
    if (LD == LD_X0 && first) map1 = map0;       // u^{-1} unused: keep the byte count fixed
    HF_TR(1);

    Real(*seam)[NW][32] = reinterpret_cast<Real(*)[NW][32]>(stage + NS * SH::STAGE_DBL + (16 / ES) * NS);
    // EL_Q1P: per material the (a, b) coefficients of the fused z butterfly, as the pair path
    // computes them from (k, c) (bit-identical): palt[m] = {a0, b0, a1, b1, a2, b2, a3, b3}
    double(*palt)[8] = reinterpret_cast<double(*)[8]>(seam + 2);
    Real *const ubuf = reinterpret_cast<Real *>(reinterpret_cast<char *>(palt) + SH::PAL_BYTES);   // LD_CG1

    const int X0 = blockIdx.x * TILE_X;
    const int Y0 = blockIdx.y * (NW * R - 1);
    const int xi = X0 - 1 + lane;
    // TMA box x origin must be 16-B aligned (even for fp64, a multiple of 4 for fp32): the box
    // starts at column xb <= X0-1 and lane l reads box column l + xoff (the box is SH::BW wide);
    // the (k, c) box likewise starts at kb <= 2 (X0-1) and lane l reads value 2 l + koff
    const int xb = (X0 - 1) & ~(16 / ES - 1);
    const int xoff = (X0 - 1) - xb;
    const int kb = (2 * (X0 - 1)) & ~(16 / ES - 1);
    const int koff = 2 * (X0 - 1) - kb;
    const int yb = Y0 - 1 + w * R;
    const int zsb = a.z_out0 + sj * a.zper_out;                  // output planes of this system
    const int zb = zsb + ((int)blockIdx.z - sj * nchs) * a.zchunk;
    const int ze = min(min(zb + a.zchunk, zsb + a.zper_out), a.z_out1);
    const int nplanes = ze - zb + 2;               // planes zb-1 .. ze
    // rows this thread owns (writes): lane >= 1, inside the grid, not the tile's halo row
    unsigned own = 0;
#pragma unroll
    for (int e = 0; e < R; e++)
        if (lane >= 1 && xi < g.nx1 && (w > 0 || e > 0) && yb + e < g.ny1) own |= 1u << e;
    const long long rowbase = (long long)yb * g.pitch + xi;   // node (xi, yb) within a plane

    auto issue = [&](int it) {                     // TMA of plane zb-1+it into its stage
        const int st = it % NS;
        const int p = zb - 1 + it;
        Real *sb = stage + st * SH::STAGE_DBL;
        mbar_expect_tx(&bars[st], SH::STAGE_BYTES);
        if (LD == LD_CG1 || LD == LD_CG1W) {   // single-reduction PCG: node maps 0 .. NA-1
#pragma unroll
            for (int k = 0; k < NA; k++) tma_load_3d(sb + k * SH::NODE_DBL, a.tm + k, xb, Y0 - 1, p, &bars[st]);
        } else if (LD == LD_CGD && PEER && (p == a.gz_lo || p == a.gz_hi))   // s of a neighbour's plane
            tma_load_3d(sb, a.tm + MAP_GHOST, xb, Y0 - 1, p == a.gz_lo ? 0 : 1, &bars[st]);
        else if (NA >= 1) tma_load_3d(sb, a.tm + map0, xb, Y0 - 1, p, &bars[st]);
        if (NA >= 2 && LD != LD_CG1 && LD != LD_CG1W) tma_load_3d(sb + SH::NODE_DBL, a.tm + map1, xb, Y0 - 1, p, &bars[st]);
        if (EL == EL_TETV)   // per-node (k, c) pairs of plane p, same rows as the node box
            tma_load_3d(sb + NA * SH::NODE_DBL, a.tm + MAP_KCN, 2 * xb, Y0 - 1, p, &bars[st]);
        else if (EL == EL_Q1P)   // material ids of element layer p - 1 (16-B aligned x origin)
            tma_load_3d(sb + NA * SH::NODE_DBL, a.tm + MAP_KC, (X0 - 1) & ~15, Y0 - 1, p, &bars[st]);
        else                 // element layer L = p - 1 sits at z = p in the kc tensor
            tma_load_3d(sb + NA * SH::NODE_DBL, a.tm + MAP_KC, kb, Y0 - 1, p, &bars[st]);
    };

    if (tid == 0) {
        if (smem_u32(stage) & 127u) __trap();     // TMA destinations need 128-B alignment
        if (EP != EP_CGA && EP != EP_CG1) {       // (kernel A initialised them before its wait)
            for (int i = 0; i < NS; i++) mbar_init(&bars[i], 1);
            fence_mbar_init();
        }
        if (a.tm_fence) {
            if (LD == LD_CG1 || LD == LD_CG1W) for (int k = 0; k < NA; k++) tensormap_acquire(a.tm + k);
            else if (NA >= 1) tensormap_acquire(a.tm + map0);
            if (NA >= 2 && LD != LD_CG1 && LD != LD_CG1W) tensormap_acquire(a.tm + map1);
            tensormap_acquire(a.tm + KMAP);
        }
    }
    __syncthreads();
    // slab over peer memory: a CTA whose planes include a ghost plane of s waits for the
    // neighbours' data (and every rank's sums) before its first TMA; the others wait after
    const PeerSync *const pp = PEER ? a.sy.peer : nullptr;
    double ps_peer[NPART];
    const bool peer_early = EP == EP_CGA && pp && ((a.gz_lo >= zb - 1 && a.gz_lo <= ze) || (a.gz_hi >= zb - 1 && a.gz_hi <= ze));
    if (peer_early) peer_sums<NT>(pp, ps_peer);
    if (tid == 0)
        for (int i = 0; i < NS && i < nplanes; i++) issue(i);
    HF_TR(2);
    if constexpr (EL == EL_Q1P) {
        // the material table, built while the first TMA loads are in flight (entries in use only)
        for (int i = tid; i < a.npal * 4; i += NT) {
            const int m = i >> 2, ch = i & 3;
            const double kk = a.pal[m][0], cc = a.pal[m][1];
            palt[m][2 * ch] = fma(kk, a.lam.ka[ch], cc * a.lam.ma[ch]);
            palt[m][2 * ch + 1] = fma(kk, a.lam.kb[ch], cc * a.lam.mb[ch]);
        }
        __syncthreads();
    }

    double alpha1 = 0.0, bb_fwd = 0.0;      // EP_CG1: alpha_i; EP_CG1W: ||b_F||^2 forwarded by block 0
    if (EP == EP_CG1) {
        // start of iteration i of the single-reduction PCG from the previous kernel's sums
        double ps[NPART];
        prev_sums<NT>(a.sy, npart_b, ps, sj);
        const IterStart1 is = iter_start_cg1(sst, it_i, ps, max_iter);
        if (sys_lead) {
            CgState *stw = sst;
            stw->rr = is.rr;
            if (it_i == 0) { stw->bb = is.bb; stw->thresh = is.thresh; }
            stw->delta[it_i & 1] = is.gamma;
            stw->alf[it_i & 1] = is.alpha;
            if (!is.go) {
                stw->active = 0;
                stw->status = is.status;
                stw->zero_x = is.zero_x;
                stw->iter = it_i;
                set_while(a.sy, 0);
                set_if(a.sy, 0);
            } else {
                // loop duties: the next iteration's counter (the other parity's slot) and the
                // residual replacement after this iteration (Alg. 1 line 10, R6)
                const bool replace = it_i > 0 && re_ > 0 && (it_i % re_) == 0;
                if (a.c1.par) stw->b_iter = it_i + 1;
                else stw->a_iter = it_i + 1;
                stw->replace = replace;
                set_if(a.sy, replace ? 1 : 0);
            }
        }
        if (!is.go) {
            for (int i = 0; i < NS && i < nplanes; i++) mbar_wait(&bars[i], 0);   // drain the TMA
            return;
        }
        beta = is.beta;
        alpha1 = is.alpha;
    }
    if (EP == EP_CG1W && blk == 0) {
        // ||b_F||^2 of the init kernel (slot 2 of its sums) rides along in block 0's partial
        double ps[NPART];
        prev_sums<NT>(a.sy, npart_b, ps, sj);
        bb_fwd = ps[2];
    }
    if (EP == EP_CGA) {
        // start of PCG iteration i from the previous kernel's partial sums (overlaps the TMA)
        double ps[NPART];
        if (peer_early) for (int j = 0; j < NPART; j++) ps[j] = ps_peer[j];
        else if (pp) peer_sums<NT>(pp, ps);
        else {
            const int n = pre_ok ? a.sy.pin_n : (a.sy.pin_n >= 0 ? a.sy.pin_n : npart_b);
            const double *pin = a.sy.pin + (long long)sj * n * NPART;
            if (!pre_ok) prev_load<NT>(pin, n, tid, pre);
            prev_finish<NT>(pre, pin, n, ps);
        }
        const IterStart is = iter_start(sst, it_i, ps, max_iter);
        if (!is.go) {
            if (sys_lead) {
                CgState *stw = sst;
                stw->active = 0;
                stw->status = is.status;
                stw->zero_x = is.zero_x;
                stw->iter = it_i;
                stw->rr = is.rr;
                if (it_i == 0) { stw->bb = is.bb; stw->thresh = is.thresh; }
                stw->delta[it_i & 1] = is.delta;
                if (nsys == 1) {                 // one system: its stop ends the loop here
                    set_while(a.sy, 0);
                    set_if(a.sy, 0);
                }
            }
#ifdef HF_DEBUG_WAIT
            for (int i = 0; i < NS && i < nplanes; i++) mbar_wait_dbg(&bars[i], 0, 1000 + EP * 10 + LD, -1 - i);
#else
            for (int i = 0; i < NS && i < nplanes; i++) mbar_wait(&bars[i], 0);   // drain the TMA
#endif
            return;
        }
        beta = is.beta;
        delta_i = is.delta;
        HF_TR(3);
#ifdef HF_DEBUG_WAIT
        if (blk == 0 && tid == 0 && g_dbg) {
            volatile unsigned long long *d = g_dbg;
            const int sl = ((uintptr_t)a.sy.st >> 8) & 1;
            d[10 + 3 * sl] = it_i;
            d[11 + 3 * sl] = a.sy.st->step;
            d[12 + 3 * sl] += 1;
        }
#endif
        if (sys_lead) {
            CgState *stw = sst;
            stw->delta[it_i & 1] = is.delta;
            stw->rr = is.rr;
            if (it_i == 0) { stw->bb = is.bb; stw->thresh = is.thresh; }
        }
    }

    const Real betar = (Real)beta;
    const Real alphar = (Real)alpha1;
    const bool first_it = it_i == 0;
    // planes whose owned nodes this CTA updates / stores (each plane of the run belongs to one chunk)
    auto own_plane = [&](int pl) -> bool {
        return (pl >= a.zs0 && pl < a.zs1) &&
               ((pl >= zb && pl < ze) || (pl == zb - 1 && zb == a.z_out0) || (pl == ze && ze == a.z_out1));
    };
    // LD_CG1 pre-pass: the CTA's threads form u_{i+1} once per box node (rows 0..NW R, columns
    // xoff .. xoff + TILE_X + 1) into the shared u plane; thread t takes the owned nodes
    // n = t + k NT (k < KOWN) of the tile (box rows 1..NW R - 1, columns xoff+1 .. xoff+TILE_X) and
    // t < NHALO one halo node.  p_{i-1} and x_i of its owned nodes are prefetched one plane ahead.
    constexpr int OWNR = NW * R - 1, NOWN = TILE_X * OWNR, KOWN = (NOWN + NT - 1) / NT;
    constexpr int NHALO = 2 * (TILE_X + 2) + 2 * OWNR;
    static_assert(LD != LD_CG1 || NHALO <= NT, "halo pass: one node per thread");
    Real *const c1x = EP == EP_CG1 ? reinterpret_cast<Real *>(a.c1.x ? a.c1.x : a.ring[(step_ + 1) % 3]) : nullptr;
    Real *const c1p = reinterpret_cast<Real *>(a.c1.p);
    int c1o[KOWN], c1h = 0;
    long long c1g[KOWN];
    unsigned c1own = 0;
    Real pfp[KOWN], pfx[KOWN];
    if constexpr (LD == LD_CG1) {
        constexpr int BW = SH::BW;
#pragma unroll
        for (int k = 0; k < KOWN; k++) {
            const int n = tid + k * NT;
            const int row = 1 + n / TILE_X, col = 1 + n % TILE_X;
            const int x = X0 - 1 + col, y = Y0 - 1 + row;
            c1o[k] = n < NOWN ? row * BW + xoff + col : -1;
            c1g[k] = (long long)y * g.pitch + x;
            if (n < NOWN && x < g.nx1 && y < g.ny1) c1own |= 1u << k;
        }
        int hr, hc;
        const int t = tid;
        if (t < TILE_X + 2) { hr = 0; hc = t; }
        else if (t < 2 * (TILE_X + 2)) { hr = NW * R; hc = t - (TILE_X + 2); }
        else if (t < 2 * (TILE_X + 2) + OWNR) { hr = 1 + t - 2 * (TILE_X + 2); hc = 0; }
        else { hr = 1 + t - 2 * (TILE_X + 2) - OWNR; hc = TILE_X + 1; }
        c1h = hr * BW + xoff + hc;
    }
    auto c1_prefetch = [&](int pl) {
        if (EP == EP_CG1 && own_plane(pl)) {
            const long long b0 = (long long)pl * g.plane;
#pragma unroll
            for (int k = 0; k < KOWN; k++)
                if ((c1own >> k) & 1u) {
                    pfx[k] = c1x[b0 + c1g[k]];
                    if (!first_it) pfp[k] = c1p[b0 + c1g[k]];
                }
        }
    };
    Real Fp[R][4];            // Q1: face transforms of the lower plane p-1
    Real Cy[R][4];            // contributions carried from the layer below (face / node space)
    float2 Fp2[R][2], Cy2[R][2];  // fp32 Q1: the same per channel pair (0,2), (1,3), packed math
    Real Pv[R + 1], Pv1[R + 1];   // dense: node values of plane p-1 at x and x+1
    V2 PK0[R + 1], PK1[R + 1];    // EL_TETV: node (k, c) pairs of plane p-1 at x and x+1
    Real cen[R];              // raw centre values of plane p-1 (rows 0..R-1)
    double acc[NPART] = {0.0, 0.0, 0.0, 0.0};
    if (EP == EP_CG1W && blk == 0 && tid == 0) acc[2] = bb_fwd;
    bool remote = false;                     // this thread stored into a neighbour's memory
    c1_prefetch(zb - 1);
#pragma unroll
    for (int r = 0; r < R; r++) {
#pragma unroll
        for (int ch = 0; ch < 4; ch++) { Fp[r][ch] = Real(0); Cy[r][ch] = Real(0); }
        for (int q = 0; q < 2; q++) { Fp2[r][q] = make_float2(0.f, 0.f); Cy2[r][q] = make_float2(0.f, 0.f); }
        cen[r] = Real(0);
    }
#pragma unroll
    for (int r = 0; r <= R; r++) {
        Pv[r] = Real(0);
        Pv1[r] = Real(0);
        PK0[r].x = PK0[r].y = PK1[r].x = PK1[r].y = Real(0);
    }

    // Q1 kernels without the peer protocol, at R = 2 (< 16M nodes, latency-bound) and PCG kernel
    // A at R = 4 (512^3: 2.512 vs 2.550 ms per PCG iteration): the tet and slab variants would
    // spill, and the unrolled R = 4 apply ran 9 % slower (0.805 vs 0.739 ms; with material ids
    // 0.780 vs 0.613)
    constexpr int PU = ((R == 2 || EP == EP_CGA) && (EL == EL_Q1 || EL == EL_Q1P) && !PEER) ? kPlaneUnroll : 1;
#pragma unroll PU
    for (int it = 0; it < nplanes; ++it) {
        const int p = zb - 1 + it;
        const int st = it % NS;
#ifdef HF_DEBUG_WAIT
        mbar_wait_dbg(&bars[st], (it / NS) & 1, EP * 10 + LD, it);
#else
        mbar_wait(&bars[st], (it / NS) & 1);
#endif
        if (it == 0) HF_TR(4);
        const Real *sb = stage + st * SH::STAGE_DBL;
        if constexpr (LD == LD_CG1) {
            // ---- pre-pass: s_i = w_i + beta s_{i-1}; r_{i+1} = r_i - alpha s_i; u_{i+1} = P^{-1} r_{i+1}
            const Real *sr = sb, *sw = sb + SH::NODE_DBL, *ss = sb + 2 * SH::NODE_DBL, *si = sb + 3 * SH::NODE_DBL;
            const bool ownp = own_plane(p);
            const long long pb = (long long)p * g.plane;
            Real *const sout = reinterpret_cast<Real *>(a.c1.sout);
            Real *const rout = reinterpret_cast<Real *>(a.c1.rout);
#pragma unroll
            for (int k = 0; k < KOWN; k++) {
                const int o = c1o[k];
                if (o < 0) continue;
                const Real rv = sr[o], wv = sw[o], sv = ss[o], iv = si[o];
                const Real sn = first_it ? wv : fma(betar, sv, wv);
                const Real rn = fma(-alphar, sn, rv);
                const Real u = iv * rn;
                ubuf[o] = u;
                if (ownp && ((c1own >> k) & 1u)) {
                    // owned node: s_i, r_{i+1}; p_i = u_i + beta p_{i-1}; x_{i+1} = x_i + alpha p_i
                    const long long idx = pb + c1g[k];
                    sout[idx] = sn;
                    rout[idx] = rn;
                    const Real uo = iv * rv;
                    const Real pn = first_it ? uo : fma(betar, pfp[k], uo);
                    c1p[idx] = pn;
                    c1x[idx] = fma(alphar, pn, pfx[k]);
                    acc[0] = fma((double)rn, (double)u, acc[0]);
                    acc[1] = fma((double)rn, (double)rn, acc[1]);
                }
            }
            if (tid < NHALO) {
                const int o = c1h;
                const Real sn = first_it ? sw[o] : fma(betar, ss[o], sw[o]);
                ubuf[o] = si[o] * fma(-alphar, sn, sr[o]);
            }
            c1_prefetch(p + 1);
            __syncthreads();                            // u plane complete ((k, c) still read below)
        }
        const Real *n0 = (LD == LD_CG1 ? ubuf : sb) + w * R * SH::BW + lane + xoff;   // row 0 of this warp
        const Real *n1 = sb + SH::NODE_DBL + w * R * SH::BW + lane + xoff;
        const Real *kcs = sb + NA * SH::NODE_DBL + w * R * SH::KW + koff + 2 * lane;
        const unsigned char *kis = reinterpret_cast<const unsigned char *>(sb + NA * SH::NODE_DBL) + w * R * PAL_BW +
                                   ((X0 - 1) - ((X0 - 1) & ~15)) + lane;                      // EL_Q1P
        const Real *kns = sb + NA * SH::NODE_DBL + w * R * (2 * SH::BW) + 2 * (lane + xoff);   // EL_TETV
        // ---- node values of plane p (rows 0..R), x butterfly (edges) ----------------------
        Real S[R + 1], D[R + 1], V0[R + 1], V1[R + 1], craw[R];
        // EL_Q1P: the element layer's (a, b) coefficients are looked up first (id, then table),
        // so the two dependent shared-memory round trips overlap the node loads and butterflies
        double2 pabr[EL == EL_Q1P ? R : 1][4];
        if constexpr (EL == EL_Q1P) {
            int idr[R];
#pragma unroll
            for (int r = 0; r < R; r++) idr[r] = kis[r * PAL_BW];
#pragma unroll
            for (int r = 0; r < R; r++) {
                const double2 *pe = reinterpret_cast<const double2 *>(palt[idr[r]]);
#pragma unroll
                for (int ch = 0; ch < 4; ch++) pabr[r][ch] = pe[ch];
            }
        }
        const bool store_p = (EP == EP_CGA || EP == EP_RESID_INIT || EP == EP_CG1 || EP == EP_CG1W) && own_plane(p);
        Real *cst = store_p ? cstore + (long long)p * g.plane + rowbase : nullptr;
#pragma unroll
        for (int r = 0; r <= R; r++) {
            Real v, v1;
            constexpr int BW = SH::BW;
            if (LD == LD_RAW || LD == LD_CG1) { v = n0[r * BW]; v1 = n0[r * BW + 1]; }
            else if (LD == LD_CGD) {
                v = fma(betar, n1[r * BW], n0[r * BW]);
                v1 = fma(betar, n1[r * BW + 1], n0[r * BW + 1]);
            } else if (LD == LD_CG1W) {
                // u = P^{-1} r (map 0: r, map 1: P^{-1}); owned nodes: r^T u, r^T r
                const int o = r * BW;
                const Real r0v = n0[o];
                v = n1[o] * r0v;
                v1 = n1[o + 1] * n0[o + 1];
                if (r < R && store_p && ((own >> r) & 1u)) {
                    acc[0] = fma((double)r0v, (double)v, acc[0]);
                    acc[1] = fma((double)r0v, (double)r0v, acc[1]);
                }
            } else if (LD == LD_X0) {
                v = n0[r * BW];
                v1 = n0[r * BW + 1];
                if (!first) { v = Real(2) * v - n1[r * BW]; v1 = Real(2) * v1 - n1[r * BW + 1]; }
            } else {   // LD_GT: the Dirichlet lift g~ (g on D nodes, 0 elsewhere)
                double gv = 0.0;
                const int yi = yb + r;
                const bool in = xi >= 0 && xi < g.nx1 && yi >= 0 && yi < g.ny1 && p >= 0 && p < g.nzl;
                v = (in && is_dirichlet(g, xi, yi, p, gv)) ? (Real)gv : Real(0);
                gv = 0.0;
                const bool in1 = xi + 1 < g.nx1 && yi >= 0 && yi < g.ny1 && p >= 0 && p < g.nzl;
                v1 = (in1 && is_dirichlet(g, xi + 1, yi, p, gv)) ? (Real)gv : Real(0);
            }
            if (r < R) {
                craw[r] = v;
                // d_new (CG kernel A) or the guess x0 (init) is stored once, raw, by its owner
                if ((EP == EP_CGA || EP == EP_RESID_INIT) && store_p && ((own >> r) & 1u)) cst[r * g.pitch] = v;
            }
            if (MASK) {
                double gv;
                const int yi = yb + r;
                if (is_dirichlet(g, xi, yi, p, gv)) v = Real(0);
                if (is_dirichlet(g, xi + 1, yi, p, gv)) v1 = Real(0);
            }
            S[r] = v + v1;
            D[r] = v - v1;
            V0[r] = v;
            V1[r] = v1;
        }
        const int pout = p - 1;
        const bool out_plane = pout >= zb && pout < ze;   // uniform across the CTA
        Real yv[R + 1];
        if (EL == EL_Q1 || EL == EL_Q1P) {
            // ---- element layer p-1: y butterfly, fused z butterfly + scaling -------------------
            // (lane 31's element X0+30 reads node X0+31 from the box; elements outside the domain
            //  have k = c = 0 from the TMA zero fill)
            if constexpr (ES == 4) {
                // fp32: the same algebra on channel pairs (0,2) and (1,3) with Blackwell's packed
                // FP32x2 instructions (FFMA2 / FMUL2 / FADD2), half the FP instruction count
                const float2 M1 = make_float2(-1.f, -1.f);
                const float2 LKA[2] = {make_float2(a.lamf.ka[0], a.lamf.ka[2]), make_float2(a.lamf.ka[1], a.lamf.ka[3])};
                const float2 LMA[2] = {make_float2(a.lamf.ma[0], a.lamf.ma[2]), make_float2(a.lamf.ma[1], a.lamf.ma[3])};
                const float2 LKB[2] = {make_float2(a.lamf.kb[0], a.lamf.kb[2]), make_float2(a.lamf.kb[1], a.lamf.kb[3])};
                const float2 LMB[2] = {make_float2(a.lamf.mb[0], a.lamf.mb[2]), make_float2(a.lamf.mb[1], a.lamf.mb[3])};
                float2 T2[R][2];
#pragma unroll
                for (int r = 0; r < R; r++) {
                    const float2 sd0 = make_float2(S[r], D[r]), sd1 = make_float2(S[r + 1], D[r + 1]);
                    const float2 Fc2[2] = {__fadd2_rn(sd0, sd1), __ffma2_rn(sd1, M1, sd0)};   // (0,2), (1,3)
                    const V2 kc = *reinterpret_cast<const V2 *>(kcs + r * SH::KW);
                    const float2 k2 = make_float2(kc.x, kc.x), c2 = make_float2(kc.y, kc.y);
#pragma unroll
                    for (int q = 0; q < 2; q++) {
                        const float2 av = __ffma2_rn(k2, LKA[q], __fmul2_rn(c2, LMA[q]));
                        const float2 bv = __ffma2_rn(k2, LKB[q], __fmul2_rn(c2, LMB[q]));
                        T2[r][q] = __ffma2_rn(av, Fp2[r][q], __ffma2_rn(bv, Fc2[q], Cy2[r][q]));
                        Cy2[r][q] = __ffma2_rn(bv, Fp2[r][q], __fmul2_rn(av, Fc2[q]));
                        Fp2[r][q] = Fc2[q];
                    }
                }
#pragma unroll
                for (int e = 0; e <= R; e++) {
                    float2 E;                                   // (E0, E1): channel sums (0+1, 2+3)
                    if (e == 0) E = __fadd2_rn(T2[0][0], T2[0][1]);
                    else if (e == R) E = __ffma2_rn(T2[R - 1][1], M1, T2[R - 1][0]);
                    else E = __fadd2_rn(__fadd2_rn(T2[e][0], T2[e][1]), __ffma2_rn(T2[e - 1][1], M1, T2[e - 1][0]));
                    const Real left = __shfl_up_sync(0xffffffffu, E.x - E.y, 1);
                    yv[e] = (E.x + E.y) + left;                 // lane 0's value is not owned
                }
            } else {
            Real T[R][4];
#pragma unroll
            for (int r = 0; r < R; r++) {
                Real Fc[4];
                Fc[0] = S[r] + S[r + 1];   // sx=0, sy=0
                Fc[1] = S[r] - S[r + 1];   // sx=0, sy=1
                Fc[2] = D[r] + D[r + 1];   // sx=1, sy=0
                Fc[3] = D[r] - D[r + 1];   // sx=1, sy=1
                V2 kc;
                if constexpr (EL != EL_Q1P) kc = *reinterpret_cast<const V2 *>(kcs + r * SH::KW);
#pragma unroll
                for (int ch = 0; ch < 4; ch++) {
                    Real av, bv;
                    if constexpr (EL == EL_Q1P) { av = pabr[r][ch].x; bv = pabr[r][ch].y; }
                    else {
                        av = fma(kc.x, LKA(ch), kc.y * LMA(ch));
                        bv = fma(kc.x, LKB(ch), kc.y * LMB(ch));
                    }
                    T[r][ch] = fma(av, Fp[r][ch], fma(bv, Fc[ch], Cy[r][ch]));   // bottom plane p-1
                    Cy[r][ch] = fma(bv, Fp[r][ch], av * Fc[ch]);                  // top plane p
                    Fp[r][ch] = Fc[ch];
                }
            }
            // ---- backward y and x butterflies for plane p-1 ------------------------------------
#pragma unroll
            for (int e = 0; e <= R; e++) {
                Real E0, E1;                                // sx = 0, 1
                if (e == 0) { E0 = T[0][0] + T[0][1]; E1 = T[0][2] + T[0][3]; }
                else if (e == R) { E0 = T[R - 1][0] - T[R - 1][1]; E1 = T[R - 1][2] - T[R - 1][3]; }
                else {
                    E0 = (T[e][0] + T[e][1]) + (T[e - 1][0] - T[e - 1][1]);
                    E1 = (T[e][2] + T[e][3]) + (T[e - 1][2] - T[e - 1][3]);
                }
                const Real left = __shfl_up_sync(0xffffffffu, E0 - E1, 1);
                yv[e] = (E0 + E1) + left;                   // lane 0's value is not owned
            }
            }
        } else {
            // ---- 6-tet split: u_e = 4 values of plane p-1 + 4 of p ----------------------------
            Real B4[R][4];
            V2 KN0[R + 1], KN1[R + 1];             // EL_TETV: node pairs of plane p at x, x+1
            if constexpr (EL == EL_TETV) {
#pragma unroll
                for (int r = 0; r <= R; r++) {
                    KN0[r] = *reinterpret_cast<const V2 *>(kns + r * 2 * SH::BW);
                    KN1[r] = *reinterpret_cast<const V2 *>(kns + r * 2 * SH::BW + 2);
                }
            }
#pragma unroll
            for (int r = 0; r < R; r++) {
                const Real ue[8] = {Pv[r], Pv1[r], Pv[r + 1], Pv1[r + 1], V0[r], V1[r], V0[r + 1], V1[r + 1]};
                if constexpr (EL == EL_DENSE) {
                    // one (k, c) per voxel: dense 8x8 voxel matrices
                    const V2 kc = *reinterpret_cast<const V2 *>(kcs + r * SH::KW);
#pragma unroll
                    for (int i = 0; i < 8; i++) {
                        Real yk = Real(0), ym = Real(0);
#pragma unroll
                        for (int j = 0; j < 8; j++) {
                            yk = fma(DK(i * 8 + j), ue[j], yk);
                            ym = fma(DM(i * 8 + j), ue[j], ym);
                        }
                        const Real y = fma(kc.x, yk, kc.y * ym);
                        if (i < 4) B4[r][i] = Cy[r][i] + y;      // bottom plane p-1 complete
                        else Cy[r][i - 4] = y;                   // top plane p, carried
                    }
                } else {
                    // per-tet coefficients = means of the tet's 4 vertex values
                    const V2 ke[8] = {PK0[r], PK1[r], PK0[r + 1], PK1[r + 1], KN0[r], KN1[r], KN0[r + 1], KN1[r + 1]};
                    const int ey = yb + r, ez = p - 1 + g.zg0;
                    const bool vin = xi >= 0 && xi < g.nx && ey >= 0 && ey < g.ny && ez >= 0 && ez < g.nz1g - 1;
                    Real yl[8];
#pragma unroll
                    for (int i = 0; i < 8; i++) yl[i] = Real(0);
#pragma unroll
                    for (int t = 0; t < 6; t++) {
                        const int l0 = tet_loc(t, 0), l1 = tet_loc(t, 1), l2 = tet_loc(t, 2), l3 = tet_loc(t, 3);
                        const int lv[4] = {l0, l1, l2, l3};
                        // voxels outside the domain (halo lanes, phantom layers) would average
                        // boundary vertex values: their tets carry no coefficient
                        const Real kt = vin ? Real(0.25) * ((ke[l0].x + ke[l1].x) + (ke[l2].x + ke[l3].x)) : Real(0);
                        const Real cm = vin ? Real(0.25) * ((ke[l0].y + ke[l1].y) + (ke[l2].y + ke[l3].y)) * TMS() : Real(0);
                        const Real su = (ue[l0] + ue[l1]) + (ue[l2] + ue[l3]);
#pragma unroll
                        for (int i = 0; i < 4; i++) {
                            Real ku = Real(0);
#pragma unroll
                            for (int j = 0; j < 4; j++) ku = fma(TK(t, i * 4 + j), ue[lv[j]], ku);
                            yl[lv[i]] = fma(kt, ku, fma(cm, su + ue[lv[i]], yl[lv[i]]));
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        B4[r][i] = Cy[r][i] + yl[i];
                        Cy[r][i] = yl[i + 4];
                    }
                }
            }
            if constexpr (EL == EL_TETV) {
#pragma unroll
                for (int r = 0; r <= R; r++) { PK0[r] = KN0[r]; PK1[r] = KN1[r]; }
            }
#pragma unroll
            for (int r = 0; r <= R; r++) { Pv[r] = V0[r]; Pv1[r] = V1[r]; }
            // node (x, row e) of plane p-1 collects element rows e (by = 0) and e-1 (by = 1);
            // the bx = 1 parts belong to node x+1 (next lane)
#pragma unroll
            for (int e = 0; e <= R; e++) {
                Real X0v = Real(0), X1v = Real(0);
                if (e < R) { X0v += B4[e][0]; X1v += B4[e][1]; }
                if (e > 0) { X0v += B4[e - 1][2]; X1v += B4[e - 1][3]; }
                const Real left = __shfl_up_sync(0xffffffffu, X1v, 1);
                yv[e] = X0v + left;
            }
        }
        seam[it & 1][w][lane] = yv[R];
        __syncthreads();                                // seam visible; stage `st` fully read
        if (tid == 0 && it + NS < nplanes) {
            fence_proxy_async();
            issue(it + NS);
        }
        if (out_plane) {
            if (w > 0) yv[0] += seam[it & 1][w - 1][lane];
            const long long pofs = (long long)pout * g.plane + rowbase;
#pragma unroll
            for (int e = 0; e < R; e++) {
                if (!((own >> e) & 1u)) continue;
                const long long idx = pofs + e * g.pitch;
                double gv = 0.0;
                const bool isd = DIR && is_dirichlet(g, xi, yb + e, pout, gv);
                if (EP == EP_APPLY) {
                    Real y = (Real)a.c * yv[e];
                    if (DIR && !DSET && isd) y = cen[e];
                    if (HB) y = fma((Real)a.s, bvec[idx], y);
                    if (DIR && DSET && isd) y = (Real)gv;
                    out0[idx] = y;
                } else if (EP == EP_CG1 || EP == EP_CG1W) {
                    const Real u = cen[e];
                    const Real wv = isd ? u : yv[e];        // identity rows (R3)
                    reinterpret_cast<Real *>(a.c1.wout)[idx] = wv;
                    acc[3] = fma((double)u, (double)wv, acc[3]);
                } else if (EP == EP_CGA) {
                    const Real d = cen[e];
                    const Real q = isd ? d : yv[e];         // identity rows (R3)
                    out0[idx] = q;
                    acc[0] = fma((double)d, (double)q, acc[0]);
                } else {   // EP_RESID, EP_RESID_INIT: r = b - A x (identity rows on D); s = P^{-1} r
                    const Real b = __ldg(bvec + idx);
                    const Real r = isd ? Real(0) : b - yv[e];
                    const Real sv = r * __ldg(invdv + idx);
                    out0[idx] = r;
                    out_s[idx] = sv;
                    if (pp) remote |= peer_ghost<Real>(pp, idx, sv);
                    acc[0] = fma((double)r, (double)sv, acc[0]);
                    acc[1] = fma((double)r, (double)r, acc[1]);
                    if (EP == EP_RESID_INIT && !isd) acc[2] = fma((double)b, (double)b, acc[2]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; r++) cen[r] = craw[r];
    }

    if (EP == EP_APPLY) return;
    if (EP == EP_CGA || EP == EP_CG1) pdl_trigger();
    HF_TR(5);
    // per-block partial sums for the next kernel: A -> (d^T q); init, RESID -> (r^T s, r^T r, b^T b)
    block_reduce_store<NT>(acc, a.sy.pout, blk);
    if (nsys == 1) pad_partials<NT>(a.sy, nblocks, blk, tid);
    if (pp) peer_publish<NT>(pp, a.sy.pout, nblocks, remote);
    HF_TR(6);
    if (EP == EP_RESID_INIT && sys_lead) {      // a new solve of this system starts: A_0 follows
        CgState *stw = sst;
        stw->active = 1;
        stw->status = ST_OK;
        stw->zero_x = 0;
        stw->iter = 0;
    }
    if constexpr (EP == EP_CGA && (FL & FL_FUSEB) != 0) {
        // kernel B of the same iteration in the same launch: every CTA's q, d and d^T q partial
        // are in L2 after the barrier; each block reduces them (same order as kernel B) and
        // updates its contiguous share of the nodes
        grid_barrier(a.gbar, (unsigned)nblocks, tid);
        double ps[NPART];
        reduce_prev<NT, true>(a.sy.pout, nblocks, ps);
        cg_b_work<NT, Real, true>(a.fb, a.sy.st, true, 0, blk, nblocks, blk, tid, it_i, re_, step_, delta_i, ps[0],
                                  true);
    }
}


// Local sums of the last producer's partials (slab mode: before the cross-rank allreduce).
// which = 0: kernel A's partials, 1: init / B / RESID partials.
__global__ void __launch_bounds__(256) k_localsum(Sync sy, int which, double *sums)
{
    if (threadIdx.x == 0 && sy.launches) atomicAdd(sy.launches, 1ull);
    const CgState *st = sy.st;
    double s[NPART];
    reduce_prev<256>(sy.pin, which == 0 ? st->npart_a : st->npart_b, s);
    if (threadIdx.x < NPART) sums[threadIdx.x] = s[threadIdx.x];
}

// ---- element coefficient access (compact (nx, ny, nzl + 1) layout, layer L at index L + 1) --

template <class Real>
__device__ __forceinline__ typename Vec2<Real>::type load_kc(const Geom &g, const typename Vec2<Real>::type *kc, int ex,
                                                             int ey, int L)
{
    typename Vec2<Real>::type z;
    z.x = Real(0);
    z.y = Real(0);
    if (ex < 0 || ey < 0 || ex >= g.nx || ey >= g.ny || L < -1 || L >= g.nzl) return z;
    return kc[((long long)(L + 1) * g.ny + ey) * g.kpitch + ex];
}

// ---- Jacobi diagonal (Jacobi_A P:659-662) -------------------------------------------
// diag_i = sum over the 8 elements around node i of aK k_e Kd + aM c_e Md, with
// Kd = K_ref[l][l], Md = M_ref[l][l] (the same for every l of a voxel); 1 on Dirichlet rows.

struct DiagC {              // diagonal entries K_ref[l][l], M_ref[l][l] per local node l
    double Kd[8], Md[8];
};

template <class Real>
__global__ void k_diag(Geom g, const void *kcp, double aK, double aM, DiagC dc, void *diagp, void *invdp,
                       unsigned long long *launches)
{
    using V2 = typename Vec2<Real>::type;
    const V2 *kc = reinterpret_cast<const V2 *>(kcp);
    Real *diag = reinterpret_cast<Real *>(diagp), *invd = reinterpret_cast<Real *>(invdp);
    const long long n = g.plane * g.nzl;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= n) return;
    const int x = (int)(i % g.pitch), y = (int)((i / g.pitch) % g.ny1), z = (int)(i / g.plane);
    if (x >= g.nx1) { if (diag) diag[i] = Real(0); if (invd) invd[i] = Real(0); return; }   // pitch padding
    double sk = 0.0, sc = 0.0;
    for (int l = 0; l < 8; l++) {   // node is local node l of element (x - bx, y - by, z - bz)
        const V2 v = load_kc<Real>(g, kc, x - (l & 1), y - ((l >> 1) & 1), z - ((l >> 2) & 1));
        sk = fma((double)v.x, dc.Kd[l], sk);
        sc = fma((double)v.y, dc.Md[l], sc);
    }
    double d = aK * sk + aM * sc;
    double gv;
    if (is_dirichlet(g, x, y, z, gv)) d = 1.0;
    if (diag) diag[i] = (Real)d;
    if (invd) invd[i] = (Real)(1.0 / d);
}

// EL_TETV diagonal: diag_i = sum over the voxels and tets containing node i of
// aK k_t K_t[ii] + aM c_t 2m, k_t, c_t the means of the tet's 4 vertex pairs; 1 on
// Dirichlet rows.  kd[t][v]: unit-coefficient K_t diagonal (tet_loc order), md = 2 V_tet / 20.
struct TetDiag {
    double kd[6][4];
    double md;
};

template <class Real>
__global__ void k_diag_tv(Geom g, const void *kcnp, double aK, double aM, TetDiag td, void *diagp, void *invdp,
                          unsigned long long *launches)
{
    using V2 = typename Vec2<Real>::type;
    const V2 *kcn = reinterpret_cast<const V2 *>(kcnp);
    Real *diag = reinterpret_cast<Real *>(diagp), *invd = reinterpret_cast<Real *>(invdp);
    const long long n = g.plane * g.nzl;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= n) return;
    const int x = (int)(i % g.pitch), y = (int)((i / g.pitch) % g.ny1), z = (int)(i / g.plane);
    if (x >= g.nx1) { if (diag) diag[i] = Real(0); if (invd) invd[i] = Real(0); return; }
    double d = 0.0;
    for (int l = 0; l < 8; l++) {                  // node is local node l of voxel (x-bx, y-by, z-bz)
        const int vx = x - (l & 1), vy = y - ((l >> 1) & 1), vz = z - ((l >> 2) & 1);
        if (vx < 0 || vy < 0 || vx >= g.nx || vy >= g.ny) continue;
        const int zg = vz + g.zg0;
        if (zg < 0 || zg >= g.nz1g - 1 || vz < -1 || vz + 1 >= g.nzl + 1) continue;
        for (int t = 0; t < 6; t++) {
            int me = -1;
            for (int v = 0; v < 4; v++) if (tet_loc(t, v) == l) me = v;
            if (me < 0) continue;
            double kt = 0.0, ct = 0.0;
            for (int v = 0; v < 4; v++) {
                const int lv = tet_loc(t, v);
                const int nzp = vz + ((lv >> 2) & 1);
                if (nzp < 0 || nzp >= g.nzl) continue;   // (slab ghosts carry the pairs they need)
                const V2 p = kcn[(long long)nzp * g.plane + (long long)(vy + ((lv >> 1) & 1)) * g.pitch + vx + (lv & 1)];
                kt += (double)p.x;
                ct += (double)p.y;
            }
            d += aK * 0.25 * kt * td.kd[t][me] + aM * 0.25 * ct * td.md;
        }
    }
    double gv;
    if (is_dirichlet(g, x, y, z, gv)) d = 1.0;
    if (diag) diag[i] = (Real)d;
    if (invd) invd[i] = (Real)(1.0 / d);
}

// per-node (k, c) pairs in the padded node layout (EL_TETV), from global natural node arrays
template <class Real>
__global__ void k_pack_nodes(Geom g, const double *k, const double *c, void *kcnp, unsigned long long *launches)
{
    using V2 = typename Vec2<Real>::type;
    V2 *kcn = reinterpret_cast<V2 *>(kcnp);
    const long long n = g.plane * g.nzl;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= n) return;
    const int x = (int)(i % g.pitch), y = (int)((i / g.pitch) % g.ny1), z = (int)(i / g.plane);
    V2 v;
    v.x = Real(0);
    v.y = Real(0);
    if (x < g.nx1) {
        const long long gi = x + (long long)g.nx1 * (y + (long long)g.ny1 * (z + g.zg0));
        v.x = (Real)k[gi];
        v.y = (Real)c[gi];
    }
    kcn[i] = v;
}

// per-voxel means of the 8 corner values (Q1 with vertex materials)
__global__ void k_vertex_means(Geom g, int nz, const double *kn, const double *cn, double *ke, double *ce,
                               unsigned long long *launches)
{
    const long long ne = (long long)g.nx * g.ny * nz;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e == 0 && launches) atomicAdd(launches, 1ull);
    if (e >= ne) return;
    const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
    double sk = 0.0, sc = 0.0;
    for (int l = 0; l < 8; l++) {
        const long long n = (ex + (l & 1)) + (long long)g.nx1 * ((ey + ((l >> 1) & 1)) + (long long)g.ny1 * (ez + ((l >> 2) & 1)));
        sk += kn[n];
        sc += cn[n];
    }
    ke[e] = sk / 8.0;
    ce[e] = sc / 8.0;
}

// ---- packing of the per-element coefficients into the (k, c) pair layout ------------------
// pair (ex, ey, L) for local layer L in [-1, nzl-1] = global element (ex, ey, zg0 + L), or 0;
// rows of g.kpitch pairs (the pad pairs of an fp32 row stay 0).

template <class Real>
__global__ void k_pack(Geom g, int nz, const double *k, const double *c, void *kcp, long long ntot,
                       unsigned long long *launches)
{
    using V2 = typename Vec2<Real>::type;
    V2 *kc = reinterpret_cast<V2 *>(kcp);
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= ntot) return;
    const int ex = (int)(i % g.kpitch), ey = (int)((i / g.kpitch) % g.ny);
    const int L = (int)(i / ((long long)g.kpitch * g.ny)) - 1;
    const int ez = g.zg0 + L;
    V2 v;
    v.x = Real(0);
    v.y = Real(0);
    if (ex < g.nx && ez >= 0 && ez < nz) {
        const long long e = ex + (long long)g.nx * (ey + (long long)g.ny * ez);
        v.x = (Real)k[e];
        v.y = c ? (Real)c[e] : Real(0);
    }
    kc[i] = v;
}

// ---- materials by id (hf_set_material_ids) --------------------------------------------------
struct PalTab {
    double kc[PAL_MAX][2];  // (k, c) of material m (m < n_materials)
};

// (k, c) pairs from ids, in the k_pack layout (for the kernels that read pairs: diagonal,
// extraction, the other element variants); *bad = 1 if an id is out of range
template <class Real>
__global__ void k_pack_ids(Geom g, int nz, const unsigned char *ids, int nmat, PalTab pt, void *kcp, long long ntot,
                           int *bad, unsigned long long *launches)
{
    using V2 = typename Vec2<Real>::type;
    V2 *kc = reinterpret_cast<V2 *>(kcp);
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= ntot) return;
    const int ex = (int)(i % g.kpitch), ey = (int)((i / g.kpitch) % g.ny);
    const int L = (int)(i / ((long long)g.kpitch * g.ny)) - 1;
    const int ez = g.zg0 + L;
    V2 v;
    v.x = Real(0);
    v.y = Real(0);
    if (ex < g.nx && ez >= 0 && ez < nz) {
        const int m = ids[ex + (long long)g.nx * (ey + (long long)g.ny * ez)];
        if (m < nmat) {
            v.x = (Real)pt.kc[m][0];
            v.y = (Real)pt.kc[m][1];
        } else *bad = 1;
    }
    kc[i] = v;
}

// id + 1 per element in the (kp, ny, nzl + 1) layer layout (0 = outside the domain / padding)
__global__ void k_pack_kid(Geom g, int nz, const unsigned char *ids, int kp, unsigned char *kid, long long ntot,
                           unsigned long long *launches)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= ntot) return;
    const int ex = (int)(i % kp), ey = (int)((i / kp) % g.ny);
    const int L = (int)(i / ((long long)kp * g.ny)) - 1;
    const int ez = g.zg0 + L;
    unsigned char v = 0;
    if (ex < g.nx && ez >= 0 && ez < nz) v = (unsigned char)(ids[ex + (long long)g.nx * (ey + (long long)g.ny * ez)] + 1);
    kid[i] = v;
}

// ---- flux load F_i = int_face f phi_i ds (reading R12) ----------------------------
// one thread per node of the face plane; 2x2 Gauss points per adjacent boundary quad.

struct FaceArgs {
    Geom g;
    int face, nd, ax, bx;     // normal axis, in-plane axes (increasing order)
    int na, nb;               // nodes along ax, bx (global counts of that axis)
    int plane_g;              // global index of the face along the normal axis
    double ha, hb, oa, ob;    // spacing and origin of the in-plane axes
    double f_const;
    int has_beam;
    double bP, bs, bca, bcb;
    int tets;                 // 1: boundary quads are two P1 triangles (6-tet split, f1)
    double *F;
    unsigned long long *launches;
};

__device__ __forceinline__ double phi1(int b, double t, double h) { return b ? t / h : 1.0 - t / h; }

template <class Real>
__global__ void k_face_load(const FaceArgs a)
{
    Real *const F = reinterpret_cast<Real *>(a.F);
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && a.launches) atomicAdd(a.launches, 1ull);
    const long long nface = (long long)a.na * a.nb;
    if (i >= nface) return;
    const int ia = (int)(i % a.na), ib = (int)(i / a.na);
    int idx3[3];
    idx3[a.nd] = a.plane_g;
    idx3[a.ax] = ia;
    idx3[a.bx] = ib;
    const int zl = idx3[2] - a.g.zg0;                  // local plane (slab)
    if (zl < 0 || zl >= a.g.nzl) return;
    const double gp0 = 0.5 * (1.0 - 0.57735026918962576451), gp1 = 0.5 * (1.0 + 0.57735026918962576451);
    const double w = (a.ha * 0.5) * (a.hb * 0.5);
    double sum = 0.0;
    if (a.tets) {
        // quad (qa, qb) = triangles {(0,0),(1,0),(1,1)} and {(0,0),(0,1),(1,1)} (the Kuhn tets'
        // boundary faces); P1 hat of the node; 3-point rule (barycentric 2/3,1/6,1/6; weight 1/3)
        const double area3 = (0.5 * a.ha * a.hb) / 3.0;
        for (int cb = 0; cb < 2; cb++) {
            const int qb = ib - cb;
            if (qb < 0 || qb >= a.nb - 1) continue;
            for (int ca = 0; ca < 2; ca++) {
                const int qa = ia - ca;
                if (qa < 0 || qa >= a.na - 1) continue;
                for (int t = 0; t < 2; t++) {
                    // triangle vertices in corner coordinates
                    const int va[3] = {0, t ? 0 : 1, 1}, vb[3] = {0, t ? 1 : 0, 1};
                    int me = -1;
                    for (int v = 0; v < 3; v++) if (va[v] == ca && vb[v] == cb) me = v;
                    if (me < 0) continue;                 // node not a vertex of this triangle
                    for (int gq = 0; gq < 3; gq++) {
                        double pa = 0.0, pb = 0.0, lam = 0.0;
                        for (int v = 0; v < 3; v++) {
                            const double bw = (v == gq) ? (2.0 / 3.0) : (1.0 / 6.0);
                            pa += bw * va[v];
                            pb += bw * vb[v];
                            if (v == me) lam = bw;
                        }
                        double f = a.f_const;
                        if (a.has_beam) {
                            const double xa = a.oa + (qa + pa) * a.ha - a.bca, xb = a.ob + (qb + pb) * a.hb - a.bcb;
                            f += a.bP / (2.0 * 3.14159265358979323846 * a.bs * a.bs) *
                                 exp(-(xa * xa + xb * xb) / (2.0 * a.bs * a.bs));
                        }
                        sum += area3 * f * lam;
                    }
                }
            }
        }
        const long long node = (long long)zl * a.g.plane + (long long)idx3[1] * a.g.pitch + idx3[0];
        F[node] = (Real)sum;
        return;
    }
    for (int cb = 0; cb < 2; cb++) {             // node is corner (ca, cb) of quad (ia-ca, ib-cb)
        const int qb = ib - cb;
        if (qb < 0 || qb >= a.nb - 1) continue;
        for (int ca = 0; ca < 2; ca++) {
            const int qa = ia - ca;
            if (qa < 0 || qa >= a.na - 1) continue;
            for (int gb = 0; gb < 2; gb++) {
                const double tb = (gb ? gp1 : gp0) * a.hb;
                for (int ga = 0; ga < 2; ga++) {
                    const double ta = (ga ? gp1 : gp0) * a.ha;
                    double f = a.f_const;
                    if (a.has_beam) {
                        const double xa = a.oa + qa * a.ha + ta - a.bca, xb = a.ob + qb * a.hb + tb - a.bcb;
                        f += a.bP / (2.0 * 3.14159265358979323846 * a.bs * a.bs) *
                             exp(-(xa * xa + xb * xb) / (2.0 * a.bs * a.bs));
                    }
                    sum += w * f * phi1(ca, ta, a.ha) * phi1(cb, tb, a.hb);
                }
            }
        }
    }
    const long long node = (long long)zl * a.g.plane + (long long)idx3[1] * a.g.pitch + idx3[0];
    F[node] = (Real)sum;
}

// ---- small pointwise kernels ----------------------------------------------------------------

// v_D <- src_D (src = NULL: the Dirichlet value g) on every local node.
template <class Real>
__global__ void k_set_dirichlet(Geom g, void *vp, const void *srcp, unsigned long long *launches)
{
    Real *v = reinterpret_cast<Real *>(vp);
    const Real *src = reinterpret_cast<const Real *>(srcp);
    const long long n = g.plane * g.nzl;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && launches) atomicAdd(launches, 1ull);
    if (i >= n) return;
    const int x = (int)(i % g.pitch), y = (int)((i / g.pitch) % g.ny1), z = (int)(i / g.plane);
    double gv;
    if (x < g.nx1 && is_dirichlet(g, x, y, z, gv)) v[i] = src ? src[i] : (Real)gv;
}

// End of one solve / time step: x_F <- 0 if b_F = 0; snapshot of one plane of x
// (one-system contexts).  Stacked systems: node slot i belongs to system i / sysn.
struct StepArgs {
    Geom g;
    double *x;
    double *rot[3];         // if rot[0]: x = rot[(step + 1) % 3]
    long long n;
    long long sysn;         // node slots per stacked system (= n for one system)
    double *snap;           // NULL or nsteps x plane (padded plane layout)
    int snap_plane;         // local plane index, -1 none
    int *iters_out;         // per-step iteration counts (may be NULL; one-system contexts)
    Sync sy;
};

template <class Real>
__global__ void __launch_bounds__(256) k_step_end(const StepArgs a)
{
    const int tid = threadIdx.x, blk = blockIdx.x;
    if (blk == 0 && tid == 0 && a.sy.launches) atomicAdd(a.sy.launches, 1ull);
    const CgState *st = a.sy.st;
    const int nsys = a.sy.nsys > 0 ? a.sy.nsys : 1;
    const int step = st->step;
    Real *xv = reinterpret_cast<Real *>(a.rot[0] ? a.rot[(step + 1) % 3] : a.x);
    bool any_zx = false;
    for (int j = 0; j < nsys; j++) any_zx |= st[j].first_failed < 0 && st[j].zero_x;
    if (any_zx) {
        for (long long i = (long long)blk * 256 + tid; i < a.n; i += (long long)gridDim.x * 256) {
            const CgState &sj = st[nsys == 1 ? 0 : (int)(i / a.sysn)];
            if (sj.first_failed >= 0 || !sj.zero_x) continue;
            const int x = (int)(i % a.g.pitch), y = (int)((i / a.g.pitch) % a.g.ny1), z = (int)(i / a.g.plane);
            double gv;
            if (x < a.g.nx1 && !is_dirichlet(a.g, x, y, z, gv)) xv[i] = Real(0);
        }
    }
    if (st->first_failed >= 0) return;
    const bool zx = st->zero_x;
    if (a.snap && a.snap_plane >= 0) {
        const Real *src = xv + (long long)a.snap_plane * a.g.plane;
        Real *dst = reinterpret_cast<Real *>(a.snap) + (long long)step * a.g.plane;
        for (long long i = (long long)blk * 256 + tid; i < a.g.plane; i += (long long)gridDim.x * 256) {
            Real v = src[i];
            if (zx) {
                const int x = (int)(i % a.g.pitch), y = (int)(i / a.g.pitch);
                double gv;
                if (x < a.g.nx1 && !is_dirichlet(a.g, x, y, a.snap_plane, gv)) v = Real(0);
            }
            dst[i] = v;
        }
    }
}

// Per-step bookkeeping after k_step_end (thread j: system j): iteration statistics, failure;
// thread 0 then advances the shared step counter.
__global__ void k_step_commit(Sync sy, int *iters_out)
{
    const int j = threadIdx.x;
    const int nsys = sy.nsys > 0 ? sy.nsys : 1;
    if (j == 0 && sy.launches) atomicAdd(sy.launches, 1ull);
    CgState *st0 = sy.st;
    const int step = st0->step;
    for (int k = j; k < nsys; k += blockDim.x) {
        CgState *st = st0 + k;
        if (st->first_failed >= 0) continue;
        if (iters_out && nsys == 1) iters_out[step] = st->iter;
        st->total_iters += st->iter;
        if (st->iter > st->max_iters_step) st->max_iters_step = st->iter;
        st->steps_done = step + 1;
        if (st->status != ST_OK) st->first_failed = step;
    }
    __syncthreads();
    if (j == 0) st0->step = step + 1;
}

// ---- mixed precision (hf_set_mixed, NEXT row f3): fp32 correction, fp64 finish ---------------
// The fp64 context (hi) owns an fp32 shadow (lo) with the same grid, coefficients and Dirichlet
// faces.  Per time step (defect correction): hi's RHS and init kernels give x0 = 2u^n - u^(n-1)
// (in U[(n+1) % 3]) and its fp64 residual r0 = b - A x0; k_mix_in hands r0 to the fp32 PCG,
// which solves A e = r0 from e = 0 to rtol_lo; k_mix_out adds e to x0 in fp64; hi's PCG then
// finishes from x0 + e to rtol with the fp64 residual of the fp64 operator deciding, so the
// result has the fp64 path's accuracy while most of the error reduction ran on half the bytes.
struct MixArgs {
    int nx1, ny1, nzl;
    int pitch_hi, pitch_lo;          // row pitches of the two layouts
    long long plane_hi, plane_lo;
    const double *rhi;               // hi r0 = b - A x0 (after hi's init kernel)
    double *ring[3];                 // hi time-step ring: x0 in U[(step + 1) % 3]
    const CgState *st;               // hi state (step counter)
    float *blo, *xlo;                // lo right-hand side (r0) and iterate (e)
    const CgState *stlo;             // lo state (iterations of the fp32 solve)
    unsigned long long *lo_iters;    // accumulated fp32 iterations
    unsigned long long *launches;
    int nsys, sys_planes;            // stacked systems (batched sims): planes per system
};

// a system of a stack that failed in an earlier step keeps its result: no correction
__device__ __forceinline__ bool mix_failed(const MixArgs &a, int z)
{
    const int sj = a.nsys > 1 ? z / a.sys_planes : 0;
    return a.st[sj].first_failed >= 0;
}

__global__ void k_mix_in(const MixArgs a)
{
    const long long n = (long long)a.nx1 * a.ny1 * a.nzl;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0 && a.launches) atomicAdd(a.launches, 1ull);
    if (i >= n) return;
    const int x = (int)(i % a.nx1), y = (int)((i / a.nx1) % a.ny1), z = (int)(i / ((long long)a.nx1 * a.ny1));
    const long long h = z * a.plane_hi + (long long)y * a.pitch_hi + x, l = z * a.plane_lo + (long long)y * a.pitch_lo + x;
    a.blo[l] = mix_failed(a, z) ? 0.0f : (float)a.rhi[h];
    a.xlo[l] = 0.0f;
}

__global__ void k_mix_out(const MixArgs a)
{
    const long long n = (long long)a.nx1 * a.ny1 * a.nzl;
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) {
        if (a.launches) atomicAdd(a.launches, 1ull);
        if (a.lo_iters) atomicAdd(a.lo_iters, (unsigned long long)a.stlo->iter);
    }
    if (i >= n) return;
    const int x = (int)(i % a.nx1), y = (int)((i / a.nx1) % a.ny1), z = (int)(i / ((long long)a.nx1 * a.ny1));
    const long long h = z * a.plane_hi + (long long)y * a.pitch_hi + x, l = z * a.plane_lo + (long long)y * a.pitch_lo + x;
    if (mix_failed(a, z)) return;
    double *xv = a.ring[(a.st->step + 1) % 3];
    xv[h] += (double)a.xlo[l];
}

// ---- c lane of the packed (k, c) pairs back to a plain per-element fp64 array ----------------
template <class Real>
__global__ void k_extract_c(Geom g, int nz, const void *kcp, double *c, unsigned long long *launches)
{
    using V2 = typename Vec2<Real>::type;
    const V2 *kc = reinterpret_cast<const V2 *>(kcp);
    const long long ne = (long long)g.nx * g.ny * nz;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e == 0 && launches) atomicAdd(launches, 1ull);
    if (e >= ne) return;
    const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
    c[e] = (double)kc[((long long)(ez - g.zg0 + 1) * g.ny + ey) * g.kpitch + ex].y;
}

// both lanes (k and c) of the fp64 pairs back to plain per-element arrays (the mixed-precision
// shadow of a context whose coefficients came as material ids)
__global__ void k_extract_kc(Geom g, int nz, const double2 *kc, double *k, double *c, unsigned long long *launches)
{
    const long long ne = (long long)g.nx * g.ny * nz;
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e == 0 && launches) atomicAdd(launches, 1ull);
    if (e >= ne) return;
    const int ex = (int)(e % g.nx), ey = (int)((e / g.nx) % g.ny), ez = (int)(e / ((long long)g.nx * g.ny));
    const double2 v = kc[((long long)(ez - g.zg0 + 1) * g.ny + ey) * g.kpitch + ex];
    k[e] = v.x;
    c[e] = v.y;
}

// ---- boundary conversions of the fp32 variant: user fp64 (natural pitch) <-> internal Real ----

template <class Real>
__global__ void k_cvt_in(const double *src, Real *dst, int nx1, long long rows, int pitch, unsigned long long *launches)
{
    const long long n = rows * nx1;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 == 0 && launches) atomicAdd(launches, 1ull);
    for (long long i = i0; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / nx1;
        dst[row * pitch + (i - row * nx1)] = (Real)src[i];
    }
}

template <class Real>
__global__ void k_cvt_out(const Real *src, double *dst, int nx1, long long rows, int pitch, unsigned long long *launches)
{
    const long long n = rows * nx1;
    const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 == 0 && launches) atomicAdd(launches, 1ull);
    for (long long i = i0; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long row = i / nx1;
        dst[i] = (double)src[row * pitch + (i - row * nx1)];
    }
}

}  // namespace hf
