// hf_lib.cu -- libheatfem: the C ABI of include/heatfem.h on top of hf_kernels.cuh.
//
// Host runtime: contexts, workspaces, TMA descriptors, host-pointer staging, the PCG and
// time-loop drivers (a CUDA graph with a device-side WHILE loop, or a host loop), batched
// simulations, z-slab decomposition with NCCL (dlopen'ed) or an in-process transport.
// Citations: P:n = PAPER.md line n.
//
// Internal layout: node vectors use a row pitch of nx1 rounded up to an even number of
// doubles (TMA needs 16-byte global strides); user vectors use the natural pitch nx1 and are
// converted at the boundary (no copy when nx1 is even and the pointer is on the device).
#include "heatfem.h"
#include "hf_kernels.cuh"
#include "hf_ablate.cuh"
#include "hf_resident.cuh"

#include <dlfcn.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <chrono>
#include <string>
#include <vector>

using namespace hf;

// ============================================================================================
// errors

static thread_local std::string g_err;

#ifdef HF_DEBUG_WAIT
static unsigned long long *g_dbg_host = nullptr;
static void dbg_dump()
{
    if (g_dbg_host && g_dbg_host[0])
        fprintf(stderr, "[hf debug] stuck wait: tag %llu it %lld parity %llu block (%llu,%llu,%llu) tid %llu bar 0x%llx state 0x%llx (hits %llu)\n",
                g_dbg_host[1], (long long)g_dbg_host[2], g_dbg_host[3], g_dbg_host[4], g_dbg_host[5], g_dbg_host[6],
                g_dbg_host[7], g_dbg_host[8], g_dbg_host[9], g_dbg_host[0]);
}
#endif

static hf_status fail(hf_status s, const std::string &msg)
{
    g_err = msg;
#ifdef HF_DEBUG_WAIT
    dbg_dump();
#endif
    return s;
}

#define CUCK(call)                                                                           \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            return fail(e_ == cudaErrorMemoryAllocation ? HF_E_OOM : HF_E_CUDA,              \
                        std::string(#call) + ": " + cudaGetErrorString(e_));                \
    } while (0)

#define HFCK(call)                                                                           \
    do {                                                                                     \
        hf_status s_ = (call);                                                               \
        if (s_ != HF_OK) return s_;                                                          \
    } while (0)

// ============================================================================================
// NCCL, loaded at run time (libnccl.so.2: torch's copy if torch is already loaded, else system)

namespace nccl {
typedef struct ncclComm *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { ncclFloat32 = 7, ncclFloat64 = 8, ncclSum = 0 };
typedef ncclResult_t (*GetUniqueId_t)(ncclUniqueId *);
typedef ncclResult_t (*CommInitRank_t)(ncclComm_t *, int, ncclUniqueId, int);
typedef ncclResult_t (*CommDestroy_t)(ncclComm_t);
typedef ncclResult_t (*AllReduce_t)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*Send_t)(const void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*Recv_t)(void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*Group_t)(void);
typedef const char *(*GetErrorString_t)(ncclResult_t);
typedef ncclResult_t (*CommGetAsyncError_t)(ncclComm_t, ncclResult_t *);
typedef ncclResult_t (*CommAbort_t)(ncclComm_t);
struct Api {
    void *h = nullptr;
    GetUniqueId_t getUniqueId;
    CommInitRank_t commInitRank;
    CommDestroy_t commDestroy;
    AllReduce_t allReduce;
    Send_t send;
    Recv_t recv;
    Group_t groupStart, groupEnd;
    GetErrorString_t getErrorString;
    CommGetAsyncError_t commGetAsyncError;
    CommAbort_t commAbort;
};
static Api g_api;
static std::mutex g_mu;

static hf_status load()
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_api.h) return HF_OK;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(HF_E_NCCL, std::string("dlopen libnccl.so.2: ") + dlerror());
#define SYM(field, name, type)                                                               \
    g_api.field = (type)dlsym(h, name);                                                      \
    if (!g_api.field) return fail(HF_E_NCCL, std::string("dlsym ") + name);
    SYM(getUniqueId, "ncclGetUniqueId", GetUniqueId_t)
    SYM(commInitRank, "ncclCommInitRank", CommInitRank_t)
    SYM(commDestroy, "ncclCommDestroy", CommDestroy_t)
    SYM(allReduce, "ncclAllReduce", AllReduce_t)
    SYM(send, "ncclSend", Send_t)
    SYM(recv, "ncclRecv", Recv_t)
    SYM(groupStart, "ncclGroupStart", Group_t)
    SYM(groupEnd, "ncclGroupEnd", Group_t)
    SYM(getErrorString, "ncclGetErrorString", GetErrorString_t)
    SYM(commGetAsyncError, "ncclCommGetAsyncError", CommGetAsyncError_t)
    SYM(commAbort, "ncclCommAbort", CommAbort_t)
#undef SYM
    g_api.h = h;
    return HF_OK;
}
}  // namespace nccl

#define NCCK(call)                                                                           \
    do {                                                                                     \
        nccl::ncclResult_t r_ = (call);                                                      \
        if (r_ != 0) return fail(HF_E_NCCL, std::string(#call) + ": " + nccl::g_api.getErrorString(r_)); \
    } while (0)

// ============================================================================================
// TMA descriptors (cuTensorMapEncodeTiled through the runtime's driver entry point)

typedef CUresult (*EncodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled_t g_encode = nullptr;

static hf_status get_encode()
{
    if (g_encode) return HF_OK;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUCK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) return fail(HF_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = (EncodeTiled_t)fn;
    return HF_OK;
}

// ============================================================================================
// context

struct SimKey {
    double aK = 0, aM = 0, aKL = 0, aML = 0, rtol = 0, dt = 0;
    int max_iter = 0, replace_every = 0, first = 0, snap_plane = -1, lift = 0, res = 0, cg1 = 0;
    const double *F = nullptr;
    double *snap = nullptr;
    bool operator==(const SimKey &o) const { return std::memcmp(this, &o, sizeof(SimKey)) == 0; }
};

struct Sys {                         // one system's PCG workspace (Table 3 buffers)
    void *kc = nullptr;              // (k, c) pairs of the storage type, (kpitch, ny, nzl + 1)
    void *kcn = nullptr;             // EL_TETV: per-node (k, c) pairs, padded node layout
    double *U[3] = {nullptr, nullptr, nullptr};   // time-step ring
    double *b = nullptr, *r = nullptr, *s = nullptr, *q = nullptr, *invd = nullptr;
    double *dbuf[2] = {nullptr, nullptr};
    Maps maps;                       // TMA maps of U[0..2], dbuf[0..1], s and kc
    CgState *st = nullptr;           // device, one per stacked system (hf_ctx::nsys)
    CgState *st_host = nullptr;      // pinned mirror
    double *partA = nullptr, *partB = nullptr;   // per-block partial sums of A / (init, B, RESID)
    double *sums = nullptr;                      // slab mode: allreduced sums
    unsigned long long *gbar = nullptr;          // grid-barrier counter of the fused A+B launch
    CgState *st_ring = nullptr;                  // pinned state copies of the pipelined host loop
    cudaEvent_t ev_ring[2] = {nullptr, nullptr};
    // single-reduction PCG (hf_set_cg_variant 1): r, w = A u, s = A p ping-pong by iteration
    // parity, p; node maps of the CG1 kernel of parity k (r[k], w[k], s[k], P^-1) and of the
    // w = A P^-1 r kernel reading r[k] (r[k], P^-1)
    double *c1r[2] = {nullptr, nullptr}, *c1w[2] = {nullptr, nullptr}, *c1s[2] = {nullptr, nullptr};
    double *c1p = nullptr;
    Maps c1maps[2], c1wmaps[2];

    int *iters = nullptr;
    int iters_cap = 0;
    cudaStream_t stream = nullptr;   // == ctx stream for the primary system
    bool own_stream = false;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    SimKey key;
    bool key_valid = false;
};

struct Comm {
    virtual ~Comm() {}
    // make ghost planes of `v` (local layout) equal to the neighbours' owned boundary planes
    virtual hf_status exchange(hf_ctx *c, Sys &s, double *v) = 0;
    // in-place sum of n doubles (device) across ranks
    virtual hf_status allreduce(hf_ctx *c, Sys &s, double *v, int n) = 0;
    virtual bool graph_capturable() const = 0;
    // the kernels themselves exchange sums and ghost planes (peer memory): no host step between
    // kernels, the whole solve can run in the step graph
    virtual bool in_kernel() const { return false; }
    virtual const PeerSync *peer_dev() const { return nullptr; }
    virtual bool ready() const { return true; }
    // host-side health check while waiting for device work (NCCL: asynchronous errors)
    virtual hf_status poll() { return HF_OK; }
    // start of a collective call (simulate / cg), after this rank's host-side setup and before
    // its first kernel that waits for another rank (ranks sharing one process: a barrier, so
    // that no rank's allocation -- an implicit device synchronisation -- waits for kernels that
    // themselves wait for this rank)
    virtual hf_status enter() { return HF_OK; }
};

struct hf_ctx {
    std::map<int, hf_ctx *> stacks;  // batched: contexts of G stacked systems (batched_stacked)
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int nsm = 148;
    hf_grid g{};
    int nx1 = 0, ny1 = 0, nz1g = 0;
    int prec = 64, es = 8;           // storage precision of node vectors and (k, c): 64 or 32 (f3)
    int pitch = 0;                   // internal row pitch (16-B multiple)
    int kpitch = 0;                  // (k, c) pairs per coefficient row
    int nzl = 0, zg0 = 0;            // local planes, global index of local plane 0
    int own_lo = 0, own_hi = 0;      // owned local planes [own_lo, own_hi)
    long long plane = 0, nloc = 0;   // internal plane size, local node slots (padded)
    long long kc_elems = 0;
    bool coef_set = false;
    unsigned dbits = 0;
    double gval[6] = {0, 0, 0, 0, 0, 0};
    int elem = EL_Q1;                // element variant (hf_set_element)
    bool tetv = false;               // tets with per-tet vertex-averaged coefficients (EL_TETV)
    DiagC dg;                        // diagonal entries of K_ref, M_ref per local node
    Sys sys0;
    unsigned long long *launches = nullptr;
    std::vector<void *> scratch;     // staging buffers (padded node layout unless noted)
    std::vector<size_t> scratch_cap;
    double *flush = nullptr;
    int driver = 0;                  // 0 graph, 1 host loop
    int tileR = 4;
    int zchunk = 0;                  // z planes per stencil CTA (0: sized to fill the SMs)
    int tile_r_set = 0;              // tile height set by hf_set_tuning / HF_TILE_R (0: default_tile_r)
    int batch_group = 0;             // systems per stack of hf_simulate_batched (0: stack_group's model)
    double comm_timeout_s = 120.0;   // host-loop slab transports: fail instead of waiting longer
    int check_every = 8;
    int max_blocks = 0;
    int occ = 2;                     // resident CTAs/SM of the CG stencil (occupancy API)
    int unroll = 0;                  // PCG iterations per WHILE-body launch (0: by grid size, see build_cg_graph)
    int pdl = 1;                     // programmatic A <-> B edges in the loop body (HF_PDL=0 disables)
    int fuse_ab = 0;                 // A and B of an iteration in one launch (HF_FUSE_AB=1)
    int cg1 = 0;                     // hf_set_cg_variant: 1 = single-reduction PCG (one kernel per iteration)
    int last_cg1 = 0;                // the last hf_simulate* ran the single-reduction PCG
    int tm_fence = 0;                // acquire TMA descriptors in every launch (HF_TM_FENCE=1, see maps_dev)
    int resident = 0;                // hf_set_resident: 1 = on-chip PCG when eligible, 0 = never (default)
    int last_resident = 0;           // the last hf_simulate* ran the on-chip PCG
    ResSync *rsync = nullptr;        // flags + partials of the on-chip PCG's grid reductions
    unsigned long long *res_prof = nullptr;   // per-phase timer of the on-chip PCG (hf_resident_profile)
    // mixed precision (hf_set_mixed): the fp32 shadow context, its stop tolerance, its iteration
    // counter, and the per-step graph of [RHS -> fp32 solve] (the fp64 finish is sys0's graph)
    hf_ctx *lo = nullptr;
    double mix_rtol = 1e-6;
    unsigned long long *mix_iters = nullptr;
    cudaGraph_t mix_graph = nullptr;
    cudaGraphExec_t mix_exec = nullptr;
    int nsys = 1;                    // systems stacked along z (batched forward simulations, a13)
    int sys_planes = 0;              // local node planes per system (= nzl for one system)
    int rank = 0, nranks = 1;
    Comm *comm = nullptr;
    int nsm_share = 0;               // SMs a stencil grid is sized for (< nsm when ranks share a GPU)
    void *ghost_buf = nullptr;       // peer transport: the two s ghost planes the neighbours write
    size_t ghost_pb = 0;             // bytes per plane slot of the mailbox buffers
    int step_flush = 0;              // 1: flush L2 + time every step; 2: time every step, no flush
    double last_ms_steps = 0.0;      // per-step event total of the last run (step_flush)
    double last_aK = 0.0;            // operator (aK, 1) of the last time loop (hf_time_kernel_a)
    bool prof = false;
    double prof_ms[5] = {0, 0, 0, 0, 0};
    long long prof_n[5] = {0, 0, 0, 0, 0};
    // NEXT f4 ablation (Implementation 1): stored scaled element matrices and vertex-order
    // contributions (hf_ablation_prepare)
    double *ab_A = nullptr, *ab_contrib = nullptr;
    double ab_aK = 0.0, ab_aM = 0.0;
    bool ab_ready = false;
    // materials by id (hf_set_material_ids): uint8 ids + 1 in the (k, c) layer layout, the
    // material table, and the id tensor's TMA descriptor (sys0's kc map while pal_on)
    unsigned char *kid = nullptr;
    int kid_pitch = 0;               // ids per row (nx rounded up to 16: TMA strides)
    double pal[PAL_MAX][2] = {};
    int npal = 0;                    // table entries in use (materials + 1)
    bool pal_on = false;
    CUtensorMap kid_map;
};

static const int NW = 8;             // warps per stencil CTA

// p + n elements of the context's storage type (node vectors are typed double* on the host)
static inline double *eoff(const hf_ctx *c, const double *p, long long n)
{
    return (double *)((char *)p + n * (long long)c->es);
}

static bool is_device_ptr(const void *p)
{
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// device memory of another GPU than the context's: rejected at the ABI (HF_E_ARG) instead of
// being used in TMA maps and kernels of this device
static bool foreign_ptr(const hf_ctx *c, const void *p)
{
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice && at.device != c->device;
}

static hf_status check_ptrs(const hf_ctx *c, const char *who, std::initializer_list<const void *> ps);

// user node vector usable in place: device, natural pitch == internal pitch, 16-B aligned
static bool direct_ok(const hf_ctx *c, const void *p)
{
    return c->es == 8 && c->pitch == c->nx1 && ((uintptr_t)p % 16) == 0 && is_device_ptr(p);
}

static hf_status check_ptrs(const hf_ctx *c, const char *who, std::initializer_list<const void *> ps)
{
    for (const void *p : ps)
        if (foreign_ptr(c, p))
            return fail(HF_E_ARG, std::string(who) + ": array on another CUDA device than the context's (device " +
                                      std::to_string(c->device) + ")");
    return HF_OK;
}

static hf_status scratch_get(hf_ctx *c, int slot, size_t bytes, void **out)
{
    if ((int)c->scratch.size() <= slot) {
        c->scratch.resize(slot + 1, nullptr);
        c->scratch_cap.resize(slot + 1, 0);
    }
    if (c->scratch_cap[slot] < bytes) {
        if (c->scratch[slot]) cudaFree(c->scratch[slot]);
        c->scratch[slot] = nullptr;
        c->scratch_cap[slot] = 0;
        CUCK(cudaMalloc(&c->scratch[slot], bytes));
        CUCK(cudaMemsetAsync(c->scratch[slot], 0, bytes, c->stream));   // pitch padding stays 0
        CUCK(cudaStreamSynchronize(c->stream));   // before any use on another stream
        c->scratch_cap[slot] = bytes;
    }
    *out = c->scratch[slot];
    return HF_OK;
}

static hf_status scratch_get(hf_ctx *c, int slot, size_t bytes, void **out);

// user fp64 (natural pitch) -> internal (padded pitch, storage type), nplanes planes.  fp32
// contexts convert on the device (k_cvt_in); a host source is staged in scratch `stage` first.
static hf_status copy_in(hf_ctx *c, double *dst, const double *src, int nplanes, cudaStream_t s, int stage = 30)
{
    if (c->es == 8) {
        CUCK(cudaMemcpy2DAsync(dst, (size_t)c->pitch * 8, src, (size_t)c->nx1 * 8, (size_t)c->nx1 * 8,
                               (size_t)c->ny1 * nplanes, cudaMemcpyDefault, s));
        return HF_OK;
    }
    const size_t n = (size_t)c->nx1 * c->ny1 * nplanes;
    const double *d = src;
    if (!is_device_ptr(src)) {
        void *t;
        HFCK(scratch_get(c, stage, n * 8, &t));
        CUCK(cudaMemcpyAsync(t, src, n * 8, cudaMemcpyHostToDevice, s));
        d = (const double *)t;
    }
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)c->nsm * 8);
    k_cvt_in<float><<<std::max(1u, blocks), 256, 0, s>>>(d, (float *)dst, c->nx1, (long long)c->ny1 * nplanes,
                                                         c->pitch, c->launches);
    CUCK(cudaGetLastError());
    return HF_OK;
}

static hf_status copy_out(hf_ctx *c, double *dst, const double *src, int nplanes, cudaStream_t s, int stage = 31)
{
    if (c->es == 8) {
        CUCK(cudaMemcpy2DAsync(dst, (size_t)c->nx1 * 8, src, (size_t)c->pitch * 8, (size_t)c->nx1 * 8,
                               (size_t)c->ny1 * nplanes, cudaMemcpyDefault, s));
        return HF_OK;
    }
    const size_t n = (size_t)c->nx1 * c->ny1 * nplanes;
    const bool dev = is_device_ptr(dst);
    double *d = dst;
    if (!dev) {
        void *t;
        HFCK(scratch_get(c, stage, n * 8, &t));
        d = (double *)t;
    }
    const unsigned blocks = (unsigned)std::min<size_t>((n + 255) / 256, (size_t)c->nsm * 8);
    k_cvt_out<float><<<std::max(1u, blocks), 256, 0, s>>>((const float *)src, d, c->nx1, (long long)c->ny1 * nplanes,
                                                          c->pitch, c->launches);
    CUCK(cudaGetLastError());
    if (!dev) CUCK(cudaMemcpyAsync(dst, d, n * 8, cudaMemcpyDeviceToHost, s));
    return HF_OK;
}

// internal view of a user input node vector (copied into scratch `slot` unless direct)
static hf_status node_in(hf_ctx *c, const double *p, int slot, const double **out)
{
    if (!p) { *out = nullptr; return HF_OK; }
    if (direct_ok(c, p)) { *out = p; return HF_OK; }
    void *d;
    HFCK(scratch_get(c, slot, (size_t)c->nloc * 8, &d));
    HFCK(copy_in(c, (double *)d, p, c->nzl, c->stream));
    *out = (const double *)d;
    return HF_OK;
}

// internal view of a user output (or in/out) node vector
static hf_status node_out(hf_ctx *c, double *p, int slot, bool copy, double **out)
{
    if (direct_ok(c, p)) { *out = p; return HF_OK; }
    void *d;
    HFCK(scratch_get(c, slot, (size_t)c->nloc * 8, &d));
    if (copy) HFCK(copy_in(c, (double *)d, p, c->nzl, c->stream));
    *out = (double *)d;
    return HF_OK;
}

static hf_status node_out_finish(hf_ctx *c, double *p, const double *d)
{
    if (p != d) HFCK(copy_out(c, p, d, c->nzl, c->stream));
    CUCK(cudaStreamSynchronize(c->stream));
    return HF_OK;
}

// device view of a plain (element) input array
static hf_status dev_in(hf_ctx *c, const double *p, size_t n, int slot, const double **out)
{
    if (!p) { *out = nullptr; return HF_OK; }
    if (is_device_ptr(p)) { *out = p; return HF_OK; }
    void *d;
    HFCK(scratch_get(c, slot, n * sizeof(double), &d));
    CUCK(cudaMemcpyAsync(d, p, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    *out = (const double *)d;
    return HF_OK;
}

static Geom make_geom(const hf_ctx *c)
{
    Geom g;
    std::memset(&g, 0, sizeof(g));
    g.nx1 = c->nx1; g.ny1 = c->ny1; g.nzl = c->nzl;
    g.zg0 = c->zg0; g.nz1g = c->nz1g;
    g.pitch = c->pitch;
    g.plane = c->plane;
    g.nx = (int)c->g.ne[0];
    g.ny = (int)c->g.ne[1];
    g.kpitch = c->kpitch;
    g.dbits = c->dbits;
    g.zper = c->nz1g / c->nsys;
    for (int f = 0; f < 6; f++) g.gval[f] = c->gval[f];
    return g;
}

// WHT eigenvalues of the voxel matrices (1/8 folded in): mu_d(0) = h/2, mu_d(1) = h/6 for
// (h/6)[[2,1],[1,2]]; kappa_d(0) = 0, kappa_d(1) = 2/h for (1/h)[[1,-1],[-1,1]].  Folded into
// the per-channel (a, b) coefficients of the fused z butterfly.
static Lam make_lam(const double h[3], double aK, double aM)
{
    double lm[8], lk[8];
    for (int s = 0; s < 8; s++) {
        const int b[3] = {s & 1, (s >> 1) & 1, (s >> 2) & 1};
        double mu[3], ka[3];
        for (int d = 0; d < 3; d++) {
            mu[d] = b[d] ? h[d] / 6.0 : h[d] / 2.0;
            ka[d] = b[d] ? 2.0 / h[d] : 0.0;
        }
        lm[s] = aM * (mu[0] * mu[1] * mu[2]) / 8.0;
        lk[s] = aK * (ka[0] * mu[1] * mu[2] + mu[0] * ka[1] * mu[2] + mu[0] * mu[1] * ka[2]) / 8.0;
    }
    Lam L;
    for (int ch = 0; ch < 4; ch++) {
        const int sx = ch >> 1, sy = ch & 1;
        const int s0 = sx + 2 * sy, s1 = s0 + 4;
        L.ka[ch] = lk[s0] + lk[s1];
        L.ma[ch] = lm[s0] + lm[s1];
        L.kb[ch] = lk[s0] - lk[s1];
        L.mb[ch] = lm[s0] - lm[s1];
    }
    return L;
}

// Voxel matrices of the 6-tet split (NEXT row f1): tet t follows the lattice path
// 0 -> e_a -> e_a + e_b -> 7 for the t-th axis permutation (a, b, c).  On that tet the P1
// barycentric coordinates are 1 - x_a/h_a, x_a/h_a - x_b/h_b, x_b/h_b - x_c/h_c, x_c/h_c, so
// their gradients are -e_a/h_a, e_a/h_a - e_b/h_b, e_b/h_b - e_c/h_c, e_c/h_c; V = hx hy hz / 6;
// K_ij = V g_i . g_j, M_ij = V (1 + delta_ij) / 20, summed into the voxel's 8 nodes.
static void tet_voxel(const double h[3], double K[64], double M[64])
{
    static const int perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int i = 0; i < 64; i++) { K[i] = 0.0; M[i] = 0.0; }
    const double V = h[0] * h[1] * h[2] / 6.0;
    for (int t = 0; t < 6; t++) {
        int loc[4] = {0, 0, 0, 0}, bits = 0;
        double g[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int s = 0; s < 3; s++) {
            const int ax = perm[t][s];
            bits |= 1 << ax;
            loc[s + 1] = bits;
            g[s][ax] -= 1.0 / h[ax];          // lambda_s decreases along its axis
            g[s + 1][ax] += 1.0 / h[ax];      // lambda_{s+1} increases
        }
        for (int i = 0; i < 4; i++)
            for (int j = 0; j < 4; j++) {
                K[loc[i] * 8 + loc[j]] += V * (g[i][0] * g[j][0] + g[i][1] * g[j][1] + g[i][2] * g[j][2]);
                M[loc[i] * 8 + loc[j]] += V * (i == j ? 2.0 : 1.0) / 20.0;
            }
    }
}

// Q1 voxel matrices as dense 8 x 8 (NEXT f4 ablation kernels): tensor products of the 1D
// k = (1/h)[[1,-1],[-1,1]] and m = (h/6)[[2,1],[1,2]], K = kx my mz + mx ky mz + mx my kz,
// local node l = bx + 2 by + 4 bz.
static void q1_voxel(const double h[3], double K[64], double M[64])
{
    for (int a = 0; a < 8; a++)
        for (int b = 0; b < 8; b++) {
            double m[3], k[3];
            for (int d = 0; d < 3; d++) {
                const bool same = ((a >> d) & 1) == ((b >> d) & 1);
                m[d] = h[d] / 6.0 * (same ? 2.0 : 1.0);
                k[d] = (same ? 1.0 : -1.0) / h[d];
            }
            K[a * 8 + b] = k[0] * m[1] * m[2] + m[0] * k[1] * m[2] + m[0] * m[1] * k[2];
            M[a * 8 + b] = m[0] * m[1] * m[2];
        }
}

// Unit-coefficient stiffness of each Kuhn tet in tet_loc order (gradient-path formula as in
// tet_voxel) and the tet volume (EL_TETV).
static void tet_matrices(const double h[3], double K[6][16], double *V)
{
    *V = h[0] * h[1] * h[2] / 6.0;
    for (int t = 0; t < 6; t++) {
        double g[4][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
        for (int s = 0; s < 3; s++) {
            const int prev = tet_loc(t, s), next = tet_loc(t, s + 1);
            const int ax = (prev ^ next) == 1 ? 0 : ((prev ^ next) == 2 ? 1 : 2);   // axis of this path step
            g[s][ax] -= 1.0 / h[ax];
            g[s + 1][ax] += 1.0 / h[ax];
        }
        for (int i = 0; i < 4; i++)
            for (int j = 0; j < 4; j++)
                K[t][i * 4 + j] = *V * (g[i][0] * g[j][0] + g[i][1] * g[j][1] + g[i][2] * g[j][2]);
    }
}

// node tensor map over nplanes planes of plane_bytes each (default: a local node vector)
static hf_status node_map(const hf_ctx *c, const double *p, CUtensorMap *m, int nplanes = 0, size_t plane_bytes = 0)
{
    HFCK(get_encode());
    const cuuint64_t dims[3] = {(cuuint64_t)c->nx1, (cuuint64_t)c->ny1, (cuuint64_t)(nplanes ? nplanes : c->nzl)};
    const cuuint64_t strides[2] = {(cuuint64_t)c->pitch * c->es,
                                   (cuuint64_t)(plane_bytes ? plane_bytes : (size_t)c->plane * c->es)};
    const cuuint32_t bw = c->es == 8 ? StencilShape<2, 8, LD_RAW, double>::BW : StencilShape<2, 8, LD_RAW, float>::BW;
    const cuuint32_t box[3] = {bw, (cuuint32_t)(NW * c->tileR + 1), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapDataType dt = c->es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = g_encode(m, dt, 3, (void *)p, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HF_E_CUDA, "cuTensorMapEncodeTiled(node) failed: " + std::to_string((int)r));
    return HF_OK;
}

static hf_status kc_map(const hf_ctx *c, const void *kc, CUtensorMap *m)
{
    HFCK(get_encode());
    const cuuint64_t kp = (cuuint64_t)c->kpitch, ny = (cuuint64_t)c->g.ne[1];
    const cuuint64_t dims[3] = {2 * kp, ny, (cuuint64_t)c->nzl + 1};
    const cuuint64_t strides[2] = {2 * kp * c->es, 2 * kp * ny * c->es};
    const cuuint32_t kw = c->es == 8 ? StencilShape<2, 8, LD_RAW, double>::KW : StencilShape<2, 8, LD_RAW, float>::KW;
    const cuuint32_t box[3] = {kw, (cuuint32_t)(NW * c->tileR), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapDataType dt = c->es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = g_encode(m, dt, 3, (void *)kc, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HF_E_CUDA, "cuTensorMapEncodeTiled(kc) failed: " + std::to_string((int)r));
    return HF_OK;
}

static hf_status kcn_map(const hf_ctx *c, const void *kcn, CUtensorMap *m)
{
    HFCK(get_encode());
    const cuuint64_t dims[3] = {2 * (cuuint64_t)c->nx1, (cuuint64_t)c->ny1, (cuuint64_t)c->nzl};
    const cuuint64_t strides[2] = {2 * (cuuint64_t)c->pitch * c->es, 2 * (cuuint64_t)c->plane * c->es};
    const cuuint32_t bw = c->es == 8 ? StencilShape<2, 8, LD_RAW, double>::BW : StencilShape<2, 8, LD_RAW, float>::BW;
    const cuuint32_t box[3] = {2 * bw, (cuuint32_t)(NW * c->tileR + 1), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    const CUtensorMapDataType dt = c->es == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
    CUresult r = g_encode(m, dt, 3, (void *)kcn, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HF_E_CUDA, "cuTensorMapEncodeTiled(kcn) failed: " + std::to_string((int)r));
    return HF_OK;
}

// material ids (EL_Q1P): uint8 view (kid_pitch, ny, nzl + 1), layer L at z = L + 1 as kc
static hf_status kid_map_enc(const hf_ctx *c, const void *kid, CUtensorMap *m)
{
    HFCK(get_encode());
    const cuuint64_t kp = (cuuint64_t)c->kid_pitch, ny = (cuuint64_t)c->g.ne[1];
    const cuuint64_t dims[3] = {kp, ny, (cuuint64_t)c->nzl + 1};
    const cuuint64_t strides[2] = {kp, kp * ny};
    const cuuint32_t box[3] = {(cuuint32_t)PAL_BW, (cuuint32_t)(NW * c->tileR), 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void *)kid, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(HF_E_CUDA, "cuTensorMapEncodeTiled(kid) failed: " + std::to_string((int)r));
    return HF_OK;
}

// ============================================================================================
// launches (one spec -> direct launch, or a graph kernel node)

struct Launch {
    const void *fn = nullptr;
    dim3 grid, block;
    size_t smem = 0;
    std::vector<std::vector<char>> args;
    int cls = 4;
    template <class T> void add(const T &v)
    {
        std::vector<char> b(sizeof(T));
        std::memcpy(b.data(), &v, sizeof(T));
        args.push_back(std::move(b));
    }
    template <class T> T get(int i) const
    {
        check<T>(i);
        T v;
        std::memcpy(&v, args[i].data(), sizeof(T));
        return v;
    }
    template <class T> void put(int i, const T &v)
    {
        check<T>(i);
        std::memcpy(args[i].data(), &v, sizeof(T));
    }
    template <class T> void check(int i) const
    {
        if (i < 0 || i >= (int)args.size() || args[i].size() != sizeof(T)) {
            fprintf(stderr, "libheatfem: internal error: launch argument %d has the wrong type\n", i);
            abort();
        }
    }
};

#ifndef HF_NS_R2
#define HF_NS_R2 4
#endif
template <int R, int LD> constexpr int ns_of()
{
    return (LD == LD_CG1 || (R >= 4 && StencilShape<R, NW, LD>::NA >= 2)) ? 3 : (R == 2 ? HF_NS_R2 : 4);
}

struct StencilFn {
    const void *fn;
    size_t smem;
    int nw = NW;             // warps per CTA
};

template <int R, int LD, int EP, int FL, int EL, class Real> static StencilFn stencil_fn_t()
{
    constexpr int NS = ns_of<R, LD>();
    return {(const void *)k_stencil<R, NW, NS, LD, EP, FL, EL, Real>, StencilShape<R, NW, LD, Real, EL>::smem_bytes(NS), NW};
}

// every (loader, epilogue, flags) variant the library launches, for tile heights R = 2 and 4
#define HF_STENCIL_VARIANTS(X)                                                                  \
    X(LD_RAW, EP_APPLY, 0)                                                                      \
    X(LD_RAW, EP_APPLY, FL_HB)                                                                  \
    X(LD_RAW, EP_APPLY, FL_HB | FL_DIR | FL_DSET)                                               \
    X(LD_GT, EP_APPLY, FL_HB | FL_DIR | FL_DSET)                                                \
    X(LD_CGD, EP_CGA, 0)                                                                        \
    X(LD_CGD, EP_CGA, FL_DIR)                                                                   \
    X(LD_CGD, EP_CGA, FL_FUSEB)                                                                 \
    X(LD_CGD, EP_CGA, FL_DIR | FL_FUSEB)                                                        \
    X(LD_X0, EP_RESID_INIT, 0)                                                                  \
    X(LD_X0, EP_RESID_INIT, FL_MASK | FL_DIR)                                                   \
    X(LD_RAW, EP_RESID_INIT, 0)                                                                 \
    X(LD_RAW, EP_RESID_INIT, FL_MASK | FL_DIR)                                                  \
    X(LD_RAW, EP_RESID, 0)                                                                      \
    X(LD_RAW, EP_RESID, FL_MASK | FL_DIR)                                                       \
    X(LD_CGD, EP_CGA, FL_PEER)                                                                  \
    X(LD_CGD, EP_CGA, FL_DIR | FL_PEER)                                                         \
    X(LD_X0, EP_RESID_INIT, FL_PEER)                                                            \
    X(LD_X0, EP_RESID_INIT, FL_MASK | FL_DIR | FL_PEER)                                         \
    X(LD_RAW, EP_RESID_INIT, FL_PEER)                                                           \
    X(LD_RAW, EP_RESID_INIT, FL_MASK | FL_DIR | FL_PEER)                                        \
    X(LD_RAW, EP_RESID, FL_PEER)                                                                \
    X(LD_RAW, EP_RESID, FL_MASK | FL_DIR | FL_PEER)

template <class Real> static StencilFn stencil_fn_p(int R, int LD, int EP, int FL, int EL)
{
#define X(ld, ep, fl)                                                                           \
    if (LD == (ld) && EP == (ep) && FL == (fl)) {                                               \
        if (EL == EL_DENSE) return stencil_fn_t<2, ld, ep, fl, EL_DENSE, Real>();              \
        if (EL == EL_TETV) return stencil_fn_t<2, ld, ep, fl, EL_TETV, Real>();                \
        if constexpr (sizeof(Real) == 8)                                                        \
            if (EL == EL_Q1P)                                                                   \
                return R >= 4 ? stencil_fn_t<4, ld, ep, fl, EL_Q1P, Real>() : stencil_fn_t<2, ld, ep, fl, EL_Q1P, Real>(); \
        return R >= 4 ? stencil_fn_t<4, ld, ep, fl, EL_Q1, Real>() : stencil_fn_t<2, ld, ep, fl, EL_Q1, Real>(); \
    }
    HF_STENCIL_VARIANTS(X)
#undef X
    // single-reduction PCG kernels: fp64, Q1 elements ((k, c) pairs or material ids)
    if constexpr (sizeof(Real) == 8) {
#define Y(ld, ep, fl)                                                                           \
        if (LD == (ld) && EP == (ep) && FL == (fl) && (EL == EL_Q1 || EL == EL_Q1P)) {          \
            if (EL == EL_Q1P)                                                                   \
                return R >= 4 ? stencil_fn_t<4, ld, ep, fl, EL_Q1P, Real>() : stencil_fn_t<2, ld, ep, fl, EL_Q1P, Real>(); \
            return R >= 4 ? stencil_fn_t<4, ld, ep, fl, EL_Q1, Real>() : stencil_fn_t<2, ld, ep, fl, EL_Q1, Real>(); \
        }
        Y(LD_CG1, EP_CG1, 0)
        Y(LD_CG1, EP_CG1, FL_DIR)
        Y(LD_CG1W, EP_CG1W, 0)
        Y(LD_CG1W, EP_CG1W, FL_DIR)
#undef Y
    }
    return {nullptr, 0};
}

// es: element size of the storage type (8: fp64, 4: the fp32 variant, NEXT row f3)
static StencilFn stencil_fn(int R, int LD, int EP, int FL, int EL, int es)
{
    return es == 8 ? stencil_fn_p<double>(R, LD, EP, FL, EL) : stencil_fn_p<float>(R, LD, EP, FL, EL);
}

// element variant of the stencil kernels on this context
static int kernel_elem(const hf_ctx *c) { return c->elem == EL_DENSE && c->tetv ? EL_TETV : c->elem; }

// flags of a launch on this context
static int dir_flags(const hf_ctx *c, int EP, bool has_b, bool dset);

static std::mutex g_attr_mu;
static std::map<std::pair<const void *, int>, size_t> g_attr_done;

static hf_status ensure_smem_attr(const void *fn, size_t smem, int device)
{
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto key = std::make_pair(fn, device);
    auto it = g_attr_done.find(key);
    if (it != g_attr_done.end() && it->second >= smem) return HF_OK;
    CUCK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    g_attr_done[key] = smem;
    return HF_OK;
}

// resident CTAs per SM of this context's PCG kernel A (grid sizing of every stencil launch).
// The material-id variant (EL_Q1P) uses fewer registers and could fit 3 CTAs per SM at R = 2,
// but more, shorter z-chunks cost more than they hide (measured at C3: kernel A 18.5 vs 16.4 us),
// so grids are sized by the pair kernel for both layouts.
static hf_status update_occ(hf_ctx *c)
{
    const int el = kernel_elem(c);
    StencilFn f = stencil_fn(c->tileR, LD_CGD, EP_CGA, 0, el, c->es);
    HFCK(ensure_smem_attr(f.fn, f.smem, c->device));
    int occ = 0;
    CUCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f.fn, 32 * f.nw, f.smem));
    c->occ = std::max(1, occ);
    return HF_OK;
}

static int rows_per_tile(int R) { return NW * R - 1; }

// Tile height: R = 4 amortises the halo rows best when the stencil streams from HBM (large
// grids); below ~16M local nodes the kernel is latency-bound and R = 2 (more, shorter tiles,
// 2 CTAs/SM, less y padding at 100^3) is faster (tools/sweep_c3.py).  The dense (tet) element
// keeps R = 2 (R = 4 spills).
static int default_tile_r(const hf_ctx *c, int elem)
{
    if (elem == EL_DENSE) return 2;
    return c->nloc < (16LL << 20) ? 2 : 4;
}

// grid of the stencil over output planes [z0, z1): one (x, y) tile column per CTA, z split
// into chunks so that the grid fills the resident slots (occupancy x SMs) once.
// Stacked systems (nsys > 1): every system's planes get their own chunks (blockIdx.z = system *
// chunks + chunk), so no CTA straddles two systems and the partial sums stay per system; *zper
// receives the output planes per system.
static void stencil_grid(const hf_ctx *c, int z0, int z1, dim3 *grid, int *zchunk, int *zper)
{
    const int tx = (c->nx1 + TILE_X - 1) / TILE_X;
    const int ty = (c->ny1 + rows_per_tile(c->tileR) - 1) / rows_per_tile(c->tileR);
    const int ns = c->nsys;
    const int planes = ns > 1 ? c->sys_planes : std::max(1, z1 - z0);
    const long long cols = (long long)tx * ty;
    const long long slots = (long long)(c->nsm_share ? c->nsm_share : c->nsm) * c->occ;
    long long nch = std::max(1LL, slots / (cols * ns));
    int chunk = (int)std::max(1LL, ((long long)planes + nch - 1) / nch);
    if (c->zchunk > 0) chunk = c->zchunk;
    chunk = std::min(chunk, planes);
    nch = (planes + chunk - 1) / chunk;
    *grid = dim3(tx, ty, (unsigned)(nch * ns));
    *zchunk = chunk;
    *zper = planes;
}

// which = 0: consumes kernel A's partials, 1: consumes init/B/RESID partials, -1: none.
// pout = 0: writes A partials, 1: writes init/B/RESID partials, -1: none.  In slab mode the
// consumer reads the allreduced sums instead (count 1).
static int b_blocks(const hf_ctx *c);

// CTAs of this context's stencil launches over its owned planes (every stencil launch of a
// context has this grid)
static int stencil_blocks(const hf_ctx *c)
{
    dim3 grid;
    int chunk, zper;
    stencil_grid(c, c->own_lo, c->own_hi, &grid, &chunk, &zper);
    return (int)(grid.x * grid.y * grid.z);
}

// Fixed partial counts (one system, no slab transport): every producer of the init / B / RESID
// buffer writes max(B blocks, stencil blocks) entries (zero-padded), the A buffer holds the
// stencil grid's, so consumers know the count before they read the state header.
static Sync make_sync(hf_ctx *c, Sys &s, int consumes = -1, int produces = -1)
{
    Sync y;
    std::memset(&y, 0, sizeof(y));
    y.st = s.st;
    y.launches = c->launches;
    y.nsys = c->nsys;
    const bool fixed = c->nsys == 1 && !c->comm;
    const int nb_st = fixed ? stencil_blocks(c) : 0;
    const int nb_b = fixed ? std::max(b_blocks(c), nb_st) : 0;
    if (consumes >= 0) {
        if (c->comm && !c->comm->in_kernel()) { y.pin = s.sums; y.pin_n = 1; }
        else { y.pin = consumes == 0 ? s.partA : s.partB; y.pin_n = fixed ? (consumes == 0 ? nb_st : nb_b) : -1; }
    }
    if (produces >= 0) {
        y.pout = produces == 0 ? s.partA : s.partB;
        if (fixed && produces == 1) y.pout_pad = nb_b;
    }
    y.peer = c->comm ? c->comm->peer_dev() : nullptr;
    return y;
}

static StencilArgs base_args(hf_ctx *c, double aK, double aM)
{
    StencilArgs a;
    std::memset(&a, 0, sizeof(a));
    a.g = make_geom(c);
    a.lam = make_lam(c->g.h, aK, aM);
    for (int ch = 0; ch < 4; ch++) {
        a.lamf.ka[ch] = (float)a.lam.ka[ch];
        a.lamf.ma[ch] = (float)a.lam.ma[ch];
        a.lamf.kb[ch] = (float)a.lam.kb[ch];
        a.lamf.mb[ch] = (float)a.lam.mb[ch];
    }
    if (c->elem == EL_DENSE && c->tetv) {
        double K[6][16], V;
        tet_matrices(c->g.h, K, &V);
        for (int t = 0; t < 6; t++)
            for (int i = 0; i < 16; i++) {
                a.tv.K[t][i] = aK * K[t][i];
                a.tvf.K[t][i] = (float)a.tv.K[t][i];
            }
        a.tv.m = aM * V / 20.0;
        a.tvf.m = (float)a.tv.m;
    }
    if (c->elem == EL_DENSE) {
        double K[64], M[64];
        tet_voxel(c->g.h, K, M);
        for (int i = 0; i < 64; i++) {
            a.dn.K[i] = aK * K[i];
            a.dn.M[i] = aM * M[i];
            a.dnf.K[i] = (float)a.dn.K[i];
            a.dnf.M[i] = (float)a.dn.M[i];
        }
    }
    a.c = 1.0;
    a.s = 0.0;
    a.z_out0 = c->own_lo;
    a.z_out1 = c->own_hi;
    a.zs0 = c->own_lo;
    a.zs1 = c->own_hi;
    a.gz_lo = a.gz_hi = -1000;
    return a;
}

static int dir_flags(const hf_ctx *c, int EP, bool has_b, bool dset)
{
    int fl = has_b && EP == EP_APPLY ? FL_HB : 0;
    if (EP != EP_APPLY && c->comm && c->comm->in_kernel()) fl |= FL_PEER;   // mailbox sums / ghosts
    if (c->dbits) {
        if (EP == EP_APPLY) { if (dset) fl |= FL_DIR | FL_DSET; }
        else if (EP == EP_CGA || EP == EP_CG1 || EP == EP_CG1W) fl |= FL_DIR;
        else fl |= FL_MASK | FL_DIR;
    }
    return fl;
}

// Device copies of TMA descriptor sets.  They live in a per-device arena that is never freed and
// is deduplicated by content, so a descriptor address is written exactly once in the life of the
// process: an SM's descriptor cache can never hold a stale entry for it, and the kernels need no
// fence.proxy.tensormap acquire (which cost 1.6 us per C3 PCG iteration: every CTA re-fetched its
// 3 descriptors).  Growth is bounded by the number of distinct descriptor sets the process
// creates (1 KB each; a context creates a few, hf_apply one per distinct user buffer).
// Descriptors in kernel parameter space were not reliable for kernels launched from graph
// conditional bodies of concurrently running graphs (intermittent TMA transaction-count faults
// and hangs with two batched streams; tools/stress_batched.sh), hence device memory.
static std::mutex g_maps_mu;
static std::map<std::pair<int, std::string>, void *> g_maps;       // (device, content) -> address
static std::map<int, std::pair<char *, size_t>> g_maps_chunk;      // device -> (chunk, used bytes)

static hf_status maps_dev(hf_ctx *c, const Maps &m, const CUtensorMap **out)
{
    std::lock_guard<std::mutex> lk(g_maps_mu);
    auto key = std::make_pair(c->device, std::string((const char *)&m, sizeof(Maps)));
    auto it = g_maps.find(key);
    if (it != g_maps.end()) { *out = (const CUtensorMap *)it->second; return HF_OK; }
    const size_t chunk = 256 * sizeof(Maps);
    auto &ch = g_maps_chunk[c->device];
    if (!ch.first || ch.second + sizeof(Maps) > chunk) {
        void *p = nullptr;
        CUCK(cudaMalloc(&p, chunk));                                // never freed (see above)
        ch = {(char *)p, 0};
    }
    void *d = ch.first + ch.second;
    ch.second += sizeof(Maps);
    CUCK(cudaMemcpy(d, &m, sizeof(Maps), cudaMemcpyHostToDevice));
    g_maps.emplace(key, d);
    *out = (const CUtensorMap *)d;
    return HF_OK;
}

// stencil launch spec.  dset: EP_APPLY writes g on Dirichlet rows (RHS / lift); the plain
// apply (hf_apply) is the unconstrained operator.
static hf_status stencil_launch(hf_ctx *c, int LD, int EP, bool dset, const Maps &maps, StencilArgs a, int cls,
                                Launch *out, int extra_fl = 0)
{
    const int FL = dir_flags(c, EP, a.bvec != nullptr, dset) | extra_fl;
    int el = kernel_elem(c);
    if (el == EL_Q1 && c->pal_on && std::memcmp(&maps.kc, &c->kid_map, sizeof(CUtensorMap)) == 0) {
        el = EL_Q1P;                          // this map set streams material ids (sys0 of the context)
        std::memcpy(a.pal, c->pal, sizeof(a.pal));
        a.npal = c->npal;
    }
    StencilFn f = stencil_fn(c->tileR, LD, EP, FL, el, c->es);
    if (!f.fn) return fail(HF_E_ARG, "internal: no stencil instantiation");
    HFCK(ensure_smem_attr(f.fn, f.smem, c->device));
    dim3 grid;
    int chunk, zper;
    stencil_grid(c, a.z_out0, a.z_out1, &grid, &chunk, &zper);
    a.zchunk = chunk;
    a.zper_out = zper;
    Launch L;
    L.fn = f.fn;
    L.grid = grid;
    L.block = dim3(32, f.nw, 1);
    L.smem = f.smem;
    HFCK(maps_dev(c, maps, &a.tm));
    a.tm_fence = c->tm_fence;
    L.add(a);
    L.cls = cls;
    *out = L;
    return HF_OK;
}

// Kernel B's grid: 3 CTAs per SM.  Every CTA first reduces kernel A's partials (~9 KB of L2
// reads each); fewer CTAs doing more sweeps measured best at C3 (per-iteration 25.3 / 24.3 / 24.7 /
// 25.9 / 27.2 us for 4 / 3 / 2 / 6 / 8 per SM; 4 pairs per thread per sweep instead of 2: no gain).
static int b_blocks(const hf_ctx *c)
{
    const int per_sm = 3;
    const long long sysn = c->nloc / c->nsys;
    const int nsm = c->nsm_share ? c->nsm_share : c->nsm;
    const int bps = std::max(1, std::min((int)((sysn + 1023) / 1024), nsm * per_sm / c->nsys));
    return bps * c->nsys;                  // bps blocks per system, contiguous
}

static hf_status run(hf_ctx *c, const Launch &L, cudaStream_t s)
{
    void *args[4];
    for (size_t i = 0; i < L.args.size(); i++) args[i] = (void *)L.args[i].data();
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->prof) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s);
    }
    CUCK(cudaLaunchKernel(L.fn, L.grid, L.block, args, L.smem, s));
    if (c->prof) {
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        c->prof_ms[L.cls] += ms;
        c->prof_n[L.cls] += 1;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    return HF_OK;
}

static hf_status add_node(cudaGraph_t g, const Launch &L, cudaGraphNode_t *dep, cudaGraphNode_t *out)
{
    cudaKernelNodeParams p;
    std::memset(&p, 0, sizeof(p));
    void *args[4];
    for (size_t i = 0; i < L.args.size(); i++) args[i] = (void *)L.args[i].data();
    p.func = (void *)L.fn;
    p.gridDim = L.grid;
    p.blockDim = L.block;
    p.sharedMemBytes = (unsigned)L.smem;
    p.kernelParams = args;
    CUCK(cudaGraphAddKernelNode(out, g, dep, dep ? 1 : 0, &p));
    return HF_OK;
}

// edge from -> to of type Programmatic: `to` may launch once every CTA of `from` has called
// griddepcontrol.launch_dependents (or exited); it waits for `from` with griddepcontrol.wait
static hf_status add_pdl_edge(cudaGraph_t g, cudaGraphNode_t from, cudaGraphNode_t to)
{
    cudaGraphEdgeData e;
    std::memset(&e, 0, sizeof(e));
    e.from_port = cudaGraphKernelNodePortProgrammatic;
    e.type = cudaGraphDependencyTypeProgrammatic;
    CUCK(cudaGraphAddDependencies_v2(g, &from, &to, &e, 1));
    return HF_OK;
}

// ============================================================================================
// workspace

static hf_status sys_maps(hf_ctx *c, Sys &s)
{
    for (int i = 0; i < 3; i++) HFCK(node_map(c, s.U[i], &s.maps.node[MAP_U0 + i]));
    for (int i = 0; i < 2; i++) HFCK(node_map(c, s.dbuf[i], &s.maps.node[MAP_D0 + i]));
    HFCK(node_map(c, s.s, &s.maps.node[MAP_S]));
    if (&s == &c->sys0 && c->pal_on && c->elem == EL_Q1 && c->es == 8) {
        HFCK(kid_map_enc(c, c->kid, &c->kid_map));
        s.maps.kc = c->kid_map;
    } else HFCK(kc_map(c, s.kc, &s.maps.kc));
    if (s.kcn) HFCK(kcn_map(c, s.kcn, &s.maps.kcn));
    else s.maps.kcn = s.maps.kc;            // unused unless EL_TETV
    if (c->ghost_buf) HFCK(node_map(c, (const double *)c->ghost_buf, &s.maps.ghost, 2, c->ghost_pb));
    else s.maps.ghost = s.maps.node[MAP_S];  // unused without the peer transport
    return HF_OK;
}

static hf_status sys_alloc(hf_ctx *c, Sys &s, cudaStream_t stream)
{
    const size_t vb = (size_t)c->nloc * c->es;
    double **vecs[] = {&s.U[0], &s.U[1], &s.U[2], &s.b, &s.r, &s.s, &s.q, &s.invd, &s.dbuf[0], &s.dbuf[1]};
    for (double **v : vecs) {
        CUCK(cudaMalloc(v, vb));
        CUCK(cudaMemsetAsync(*v, 0, vb, stream));   // pitch padding must stay zero
    }
    CUCK(cudaMalloc(&s.kc, (size_t)c->kc_elems * 2 * c->es));
    CUCK(cudaMemsetAsync(s.kc, 0, (size_t)c->kc_elems * 2 * c->es, stream));
    CUCK(cudaMalloc(&s.st, c->nsys * sizeof(CgState)));
    CUCK(cudaMallocHost(&s.st_host, c->nsys * sizeof(CgState)));
    CUCK(cudaMalloc(&s.partA, (size_t)c->max_blocks * NPART * sizeof(double)));
    CUCK(cudaMalloc(&s.partB, (size_t)c->max_blocks * NPART * sizeof(double)));
    CUCK(cudaMalloc(&s.sums, NPART * sizeof(double)));
    CUCK(cudaMalloc(&s.gbar, sizeof(unsigned long long)));
    CUCK(cudaMemsetAsync(s.gbar, 0, sizeof(unsigned long long), stream));
    std::memset(s.st_host, 0, c->nsys * sizeof(CgState));
    for (int j = 0; j < c->nsys; j++) s.st_host[j].first_failed = -1;
    CUCK(cudaMemcpyAsync(s.st, s.st_host, c->nsys * sizeof(CgState), cudaMemcpyHostToDevice, stream));
    s.stream = stream;
    HFCK(sys_maps(c, s));
    CUCK(cudaStreamSynchronize(stream));
    return HF_OK;
}

static void sys_free(Sys &s)
{
    for (int i = 0; i < 3; i++) cudaFree(s.U[i]);
    cudaFree(s.b); cudaFree(s.r); cudaFree(s.s); cudaFree(s.q); cudaFree(s.invd);
    cudaFree(s.dbuf[0]); cudaFree(s.dbuf[1]);
    for (int k = 0; k < 2; k++) { cudaFree(s.c1r[k]); cudaFree(s.c1w[k]); cudaFree(s.c1s[k]); }
    cudaFree(s.c1p);
    cudaFree(s.st); cudaFreeHost(s.st_host);
    cudaFree(s.partA); cudaFree(s.partB); cudaFree(s.sums); cudaFree(s.iters); cudaFree(s.gbar);
    if (s.st_ring) cudaFreeHost(s.st_ring);
    for (int i = 0; i < 2; i++) if (s.ev_ring[i]) cudaEventDestroy(s.ev_ring[i]);
    cudaFree(s.kc);
    cudaFree(s.kcn);
    if (s.gexec) cudaGraphExecDestroy(s.gexec);
    if (s.graph) cudaGraphDestroy(s.graph);
    if (s.own_stream && s.stream) cudaStreamDestroy(s.stream);
    s = Sys();
}

// padded layouts of the storage type: node rows 16-B multiples (TMA strides), fp32 (k, c) rows
// an even number of pairs
static void set_layout(hf_ctx *c)
{
    const int q = 16 / c->es;
    c->pitch = (c->nx1 + q - 1) / q * q;
    c->kpitch = c->es == 8 ? (int)c->g.ne[0] : ((int)c->g.ne[0] + 1) & ~1;
    c->plane = (long long)c->pitch * c->ny1;
    c->nloc = c->plane * c->nzl;
    c->kc_elems = (long long)c->kpitch * c->g.ne[1] * (c->nzl + 1);
}

// The library's only reads of the environment: defaults of the tuning knobs for tools and
// experiments, read once when a context is created (hf_set_tuning / hf_set_driver /
// hf_set_resident override them per context; see heatfem.h).
static void tuning_from_env(hf_ctx *c)
{
    if (const char *e = getenv("HF_TILE_R")) c->tile_r_set = atoi(e) >= 4 ? 4 : 2;
    if (const char *e = getenv("HF_ZCHUNK")) c->zchunk = std::max(0, atoi(e));
    if (const char *e = getenv("HF_DRIVER")) c->driver = atoi(e) != 0;
    if (const char *e = getenv("HF_UNROLL")) c->unroll = std::min(50, std::max(1, atoi(e)));
    if (const char *e = getenv("HF_PDL")) c->pdl = atoi(e) != 0;
    if (const char *e = getenv("HF_FUSE_AB")) c->fuse_ab = atoi(e) != 0;
    if (const char *e = getenv("HF_CHECK_EVERY")) c->check_every = std::max(1, atoi(e));
    if (const char *e = getenv("HF_TM_FENCE")) c->tm_fence = atoi(e) != 0;
    if (const char *e = getenv("HF_RESIDENT")) c->resident = atoi(e) != 0;
    if (const char *e = getenv("HF_BATCH_GROUP")) c->batch_group = std::max(0, atoi(e));
    if (const char *e = getenv("HF_COMM_TIMEOUT_S")) c->comm_timeout_s = atof(e);
}

static hf_status ctx_init(hf_ctx *c, const hf_grid *g, int device, void *stream, int rank, int nranks, int nsys = 1)
{
    for (int d = 0; d < 3; d++)
        if (g->ne[d] < 1 || !(g->h[d] > 0.0)) return fail(HF_E_ARG, "grid: ne must be >= 1 and h > 0");
    if (g->ne[0] > 1000000 || g->ne[1] > 1000000) return fail(HF_E_ARG, "grid too large");
    c->g = *g;
    c->device = device;
#ifdef HF_DEBUG_WAIT
    if (!g_dbg_host) {
        cudaSetDevice(device);
        cudaHostAlloc((void **)&g_dbg_host, 16 * sizeof(unsigned long long), cudaHostAllocMapped);
        std::memset(g_dbg_host, 0, 16 * sizeof(unsigned long long));
        unsigned long long *dp = nullptr;
        cudaHostGetDevicePointer((void **)&dp, g_dbg_host, 0);
        cudaMemcpyToSymbol(g_dbg, &dp, sizeof(dp));
        std::thread([] {
            for (;;) {
                std::this_thread::sleep_for(std::chrono::seconds(4));
                volatile unsigned long long *h = g_dbg_host;
                fprintf(stderr, "[hf debug] heartbeat sysA it %llu step %llu n %llu | sysB it %llu step %llu n %llu | stuck %llu\n",
                        h[10], h[11], h[12], h[13], h[14], h[15], h[0]);
                dbg_dump();
            }
        }).detach();
    }
#endif
    CUCK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUCK(cudaGetDeviceProperties(&prop, device));
    c->nsm = prop.multiProcessorCount;
    if (stream) c->stream = (cudaStream_t)stream;
    else { CUCK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)); c->own_stream = true; }
    c->nx1 = (int)g->ne[0] + 1;
    c->ny1 = (int)g->ne[1] + 1;
    c->nz1g = (int)g->ne[2] + 1;
    c->rank = rank;
    c->nranks = nranks;
    int64_t lo = 0, hi = c->nz1g;
    if (nranks > 1) HFCK(hf_slab_plan(c->nz1g, rank, nranks, &lo, &hi));
    const int glo = (int)lo - (rank > 0 ? 1 : 0);
    const int ghi = (int)hi + (rank < nranks - 1 ? 1 : 0);
    c->zg0 = glo;
    c->nzl = ghi - glo;
    c->own_lo = (int)lo - glo;
    c->own_hi = (int)hi - glo;
    c->nsys = std::max(1, nsys);
    if (c->nz1g % c->nsys != 0 || (c->nsys > 1 && nranks > 1)) return fail(HF_E_ARG, "internal: bad system stack");
    c->sys_planes = c->nzl / c->nsys;
    set_layout(c);
    const double hx = g->h[0], hy = g->h[1], hz = g->h[2];
    for (int l = 0; l < 8; l++) {     // Q1: the same for every local node
        c->dg.Kd[l] = (hy * hz / hx + hx * hz / hy + hx * hy / hz) / 9.0;
        c->dg.Md[l] = hx * hy * hz / 27.0;
    }
    tuning_from_env(c);
    c->tileR = c->tile_r_set ? c->tile_r_set : default_tile_r(c, EL_Q1);
    // resident CTAs per SM of the CG stencil decide the z split of the grid
    StencilFn f = stencil_fn(c->tileR, LD_CGD, EP_CGA, 0, c->elem, c->es);
    HFCK(ensure_smem_attr(f.fn, f.smem, device));
    int occ = 0;
    CUCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f.fn, 32 * f.nw, f.smem));
    c->occ = std::max(1, occ);
    // partial-sum buffers sized for any tile height / z split (upper bound: one plane per CTA)
    {
        const long long tx = (c->nx1 + TILE_X - 1) / TILE_X, ty = (c->ny1 + rows_per_tile(2) - 1) / rows_per_tile(2);
        const long long worst = tx * ty * std::max(1, c->own_hi - c->own_lo);
        c->max_blocks = (int)std::max<long long>(worst, std::max(b_blocks(c), c->nsm * 4));
    }
    CUCK(cudaMalloc(&c->launches, sizeof(unsigned long long)));
    CUCK(cudaMemsetAsync(c->launches, 0, sizeof(unsigned long long), c->stream));
    HFCK(sys_alloc(c, c->sys0, c->stream));
    return HF_OK;
}

static void ctx_free(hf_ctx *c);

// batched stacks copy the operator settings (Dirichlet faces, element, precision, driver) of
// their parent when created: every setter that changes them drops the stacks
static void drop_stacks(hf_ctx *c)
{
    for (auto &kv : c->stacks) { ctx_free(kv.second); delete kv.second; }
    c->stacks.clear();
}

static void ctx_free(hf_ctx *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    sys_free(c->sys0);
    for (void *p : c->scratch) cudaFree(p);
    cudaFree(c->launches);
    cudaFree(c->flush);
    cudaFree(c->ab_A);
    cudaFree(c->ab_contrib);
    cudaFree(c->kid);
    cudaFree(c->rsync);
    cudaFree(c->res_prof);
    cudaFree(c->mix_iters);
    if (c->mix_exec) cudaGraphExecDestroy(c->mix_exec);
    if (c->mix_graph) cudaGraphDestroy(c->mix_graph);
    if (c->lo) { ctx_free(c->lo); delete c->lo; c->lo = nullptr; }
    for (auto &kv : c->stacks) { ctx_free(kv.second); delete kv.second; }
    c->stacks.clear();
    delete c->comm;
    if (c->own_stream) cudaStreamDestroy(c->stream);
}

// ============================================================================================
// building blocks

static hf_status enqueue_pack(hf_ctx *c, Sys &s, const double *k, const double *cc)
{
    const long long n = c->kc_elems;
    const int bs = 256;
    if (c->es == 8)
        k_pack<double><<<(unsigned)((n + bs - 1) / bs), bs, 0, s.stream>>>(make_geom(c), (int)c->g.ne[2], k, cc, s.kc,
                                                                           n, c->launches);
    else
        k_pack<float><<<(unsigned)((n + bs - 1) / bs), bs, 0, s.stream>>>(make_geom(c), (int)c->g.ne[2], k, cc, s.kc,
                                                                          n, c->launches);
    CUCK(cudaGetLastError());
    return HF_OK;
}

static hf_status enqueue_diag(hf_ctx *c, Sys &s, double aK, double aM, double *diag, double *invd)
{
    const int bs = 256;
    const unsigned nb = (unsigned)((c->nloc + bs - 1) / bs);
    if (kernel_elem(c) == EL_TETV) {
        TetDiag td;
        double K[6][16], V;
        tet_matrices(c->g.h, K, &V);
        for (int t = 0; t < 6; t++)
            for (int v = 0; v < 4; v++) td.kd[t][v] = K[t][v * 5];
        td.md = 2.0 * V / 20.0;
        if (c->es == 8) k_diag_tv<double><<<nb, bs, 0, s.stream>>>(make_geom(c), s.kcn, aK, aM, td, diag, invd, c->launches);
        else k_diag_tv<float><<<nb, bs, 0, s.stream>>>(make_geom(c), s.kcn, aK, aM, td, diag, invd, c->launches);
    } else if (c->es == 8) k_diag<double><<<nb, bs, 0, s.stream>>>(make_geom(c), s.kc, aK, aM, c->dg, diag, invd, c->launches);
    else k_diag<float><<<nb, bs, 0, s.stream>>>(make_geom(c), s.kc, aK, aM, c->dg, diag, invd, c->launches);
    CUCK(cudaGetLastError());
    return HF_OK;
}

static hf_status enqueue_set_dirichlet(hf_ctx *c, Sys &s, double *v, const double *src)
{
    if (!c->dbits) return HF_OK;
    const int bs = 256;
    const unsigned nb = (unsigned)((c->nloc + bs - 1) / bs);
    if (c->es == 8) k_set_dirichlet<double><<<nb, bs, 0, s.stream>>>(make_geom(c), v, src, c->launches);
    else k_set_dirichlet<float><<<nb, bs, 0, s.stream>>>(make_geom(c), v, src, c->launches);
    CUCK(cudaGetLastError());
    return HF_OK;
}

// PCG kernels of one iteration for system s, in order.
struct CgLaunches {
    Launch A, B, RES;
    Launch AB;                       // A and B in one launch with a grid barrier (FL_FUSEB)
    bool has_ab = false;
};

// x: the iterate (NULL: the time-step ring slot U[(step+1)%3]); xmaps: maps with node[0] = x
static hf_status cg_launches(hf_ctx *c, Sys &s, double aK, double aM, double *x, const Maps &xmaps, CgLaunches *L)
{
    const bool rot = x == nullptr;
    // kernel A: d = s + beta d; q = A d; d^T q -> alpha   (Alg. 1 lines 7-8, 15, 18)
    StencilArgs a = base_args(c, aK, aM);
    a.dbuf[0] = s.dbuf[0];
    a.dbuf[1] = s.dbuf[1];
    a.out0 = s.q;
    a.zs0 = c->own_lo - (c->own_lo > 0 ? 1 : 0);   // store d on ghost planes too (slab)
    a.zs1 = c->own_hi + (c->own_hi < c->nzl ? 1 : 0);
    a.dmode = 1;
    a.sy = make_sync(c, s, 1, 0);
    if (a.sy.peer) {                               // s of the ghost planes: the neighbours' stores
        a.gz_lo = c->own_lo > 0 ? c->own_lo - 1 : -1000;
        a.gz_hi = c->own_hi < c->nzl ? c->own_hi : -1000;
    }
    HFCK(stencil_launch(c, LD_CGD, EP_CGA, false, s.maps, a, 0, &L->A));
    // kernel B: x += alpha d; r -= alpha q; s = P^{-1} r; r^T s, r^T r -> beta   (lines 9-19)
    BArgs b;
    std::memset(&b, 0, sizeof(b));
    b.x = x;
    b.q = s.q;
    b.invd = s.invd;
    b.dbuf[0] = s.dbuf[0];
    b.dbuf[1] = s.dbuf[1];
    b.r = s.r;
    b.s = s.s;
    b.n = c->nloc;
    b.sysn = c->nloc / c->nsys;
    b.own0 = (long long)c->own_lo * c->plane;
    b.own1 = (long long)c->own_hi * c->plane;
    if (rot) for (int i = 0; i < 3; i++) b.rot[i] = s.U[i];
    b.sy = make_sync(c, s, 0, 1);
    L->B = Launch();
    const bool peer = c->comm && c->comm->in_kernel();
    L->B.fn = c->es == 8 ? (peer ? (const void *)k_cg_b<256, double, true> : (const void *)k_cg_b<256, double, false>)
                         : (peer ? (const void *)k_cg_b<256, float, true> : (const void *)k_cg_b<256, float, false>);
    L->B.grid = dim3(b_blocks(c));
    L->B.block = dim3(256);
    L->B.add(b);
    L->B.cls = 1;
    // the fused A+B launch for graph loop bodies of the context's own system (no slabs: their
    // exchange and allreduce sit between A and B).  Its grid barrier needs every CTA resident
    // at once: used only if the occupancy API says the whole grid fits.
    L->has_ab = false;
    if (c->fuse_ab && !c->comm && c->nsys == 1) {
        StencilArgs f = a;
        f.fb = b;
        f.gbar = s.gbar;
        HFCK(stencil_launch(c, LD_CGD, EP_CGA, false, s.maps, f, 0, &L->AB, FL_FUSEB));
        int occ = 0;
        CUCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, L->AB.fn, 32 * L->AB.block.y, L->AB.smem));
        const long long grid = (long long)L->AB.grid.x * L->AB.grid.y * L->AB.grid.z;
        L->has_ab = (long long)occ * c->nsm >= grid;
    }
    // residual replacement r = b - A x every replace_every iterations (Alg. 1 lines 10-11)
    StencilArgs rr = base_args(c, aK, aM);
    rr.invd = s.invd;
    rr.bvec = s.b;
    rr.out0 = s.r;
    rr.out_s = s.s;
    rr.sy = make_sync(c, s, -1, 1);
    if (rot) rr.rot_role = ROT_X;
    HFCK(stencil_launch(c, LD_RAW, EP_RESID, true, rot ? s.maps : xmaps, rr, 2, &L->RES));
    return HF_OK;
}

// slab mode, after a producer kernel: local sums -> allreduce -> (ghosts of s for the next apply)
static hf_status comm_after(hf_ctx *c, Sys &s, int which, bool exch)
{
    if (!c->comm || c->comm->in_kernel()) return HF_OK;
    Sync sy = make_sync(c, s);
    sy.pin = which == 0 ? s.partA : s.partB;
    k_localsum<<<1, 256, 0, s.stream>>>(sy, which, s.sums);
    CUCK(cudaGetLastError());
    HFCK(c->comm->allreduce(c, s, s.sums, NPART));
    if (exch) HFCK(c->comm->exchange(c, s, s.s));
    return HF_OK;
}

static hf_status read_state(hf_ctx *c, Sys &s)
{
    CUCK(cudaMemcpyAsync(s.st_host, s.st, c->nsys * sizeof(CgState), cudaMemcpyDeviceToHost, s.stream));
    CUCK(cudaStreamSynchronize(s.stream));
    return HF_OK;
}

// options and counters of a new solve / run, written without a device round trip
// replace_every < 0: the context default, 50 (Alg. 1, R6) in fp64, 0 in the fp32 variant (R18)
static hf_cg_opts resolved(const hf_ctx *c, hf_cg_opts o)
{
    if (o.replace_every < 0) o.replace_every = c->es == 8 ? 50 : 0;
    return o;
}

static hf_status set_solver_opts(hf_ctx *c, Sys &s, const hf_cg_opts &d0)
{
    const hf_cg_opts d = resolved(c, d0);
    if (!(d.rtol >= 0.0) || d.max_iter < 0) return fail(HF_E_ARG, "bad hf_cg_opts");
    CUCK(cudaStreamSynchronize(s.stream));     // the pinned image may still be in flight
    for (int j = 0; j < c->nsys; j++) {       // every system: its own scalars, the same options
        CgState &h = s.st_host[j];
        std::memset(&h, 0, sizeof(h));
        h.rtol2 = d.rtol * d.rtol;
        h.max_iter = d.max_iter;
        h.replace_every = d.replace_every;
        h.first_failed = -1;
    }
    CUCK(cudaMemcpyAsync(s.st, s.st_host, c->nsys * sizeof(CgState), cudaMemcpyHostToDevice, s.stream));
    return HF_OK;
}

static StepArgs step_args(hf_ctx *c, Sys &s, double *x, double *snapdev, int snap_local)
{
    StepArgs a;
    std::memset(&a, 0, sizeof(a));
    a.g = make_geom(c);
    a.x = x;
    if (!x) for (int i = 0; i < 3; i++) a.rot[i] = s.U[i];
    a.n = c->nloc;
    a.sysn = c->nloc / c->nsys;
    a.snap = snapdev;
    a.snap_plane = snap_local;
    a.iters_out = s.iters;
    a.sy = make_sync(c, s);
    return a;
}

// end of a solve / time step: k_step_end (x_F = 0 if b_F = 0, snapshot) + k_step_commit
static std::vector<Launch> step_launches(hf_ctx *c, const StepArgs &a, bool commit)
{
    std::vector<Launch> v;
    Launch L;
    L.fn = c->es == 8 ? (const void *)k_step_end<double> : (const void *)k_step_end<float>;
    L.grid = dim3(std::max(1, std::min(c->nsm, (int)((c->nloc + 255) / 256))));
    L.block = dim3(256);
    L.add(a);
    L.cls = 4;
    v.push_back(L);
    if (commit) {
        Launch C;
        C.fn = (const void *)k_step_commit;
        C.grid = dim3(1);
        C.block = dim3(std::min(256, ((c->nsys + 31) / 32) * 32));
        C.add(a.sy);
        C.add(a.iters_out);
        C.cls = 4;
        v.push_back(C);
    }
    return v;
}

// ---- host-loop PCG (profiling, slab transports) ------------------------------------------
// one PCG iteration on the host-loop driver (slab transports exchange / allreduce in between)
static hf_status host_cg_iter(hf_ctx *c, Sys &s, CgLaunches &L, int i, int replace_every)
{
    HFCK(run(c, L.A, s.stream));
    HFCK(comm_after(c, s, 0, false));
    const bool rep = i > 0 && replace_every > 0 && i % replace_every == 0;
    HFCK(run(c, L.B, s.stream));
    if (!rep) HFCK(comm_after(c, s, 1, true));
    if (rep) {
        HFCK(run(c, L.RES, s.stream));
        HFCK(comm_after(c, s, 1, true));
    }
    return HF_OK;
}

// Host loop without a stall per check: after every batch of `check` iterations the state is
// copied to pinned memory with an event behind it, and batch k + 1 is enqueued before batch
// k - 1's copy is waited on, so the stream always holds queued work.  Iterations enqueued after
// convergence exit at their first instruction (the kernels test `active`); every rank of a slab
// run enqueues the same sequence (the stop decision comes from allreduced sums).
// wait for an event of the host loop; slab transports are polled for asynchronous errors, and a
// wait beyond HF_COMM_TIMEOUT_S (default 120 s) fails instead of hanging on a dead peer
static hf_status wait_event(hf_ctx *c, cudaEvent_t ev)
{
    if (!c->comm) { CUCK(cudaEventSynchronize(ev)); return HF_OK; }
    const double limit = c->comm_timeout_s;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t q = cudaEventQuery(ev);
        if (q == cudaSuccess) return HF_OK;
        if (q != cudaErrorNotReady) CUCK(q);
        HFCK(c->comm->poll());
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
            return fail(HF_E_NCCL, "slab transport: no progress within HF_COMM_TIMEOUT_S");
        std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
}

static hf_status host_cg_loop_pipelined(hf_ctx *c, Sys &s, CgLaunches &L, int max_iter, int replace_every,
                                        int check)
{
    if (!s.st_ring) {
        CUCK(cudaMallocHost(&s.st_ring, 2 * sizeof(CgState)));
        CUCK(cudaEventCreateWithFlags(&s.ev_ring[0], cudaEventDisableTiming));
        CUCK(cudaEventCreateWithFlags(&s.ev_ring[1], cudaEventDisableTiming));
    }
    int i = 0, batch = 0;
    bool pending[2] = {false, false};
    for (;;) {
        const int slot = batch & 1;
        // the device ends the solve itself (kernel A of iteration max_iter records NOCONV), so
        // batches are enqueued until a copied state says inactive; the bound is a safety net
        for (int k = 0; k < check; k++, i++) HFCK(host_cg_iter(c, s, L, i, replace_every));
        CUCK(cudaMemcpyAsync(&s.st_ring[slot], s.st, sizeof(CgState), cudaMemcpyDeviceToHost, s.stream));
        CUCK(cudaEventRecord(s.ev_ring[slot], s.stream));
        pending[slot] = true;
        const int prev = slot ^ 1;
        if (i > max_iter + 2 * check + 2) break;
        if (pending[prev]) {                      // the batch before this one
            HFCK(wait_event(c, s.ev_ring[prev]));
            pending[prev] = false;
            if (!s.st_ring[prev].active) break;
        }
        batch++;
    }
    CUCK(cudaStreamSynchronize(s.stream));
    *s.st_host = s.st_ring[batch & 1];
    return HF_OK;
}

static hf_status host_cg_loop(hf_ctx *c, Sys &s, CgLaunches &L, int max_iter, int replace_every)
{
    HFCK(read_state(c, s));
    if (!s.st_host->active) return HF_OK;
    const bool slab = c->comm != nullptr;
    const int check = slab && !c->comm->graph_capturable() ? 1 : c->check_every;
    if (check > 1) return host_cg_loop_pipelined(c, s, L, max_iter, replace_every, check);
    for (int i = 0;;) {
        HFCK(run(c, L.A, s.stream));
        HFCK(comm_after(c, s, 0, false));
        const bool rep = i > 0 && replace_every > 0 && i % replace_every == 0;
        HFCK(run(c, L.B, s.stream));
        if (!rep) HFCK(comm_after(c, s, 1, true));
        if (rep) {
            HFCK(run(c, L.RES, s.stream));
            HFCK(comm_after(c, s, 1, true));
        }
        i++;
        if (i % check == 0 || i >= max_iter) {
            HFCK(read_state(c, s));
            if (!s.st_host->active) break;
        }
    }
    return HF_OK;
}

// ---- graph with the device-side WHILE loop -------------------------------------------------
// root: [pre...] -> init -> WHILE(active){ A -> B -> IF(replace){ RESID } } -> [post]
// (all stencil launches carry (Maps, StencilArgs); B carries BArgs)
static hf_status build_cg_graph(hf_ctx *c, std::vector<Launch> pre, Launch init, CgLaunches L, std::vector<Launch> post,
                                int replace_every, cudaGraph_t *out, bool pdl_ok = true)
{
    const bool pdl = c->pdl && pdl_ok;
    cudaGraph_t g;
    CUCK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw, hi;
    CUCK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t prev = nullptr, n;
    if (pdl && L.has_ab) {
        // the fused A+B launch's grid barrier counts arrivals in multiples of its grid size: every
        // launch of this graph starts it from zero (the grid may differ from an earlier graph's)
        unsigned long long *ctr = L.AB.get<StencilArgs>(0).gbar;
        cudaMemsetParams mp;
        std::memset(&mp, 0, sizeof(mp));
        mp.dst = ctr;
        mp.elementSize = 4;
        mp.width = 2;
        mp.height = 1;
        mp.value = 0;
        CUCK(cudaGraphAddMemsetNode(&n, g, nullptr, 0, &mp));
        prev = n;
    }
    for (auto &p : pre) { HFCK(add_node(g, p, prev ? &prev : nullptr, &n)); prev = n; }
    // the loop is entered once at least; kernel A of the iteration after the last decides to
    // stop (it clears the WHILE handle), kernel B sets the IF handle of the replacement
    HFCK(add_node(g, init, prev ? &prev : nullptr, &n));
    prev = n;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hw;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CUCK(cudaGraphAddNode(&wnode, g, &prev, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // the body holds `unroll` copies of [A -> B -> IF(RES)]; copies after convergence exit at once.
    // Every body starts at an iteration that is a multiple of `unroll`, so when unroll divides the
    // replacement period only the first copy can meet a replacement iteration: the others get no
    // IF node (an IF node costs about a microsecond per evaluation).
    // Copies per body: with programmatic edges a long chain of copies keeps the GPU fed (C3:
    // 25.0 / 23.9 / 23.4 / 23.5 us per iteration for 5 / 10 / 25 / 50), but copies after
    // convergence still launch, which small grids (short iterations, few per step) feel more:
    // 25 from 0.5M nodes, else 5.  Reduced to a divisor of the replacement period so that only
    // the first copy needs an IF node.
    int U = c->unroll > 0 ? c->unroll : (c->nloc >= 500000 ? 25 : 5);
    if (replace_every > 0)
        while (U > 1 && replace_every % U != 0) U--;
    const bool if_first_only = replace_every > 0 && replace_every % U == 0;
    cudaGraphNode_t bprev = nullptr;
    bool bprev_is_b = false;
    for (int u = 0; u < U; u++) {
        const bool with_if = replace_every > 0 && !(u > 0 && if_first_only);
        if (with_if) CUCK(cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault));
        Launch A = L.A, B = L.B, RES = L.RES;
        StencilArgs aa = A.get<StencilArgs>(0);
        aa.sy.h_while = hw; aa.sy.h_if = hi; aa.sy.use_handles = 1; aa.sy.use_if = with_if;
        A.put(0, aa);
        const bool fused = pdl && L.has_ab;
        Launch AB = L.AB;
        if (fused) {
            StencilArgs fa = AB.get<StencilArgs>(0);
            fa.sy.h_while = hw; fa.sy.h_if = hi; fa.sy.use_handles = 1; fa.sy.use_if = with_if;
            fa.fb.sy.h_while = hw; fa.fb.sy.h_if = hi; fa.fb.sy.use_handles = 1; fa.fb.sy.use_if = with_if;
            AB.put(0, fa);
        }
        BArgs bb = B.get<BArgs>(0);
        bb.sy.h_while = hw; bb.sy.h_if = hi; bb.sy.use_handles = 1; bb.sy.use_if = with_if;
        B.put(0, bb);
        StencilArgs ra = RES.get<StencilArgs>(0);
        ra.sy.h_while = hw; ra.sy.h_if = hi; ra.sy.use_handles = 1; ra.sy.use_if = with_if;
        RES.put(0, ra);
        cudaGraphNode_t na, nb;
        if (fused) {
            // one launch per iteration: A, grid barrier, B (programmatic edge from the previous
            // copy's launch when no IF node sits between them)
            const bool prog_in = bprev && bprev_is_b;
            HFCK(add_node(body, AB, (bprev && !prog_in) ? &bprev : nullptr, &nb));
            if (prog_in) HFCK(add_pdl_edge(body, bprev, nb));
        } else if (pdl) {
            // A after B of the previous copy (when no IF node sits between them) and B after A
            // through programmatic edges: the next kernel's launch and prologue overlap the tail
            const bool prog_in = bprev && bprev_is_b;
            HFCK(add_node(body, A, (bprev && !prog_in) ? &bprev : nullptr, &na));
            if (prog_in) HFCK(add_pdl_edge(body, bprev, na));
            HFCK(add_node(body, B, nullptr, &nb));
            HFCK(add_pdl_edge(body, na, nb));
        } else {
            HFCK(add_node(body, A, bprev ? &bprev : nullptr, &na));
            HFCK(add_node(body, B, &na, &nb));
        }
        bprev_is_b = true;
        if (!with_if) {                          // no replacement can occur in this copy
            bprev = nb;
            continue;
        }
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hi;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t inode;
        CUCK(cudaGraphAddNode(&inode, body, &nb, 1, &ip));
        cudaGraphNode_t nr;
        HFCK(add_node(ip.conditional.phGraph_out[0], RES, nullptr, &nr));
        bprev = inode;
        bprev_is_b = false;
    }
    prev = wnode;
    for (auto &p : post) { HFCK(add_node(g, p, &prev, &n)); prev = n; }
    *out = g;
    return HF_OK;
}

// ---- single-reduction PCG (hf_set_cg_variant 1) -----------------------
// One stencil kernel per iteration (EP_CG1): the Chronopoulos-Gear arrangement of Alg. 1 keeps
// w = A u and s = A p by recurrence, so alpha_i and beta_i both follow from ONE set of sums
// (r^T u, w^T u) of the previous kernel, and the vector updates of Alg. 1 lines 9, 13, 15, 18 run
// inside the stencil kernel that computes the next w.  Kernel i has the parity k = i & 1, fixed
// per graph node (every WHILE body starts at an even iteration and holds an even number of
// copies), so its TMA maps, output buffers and partial-sum slots are bound at build time:
//   CG1(k): reads r[k], w[k], s[k] (+ P^-1) and partials P[k^1]; writes r[k^1], w[k^1], s[k^1], p,
//           x and partials P[k]
//   RES(k): r[k] = b - A x (replacement, Alg. 1 line 10); partials P[k]
//   W(k):   w[k] = A P^-1 r[k]; reads partials P[k], writes P[k^1]
// Solve: init (r[0], partials P[0]) -> W(0) -> WHILE{ CG1(0) -> [IF: RES(1) -> W(1)] -> CG1(1) -> ... }.
static bool cg1_eligible(const hf_ctx *c, const Sys &s)
{
    return c->cg1 && c->es == 8 && c->elem == EL_Q1 && c->nsys == 1 && !c->comm && &s == &c->sys0;
}

static hf_status c1_alloc(hf_ctx *c, Sys &s)
{
    if (s.c1p) return HF_OK;
    const size_t vb = (size_t)c->nloc * c->es;
    double **vecs[] = {&s.c1r[0], &s.c1r[1], &s.c1w[0], &s.c1w[1], &s.c1s[0], &s.c1s[1], &s.c1p};
    for (double **v : vecs) {
        CUCK(cudaMalloc(v, vb));
        CUCK(cudaMemsetAsync(*v, 0, vb, s.stream));   // pitch padding must stay zero
    }
    return HF_OK;
}

struct Cg1Launches {
    Launch C[2];      // iteration of parity k
    Launch W[2];      // w[k] = A P^-1 r[k]
    Launch RES[2];    // r[k] = b - A x
};

static hf_status cg1_launches(hf_ctx *c, Sys &s, double aK, double aM, Cg1Launches *L)
{
    HFCK(c1_alloc(c, s));
    dim3 grid;
    int chunk, zper;
    stencil_grid(c, c->own_lo, c->own_hi, &grid, &chunk, &zper);
    const int nb = (int)(grid.x * grid.y * grid.z);     // partials per stencil launch (same grid for all)
    double *P[2] = {s.partA, s.partB};
    for (int k = 0; k < 2; k++) {
        Maps m = s.maps, mw = s.maps;
        HFCK(node_map(c, s.c1r[k], &m.node[0]));
        HFCK(node_map(c, s.c1w[k], &m.node[1]));
        HFCK(node_map(c, s.c1s[k], &m.node[2]));
        HFCK(node_map(c, s.invd, &m.node[3]));
        for (int j = 4; j < NMAPS; j++) m.node[j] = m.node[0];    // unused (valid for the prefetch)
        mw.node[0] = m.node[0];
        mw.node[1] = m.node[3];
        for (int j = 2; j < NMAPS; j++) mw.node[j] = m.node[0];
        StencilArgs a = base_args(c, aK, aM);
        a.c1.rout = s.c1r[k ^ 1];
        a.c1.sout = s.c1s[k ^ 1];
        a.c1.wout = s.c1w[k ^ 1];
        a.c1.p = s.c1p;
        a.c1.x = nullptr;                                  // the time-step ring slot
        a.c1.par = k;
        for (int i = 0; i < 3; i++) a.ring[i] = s.U[i];
        a.sy = make_sync(c, s);
        a.sy.pin = P[k ^ 1];
        a.sy.pin_n = nb;
        a.sy.pout = P[k];
        HFCK(stencil_launch(c, LD_CG1, EP_CG1, false, m, a, 0, &L->C[k]));
        StencilArgs w = base_args(c, aK, aM);
        w.c1.wout = s.c1w[k];
        w.sy = make_sync(c, s);
        w.sy.pin = P[k];
        w.sy.pin_n = nb;
        w.sy.pout = P[k ^ 1];
        HFCK(stencil_launch(c, LD_CG1W, EP_CG1W, false, mw, w, 2, &L->W[k]));
        StencilArgs rr = base_args(c, aK, aM);
        rr.invd = s.invd;
        rr.bvec = s.b;
        rr.out0 = s.c1r[k];
        rr.out_s = s.s;                                    // (s = P^-1 r: not used by this variant)
        rr.sy = make_sync(c, s, -1, 0);
        rr.sy.pout = P[k];
        rr.rot_role = ROT_X;
        HFCK(stencil_launch(c, LD_RAW, EP_RESID, true, s.maps, rr, 2, &L->RES[k]));
    }
    return HF_OK;
}

// root: [pre...] -> init -> W(0) -> WHILE(active){ CG1(0) -> IF(replace){ RES(1) -> W(1) } -> CG1(1) -> ... }
static hf_status build_cg1_graph(hf_ctx *c, const std::vector<Launch> &pre, const Launch &init, const Cg1Launches &L,
                                 const std::vector<Launch> &post, int replace_every, cudaGraph_t *out)
{
    cudaGraph_t g;
    CUCK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw, hi = 0;
    CUCK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t prev = nullptr, n;
    for (auto &p : pre) { HFCK(add_node(g, p, prev ? &prev : nullptr, &n)); prev = n; }
    HFCK(add_node(g, init, prev ? &prev : nullptr, &n));
    prev = n;
    HFCK(add_node(g, L.W[0], &prev, &n));
    prev = n;
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hw;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t wnode;
    CUCK(cudaGraphAddNode(&wnode, g, &prev, 1, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    // an even number of copies per body (static parities), a divisor of the replacement period
    // when one exists (then only the first copy can meet a replacement iteration: one IF node)
    int U = c->unroll > 0 ? c->unroll : (c->nloc >= 500000 ? 50 : 10);
    U = std::max(2, U & ~1);
    if (replace_every > 0)
        while (U > 2 && replace_every % U != 0) U -= 2;
    const bool if_first_only = replace_every > 0 && replace_every % U == 0;
    cudaGraphNode_t bprev = nullptr;
    bool bprev_is_k = false;
    for (int u = 0; u < U; u++) {
        const int k = u & 1;
        const bool with_if = replace_every > 0 && !(u > 0 && if_first_only);
        if (with_if) CUCK(cudaGraphConditionalHandleCreate(&hi, body, 0, cudaGraphCondAssignDefault));
        Launch C = L.C[k];
        StencilArgs ca = C.get<StencilArgs>(0);
        ca.sy.h_while = hw; ca.sy.h_if = hi; ca.sy.use_handles = 1; ca.sy.use_if = with_if;
        C.put(0, ca);
        cudaGraphNode_t nc;
        if (c->pdl && bprev && bprev_is_k) {
            HFCK(add_node(body, C, nullptr, &nc));
            HFCK(add_pdl_edge(body, bprev, nc));
        } else
            HFCK(add_node(body, C, bprev ? &bprev : nullptr, &nc));
        bprev = nc;
        bprev_is_k = true;
        if (!with_if) continue;
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hi;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t inode;
        CUCK(cudaGraphAddNode(&inode, body, &nc, 1, &ip));
        cudaGraphNode_t nr, nw;
        HFCK(add_node(ip.conditional.phGraph_out[0], L.RES[k ^ 1], nullptr, &nr));
        HFCK(add_node(ip.conditional.phGraph_out[0], L.W[k ^ 1], &nr, &nw));
        bprev = inode;
        bprev_is_k = false;
    }
    prev = wnode;
    for (auto &p : post) { HFCK(add_node(g, p, &prev, &n)); prev = n; }
    *out = g;
    return HF_OK;
}

// host-loop driver of the same sequence (profiling, sanitizers)
static hf_status host_cg1_loop(hf_ctx *c, Sys &s, const Cg1Launches &L, int max_iter, int replace_every)
{
    HFCK(read_state(c, s));
    if (!s.st_host->active) return HF_OK;
    for (int i = 0;;) {
        const int k = i & 1;
        HFCK(run(c, L.C[k], s.stream));
        if (i > 0 && replace_every > 0 && i % replace_every == 0) {
            HFCK(run(c, L.RES[k ^ 1], s.stream));
            HFCK(run(c, L.W[k ^ 1], s.stream));
        }
        i++;
        if (i % c->check_every == 0 || i > max_iter) {
            HFCK(read_state(c, s));
            if (!s.st_host->active) break;
        }
    }
    return HF_OK;
}

// ============================================================================================
// C ABI

extern "C" {

const char *hf_version(void) { return "heatfem-b200 0.2 (sm_100a, TMA stencil)"; }

const char *hf_last_error(void) { return g_err.c_str(); }

hf_status hf_create(const hf_grid *g, int device, void *cuda_stream, hf_ctx **out)
{
    if (!g || !out) return fail(HF_E_ARG, "hf_create: NULL argument");
    hf_ctx *c = new hf_ctx();
    hf_status st = ctx_init(c, g, device, cuda_stream, 0, 1);
    if (st != HF_OK) { ctx_free(c); delete c; return st; }
    *out = c;
    return HF_OK;
}

void hf_destroy(hf_ctx *c)
{
    if (!c) return;
    ctx_free(c);
    delete c;
}

hf_status hf_set_coefficients(hf_ctx *c, const double *k, const double *cc)
{
    if (!c || !k || !cc) return fail(HF_E_ARG, "hf_set_coefficients: NULL argument");
    HFCK(check_ptrs(c, "hf_set_coefficients", {k, cc}));
    CUCK(cudaSetDevice(c->device));
    const size_t ne = (size_t)(c->g.ne[0] * c->g.ne[1] * c->g.ne[2]);
    const double *dk, *dc;
    HFCK(dev_in(c, k, ne, 0, &dk));
    HFCK(dev_in(c, cc, ne, 1, &dc));
    HFCK(enqueue_pack(c, c->sys0, dk, dc));
    CUCK(cudaStreamSynchronize(c->stream));
    if (c->tetv) {                              // back to one coefficient per element
        c->tetv = false;
        c->sys0.key_valid = false;
    }
    if (c->pal_on) {                            // back to (k, c) pairs from material ids
        c->pal_on = false;
        HFCK(update_occ(c));
        HFCK(sys_maps(c, c->sys0));
        c->sys0.key_valid = false;
    }
    c->coef_set = true;
    c->ab_ready = false;
    if (c->lo) HFCK(hf_set_coefficients(c->lo, k, cc));    // mixed precision: the fp32 shadow
    return HF_OK;
}

hf_status hf_set_material_ids(hf_ctx *c, const uint8_t *ids, int32_t nmat, const double *k_mat, const double *c_mat)
{
    if (!c || !ids || !k_mat || !c_mat) return fail(HF_E_ARG, "hf_set_material_ids: NULL argument");
    if (nmat < 1 || nmat > PAL_MAX - 1)
        return fail(HF_E_ARG, "hf_set_material_ids: n_materials must be in [1, " + std::to_string(PAL_MAX - 1) + "]");
    HFCK(check_ptrs(c, "hf_set_material_ids", {ids}));
    CUCK(cudaSetDevice(c->device));
    const size_t ne = (size_t)(c->g.ne[0] * c->g.ne[1] * c->g.ne[2]);
    const uint8_t *dids = ids;
    if (!is_device_ptr(ids)) {
        void *d;
        HFCK(scratch_get(c, 57, ne, &d));
        CUCK(cudaMemcpyAsync(d, ids, ne, cudaMemcpyHostToDevice, c->stream));
        dids = (const uint8_t *)d;
    }
    const int nx = (int)c->g.ne[0];
    const int kp = (nx + 15) & ~15;
    const long long nkid = (long long)kp * c->g.ne[1] * (c->nzl + 1);
    if (!c->kid || c->kid_pitch != kp) {
        cudaFree(c->kid);
        c->kid = nullptr;
        CUCK(cudaMalloc(&c->kid, (size_t)nkid));
        c->kid_pitch = kp;
    }
    PalTab pt;
    std::memset(&pt, 0, sizeof(pt));
    for (int m = 0; m < nmat; m++) { pt.kc[m][0] = k_mat[m]; pt.kc[m][1] = c_mat[m]; }
    int *bad;
    HFCK(scratch_get(c, 58, sizeof(int), (void **)&bad));
    CUCK(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    const long long nkc = c->kc_elems;
    if (c->es == 8)
        k_pack_ids<double><<<(unsigned)((nkc + 255) / 256), 256, 0, c->stream>>>(make_geom(c), (int)c->g.ne[2], dids, nmat,
                                                                                pt, c->sys0.kc, nkc, bad, c->launches);
    else
        k_pack_ids<float><<<(unsigned)((nkc + 255) / 256), 256, 0, c->stream>>>(make_geom(c), (int)c->g.ne[2], dids, nmat,
                                                                               pt, c->sys0.kc, nkc, bad, c->launches);
    CUCK(cudaGetLastError());
    k_pack_kid<<<(unsigned)((nkid + 255) / 256), 256, 0, c->stream>>>(make_geom(c), (int)c->g.ne[2], dids, kp,
                                                                      c->kid, nkid, c->launches);
    CUCK(cudaGetLastError());
    int hbad = 0;
    CUCK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CUCK(cudaStreamSynchronize(c->stream));
    if (hbad) return fail(HF_E_INDEX, "hf_set_material_ids: a material id >= n_materials");
    // material 0 of the table is the void outside the domain; ids are stored + 1
    std::memset(c->pal, 0, sizeof(c->pal));
    for (int m = 0; m < nmat; m++) { c->pal[m + 1][0] = k_mat[m]; c->pal[m + 1][1] = c_mat[m]; }
    c->npal = nmat + 1;
    c->pal_on = true;
    HFCK(update_occ(c));
    c->tetv = false;
    HFCK(sys_maps(c, c->sys0));
    c->sys0.key_valid = false;
    c->coef_set = true;
    c->ab_ready = false;
    if (c->lo) {                                // mixed precision: the fp32 shadow takes (k, c) pairs
        const size_t ne = (size_t)(c->g.ne[0] * c->g.ne[1] * c->g.ne[2]);
        void *kp, *cp;
        HFCK(scratch_get(c, 55, ne * sizeof(double), &kp));
        HFCK(scratch_get(c, 56, ne * sizeof(double), &cp));
        k_extract_kc<<<(unsigned)((ne + 255) / 256), 256, 0, c->stream>>>(make_geom(c), (int)c->g.ne[2],
            (const double2 *)c->sys0.kc, (double *)kp, (double *)cp, c->launches);
        CUCK(cudaGetLastError());
        CUCK(cudaStreamSynchronize(c->stream));
        HFCK(hf_set_coefficients(c->lo, (const double *)kp, (const double *)cp));
    }
    return HF_OK;
}

hf_status hf_set_vertex_coefficients(hf_ctx *c, const double *k, const double *cc)
{
    if (!c || !k || !cc) return fail(HF_E_ARG, "hf_set_vertex_coefficients: NULL argument");
    HFCK(check_ptrs(c, "hf_set_vertex_coefficients", {k, cc}));
    CUCK(cudaSetDevice(c->device));
    const size_t nng = (size_t)c->nx1 * c->ny1 * c->nz1g;     // global natural nodes
    const double *dk, *dc;
    HFCK(dev_in(c, k, nng, 0, &dk));
    HFCK(dev_in(c, cc, nng, 1, &dc));
    if (c->elem == EL_Q1) {
        // Q1: each voxel's coefficient is the mean of its 8 corners
        const size_t ne = (size_t)(c->g.ne[0] * c->g.ne[1] * c->g.ne[2]);
        void *ke, *ce;
        HFCK(scratch_get(c, 55, ne * sizeof(double), &ke));
        HFCK(scratch_get(c, 56, ne * sizeof(double), &ce));
        k_vertex_means<<<(unsigned)((ne + 255) / 256), 256, 0, c->stream>>>(make_geom(c), (int)c->g.ne[2], dk, dc,
                                                                            (double *)ke, (double *)ce, c->launches);
        CUCK(cudaGetLastError());
        return hf_set_coefficients(c, (const double *)ke, (const double *)ce);
    }
    // tets: per-node pairs; each tet averages its 4 vertices inside the stencil (EL_TETV)
    Sys &s = c->sys0;
    if (!s.kcn) {
        CUCK(cudaMalloc(&s.kcn, (size_t)c->nloc * 2 * c->es));
        CUCK(cudaMemsetAsync(s.kcn, 0, (size_t)c->nloc * 2 * c->es, c->stream));
    }
    const unsigned nb = (unsigned)((c->nloc + 255) / 256);
    if (c->es == 8) k_pack_nodes<double><<<nb, 256, 0, c->stream>>>(make_geom(c), dk, dc, s.kcn, c->launches);
    else k_pack_nodes<float><<<nb, 256, 0, c->stream>>>(make_geom(c), dk, dc, s.kcn, c->launches);
    CUCK(cudaGetLastError());
    HFCK(sys_maps(c, s));
    CUCK(cudaStreamSynchronize(c->stream));
    c->tetv = true;
    s.key_valid = false;
    c->coef_set = true;
    c->ab_ready = false;
    if (c->lo) HFCK(hf_set_vertex_coefficients(c->lo, k, cc));
    return HF_OK;
}

hf_status hf_set_dirichlet_faces(hf_ctx *c, uint32_t bits, const double values[6])
{
    if (!c || bits > 63u) return fail(HF_E_ARG, "hf_set_dirichlet_faces: bad argument");
    c->dbits = bits;
    for (int f = 0; f < 6; f++) c->gval[f] = values ? values[f] : 0.0;
    drop_stacks(c);
    c->sys0.key_valid = false;
    if (c->lo) HFCK(hf_set_dirichlet_faces(c->lo, bits, values));
    return HF_OK;
}

hf_status hf_face_load(hf_ctx *c, int face, double f_const, const double beam[4], double *F)
{
    if (!c || !F || face < 0 || face > 5) return fail(HF_E_ARG, "hf_face_load: bad argument");
    if (beam && !(beam[1] > 0.0)) return fail(HF_E_ARG, "hf_face_load: beam sigma must be > 0");
    HFCK(check_ptrs(c, "hf_face_load", {F}));
    CUCK(cudaSetDevice(c->device));
    double *dF;
    HFCK(node_out(c, F, 2, false, &dF));
    CUCK(cudaMemsetAsync(dF, 0, c->nloc * c->es, c->stream));
    FaceArgs a;
    std::memset(&a, 0, sizeof(a));
    a.g = make_geom(c);
    a.face = face;
    a.nd = face / 2;
    a.ax = a.nd == 0 ? 1 : 0;
    a.bx = a.nd == 2 ? 1 : 2;
    const int n1[3] = {c->nx1, c->ny1, c->nz1g};
    a.na = n1[a.ax];
    a.nb = n1[a.bx];
    a.plane_g = (face & 1) ? (int)c->g.ne[a.nd] : 0;
    a.ha = c->g.h[a.ax]; a.hb = c->g.h[a.bx];
    a.oa = c->g.origin[a.ax]; a.ob = c->g.origin[a.bx];
    a.f_const = f_const;
    if (beam) { a.has_beam = 1; a.bP = beam[0]; a.bs = beam[1]; a.bca = beam[2]; a.bcb = beam[3]; }
    a.tets = c->elem == EL_DENSE;
    a.F = dF;
    a.launches = c->launches;
    const long long n = (long long)a.na * a.nb;
    if (c->es == 8) k_face_load<double><<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(a);
    else k_face_load<float><<<(unsigned)((n + 255) / 256), 256, 0, c->stream>>>(a);
    CUCK(cudaGetLastError());
    return node_out_finish(c, F, dF);
}

hf_status hf_apply_axpby(hf_ctx *c, double aK, double aM, double cc, const double *u, const double *b, double *y)
{
    if (!c || !u || !y) return fail(HF_E_ARG, "hf_apply: NULL argument");
    if (!c->coef_set) return fail(HF_E_STATE, "hf_apply: coefficients not set");
    if ((const double *)y == u) return fail(HF_E_ARG, "hf_apply: u and y must not alias");
    HFCK(check_ptrs(c, "hf_apply", {u, b, y}));
    CUCK(cudaSetDevice(c->device));
    const double *du, *db = nullptr;
    double *dy;
    HFCK(node_in(c, u, 3, &du));
    if (b) HFCK(node_in(c, b, 4, &db));
    HFCK(node_out(c, y, 5, false, &dy));
    Maps maps = c->sys0.maps;
    HFCK(node_map(c, du, &maps.node[MAP_U0]));
    StencilArgs a = base_args(c, aK, aM);
    a.out0 = dy;
    a.bvec = db;
    a.c = cc;
    a.s = 1.0;
    Launch L;
    HFCK(stencil_launch(c, LD_RAW, EP_APPLY, false, maps, a, 3, &L));
    HFCK(run(c, L, c->stream));
    if (y == dy) return HF_OK;               // fully asynchronous on device buffers
    return node_out_finish(c, y, dy);
}

hf_status hf_apply(hf_ctx *c, double aK, double aM, const double *u, double *y)
{
    return hf_apply_axpby(c, aK, aM, 1.0, u, nullptr, y);
}

hf_status hf_diag(hf_ctx *c, double aK, double aM, double *diag)
{
    if (!c || !diag) return fail(HF_E_ARG, "hf_diag: NULL argument");
    if (!c->coef_set) return fail(HF_E_STATE, "hf_diag: coefficients not set");
    HFCK(check_ptrs(c, "hf_diag", {diag}));
    CUCK(cudaSetDevice(c->device));
    double *dd;
    HFCK(node_out(c, diag, 5, false, &dd));
    HFCK(enqueue_diag(c, c->sys0, aK, aM, dd, nullptr));
    if (diag == dd) return HF_OK;
    return node_out_finish(c, diag, dd);
}

// ---- NEXT f4: the paper's earlier interpretations of the assembly operator (hf_ablate.cuh) ----

static hf_status ablation_ok(const hf_ctx *c, const char *who)
{
    if (!c->coef_set) return fail(HF_E_STATE, std::string(who) + ": coefficients not set");
    if (c->es != 8) return fail(HF_E_STATE, std::string(who) + ": the ablation kernels are fp64 only");
    if (c->nranks > 1 || c->comm) return fail(HF_E_STATE, std::string(who) + ": not available on a slab context");
    if (c->elem == EL_DENSE && c->tetv)
        return fail(HF_E_STATE, std::string(who) + ": not available with per-tet vertex-averaged coefficients");
    return HF_OK;
}

static Dense ablation_dense(const hf_ctx *c, double aK, double aM)
{
    double K[64], M[64];
    if (c->elem == EL_DENSE) tet_voxel(c->g.h, K, M);
    else q1_voxel(c->g.h, K, M);
    Dense dn;
    for (int i = 0; i < 64; i++) {
        dn.K[i] = aK * K[i];
        dn.M[i] = aM * M[i];
    }
    return dn;
}

hf_status hf_ablation_prepare(hf_ctx *c, double aK, double aM)
{
    if (!c) return fail(HF_E_ARG, "hf_ablation_prepare: NULL context");
    HFCK(ablation_ok(c, "hf_ablation_prepare"));
    CUCK(cudaSetDevice(c->device));
    const long long nelem = c->g.ne[0] * c->g.ne[1] * c->g.ne[2];
    if (!c->ab_A) {
        CUCK(cudaMalloc(&c->ab_A, (size_t)nelem * 64 * sizeof(double)));
        CUCK(cudaMalloc(&c->ab_contrib, (size_t)c->nloc * 8 * sizeof(double)));
    }
    const long long nrows = nelem * 8;
    k_ebe_store<<<(unsigned)((nrows + 255) / 256), 256, 0, c->stream>>>(make_geom(c), c->sys0.kc,
                                                                      ablation_dense(c, aK, aM), c->ab_A, nrows,
                                                                      c->launches);
    CUCK(cudaGetLastError());
    c->ab_aK = aK;
    c->ab_aM = aM;
    c->ab_ready = true;
    return HF_OK;
}

hf_status hf_apply_impl(hf_ctx *c, int32_t impl, double aK, double aM, double cc, const double *u, const double *b,
                        double *y)
{
    if (impl == 3) return hf_apply_axpby(c, aK, aM, cc, u, b, y);
    if (!c || !u || !y) return fail(HF_E_ARG, "hf_apply_impl: NULL argument");
    if (impl != 1 && impl != 2) return fail(HF_E_ARG, "hf_apply_impl: impl must be 1, 2 or 3");
    if ((const double *)y == u) return fail(HF_E_ARG, "hf_apply_impl: u and y must not alias");
    HFCK(ablation_ok(c, "hf_apply_impl"));
    HFCK(check_ptrs(c, "hf_apply_impl", {u, b, y}));
    if (impl == 1 && (!c->ab_ready || aK != c->ab_aK || aM != c->ab_aM))
        return fail(HF_E_STATE, "hf_apply_impl: Implementation 1 needs hf_ablation_prepare with the same (aK, aM)");
    CUCK(cudaSetDevice(c->device));
    const double *du, *db = nullptr;
    double *dy;
    HFCK(node_in(c, u, 3, &du));
    if (b) HFCK(node_in(c, b, 4, &db));
    HFCK(node_out(c, y, 5, false, &dy));
    const Geom g = make_geom(c);
    const int nz = (int)c->g.ne[2];
    if (impl == 1) {
        const long long nelem = c->g.ne[0] * c->g.ne[1] * c->g.ne[2];
        k_ebe_pass1<<<(unsigned)((nelem + 31) / 32), 256, 0, c->stream>>>(g, du, c->ab_A, c->ab_contrib, nelem,
                                                                         c->launches);
        CUCK(cudaGetLastError());
        k_ebe_pass2<<<(unsigned)((c->nloc + 255) / 256), 256, 0, c->stream>>>(g, nz, c->ab_contrib, cc, db, dy,
                                                                             c->nloc, c->launches);
    } else {
        const dim3 grid((unsigned)((c->nx1 + DBD_W - 1) / DBD_W), (unsigned)c->ny1, (unsigned)c->nzl);
        k_dbd<<<grid, DBD_W, 0, c->stream>>>(g, nz, du, c->sys0.kc, ablation_dense(c, aK, aM), cc, db, dy,
                                             c->launches);
    }
    CUCK(cudaGetLastError());
    if (y == dy) return HF_OK;
    return node_out_finish(c, y, dy);
}

hf_status hf_cg(hf_ctx *c, double aK, double aM, const double *b, double *x, const hf_cg_opts *opts,
                hf_cg_info *info)
{
    if (!c || !b || !x) return fail(HF_E_ARG, "hf_cg: NULL argument");
    if (!c->coef_set) return fail(HF_E_STATE, "hf_cg: coefficients not set");
    if (c->comm && !c->comm->ready()) return fail(HF_E_STATE, "hf_cg: peer transport not connected (hf_peer_connect)");
    HFCK(check_ptrs(c, "hf_cg", {b, x}));
    CUCK(cudaSetDevice(c->device));
    Sys &s = c->sys0;
    hf_cg_opts o = {1e-12, 10000, -1};
    if (opts) o = *opts;
    o = resolved(c, o);
    HFCK(set_solver_opts(c, s, o));
    const double *db;
    double *dx;
    HFCK(node_in(c, b, 4, &db));
    HFCK(node_out(c, x, 6, true, &dx));
    CUCK(cudaMemcpyAsync(s.b, db, c->nloc * c->es, cudaMemcpyDeviceToDevice, s.stream));
    HFCK(enqueue_diag(c, s, aK, aM, nullptr, s.invd));
    HFCK(enqueue_set_dirichlet(c, s, dx, s.b));           // x_D = b_D
    Maps xm = s.maps;
    HFCK(node_map(c, dx, &xm.node[MAP_U0]));
    // init: r = b - A x0; s = P^{-1} r; delta; ||b_F||   (Alg. 1 lines 2-4)
    StencilArgs ia = base_args(c, aK, aM);
    ia.invd = s.invd;
    ia.bvec = s.b;
    ia.out0 = s.r;
    ia.out_s = s.s;
    ia.xout = dx;
    ia.sy = make_sync(c, s, -1, 1);
    Launch init;
    HFCK(stencil_launch(c, LD_RAW, EP_RESID_INIT, true, xm, ia, 2, &init));
    CgLaunches L;
    HFCK(cg_launches(c, s, aK, aM, dx, xm, &L));
    StepArgs sa = step_args(c, s, dx, nullptr, -1);
    sa.iters_out = nullptr;
    std::vector<Launch> post = step_launches(c, sa, false);
    const bool use_graph = c->driver == 0 && (!c->comm || c->comm->in_kernel()) && !c->prof;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    if (use_graph) {
        HFCK(build_cg_graph(c, {}, init, L, post, o.replace_every, &g));
        cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
        if (e != cudaSuccess) { cudaGraphDestroy(g); CUCK(e); }
    }
    if (c->comm) {                 // collective part: the iterate's ghost planes, then the solve
        hf_status cs = c->comm->enter();
        if (cs == HF_OK) cs = c->comm->exchange(c, s, dx);
        if (cs != HF_OK) {
            if (ge) cudaGraphExecDestroy(ge);
            if (g) cudaGraphDestroy(g);
            return cs;
        }
    }
    if (use_graph) {
        cudaError_t e = cudaGraphLaunch(ge, s.stream);
        cudaStreamSynchronize(s.stream);
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        CUCK(e);
    } else {
        HFCK(run(c, init, s.stream));
        HFCK(comm_after(c, s, 1, true));
        HFCK(host_cg_loop(c, s, L, o.max_iter, o.replace_every));
        for (auto &p : post) HFCK(run(c, p, s.stream));
    }
    HFCK(read_state(c, s));
    if (x != dx) HFCK(node_out_finish(c, x, dx));
    const CgState &h = *s.st_host;
    if (info) {
        info->iters = h.iter;
        info->status = h.status;
        info->relres = h.bb > 0 ? std::sqrt(h.rr / h.bb) : 0.0;
        info->delta = h.delta[h.iter & 1];
    }
    if (h.status == ST_NOCONV) return fail(HF_E_NOCONV, "hf_cg: max_iter reached");
    if (h.status == ST_BREAKDOWN) return fail(HF_E_BREAKDOWN, "hf_cg: breakdown (d^T q <= 0 or non-finite)");
    return HF_OK;
}

}  // extern "C"

// One system's time loop; U[0] holds u^0 (and U[2] u^{-1} when resuming) on entry, F (padded)
// the flux load.
// ---- on-chip PCG (hf_resident.cuh): eligibility, brick partition, launch ------------------
struct ResPlan {
    int ok = 0, px = 0, py = 0, pz = 0, bxm = 0, bym = 0, bzm = 0, BZ = 0, P = 0;
    size_t smem = 0;
    const void *fn = nullptr;
    const char *why = "";
};

// Eligible: fp64 Q1 with materials by id (hf_set_material_ids), one system, no slab transport,
// graph driver, and a brick partition that fits one CTA per SM: bricks <= 31 x (RES_NW - 1) x
// RES_BZ_MAX nodes, px py pz <= SMs, shared memory <= the opt-in limit.
static ResPlan res_plan(hf_ctx *c)
{
    ResPlan p;
    if (!c->resident) { p.why = "disabled"; return p; }
    if (!c->pal_on || c->elem != EL_Q1 || c->tetv || c->es != 8) { p.why = "needs fp64 Q1 materials by id"; return p; }
    if (c->nsys != 1 || c->comm) { p.why = "stacked systems / slabs"; return p; }
    if (c->driver != 0 || c->prof) { p.why = "host-loop driver / profiling"; return p; }
    const int RW = 31, RH = RES_ROWS - 1;
    p.px = (c->nx1 + RW - 1) / RW;
    p.py = (c->ny1 + RH - 1) / RH;
    const int cols = p.px * p.py;
    if (cols > c->nsm) { p.why = "cross-section too large"; return p; }
    p.pz = std::max(1, std::min(c->nzl, c->nsm / cols));
    p.bxm = (c->nx1 + p.px - 1) / p.px;
    p.bym = (c->ny1 + p.py - 1) / p.py;
    p.bzm = (c->nzl + p.pz - 1) / p.pz;
    if (p.bzm > RES_BZ_MAX) { p.why = "grid too large for on-chip PCG"; return p; }
    p.BZ = RES_BZ_MAX;
    p.fn = (const void *)k_pcg_res;
    p.smem = res_smem(p.bxm, p.bym, p.bzm, c->npal).total;
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, c->device) != cudaSuccess ||
        p.smem > (size_t)optin) { p.why = "shared memory"; return p; }
    p.P = p.px * p.py * p.pz;
    if (p.P > RES_PMAX) { p.why = "too many bricks"; return p; }
    if (ensure_smem_attr(p.fn, p.smem, c->device) != HF_OK) { p.why = "smem attribute"; return p; }
    int occ = 0;
    const cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, p.fn, RES_NT, p.smem);
    if (oe != cudaSuccess || occ * c->nsm < p.P) {
        static thread_local char buf[160];
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, p.fn);
        snprintf(buf, sizeof(buf), "occupancy: %d CTAs/SM (%s), %d registers, %zu B smem", occ, cudaGetErrorString(oe),
                 fa.numRegs, p.smem);
        cudaGetLastError();
        p.why = buf;
        return p;
    }
    p.ok = 1;
    return p;
}

static hf_status res_launch(hf_ctx *c, Sys &s, const ResPlan &p, double aK, double aM, bool first, Launch *out)
{
    if (!c->rsync) CUCK(cudaMalloc(&c->rsync, sizeof(ResSync)));
    ResArgs a;
    std::memset(&a, 0, sizeof(a));
    a.g = make_geom(c);
    a.lam = make_lam(c->g.h, aK, aM);
    a.px = p.px; a.py = p.py; a.pz = p.pz;
    a.bxm = p.bxm; a.bym = p.bym; a.bzm = p.bzm;
    a.kid = c->kid;
    a.kid_pitch = c->kid_pitch;
    std::memcpy(a.pal, c->pal, sizeof(a.pal));
    a.npal = c->npal;
    a.b = s.b;
    a.invd = s.invd;
    for (int i = 0; i < 3; i++) a.ring[i] = s.U[i];
    a.sg = s.s;
    a.dsave = s.dbuf[0];
    a.st = s.st;
    a.rs = c->rsync;
    a.first = first ? 1 : 0;
    a.launches = c->launches;
    a.prof = c->res_prof;
    Launch L;
    L.fn = p.fn;
    L.grid = dim3(p.P, 1, 1);
    L.block = dim3(RES_NT, 1, 1);
    L.smem = p.smem;
    L.add(a);
    L.cls = 0;
    *out = L;
    return HF_OK;
}

// graph of one time step with the on-chip PCG: [RHS] -> [lift] -> zero the reduction flags ->
// k_pcg_res (cooperative: every CTA co-resident, or the launch fails) -> step end, commit
static hf_status build_res_graph(hf_ctx *c, const std::vector<Launch> &pre, const Launch &res,
                                 const std::vector<Launch> &post, cudaGraph_t *out)
{
    cudaGraph_t g;
    CUCK(cudaGraphCreate(&g, 0));
    cudaGraphNode_t prev = nullptr, n;
    for (auto &p : pre) { HFCK(add_node(g, p, prev ? &prev : nullptr, &n)); prev = n; }
    cudaMemsetParams mp;
    std::memset(&mp, 0, sizeof(mp));
    mp.dst = c->rsync;
    mp.elementSize = 4;
    mp.width = sizeof(ResSync) / 4;
    mp.height = 1;
    mp.value = 0;
    CUCK(cudaGraphAddMemsetNode(&n, g, prev ? &prev : nullptr, prev ? 1 : 0, &mp));
    prev = n;
    HFCK(add_node(g, res, &prev, &n));
    cudaKernelNodeAttrValue v;
    std::memset(&v, 0, sizeof(v));
    v.cooperative = 1;
    CUCK(cudaGraphKernelNodeSetAttribute(n, cudaKernelNodeAttributeCooperative, &v));
    prev = n;
    for (auto &p : post) { HFCK(add_node(g, p, &prev, &n)); prev = n; }
    *out = g;
    return HF_OK;
}

static hf_status simulate_sys(hf_ctx *c, Sys &s, double theta, double dt, int nsteps, const double *dF,
                              bool first, int snap_local, double *snapdev, const hf_cg_opts &o)
{
    if (c->comm && c->step_flush && !c->flush) CUCK(cudaMalloc(&c->flush, 512ull << 20));
    const double aK = theta * dt, aM = 1.0;             // A = M + theta dt K
    c->last_aK = aK;
    const double aKL = -(1.0 - theta) * dt, aML = 1.0;  // L = M - (1-theta) dt K   (R8)
    HFCK(set_solver_opts(c, s, o));
    if (s.iters_cap < nsteps) {
        cudaFree(s.iters);
        s.iters = nullptr;
        CUCK(cudaMalloc(&s.iters, (size_t)std::max(1, nsteps) * sizeof(int)));
        s.iters_cap = nsteps;
        s.key_valid = false;
    }
    HFCK(enqueue_diag(c, s, aK, aM, nullptr, s.invd));
    HFCK(enqueue_set_dirichlet(c, s, s.U[0], nullptr));       // u^0_D = g
    if (!first) HFCK(enqueue_set_dirichlet(c, s, s.U[2], nullptr));
    bool lift = false;
    for (int f = 0; f < 6; f++) if ((c->dbits >> f & 1u) && c->gval[f] != 0.0) lift = true;
    const bool use_graph = c->driver == 0 && (!c->comm || c->comm->in_kernel()) && !c->prof;
    c->last_ms_steps = 0.0;
    SimKey key;
    std::memset(&key, 0, sizeof(key));
    key.aK = aK; key.aM = aM; key.aKL = aKL; key.aML = aML; key.rtol = o.rtol; key.dt = dt;
    key.max_iter = o.max_iter; key.replace_every = o.replace_every; key.first = first;
    key.snap_plane = snap_local; key.lift = lift; key.F = dF; key.snap = snapdev;
    ResPlan rp;
    if (use_graph && &s == &c->sys0) rp = res_plan(c);
    // mixed precision (hf_set_mixed): [RHS -> fp32 solve] graph + the fp64 finish graph
    const bool mixed = c->lo && use_graph && &s == &c->sys0 && !rp.ok;
    key.res = rp.ok + 2 * (int)mixed;
    c->last_resident = rp.ok;
    const bool use_cg1 = cg1_eligible(c, s) && !mixed && !rp.ok;
    key.cg1 = use_cg1;
    c->last_cg1 = use_cg1;
    const bool cached = use_graph && s.key_valid && s.key == key && s.gexec && (!mixed || c->mix_exec);
    if (mixed) {
        // the fp32 shadow's solver state and Jacobi diagonal (same operator, fp32 storage)
        hf_cg_opts lo_o = {std::max(c->mix_rtol, o.rtol), o.max_iter, -1};
        HFCK(set_solver_opts(c->lo, c->lo->sys0, lo_o));
        HFCK(enqueue_diag(c->lo, c->lo->sys0, aK, aM, nullptr, c->lo->sys0.invd));
    }

    std::vector<Launch> pre, post;
    Launch init;
    CgLaunches L;
    Cg1Launches L1;
    if (!cached) {
        Sync sy = make_sync(c, s);
        // b = L u^n + dt F  (knl_RHS_A/B P:678-681), b_D = g
        StencilArgs ra = base_args(c, aKL, aML);
        ra.bvec = dF;
        ra.s = dt;
        ra.out0 = s.b;
        ra.dmode = 2;
        ra.rot_role = ROT_RHS;
        ra.sy = sy;
        Launch rhs;
        HFCK(stencil_launch(c, LD_RAW, EP_APPLY, true, s.maps, ra, 3, &rhs));
        pre.push_back(rhs);
        if (lift) {  // b_F -= (A g~)_F  (Dirichlet lift, R3)
            StencilArgs la = base_args(c, aK, aM);
            la.bvec = s.b;
            la.s = 1.0;
            la.c = -1.0;
            la.out0 = s.b;
            la.dmode = 2;
            la.sy = sy;
            Launch lf;
            HFCK(stencil_launch(c, LD_GT, EP_APPLY, true, s.maps, la, 3, &lf));
            pre.push_back(lf);
        }
        // init with the extrapolated guess x0 = 2u^n - u^{n-1} (u0_update)
        StencilArgs ia = base_args(c, aK, aM);
        ia.invd = s.invd;
        ia.bvec = s.b;
        ia.out0 = s.r;
        ia.out_s = s.s;
        ia.first = first ? 1 : 0;
        ia.rot_role = ROT_INIT;
        for (int i = 0; i < 3; i++) ia.ring[i] = s.U[i];
        ia.sy = make_sync(c, s, -1, 1);
        ia.zs0 = c->own_lo - (c->own_lo > 0 ? 1 : 0);
        ia.zs1 = c->own_hi + (c->own_hi < c->nzl ? 1 : 0);
        HFCK(stencil_launch(c, LD_X0, EP_RESID_INIT, true, s.maps, ia, 2, &init));
        if (mixed) {
            // fp32 stage (defect correction): r0 of the extrapolated guess to fp32 (k_mix_in),
            // the fp32 PCG for A e = r0 from e = 0, x0 += e in fp64 (k_mix_out)
            hf_ctx *lo = c->lo;
            Sys &ls = lo->sys0;
            MixArgs ma;
            std::memset(&ma, 0, sizeof(ma));
            ma.nx1 = c->nx1; ma.ny1 = c->ny1; ma.nzl = c->nzl;
            ma.pitch_hi = c->pitch; ma.pitch_lo = lo->pitch;
            ma.plane_hi = c->plane; ma.plane_lo = lo->plane;
            ma.rhi = s.r;
            for (int i = 0; i < 3; i++) ma.ring[i] = s.U[i];
            ma.st = s.st;
            ma.blo = (float *)ls.b;
            ma.xlo = (float *)ls.U[0];
            ma.stlo = ls.st;
            ma.lo_iters = c->mix_iters;
            ma.launches = c->launches;
            ma.nsys = c->nsys;
            ma.sys_planes = c->sys_planes;
            const long long nn = (long long)c->nx1 * c->ny1 * c->nzl;
            Launch Min, Mout;
            Min.fn = (const void *)k_mix_in;
            Mout.fn = (const void *)k_mix_out;
            Min.grid = Mout.grid = dim3((unsigned)((nn + 255) / 256));
            Min.block = Mout.block = dim3(256);
            Min.add(ma);
            Mout.add(ma);
            std::vector<Launch> mpre = pre;
            mpre.push_back(init);                     // x0 -> U[(n+1) % 3], r0 = b - A x0 (fp64)
            mpre.push_back(Min);
            pre.clear();
            StencilArgs li = base_args(lo, aK, aM);
            li.invd = ls.invd;
            li.bvec = ls.b;
            li.out0 = ls.r;
            li.out_s = ls.s;
            li.xout = ls.U[0];
            li.sy = make_sync(lo, ls, -1, 1);
            Launch linit;
            HFCK(stencil_launch(lo, LD_RAW, EP_RESID_INIT, true, ls.maps, li, 2, &linit));
            CgLaunches LL;
            HFCK(cg_launches(lo, ls, aK, aM, ls.U[0], ls.maps, &LL));
            if (c->mix_exec) { cudaGraphExecDestroy(c->mix_exec); c->mix_exec = nullptr; }
            if (c->mix_graph) { cudaGraphDestroy(c->mix_graph); c->mix_graph = nullptr; }
            HFCK(build_cg_graph(lo, mpre, linit, LL, {Mout}, resolved(lo, hf_cg_opts{0.0, 0, -1}).replace_every,
                                 &c->mix_graph));
            CUCK(cudaGraphInstantiate(&c->mix_exec, c->mix_graph, 0));
        }
        if (mixed) {
            // the fp64 finish: init from x0 + e, already in U[(n+1) % 3]
            ia.rot_role = ROT_X;
            ia.zs0 = ia.zs1 = 0;
            HFCK(stencil_launch(c, LD_RAW, EP_RESID_INIT, true, s.maps, ia, 2, &init));
        }
        if (use_cg1) {
            // single-reduction PCG: the init kernel writes r[0] and its partials into P[0] (partA)
            HFCK(cg1_launches(c, s, aK, aM, &L1));
            ia.out0 = s.c1r[0];
            ia.sy = make_sync(c, s, -1, 0);
            HFCK(stencil_launch(c, LD_X0, EP_RESID_INIT, true, s.maps, ia, 2, &init));
        } else if (!rp.ok) HFCK(cg_launches(c, s, aK, aM, nullptr, s.maps, &L));
        post = step_launches(c, step_args(c, s, nullptr, snapdev, snap_local), true);
    }

    if (use_graph && !cached) {
        if (s.gexec) { cudaGraphExecDestroy(s.gexec); s.gexec = nullptr; }
        if (s.graph) { cudaGraphDestroy(s.graph); s.graph = nullptr; }
        s.key_valid = false;
        if (rp.ok) {
            Launch RL;
            HFCK(res_launch(c, s, rp, aK, aM, first, &RL));
            HFCK(build_res_graph(c, pre, RL, post, &s.graph));
        } else if (use_cg1)
            HFCK(build_cg1_graph(c, pre, init, L1, post, resolved(c, o).replace_every, &s.graph));
        else
            HFCK(build_cg_graph(c, pre, init, L, post, o.replace_every, &s.graph));
        CUCK(cudaGraphInstantiate(&s.gexec, s.graph, 0));
        s.key = key;
        s.key_valid = true;
    }
    if (c->comm) {
        // collective part: every rank's setup is done; make the ghost planes of the input state
        // consistent (u^n, and u^{n-1} when resuming), then the steps
        HFCK(c->comm->enter());
        HFCK(c->comm->exchange(c, s, s.U[0]));
        if (!first) HFCK(c->comm->exchange(c, s, s.U[2]));
    }
    if (nsteps <= 0) return HF_OK;
    if (use_graph) {
        if (c->step_flush) {
            // L2 eviction between steps, each step timed alone (no host synchronisation)
            const size_t fb = 512ull << 20;
            if (!c->flush) CUCK(cudaMalloc(&c->flush, fb));
            std::vector<cudaEvent_t> ev(2 * (size_t)nsteps);
            for (auto &e : ev) CUCK(cudaEventCreate(&e));
            for (int n = 0; n < nsteps; n++) {
                if (c->step_flush == 1) CUCK(cudaMemsetAsync(c->flush, n & 1, fb, s.stream));
                CUCK(cudaEventRecord(ev[2 * n], s.stream));
                if (mixed) CUCK(cudaGraphLaunch(c->mix_exec, s.stream));
                CUCK(cudaGraphLaunch(s.gexec, s.stream));
                CUCK(cudaEventRecord(ev[2 * n + 1], s.stream));
            }
            CUCK(cudaEventSynchronize(ev.back()));
            double tot = 0.0;
            for (int n = 0; n < nsteps; n++) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, ev[2 * n], ev[2 * n + 1]);
                tot += ms;
            }
            for (auto &e : ev) cudaEventDestroy(e);
            c->last_ms_steps = tot;
        } else {
            for (int n = 0; n < nsteps; n++) {
                if (mixed) CUCK(cudaGraphLaunch(c->mix_exec, s.stream));
                CUCK(cudaGraphLaunch(s.gexec, s.stream));
            }
        }
    } else {
        for (int n = 0; n < nsteps; n++) {
            for (auto &p : pre) HFCK(run(c, p, s.stream));
            HFCK(run(c, init, s.stream));
            if (use_cg1) {
                HFCK(run(c, L1.W[0], s.stream));
                HFCK(host_cg1_loop(c, s, L1, o.max_iter, resolved(c, o).replace_every));
            } else {
                HFCK(comm_after(c, s, 1, true));
                HFCK(host_cg_loop(c, s, L, o.max_iter, o.replace_every));
            }
            for (auto &p : post) HFCK(run(c, p, s.stream));
            if (c->comm) {
                // the next RHS reads u^{n+1} ghosts: kernel B keeps the iterate's ghost planes
                // consistent (x update on every local plane)
                HFCK(read_state(c, s));
                if (s.st_host->first_failed >= 0) break;
            }
        }
    }
    return HF_OK;
}

static hf_status finish_stats(hf_ctx *c, Sys &s, hf_sim_stats *stats, float ms)
{
    HFCK(read_state(c, s));
    const CgState &h = *s.st_host;
    if (stats) {
        stats->steps_done = h.steps_done;
        stats->total_iters = h.total_iters;
        stats->max_iters_step = h.max_iters_step;
        stats->first_failed_step = h.first_failed;
        stats->ms_total = ms;
        stats->ms_steps = c->step_flush ? c->last_ms_steps : ms;
    }
    if (c->nsys > 1) return HF_OK;             // stacked systems: per-system results (batched_stacked)
    if (h.first_failed >= 0) {
        if (h.status == ST_BREAKDOWN) return fail(HF_E_BREAKDOWN, "hf_simulate: PCG breakdown");
        return fail(HF_E_NOCONV, "hf_simulate: PCG did not converge");
    }
    return HF_OK;
}

static hf_status simulate_common(hf_ctx *c, double theta, double dt, int32_t nsteps, const double *F, double *u,
                                 double *u_prev, int64_t step0, int64_t snap_plane, double *snap,
                                 const hf_cg_opts *opts, hf_sim_stats *stats)
{
    if (!c || !u || nsteps < 0 || !(dt > 0.0) || !(theta >= 0.0 && theta <= 1.0))
        return fail(HF_E_ARG, "hf_simulate: bad argument");
    if (!c->coef_set) return fail(HF_E_STATE, "hf_simulate: coefficients not set");
    if (c->comm && !c->comm->ready()) return fail(HF_E_STATE, "hf_simulate: peer transport not connected (hf_peer_connect)");
    if (snap && (snap_plane < 0 || snap_plane >= c->nz1g)) return fail(HF_E_INDEX, "hf_simulate: snap_plane");
    HFCK(check_ptrs(c, "hf_simulate", {F, u, u_prev, snap}));
    CUCK(cudaSetDevice(c->device));
    Sys &s = c->sys0;
    hf_cg_opts o = {1e-12, 10000, -1};
    if (opts) o = *opts;
    o = resolved(c, o);
    // the flux load lives in a stable internal buffer (graph parameters point at it)
    void *fbuf;
    HFCK(scratch_get(c, 7, (size_t)c->nloc * 8, &fbuf));
    if (F) HFCK(copy_in(c, (double *)fbuf, F, c->nzl, s.stream));
    else CUCK(cudaMemsetAsync(fbuf, 0, c->nloc * c->es, s.stream));
    HFCK(copy_in(c, s.U[0], u, c->nzl, s.stream));
    const bool first = step0 <= 0 || !u_prev;
    if (!first) HFCK(copy_in(c, s.U[2], u_prev, c->nzl, s.stream));
    int snap_local = -1;
    double *snapdev = nullptr;
    if (snap) {
        snap_local = (int)(snap_plane - c->zg0);
        if (snap_local < 0 || snap_local >= c->nzl) snap_local = -1;
        void *z;
        HFCK(scratch_get(c, 8, (size_t)std::max(1, nsteps) * c->plane * c->es, &z));
        snapdev = (double *)z;
    }
    cudaEvent_t e0, e1;
    CUCK(cudaEventCreate(&e0));
    CUCK(cudaEventCreate(&e1));
    CUCK(cudaEventRecord(e0, s.stream));
    hf_status st = simulate_sys(c, s, theta, dt, nsteps, (const double *)fbuf, first, snap_local, snapdev, o);
    CUCK(cudaEventRecord(e1, s.stream));
    if (st != HF_OK) { cudaStreamSynchronize(s.stream); cudaEventDestroy(e0); cudaEventDestroy(e1); return st; }
    CUCK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    hf_status fs = finish_stats(c, s, stats, ms);
    // the newest iterate sits in U[steps % 3] (or U[(failed+1) % 3]); stacked systems: the
    // converged ones in U[nsteps % 3], a failed system's slice is fetched by batched_stacked
    const CgState &h = *s.st_host;
    const int last = c->nsys > 1 ? nsteps : (h.first_failed >= 0 ? h.first_failed + 1 : h.steps_done);
    HFCK(copy_out(c, u, s.U[last % 3], c->nzl, s.stream));
    if (u_prev && nsteps > 0) HFCK(copy_out(c, u_prev, s.U[(last + 2) % 3], c->nzl, s.stream));
    if (snap && snap_local >= 0) HFCK(copy_out(c, snap, snapdev, nsteps, s.stream));
    CUCK(cudaStreamSynchronize(s.stream));
    return fs;
}

extern "C" {

hf_status hf_simulate(hf_ctx *c, double theta, double dt, int32_t nsteps, const double *F, double *u,
                      int64_t snap_plane, double *snap, const hf_cg_opts *opts, hf_sim_stats *stats)
{
    return simulate_common(c, theta, dt, nsteps, F, u, nullptr, 0, snap_plane, snap, opts, stats);
}

hf_status hf_simulate_resume(hf_ctx *c, double theta, double dt, int32_t nsteps, const double *F, double *u,
                             double *u_prev, int64_t step0, const hf_cg_opts *opts, hf_sim_stats *stats)
{
    if (!c || !u) return fail(HF_E_ARG, "hf_simulate_resume: NULL argument");
    if (step0 > 0 && !u_prev) return fail(HF_E_ARG, "hf_simulate_resume: u_prev needed for step0 > 0");
    return simulate_common(c, theta, dt, nsteps, F, u, u_prev, step0, -1, nullptr, opts, stats);
}

}  // extern "C"

// ---- batched simulations: independent systems stacked along z ------------------------------
// G independent systems on the same grid are stacked along z into one context of G (nz + 1)
// node planes; the element layer between two systems gets k = c = 0, so no element couples two
// systems and the stacked operator is exactly block diagonal ("rapid successive solutions":
// the GPU sees G times the parallelism of one 1M-DoF system, which alone is latency-bound).
// Each system keeps its own PCG (Alg. 1): its own delta, alpha, beta, ||b_j|| and stop test
// ||r_j|| <= rtol ||b_j||, its own iteration count and failure status.  Every stencil CTA and
// every kernel-B block works inside one system and writes that system's partial sums; a system
// that has converged (or failed) stops while the others iterate on; the loop ends when none
// iterates.  z-face Dirichlet values apply to each system's own z faces (Geom::zper).
static hf_status stack_ctx(hf_ctx *c, int G, hf_ctx **out)
{
    auto it = c->stacks.find(G);
    if (it != c->stacks.end()) { *out = it->second; return HF_OK; }
    hf_grid g2 = c->g;
    g2.ne[2] = (int64_t)G * (c->g.ne[2] + 1) - 1;
    hf_ctx *s = new hf_ctx();
    hf_status st = ctx_init(s, &g2, c->device, c->stream, 0, 1, G);
    if (st == HF_OK && c->prec != 64) st = hf_set_precision(s, c->prec);
    if (st == HF_OK && c->elem != EL_Q1) st = hf_set_element(s, c->elem);
    if (st != HF_OK) { ctx_free(s); delete s; return st; }
    s->dbits = c->dbits;
    for (int f = 0; f < 6; f++) s->gval[f] = c->gval[f];
    s->driver = c->driver;
    s->unroll = c->unroll;
    s->zchunk = c->zchunk;
    s->pdl = c->pdl;
    s->check_every = c->check_every;
    s->tm_fence = c->tm_fence;
    if (c->lo) {                            // mixed precision: the stack gets its own fp32 shadow
        const hf_status sm = hf_set_mixed(s, 1, c->mix_rtol);
        if (sm != HF_OK) { ctx_free(s); delete s; return sm; }
    }
    c->stacks[G] = s;
    *out = s;
    return HF_OK;
}

static hf_status simulate_common(hf_ctx *c, double theta, double dt, int32_t nsteps, const double *F, double *u,
                                 double *u_prev, int64_t step0, int64_t snap_plane, double *snap,
                                 const hf_cg_opts *opts, hf_sim_stats *stats);

// systems per stack: about 8M stacked nodes (a 1M-DoF system alone is latency-bound, a stack of
// 8 streams at the HBM roofline), at most 256 (kernel B's loop duties scan the systems with one
// block) and at most B
// Systems per stack (batched sims, a13).  A stack of G systems runs its stencil kernels on
// tx * ty * G * nch CTAs, each system's z-range cut into nch chunks (stencil_grid); CTAs are
// dispatched in waves of (SMs x resident CTAs per SM) slots, and every chunk carries ~4 planes of
// warm-up / prologue.  The group size is the one that minimises the modelled time of the whole
// batch: sum over groups of (systems / slot efficiency).  E.g. C5 (100^3 nodes, 28 tile
// columns, 296 slots): a stack of 8 fills 224 of 296 slots (efficiency 0.72), a stack of 5 with
// two chunks per system 280 (0.86), a stack of 10 280 (0.91).  Measured C5 sim-steps/s, B = 20:
// groups of 10: 193, 5: 189, 4: 176, 7: 161, 20: 152; B = 8: 5 + 3: 196, one stack of 8: 185.
static int stack_group(const hf_ctx *c, int B)
{
    if (c->batch_group > 0) return std::min(c->batch_group, B);
    const long long nn = (long long)c->pitch * c->ny1 * c->nz1g;     // nodes per system (padded)
    const int planes = c->nz1g;
    // stacks stay below the R = 4 tile threshold (default_tile_r): measured at C5, stacks of 16-20
    // systems on R = 4 tiles ran 20 % slower than stacks of 10 on R = 2 tiles
    const int gmax = (int)std::min<long long>(std::min<long long>(B, 64), std::max(1LL, ((16LL << 20) - 1) / nn));
    auto eff = [&](int G) -> double {
        const int R = 2;
        const int occ = std::max(1, c->tileR == 2 ? c->occ : 2);
        const long long tx = (c->nx1 + TILE_X - 1) / TILE_X, ty = (c->ny1 + NW * R - 2) / (NW * R - 1);
        const long long cols = tx * ty, slots = (long long)c->nsm * occ;
        long long nch = std::max(1LL, slots / (cols * G));
        const long long chunk = (planes + nch - 1) / nch;
        nch = (planes + chunk - 1) / chunk;
        const long long ctas = cols * G * nch, waves = (ctas + slots - 1) / slots;
        return (double)(G * (long long)planes * cols) / ((double)waves * slots * (chunk + 4));
    };
    int best = 1;
    double tbest = 1e300;
    for (int G = 1; G <= gmax; G++) {
        const int full = B / G, rem = B % G;
        const double t = full * (G / eff(G)) + (rem ? rem / eff(rem) : 0.0);
        if (t < tbest * (1.0 - 1e-9)) { tbest = t; best = G; }
    }
    return best;
}

static hf_status batched_stacked(hf_ctx *c, int32_t B, const double *k_batch, const double *c_batch, double theta,
                                 double dt, int32_t nsteps, const double *F, double *u_batch, int64_t snap_plane,
                                 double *front_out, const hf_cg_opts &o, hf_sim_stats *stats)
{
    const size_t nxy = (size_t)c->g.ne[0] * c->g.ne[1];
    const size_t ne = nxy * (size_t)c->g.ne[2];
    const size_t pl = (size_t)c->nx1 * c->ny1;
    const size_t nn = pl * (size_t)c->nz1g;             // natural nodes of one system
    const int G = stack_group(c, B);
    const double *cshared = nullptr;
    if (!c_batch) {                                   // the context's c, unpacked once
        void *p;
        HFCK(scratch_get(c, 50, ne * sizeof(double), &p));
        const unsigned nb = (unsigned)((ne + 255) / 256);
        if (c->es == 8) k_extract_c<double><<<nb, 256, 0, c->stream>>>(make_geom(c), (int)c->g.ne[2], c->sys0.kc, (double *)p, c->launches);
        else k_extract_c<float><<<nb, 256, 0, c->stream>>>(make_geom(c), (int)c->g.ne[2], c->sys0.kc, (double *)p, c->launches);
        CUCK(cudaGetLastError());
        cshared = (const double *)p;
    }
    hf_status first_err = HF_OK;
    for (int j0 = 0; j0 < B; j0 += G) {
        const int g = std::min(G, B - j0);
        hf_ctx *s;
        HFCK(stack_ctx(c, g, &s));
        const size_t nes = (size_t)g * ne + (size_t)(g - 1) * nxy;
        void *kp, *cp, *fp, *up;
        HFCK(scratch_get(c, 51, nes * sizeof(double), &kp));
        HFCK(scratch_get(c, 52, nes * sizeof(double), &cp));
        HFCK(scratch_get(c, 53, (size_t)g * nn * sizeof(double), &fp));
        HFCK(scratch_get(c, 54, (size_t)g * nn * sizeof(double), &up));
        double *ks = (double *)kp, *cs = (double *)cp, *fs = (double *)fp, *us = (double *)up;
        for (int i = 0; i < g; i++) {
            const size_t o1 = (size_t)i * (ne + nxy);
            const int j = j0 + i;
            CUCK(cudaMemcpyAsync(ks + o1, k_batch + (size_t)j * ne, ne * sizeof(double), cudaMemcpyDefault, c->stream));
            const double *cj = c_batch ? c_batch + (size_t)j * ne : cshared;
            CUCK(cudaMemcpyAsync(cs + o1, cj, ne * sizeof(double), cudaMemcpyDefault, c->stream));
            if (i + 1 < g) {                            // separator element layer: k = c = 0
                CUCK(cudaMemsetAsync(ks + o1 + ne, 0, nxy * sizeof(double), c->stream));
                CUCK(cudaMemsetAsync(cs + o1 + ne, 0, nxy * sizeof(double), c->stream));
            }
            if (F) CUCK(cudaMemcpyAsync(fs + (size_t)i * nn, F, nn * sizeof(double), cudaMemcpyDefault, c->stream));
            else CUCK(cudaMemsetAsync(fs + (size_t)i * nn, 0, nn * sizeof(double), c->stream));
            CUCK(cudaMemcpyAsync(us + (size_t)i * nn, u_batch + (size_t)j * nn, nn * sizeof(double), cudaMemcpyDefault,
                                 c->stream));
        }
        HFCK(hf_set_coefficients(s, ks, cs));
        hf_sim_stats st;
        std::memset(&st, 0, sizeof(st));
        hf_status rs = simulate_common(s, theta, dt, nsteps, fs, us, nullptr, 0, -1, nullptr, &o, &st);
        if (rs != HF_OK && rs != HF_E_NOCONV && rs != HF_E_BREAKDOWN) return rs;
        // per-system results: each system's newest iterate is in U[steps % 3] (all steps done) or
        // U[(failed + 1) % 3] of its own slice (simulate_common copied the former into us)
        const CgState *h = s->sys0.st_host;             // read back by simulate_common
        for (int i = 0; i < g; i++) {
            const int j = j0 + i;
            const double *src = us + (size_t)i * nn;
            if (h[i].first_failed >= 0) {
                // the failed system's slice of U[(failed + 1) % 3] (padded layout of the stack)
                const double *ring = s->sys0.U[(h[i].first_failed + 1) % 3];
                HFCK(copy_out(s, us + (size_t)i * nn, eoff(s, ring, (long long)i * s->sys_planes * s->plane),
                              s->sys_planes, c->stream));
                if (first_err == HF_OK) first_err = h[i].status == ST_BREAKDOWN ? HF_E_BREAKDOWN : HF_E_NOCONV;
            }
            CUCK(cudaMemcpyAsync(u_batch + (size_t)j * nn, src, nn * sizeof(double), cudaMemcpyDefault, c->stream));
            if (front_out)
                CUCK(cudaMemcpyAsync(front_out + (size_t)j * pl, src + (size_t)snap_plane * pl, pl * sizeof(double),
                                     cudaMemcpyDefault, c->stream));
            if (stats) {
                stats[j].steps_done = h[i].steps_done;
                stats[j].total_iters = h[i].total_iters;
                stats[j].max_iters_step = h[i].max_iters_step;
                stats[j].first_failed_step = h[i].first_failed;
                stats[j].ms_total = st.ms_total;
                stats[j].ms_steps = st.ms_steps;
            }
        }
        CUCK(cudaStreamSynchronize(c->stream));
    }
    if (first_err != HF_OK) return fail(first_err, "hf_simulate_batched: a system failed to converge");
    return HF_OK;
}

extern "C" {

hf_status hf_simulate_batched(hf_ctx *c, int32_t B, const double *k_batch, const double *c_batch, double theta,
                              double dt, int32_t nsteps, const double *F, double *u_batch, int64_t snap_plane,
                              double *front_out, const hf_cg_opts *opts, hf_sim_stats *stats)
{
    if (!c || B < 0 || nsteps < 0 || !(dt > 0.0)) return fail(HF_E_ARG, "hf_simulate_batched: bad argument");
    if (B == 0) return HF_OK;                    // an empty batch (its arrays may be NULL)
    if (!k_batch || !u_batch) return fail(HF_E_ARG, "hf_simulate_batched: NULL k_batch / u_batch");
    if (!c_batch && !c->coef_set) return fail(HF_E_STATE, "hf_simulate_batched: no capacity field");
    if (c->comm) return fail(HF_E_ARG, "hf_simulate_batched: not available on slab contexts");
    if (c->tetv) return fail(HF_E_STATE, "hf_simulate_batched: per-element coefficients only (not vertex materials)");
    if (front_out && (snap_plane < 0 || snap_plane >= c->nz1g)) return fail(HF_E_INDEX, "snap_plane");
    HFCK(check_ptrs(c, "hf_simulate_batched", {k_batch, c_batch, F, u_batch, front_out}));
    CUCK(cudaSetDevice(c->device));
    hf_cg_opts o = {1e-12, 10000, -1};
    if (opts) o = *opts;
    o = resolved(c, o);
    return batched_stacked(c, B, k_batch, c_batch, theta, dt, nsteps, F, u_batch, snap_plane, front_out, o, stats);
}

// ============================================================================================
// slabs

hf_status hf_slab_plan(int64_t nz1, int32_t rank, int32_t nranks, int64_t *z_lo, int64_t *z_hi)
{
    if (nranks < 1 || rank < 0 || rank >= nranks || !z_lo || !z_hi) return fail(HF_E_ARG, "hf_slab_plan: bad argument");
    if (nz1 < 2LL * nranks) return fail(HF_E_PARTITION, "hf_slab_plan: fewer than 2 node planes per rank");
    const int64_t base = nz1 / nranks, rem = nz1 % nranks;
    *z_lo = rank * base + std::min<int64_t>(rank, rem);
    *z_hi = *z_lo + base + (rank < rem ? 1 : 0);
    return HF_OK;
}

hf_status hf_nccl_unique_id(uint8_t id[128])
{
    if (!id) return fail(HF_E_ARG, "hf_nccl_unique_id: NULL");
    HFCK(nccl::load());
    nccl::ncclUniqueId u;
    NCCK(nccl::g_api.getUniqueId(&u));
    std::memcpy(id, u.internal, 128);
    return HF_OK;
}

}  // extern "C"

// ---- NCCL transport ------------------------------------------------------------------------
struct NcclComm : Comm {
    nccl::ncclComm_t comm = nullptr;
    bool aborted = false;
    ~NcclComm() override { if (comm && !aborted) nccl::g_api.commDestroy(comm); }
    bool graph_capturable() const override { return true; }
    hf_status poll() override
    {
        nccl::ncclResult_t ae = 0;
        if (comm && !aborted && nccl::g_api.commGetAsyncError(comm, &ae) == 0 && ae != 0 && ae != 7 /* inProgress */) {
            nccl::g_api.commAbort(comm);
            aborted = true;
            return fail(HF_E_NCCL, std::string("NCCL asynchronous error: ") + nccl::g_api.getErrorString(ae));
        }
        return HF_OK;
    }
    hf_status exchange(hf_ctx *c, Sys &s, double *v) override
    {
        const long long P = c->plane;
        const int dt = c->es == 8 ? nccl::ncclFloat64 : nccl::ncclFloat32;
        NCCK(nccl::g_api.groupStart());
        if (c->rank > 0) {
            NCCK(nccl::g_api.send(eoff(c, v, c->own_lo * P), P, dt, c->rank - 1, comm, s.stream));
            NCCK(nccl::g_api.recv(eoff(c, v, (c->own_lo - 1) * P), P, dt, c->rank - 1, comm, s.stream));
        }
        if (c->rank < c->nranks - 1) {
            NCCK(nccl::g_api.send(eoff(c, v, (c->own_hi - 1) * P), P, dt, c->rank + 1, comm, s.stream));
            NCCK(nccl::g_api.recv(eoff(c, v, c->own_hi * P), P, dt, c->rank + 1, comm, s.stream));
        }
        NCCK(nccl::g_api.groupEnd());
        return HF_OK;
    }
    hf_status allreduce(hf_ctx *c, Sys &s, double *v, int n) override
    {
        (void)c;
        NCCK(nccl::g_api.allReduce(v, v, (size_t)n, nccl::ncclFloat64, nccl::ncclSum, comm, s.stream));
        return HF_OK;
    }
};

// ---- peer-memory transport (the product path for N > 1; see PeerSync in hf_kernels.cuh) -----
// Mailbox of a rank (one device allocation, exported by CUDA IPC across processes):
//   [MailHdr | pad to 4 KB][ghost lo | ghost hi][xbuf lo: 2 parity slots][xbuf hi: 2 parity slots]
// each plane slot pb bytes (the fp64 plane rounded up to 256 B; the fp32 planes fit too).
static const size_t MAIL_HDR = 4096;

struct PeerBlob {                     // what a rank tells the others (hf_peer_export)
    uint32_t magic, version;
    int32_t pid, rank, nranks, device;
    char bus[32];                     // PCI bus id of the rank's GPU
    uint64_t mail_ptr, mail_bytes, pb;
    cudaIpcMemHandle_t handle;
};
static_assert(sizeof(PeerBlob) <= 256, "peer blob");
static const uint32_t PEER_MAGIC = 0x48465052u;   // "HFPR"

struct hf_local_group;
static void group_barrier(hf_local_group *g);

struct PeerComm : Comm {
    int transport = 1;                // 1: ranks in this process, 2: ranks in separate processes (IPC)
    hf_local_group *grp = nullptr;    // transport 1
    char *mail = nullptr;
    size_t mail_bytes = 0, pb = 0;
    PeerSync host;
    PeerSync *dev = nullptr;
    std::vector<void *> opened;       // IPC mappings of the peers' mailboxes
    bool connected = false;
    ~PeerComm() override
    {
        for (void *p : opened) cudaIpcCloseMemHandle(p);
        cudaFree(dev);
        cudaFree(mail);
    }
    bool graph_capturable() const override { return true; }
    bool in_kernel() const override { return true; }
    bool ready() const override { return connected; }
    hf_status enter() override
    {
        if (grp) group_barrier(grp);
        return HF_OK;
    }
    const PeerSync *peer_dev() const override { return connected ? dev : nullptr; }
    hf_status allreduce(hf_ctx *, Sys &, double *, int) override { return HF_OK; }   // in the kernels
    hf_status exchange(hf_ctx *c, Sys &s, double *v) override
    {
        const long long P = c->plane;
        const long long glo = c->own_lo > 0 ? 0 : -1, ghi = c->own_hi < c->nzl ? (long long)c->own_hi * P : -1;
        const unsigned nb = (unsigned)std::max(1LL, std::min<long long>((P + 255) / 256, 64));
        if (c->es == 8) {
            k_xsend<double><<<nb, 256, 0, s.stream>>>(dev, v, c->launches);
            k_xrecv<double><<<nb, 256, 0, s.stream>>>(dev, v, glo, ghi, c->launches);
        } else {
            k_xsend<float><<<nb, 256, 0, s.stream>>>(dev, v, c->launches);
            k_xrecv<float><<<nb, 256, 0, s.stream>>>(dev, v, glo, ghi, c->launches);
        }
        CUCK(cudaGetLastError());
        return HF_OK;
    }
    // device copy of the protocol state for the context's current layout (precision)
    hf_status refresh(hf_ctx *c)
    {
        host.lo0 = (long long)c->own_lo * c->plane;
        host.hi0 = (long long)(c->own_hi - 1) * c->plane;
        host.plane = c->plane;
        host.xslot = (long long)(pb / c->es);
        if (!dev) CUCK(cudaMalloc(&dev, sizeof(PeerSync)));
        CUCK(cudaMemcpy(dev, &host, sizeof(PeerSync), cudaMemcpyHostToDevice));
        return HF_OK;
    }
    // every rank's mailbox, mapped in this process: fill the protocol state
    hf_status connect(hf_ctx *c, const std::vector<char *> &mb, int share)
    {
        const int R = c->nranks, r = c->rank;
        std::memset(&host, 0, sizeof(host));
        host.nranks = R;
        host.rank = r;
        host.mine = (MailHdr *)mb[r];
        for (int q = 0; q < R; q++) host.peer[q] = (MailHdr *)mb[q];
        const size_t G0 = MAIL_HDR, X0 = MAIL_HDR + 2 * pb, X1 = MAIL_HDR + 4 * pb;
        host.gdst_lo = r > 0 ? mb[r - 1] + G0 + pb : nullptr;      // lower neighbour's hi ghost
        host.gdst_hi = r + 1 < R ? mb[r + 1] + G0 : nullptr;       // upper neighbour's lo ghost
        host.xdst_lo = r > 0 ? mb[r - 1] + X1 : nullptr;
        host.xdst_hi = r + 1 < R ? mb[r + 1] + X0 : nullptr;
        host.xsrc_lo = mb[r] + X0;
        host.xsrc_hi = mb[r] + X1;
        HFCK(refresh(c));
        if (share > 1) {
            // ranks sharing one GPU (tests): every rank's grids fit on the GPU at once, so a rank
            // waiting inside a kernel never starves the rank it waits for; no early launches
            c->nsm_share = std::max(1, c->nsm / share);
            c->pdl = 0;
        }
        connected = true;
        c->ghost_buf = mail + MAIL_HDR;
        c->ghost_pb = pb;
        return sys_maps(c, c->sys0);
    }
};

// mailbox of a new slab context (zeroed: flags and counters start at 0)
static hf_status peer_alloc(hf_ctx *c, PeerComm *pc)
{
    const size_t plane64 = (size_t)((c->nx1 + 1) / 2 * 2) * c->ny1 * 8;
    const size_t plane32 = (size_t)((c->nx1 + 3) / 4 * 4) * c->ny1 * 4;
    pc->pb = (std::max(plane64, plane32) + 255) / 256 * 256;
    pc->mail_bytes = MAIL_HDR + 6 * pc->pb;
    CUCK(cudaMalloc(&pc->mail, pc->mail_bytes));
    CUCK(cudaMemset(pc->mail, 0, pc->mail_bytes));
    return HF_OK;
}

static void bus_id(int device, char out[32])
{
    std::memset(out, 0, 32);
    if (cudaDeviceGetPCIBusId(out, 31, device) != cudaSuccess) {
        cudaGetLastError();
        std::snprintf(out, 32, "dev%d", device);
    }
}

struct hf_local_group {               // ranks of one process (transport 1)
    int n = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long long gen = 0;
    std::vector<char *> mail;
    std::vector<int> device;
    void barrier()
    {
        std::unique_lock<std::mutex> lk(mu);
        const long long g = gen;
        if (++arrived == n) { arrived = 0; gen++; cv.notify_all(); }
        else cv.wait(lk, [&] { return gen != g; });
    }
};

static void group_barrier(hf_local_group *g) { g->barrier(); }

extern "C" {

hf_status hf_local_group_create(int32_t nranks, hf_local_group **out)
{
    if (nranks < 1 || nranks > HF_MAX_RANKS || !out) return fail(HF_E_ARG, "hf_local_group_create: bad argument");
    hf_local_group *g = new hf_local_group();
    g->n = nranks;
    g->mail.assign(nranks, nullptr);
    g->device.assign(nranks, 0);
    *out = g;
    return HF_OK;
}

void hf_local_group_destroy(hf_local_group *g) { delete g; }

hf_status hf_create_slab(const hf_grid *g, int32_t rank, int32_t nranks, const uint8_t *id, int32_t transport,
                         int device, void *cuda_stream, hf_ctx **out)
{
    if (!g || !out || nranks < 1 || rank < 0 || rank >= nranks) return fail(HF_E_ARG, "hf_create_slab: bad argument");
    if ((transport == 0 || transport == 1) && !id) return fail(HF_E_ARG, "hf_create_slab: NULL id");
    if (transport != 0 && nranks > HF_MAX_RANKS)
        return fail(HF_E_ARG, "hf_create_slab: at most " + std::to_string(HF_MAX_RANKS) + " ranks (one node)");
    hf_ctx *c = new hf_ctx();
    hf_status st = ctx_init(c, g, device, cuda_stream, rank, nranks);
    if (st != HF_OK) { ctx_free(c); delete c; return st; }
    if (transport == 0) {
        st = nccl::load();
        if (st == HF_OK) {
            NcclComm *nc = new NcclComm();
            nccl::ncclUniqueId u;
            std::memcpy(u.internal, id, 128);
            nccl::ncclResult_t r = nccl::g_api.commInitRank(&nc->comm, nranks, u, rank);
            if (r != 0) { st = fail(HF_E_NCCL, std::string("ncclCommInitRank: ") + nccl::g_api.getErrorString(r)); delete nc; }
            else c->comm = nc;
        }
    } else if (transport == 1 || transport == 2) {
        PeerComm *pc = new PeerComm();
        pc->transport = transport;
        c->comm = pc;
        st = peer_alloc(c, pc);
        if (st == HF_OK && transport == 1) {
            // in-process group: publish the mailbox, wait for every rank, connect with plain pointers
            hf_local_group *grp = (hf_local_group *)id;
            if (grp->n != nranks) st = fail(HF_E_ARG, "hf_create_slab: group size != nranks");
            else {
                {
                    std::lock_guard<std::mutex> lk(grp->mu);
                    grp->mail[rank] = pc->mail;
                    grp->device[rank] = device;
                }
                grp->barrier();
                pc->grp = grp;
                int share = 0;
                for (int q = 0; q < nranks; q++) share += grp->device[q] == device;
                const uintptr_t sh = (uintptr_t)cuda_stream;
                if (share > 1 && (sh == 1 || sh == 2))
                    st = fail(HF_E_ARG, "hf_create_slab: ranks sharing a GPU need their own streams (not the legacy or "
                                        "per-thread default stream): a rank waiting inside a kernel would block the others");
                for (int q = 0; q < nranks && st == HF_OK; q++)
                    if (grp->device[q] != device) {
                        cudaError_t e = cudaDeviceEnablePeerAccess(grp->device[q], 0);
                        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
                            st = fail(HF_E_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
                        cudaGetLastError();
                    }
                if (st == HF_OK) st = pc->connect(c, grp->mail, share);
                grp->barrier();
            }
        }
    } else st = fail(HF_E_ARG, "hf_create_slab: unknown transport");
    if (st != HF_OK) { ctx_free(c); delete c; return st; }
    *out = c;
    return HF_OK;
}

hf_status hf_peer_export(hf_ctx *c, uint8_t blob[HF_PEER_BLOB_BYTES])
{
    PeerComm *pc = c ? dynamic_cast<PeerComm *>(c->comm) : nullptr;
    if (!pc || !blob) return fail(HF_E_ARG, "hf_peer_export: not a peer-transport slab context");
    CUCK(cudaSetDevice(c->device));
    PeerBlob b;
    std::memset(&b, 0, sizeof(b));
    b.magic = PEER_MAGIC;
    b.version = 1;
    b.pid = (int32_t)getpid();
    b.rank = c->rank;
    b.nranks = c->nranks;
    b.device = c->device;
    bus_id(c->device, b.bus);
    b.mail_ptr = (uint64_t)(uintptr_t)pc->mail;
    b.mail_bytes = pc->mail_bytes;
    b.pb = pc->pb;
    CUCK(cudaIpcGetMemHandle(&b.handle, pc->mail));
    std::memset(blob, 0, HF_PEER_BLOB_BYTES);
    std::memcpy(blob, &b, sizeof(b));
    return HF_OK;
}

hf_status hf_peer_connect(hf_ctx *c, const uint8_t *blobs)
{
    PeerComm *pc = c ? dynamic_cast<PeerComm *>(c->comm) : nullptr;
    if (!pc || !blobs) return fail(HF_E_ARG, "hf_peer_connect: not a peer-transport slab context");
    if (pc->connected) return fail(HF_E_STATE, "hf_peer_connect: already connected");
    CUCK(cudaSetDevice(c->device));
    const int R = c->nranks;
    char mybus[32];
    bus_id(c->device, mybus);
    std::vector<char *> mb(R, nullptr);
    int share = 0;
    for (int q = 0; q < R; q++) {
        PeerBlob b;
        std::memcpy(&b, blobs + (size_t)q * HF_PEER_BLOB_BYTES, sizeof(b));
        if (b.magic != PEER_MAGIC || b.version != 1 || b.rank != q || b.nranks != R || b.pb != pc->pb)
            return fail(HF_E_ARG, "hf_peer_connect: blob " + std::to_string(q) + " does not belong to this group");
        share += std::strncmp(b.bus, mybus, 32) == 0;
        if (q == c->rank) { mb[q] = pc->mail; continue; }
        if (b.pid == (int32_t)getpid()) { mb[q] = (char *)(uintptr_t)b.mail_ptr; continue; }
        void *p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess)
            return fail(HF_E_CUDA, "hf_peer_connect: cudaIpcOpenMemHandle(rank " + std::to_string(q) + "): " +
                                       cudaGetErrorString(e));
        pc->opened.push_back(p);
        mb[q] = (char *)p;
    }
    return pc->connect(c, mb, share);
}

hf_status hf_slab_range(const hf_ctx *c, int64_t *z_lo, int64_t *z_hi, int64_t *local_planes, int64_t *local_z0)
{
    if (!c) return fail(HF_E_ARG, "hf_slab_range: NULL");
    if (z_lo) *z_lo = c->zg0 + c->own_lo;
    if (z_hi) *z_hi = c->zg0 + c->own_hi;
    if (local_planes) *local_planes = c->nzl;
    if (local_z0) *local_z0 = c->zg0;
    return HF_OK;
}

hf_status hf_get_launch_count(hf_ctx *c, int64_t *count)
{
    if (!c || !count) return fail(HF_E_ARG, "hf_get_launch_count: NULL");
    unsigned long long v = 0;
    CUCK(cudaMemcpyAsync(&v, c->launches, sizeof(v), cudaMemcpyDeviceToHost, c->stream));
    CUCK(cudaStreamSynchronize(c->stream));
    *count = (int64_t)v;
    return HF_OK;
}

hf_status hf_profile(hf_ctx *c, int32_t enable)
{
    if (!c) return fail(HF_E_ARG, "hf_profile: NULL");
    c->prof = enable != 0;
    for (int i = 0; i < 5; i++) { c->prof_ms[i] = 0; c->prof_n[i] = 0; }
    return HF_OK;
}

hf_status hf_profile_read(hf_ctx *c, double ms[5], int64_t n[5])
{
    if (!c) return fail(HF_E_ARG, "hf_profile_read: NULL");
    for (int i = 0; i < 5; i++) {
        if (ms) ms[i] = c->prof_ms[i];
        if (n) n[i] = c->prof_n[i];
    }
    return HF_OK;
}

hf_status hf_time_kernel_a(hf_ctx *c, int32_t reps, double *ms_per_launch)
{
    if (!c || reps < 1 || !ms_per_launch) return fail(HF_E_ARG, "hf_time_kernel_a: bad argument");
    if (!(c->last_aK > 0.0)) return fail(HF_E_STATE, "hf_time_kernel_a: no previous simulation");
    CUCK(cudaSetDevice(c->device));
    Sys &s = c->sys0;
    hf_cg_opts o = resolved(c, {1e-12, 10000, -1});
    o.max_iter = 1 << 30;                       // every replayed launch must run:
    o.rtol = 0.0;                               // no stop test either (the guess may already
                                                // be the converged solution of the last step)
    HFCK(set_solver_opts(c, s, o));
    StencilArgs ia = base_args(c, c->last_aK, 1.0);
    ia.invd = s.invd;
    ia.bvec = s.b;
    ia.out0 = s.r;
    ia.out_s = s.s;
    ia.first = 1;
    ia.rot_role = ROT_INIT;
    for (int i = 0; i < 3; i++) ia.ring[i] = s.U[i];
    ia.sy = make_sync(c, s, -1, 1);
    ia.zs0 = c->own_lo;
    ia.zs1 = c->own_hi;
    Launch init;
    HFCK(stencil_launch(c, LD_X0, EP_RESID_INIT, true, s.maps, ia, 2, &init));
    CgLaunches L;
    HFCK(cg_launches(c, s, c->last_aK, 1.0, nullptr, s.maps, &L));
    const bool prof = c->prof;
    c->prof = false;
    HFCK(run(c, init, s.stream));
    HFCK(run(c, L.A, s.stream));                // warm
    cudaEvent_t e0, e1;
    CUCK(cudaEventCreate(&e0));
    CUCK(cudaEventCreate(&e1));
    CUCK(cudaEventRecord(e0, s.stream));
    for (int i = 0; i < reps; i++) HFCK(run(c, L.A, s.stream));
    CUCK(cudaEventRecord(e1, s.stream));
    CUCK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->prof = prof;
    *ms_per_launch = ms / reps;
    return HF_OK;
}

// Kernel A replayed as a CUDA graph of `reps` kernel-A nodes joined by the programmatic edges of
// the PCG loop body (each launch's prologue overlaps the previous launch's tail, as behind
// kernel B in the loop), timed as one graph launch after a warm-up launch.
hf_status hf_time_kernel_a_graph(hf_ctx *c, int32_t reps, double *ms_per_launch)
{
    if (!c || reps < 1 || !ms_per_launch) return fail(HF_E_ARG, "hf_time_kernel_a_graph: bad argument");
    if (!(c->last_aK > 0.0)) return fail(HF_E_STATE, "hf_time_kernel_a_graph: no previous simulation");
    CUCK(cudaSetDevice(c->device));
    Sys &s = c->sys0;
    hf_cg_opts o = resolved(c, {1e-12, 10000, -1});
    o.max_iter = 1 << 30;                       // every launch runs (no stop test)
    o.rtol = 0.0;
    HFCK(set_solver_opts(c, s, o));
    StencilArgs ia = base_args(c, c->last_aK, 1.0);
    ia.invd = s.invd;
    ia.bvec = s.b;
    ia.out0 = s.r;
    ia.out_s = s.s;
    ia.first = 1;
    ia.rot_role = ROT_INIT;
    for (int i = 0; i < 3; i++) ia.ring[i] = s.U[i];
    ia.sy = make_sync(c, s, -1, 1);
    ia.zs0 = c->own_lo;
    ia.zs1 = c->own_hi;
    Launch init;
    HFCK(stencil_launch(c, LD_X0, EP_RESID_INIT, true, s.maps, ia, 2, &init));
    CgLaunches L;
    HFCK(cg_launches(c, s, c->last_aK, 1.0, nullptr, s.maps, &L));
    const bool prof = c->prof;
    c->prof = false;
    HFCK(run(c, init, s.stream));
    cudaGraph_t g;
    CUCK(cudaGraphCreate(&g, 0));
    cudaGraphNode_t prev = nullptr, n;
    for (int i = 0; i < reps; i++) {
        if (prev && c->pdl) {
            HFCK(add_node(g, L.A, nullptr, &n));
            HFCK(add_pdl_edge(g, prev, n));
        } else
            HFCK(add_node(g, L.A, prev ? &prev : nullptr, &n));
        prev = n;
    }
    cudaGraphExec_t ge;
    CUCK(cudaGraphInstantiate(&ge, g, 0));
    CUCK(cudaGraphLaunch(ge, s.stream));            // warm
    cudaEvent_t e0, e1;
    CUCK(cudaEventCreate(&e0));
    CUCK(cudaEventCreate(&e1));
    CUCK(cudaEventRecord(e0, s.stream));
    CUCK(cudaGraphLaunch(ge, s.stream));
    CUCK(cudaEventRecord(e1, s.stream));
    CUCK(cudaEventSynchronize(e1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    c->prof = prof;
    *ms_per_launch = ms / reps;
    return HF_OK;
}

#ifdef HF_TRACE
// debug builds only (not part of the ABI): kernel-A timestamps of the last traced launch
hf_status hf_trace_read(unsigned long long *out, int32_t nblocks)
{
    CUCK(cudaDeviceSynchronize());
    CUCK(cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 8 * (size_t)std::min(nblocks, 4096)));
    return HF_OK;
}
#endif

hf_status hf_set_driver(hf_ctx *c, int32_t driver)
{
    if (!c || driver < 0 || driver > 1) return fail(HF_E_ARG, "hf_set_driver: bad argument");
    c->driver = driver;
    drop_stacks(c);
    return HF_OK;
}

hf_status hf_set_element(hf_ctx *c, int32_t type)
{
    if (!c || type < 0 || type > 1) return fail(HF_E_ARG, "hf_set_element: type must be 0 (Q1) or 1 (6 P1 tets)");
    CUCK(cudaSetDevice(c->device));
    c->elem = type;
    c->ab_ready = false;
    drop_stacks(c);
    const double *h = c->g.h;
    // the dense (tet) element keeps R = 2 tiles (R = 4 spills); TMA boxes follow the tile height
    int want_r = default_tile_r(c, type);
    if (type != EL_DENSE && c->tile_r_set) want_r = c->tile_r_set;
    CUCK(cudaStreamSynchronize(c->stream));
    if (want_r != c->tileR) c->tileR = want_r;
    HFCK(sys_maps(c, c->sys0));              // also selects the material-id map (Q1 only)
    if (type == EL_DENSE) {
        double K[64], M[64];
        tet_voxel(h, K, M);
        for (int l = 0; l < 8; l++) { c->dg.Kd[l] = K[l * 9]; c->dg.Md[l] = M[l * 9]; }
    } else {
        for (int l = 0; l < 8; l++) {
            c->dg.Kd[l] = (h[1] * h[2] / h[0] + h[0] * h[2] / h[1] + h[0] * h[1] / h[2]) / 9.0;
            c->dg.Md[l] = h[0] * h[1] * h[2] / 27.0;
        }
    }
    HFCK(update_occ(c));
    c->sys0.key_valid = false;
    if (c->lo) HFCK(hf_set_element(c->lo, type));
    return HF_OK;
}

hf_status hf_set_precision(hf_ctx *c, int32_t bits)
{
    if (!c || (bits != 32 && bits != 64)) return fail(HF_E_ARG, "hf_set_precision: bits must be 32 or 64");
    if (c->coef_set) return fail(HF_E_STATE, "hf_set_precision: call before hf_set_coefficients");
    if (c->lo && bits != 64) return fail(HF_E_STATE, "hf_set_precision: mixed precision is on (hf_set_mixed(ctx, 0) first)");
    if (bits == c->prec) return HF_OK;
    CUCK(cudaSetDevice(c->device));
    CUCK(cudaStreamSynchronize(c->stream));
    sys_free(c->sys0);
    drop_stacks(c);
    for (void *p : c->scratch) cudaFree(p);      // layouts change: reallocate (zeroed) on demand
    c->scratch.clear();
    c->scratch_cap.clear();
    c->prec = bits;
    c->es = bits / 8;
    set_layout(c);
    if (PeerComm *pc = dynamic_cast<PeerComm *>(c->comm))
        if (pc->connected) HFCK(pc->refresh(c));
    StencilFn f = stencil_fn(c->tileR, LD_CGD, EP_CGA, 0, c->elem, c->es);
    HFCK(ensure_smem_attr(f.fn, f.smem, c->device));
    int occ = 0;
    CUCK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, f.fn, 32 * f.nw, f.smem));
    c->occ = std::max(1, occ);
    HFCK(sys_alloc(c, c->sys0, c->stream));
    return HF_OK;
}

hf_status hf_set_tuning(hf_ctx *c, const char *key, int64_t value)
{
    if (!c || !key) return fail(HF_E_ARG, "hf_set_tuning: NULL argument");
    const std::string k(key);
    const long long v = value;
    if (k == "tile_r") {
        if (v != 0 && v != 2 && v != 4) return fail(HF_E_ARG, "hf_set_tuning: tile_r must be 0 (default), 2 or 4");
        c->tile_r_set = (int)v;
        if (c->lo) c->lo->tile_r_set = (int)v;  // the mixed-precision shadow follows
        return hf_set_element(c, c->elem);      // re-derives the tile height, TMA maps, grid occupancy
    }
    if (k == "zchunk") { if (v < 0) return fail(HF_E_ARG, "hf_set_tuning: zchunk >= 0"); c->zchunk = (int)v; }
    else if (k == "unroll") { if (v < 0 || v > 50) return fail(HF_E_ARG, "hf_set_tuning: unroll in 0..50"); c->unroll = (int)v; }
    else if (k == "pdl") { if (v < 0 || v > 1) return fail(HF_E_ARG, "hf_set_tuning: pdl 0 or 1"); c->pdl = (int)v; }
    else if (k == "fuse_ab") { if (v < 0 || v > 1) return fail(HF_E_ARG, "hf_set_tuning: fuse_ab 0 or 1"); c->fuse_ab = (int)v; }
    else if (k == "check_every") { if (v < 1) return fail(HF_E_ARG, "hf_set_tuning: check_every >= 1"); c->check_every = (int)v; }
    else if (k == "tm_fence") { if (v < 0 || v > 1) return fail(HF_E_ARG, "hf_set_tuning: tm_fence 0 or 1"); c->tm_fence = (int)v; }
    else if (k == "batch_group") { if (v < 0) return fail(HF_E_ARG, "hf_set_tuning: batch_group >= 0"); c->batch_group = (int)v; }
    else if (k == "comm_timeout_s") { if (v < 1) return fail(HF_E_ARG, "hf_set_tuning: comm_timeout_s >= 1"); c->comm_timeout_s = (double)v; }
    else return fail(HF_E_ARG, "hf_set_tuning: unknown key '" + k + "'");
    c->sys0.key_valid = false;                   // graphs are rebuilt with the new setting
    drop_stacks(c);
    return HF_OK;
}

hf_status hf_get_tuning(const hf_ctx *c, const char *key, int64_t *value)
{
    if (!c || !key || !value) return fail(HF_E_ARG, "hf_get_tuning: NULL argument");
    const std::string k(key);
    if (k == "tile_r") *value = c->tileR;
    else if (k == "zchunk") *value = c->zchunk;
    else if (k == "unroll") *value = c->unroll;
    else if (k == "pdl") *value = c->pdl;
    else if (k == "fuse_ab") *value = c->fuse_ab;
    else if (k == "check_every") *value = c->check_every;
    else if (k == "tm_fence") *value = c->tm_fence;
    else if (k == "batch_group") *value = c->batch_group;
    else if (k == "comm_timeout_s") *value = (int64_t)c->comm_timeout_s;
    else return fail(HF_E_ARG, "hf_get_tuning: unknown key '" + k + "'");
    return HF_OK;
}

hf_status hf_set_cg_variant(hf_ctx *c, int32_t variant)
{
    if (!c || variant < 0 || variant > 1) return fail(HF_E_ARG, "hf_set_cg_variant: variant must be 0 or 1");
    c->cg1 = variant;
    c->sys0.key_valid = false;
    return HF_OK;
}

hf_status hf_cg_variant(hf_ctx *c, int32_t out[2])
{
    if (!c || !out) return fail(HF_E_ARG, "hf_cg_variant: NULL argument");
    out[0] = c->cg1;
    out[1] = c->last_cg1;
    return HF_OK;
}

hf_status hf_set_resident(hf_ctx *c, int32_t mode)
{
    if (!c || mode < 0 || mode > 1) return fail(HF_E_ARG, "hf_set_resident: mode must be 0 or 1");
    c->resident = mode;
    c->sys0.key_valid = false;
    return HF_OK;
}

hf_status hf_resident_plan(hf_ctx *c, int32_t out[10])
{
    if (!c || !out) return fail(HF_E_ARG, "hf_resident_plan: NULL argument");
    CUCK(cudaSetDevice(c->device));
    const ResPlan p = res_plan(c);
    out[0] = p.ok; out[1] = p.px; out[2] = p.py; out[3] = p.pz; out[4] = p.bxm; out[5] = p.bym; out[6] = p.bzm;
    out[7] = p.BZ; out[8] = (int32_t)(p.smem / 1024); out[9] = c->last_resident;
    if (!p.ok) g_err = std::string("hf_resident_plan: not eligible: ") + p.why;
    return HF_OK;
}

hf_status hf_resident_profile(hf_ctx *c, int32_t enable, double out[24])
{
    if (!c) return fail(HF_E_ARG, "hf_resident_profile: NULL");
    CUCK(cudaSetDevice(c->device));
    const size_t n = (size_t)RES_PMAX * RES_PROF_N;
    if (out) {
        std::vector<unsigned long long> h(n, 0ull);
        if (c->res_prof) {
            CUCK(cudaStreamSynchronize(c->stream));
            CUCK(cudaMemcpy(h.data(), c->res_prof, n * 8, cudaMemcpyDeviceToHost));
        }
        // [k]: CTA 0's total of phase k (us); [12 + k]: the largest total over the CTAs
        for (int k = 0; k < 24; k++) out[k] = 0.0;
        for (int k = 0; k < RES_PROF_N && k < 12; k++) {
            const double f = k == RES_PROF_ITERS ? 1.0 : 1e-3;
            out[k] = h[k] * f;
            unsigned long long mx = 0;
            for (int b = 0; b < RES_PMAX; b++) mx = std::max(mx, h[(size_t)b * RES_PROF_N + k]);
            out[12 + k] = mx * f;
        }
    }
    if (enable && !c->res_prof) CUCK(cudaMalloc(&c->res_prof, n * 8));
    if (enable) CUCK(cudaMemset(c->res_prof, 0, n * 8));
    if (!enable && c->res_prof) { cudaFree(c->res_prof); c->res_prof = nullptr; }
    c->sys0.key_valid = false;
    return HF_OK;
}

hf_status hf_set_mixed(hf_ctx *c, int32_t enable, double rtol_lo)
{
    if (!c || (enable && !(rtol_lo > 0.0 && rtol_lo < 1.0))) return fail(HF_E_ARG, "hf_set_mixed: bad argument");
    CUCK(cudaSetDevice(c->device));
    CUCK(cudaStreamSynchronize(c->stream));
    c->sys0.key_valid = false;
    if (!enable) {
        drop_stacks(c);
        if (c->mix_exec) { cudaGraphExecDestroy(c->mix_exec); c->mix_exec = nullptr; }
        if (c->mix_graph) { cudaGraphDestroy(c->mix_graph); c->mix_graph = nullptr; }
        if (c->lo) { ctx_free(c->lo); delete c->lo; c->lo = nullptr; }
        return HF_OK;
    }
    if (c->prec != 64 || c->comm)
        return fail(HF_E_STATE, "hf_set_mixed: needs a single-GPU fp64 context");
    if (c->coef_set) return fail(HF_E_STATE, "hf_set_mixed: call before the coefficients are set");
    c->mix_rtol = rtol_lo;
    drop_stacks(c);                         // batched stacks are rebuilt with (or without) the shadow
    if (!c->lo) {
        hf_ctx *lo = new hf_ctx();
        hf_status st = ctx_init(lo, &c->g, c->device, c->stream, 0, 1, c->nsys);   // same system stack
        if (st == HF_OK) st = hf_set_precision(lo, 32);
        if (st == HF_OK && c->dbits) st = hf_set_dirichlet_faces(lo, c->dbits, c->gval);
        if (st == HF_OK && c->elem != EL_Q1) st = hf_set_element(lo, c->elem);
        if (st != HF_OK) { ctx_free(lo); delete lo; return st; }
        c->lo = lo;
    }
    if (!c->mix_iters) CUCK(cudaMalloc(&c->mix_iters, sizeof(unsigned long long)));
    CUCK(cudaMemset(c->mix_iters, 0, sizeof(unsigned long long)));
    return HF_OK;
}

hf_status hf_mixed_iters(hf_ctx *c, int64_t *lo_iters)
{
    if (!c || !lo_iters) return fail(HF_E_ARG, "hf_mixed_iters: NULL argument");
    *lo_iters = 0;
    if (!c->mix_iters) return HF_OK;
    CUCK(cudaSetDevice(c->device));
    CUCK(cudaStreamSynchronize(c->stream));
    unsigned long long v = 0;
    CUCK(cudaMemcpy(&v, c->mix_iters, sizeof(v), cudaMemcpyDeviceToHost));
    *lo_iters = (int64_t)v;
    return HF_OK;
}

hf_status hf_set_step_flush(hf_ctx *c, int32_t enable)
{
    if (!c) return fail(HF_E_ARG, "hf_set_step_flush: NULL");
    if (enable < 0 || enable > 2) return fail(HF_E_ARG, "hf_set_step_flush: enable must be 0, 1 or 2");
    c->step_flush = enable;
    return HF_OK;
}

hf_status hf_flush_l2(hf_ctx *c)
{
    if (!c) return fail(HF_E_ARG, "hf_flush_l2: NULL");
    const size_t bytes = 512ull << 20;   // 4x the 126 MB L2
    if (!c->flush) CUCK(cudaMalloc(&c->flush, bytes));
    CUCK(cudaMemsetAsync(c->flush, 1, bytes, c->stream));
    return HF_OK;
}

}  // extern "C"
