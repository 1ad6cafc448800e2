/*
 * heatfem.h -- C ABI of libheatfem.so, the B200 (sm_100a) hot path of arXiv 1905.07622,
 * "assembly-free FEM for transient heat flow through heterogeneous material".
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation / algorithm noted);
 * readings Rn = DESIGN.md section "Readings of the paper".
 *
 * Discretisation (§3.1, §3.2).  A structured voxel grid of ne[0] x ne[1] x ne[2]
 * trilinear hexahedra (reading R1; the paper's 6-tet split is not used) with spacing h and min
 * corner origin.  Each element e carries a conductivity k_e and a capacity c_e = (rho C)_e,
 * constant over the element.  The library never assembles a matrix; every operator
 * is applied element by element (Eq. (1)):
 *      y = sum_e A_e^T ( aK k_e K_ref + aM c_e M_ref ) A_e u
 * with (aK, aM) = (theta dt, 1) for A = M + theta dt K and (-(1-theta) dt, 1) for
 * L = M - (1-theta) dt K (reading R8), (1, 0) for K and (0, 1) for M.
 *
 * Layout.  Node (i,j,k) -> i + (ne0+1) * (j + (ne1+1) * k) (x fastest);
 * element (ex,ey,ez) -> ex + ne0 * (ey + ne1 * ez).  All vectors are fp64.
 *
 * Pointers.  Array arguments may be device pointers (on the context's device) or host
 * pointers (pageable or pinned); host arrays are staged through context-owned device
 * memory on the context stream.  Device arrays are borrowed for the duration of the call.
 *
 * Streams.  All device work is enqueued on the context stream (the one passed to
 * hf_create, or a library-owned stream if NULL).  hf_apply*, hf_diag and hf_face_load are
 * asynchronous when every array is on the device; calls that return host results
 * (hf_cg, hf_simulate*, hf_get_*) synchronise the context stream.
 *
 * Errors.  Every call returns an hf_status; on failure hf_last_error() returns a
 * thread-local message.  No C++ exception crosses this boundary.  Non-convergence is a
 * reported status, never a crash.
 */
#ifndef HEATFEM_H
#define HEATFEM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t hf_status;
#define HF_OK 0
#define HF_E_ARG (-1)        /* bad argument (NULL, size, value, dtype)                        */
#define HF_E_INDEX (-2)      /* index out of range                                              */
#define HF_E_NOCONV (-3)     /* PCG hit max_iter; x holds the last iterate, info is filled       */
#define HF_E_BREAKDOWN (-4)  /* d^T q <= 0 or non-finite (operator not SPD, or NaN input)         */
#define HF_E_PARTITION (-5)  /* slab decomposition impossible (fewer than 2 node planes per rank) */
#define HF_E_CUDA (-6)       /* CUDA runtime error (message has the CUDA error string)           */
#define HF_E_NCCL (-7)       /* NCCL unavailable or failed                                       */
#define HF_E_OOM (-8)        /* device allocation failed                                         */
#define HF_E_STATE (-9)      /* call out of order (e.g. hf_cg before hf_set_coefficients)        */

/* Grid: elements per axis, spacing (mm), min corner (mm).  (§4.1; Appendix C,
 * vert_scale P:408-409.) */
typedef struct {
    int64_t ne[3];
    double h[3];
    double origin[3];
} hf_grid;

/* PCG options (Alg. 1).  rtol: stop when ||r||_2 <= rtol ||b_F||_2 (reading R4);
 * max_iter: i_max (reading R10); replace_every: the "i divisible by 50" true-residual
 * replacement period of Alg. 1 line 9 (reading R6; 0 disables; negative: the context's
 * default, 50 for fp64 and 0 for the fp32 variant, whose true residual stagnates near
 * kappa eps_32 so that replacements below that level would prevent convergence, reading R18). */
typedef struct {
    double rtol;          /* default 1e-12 */
    int32_t max_iter;     /* default 10000 */
    int32_t replace_every;/* default -1: the context default (50 fp64, 0 fp32) */
} hf_cg_opts;

typedef struct {
    int32_t iters;        /* PCG iterations performed                                          */
    int32_t status;       /* HF_OK, HF_E_NOCONV or HF_E_BREAKDOWN                              */
    double relres;        /* ||r||_2 / ||b_F||_2 of the recurrence residual (0 if b_F = 0)     */
    double delta;         /* final delta = r^T P^{-1} r                                         */
} hf_cg_info;

typedef struct {
    int32_t steps_done;     /* time steps completed                                            */
    int32_t total_iters;    /* sum of PCG iterations over the steps                            */
    int32_t max_iters_step; /* largest PCG iteration count of one step                         */
    int32_t first_failed_step; /* -1 if every step converged                                  */
    double ms_total;        /* device time of the call (CUDA events on the context stream)     */
    double ms_steps;        /* sum of per-step device times (events around each step; excludes
                               the L2 flushes of hf_set_step_flush); = ms_total if not enabled */
} hf_sim_stats;

typedef struct hf_ctx hf_ctx;

/* Library version string (static storage). */
const char *hf_version(void);

/* Thread-local message of the last failing call on this thread ("" if none). */
const char *hf_last_error(void);

/* Create a context for grid g on CUDA device `device`.  cuda_stream: a cudaStream_t on that
 * device, or NULL for a library-owned stream.  *out receives the context.
 * Errors: HF_E_ARG (ne < 1, h <= 0, NULL out), HF_E_CUDA, HF_E_OOM. */
hf_status hf_create(const hf_grid *g, int device, void *cuda_stream, hf_ctx **out);

/* Destroy a context and free everything it owns (NULL is a no-op). */
void hf_destroy(hf_ctx *ctx);

/* Set the per-element coefficients (P:61, P:70 A_e = (rho C)_e M_e + theta dt k_e K_e).
 * k_elem, c_elem: n_elements fp64 each (element layout above), copied into context memory.
 * In slab mode the arrays cover the GLOBAL grid.  Errors: HF_E_ARG (NULL), HF_E_CUDA. */
hf_status hf_set_coefficients(hf_ctx *ctx, const double *k_elem, const double *c_elem);

/* Dirichlet faces (extension, reading R3).  face_bits bit f (f = 0..5 for -x,+x,-y,+y,-z,+z)
 * marks face f as Dirichlet with value values[f] (values may be NULL = all 0).  A node on
 * several flagged faces takes the value of the lowest-numbered one.  Affects hf_diag, hf_cg
 * and hf_simulate*; hf_apply is always the unconstrained operator. */
hf_status hf_set_dirichlet_faces(hf_ctx *ctx, uint32_t face_bits, const double values[6]);

/* Element variant (NEXT row f1).  type 0 (default): trilinear hexahedron per voxel (reading R1).
 * type 1: the paper's mesh -- every voxel split into 6 linear tetrahedra along its (0,0,0)-(1,1,1)
 * diagonal (Fig. 2), each tet carrying its voxel's (k_e, c_e) (reading R1b); boundary
 * quads become two P1 triangles for hf_face_load.  Affects every operator of the context.
 * Errors: HF_E_ARG. */
hf_status hf_set_element(hf_ctx *ctx, int32_t type);

/* Materials by id: element e has conductivity k_mat[ids[e]] and capacity c_mat[ids[e]] -- the
 * paper's material description (a few materials by region: steel / oxide; the corrosion
 * plate), i.e. a segmented voxel model.  The operator is exactly the one
 * hf_set_coefficients gives for k_e = k_mat[ids[e]], c_e = c_mat[ids[e]] (bit for bit); on fp64
 * Q1 contexts the stencil then streams one byte per element instead of a 16-byte (k, c) pair and
 * looks the element's coefficients up in a per-CTA shared-memory table (kernel variant EL_Q1P;
 * other element types and fp32 use the pair layout, filled from the table).
 * ids: n_elements uint8 (host or device, natural element order); n_materials in [1, 63];
 * k_mat, c_mat: n_materials fp64 (host).  hf_set_coefficients switches back to per-element pairs.
 * Synchronises.  Errors: HF_E_ARG (NULL, n_materials), HF_E_INDEX (an id >= n_materials). */
hf_status hf_set_material_ids(hf_ctx *ctx, const uint8_t *ids, int32_t n_materials, const double *k_mat,
                              const double *c_mat);

/* Materials given per node instead of per element (the paper's scheme: the material function is
 * "computed ... at each vertex and the values averaged over each element").
 * k_node, c_node: n_nodes fp64 of the GLOBAL grid (natural node order; slab contexts use their
 * planes).  Q1 elements: each voxel's (k_e, c_e) is the mean of its 8 corners.  Type-1 elements
 * (6 tets): each tet's (k_t, c_t) is the mean of its 4 vertices, evaluated inside the stencil from
 * per-node pairs (kernel variant EL_TETV).  Set the element type first; hf_set_coefficients
 * switches back to per-element values.  Not available with hf_simulate_batched (HF_E_STATE).
 * Errors: HF_E_ARG. */
hf_status hf_set_vertex_coefficients(hf_ctx *ctx, const double *k_node, const double *c_node);

/* Storage precision of the context's node vectors and (k, c) pairs: 64 (default) or 32, the
 * fp32 variant (NEXT row f3; the paper also ran single precision).  With 32 the
 * operator, the vector updates and the face load run in fp32 while every dot product, the PCG
 * scalars and the stop test stay fp64; the ABI's vectors stay fp64 (converted at the boundary).
 * Parity bar of the variant: rel-L2 <= 1e-5 against the fp64 oracle (north_star), reached with
 * rtol around 1e-6.  Must be called before hf_set_coefficients; reallocates the workspaces.
 * Errors: HF_E_ARG (bits not 32/64), HF_E_STATE (coefficients already set). */
hf_status hf_set_precision(hf_ctx *ctx, int32_t bits);

/* Flux load F_i = int_face f phi_i ds over face `face` (0..5) (P:44, P:50-52 boundary term):
 * f = f_const + beam, beam(a,b) = P/(2 pi s^2) exp(-((a-ca)^2 + (b-cb)^2) / (2 s^2)) with
 * beam = {P, s, ca, cb} (or NULL), (a, b) the face's in-plane coordinates in increasing axis
 * order (reading R12).  2x2 Gauss quadrature per boundary quad (type-1 elements: 3-point rule per
 * triangle).  F: n_nodes fp64, written
 * entirely (zero off the face).  Errors: HF_E_ARG (face, NULL F). */
hf_status hf_face_load(hf_ctx *ctx, int face, double f_const, const double beam[4], double *F);

/* y = (aK K + aM M) u, the element-by-element apply of Eq. (1) (Impl. 3 role,
 * P:210-245).  u, y: n_nodes fp64, must not alias.  Unconstrained (no Dirichlet rows). */
hf_status hf_apply(hf_ctx *ctx, double aK, double aM, const double *u, double *y);

/* y = c (aK K + aM M) u + b  (the paper's FGDbDMVM_C).  b may be NULL (= 0);
 * b may alias y. */
hf_status hf_apply_axpby(hf_ctx *ctx, double aK, double aM, double c, const double *u,
                         const double *b, double *y);

/* NEXT row f4 (ablation): the paper's earlier interpretations of the assembly operator, rebuilt
 * on sm_100a for the comparison of §5.1 (Fig. 5, Table 1).  Same result as
 * hf_apply_axpby (Eq. (1)), different data movement:
 *   impl 1 = "flexible DbD" (Eq. (3)): every scaled element matrix A_e stored in
 *            global memory in element order (512 B per element, fp64 8 x 8, written by
 *            hf_ablation_prepare); pass 1 one thread per element-DoF pair writes its row dot
 *            product in vertex order (8 contributions per node, ctx-owned, 64 B per node);
 *            pass 2 sums them per node and adds b.
 *   impl 2 = "single pass FG DbD" (Eq. (4)): one thread per output node gathers its
 *            27 inputs and 8 elements' (k, c) (3 x 3 strips staged in shared memory) and loops
 *            over the 8 element-DoF contributions; reference matrices in constant memory.
 *   impl 3 = the production stencil (= hf_apply_axpby).
 * u, b (may be NULL), y: n_nodes fp64 as hf_apply_axpby; u and y must not alias.
 * Asynchronous on the context stream.  fp64 contexts with one (k, c) per voxel, no slabs.
 * Errors: HF_E_ARG (impl, NULL, alias), HF_E_STATE (fp32 / slab / vertex-averaged tets; impl 1
 * without hf_ablation_prepare for the same (aK, aM), or coefficients changed since). */
hf_status hf_apply_impl(hf_ctx *ctx, int32_t impl, double aK, double aM, double c, const double *u,
                        const double *b, double *y);

/* Implementation 1's preprocessing: A_e = aK k_e K_ref + aM c_e M_ref for every
 * element, stored in ctx-owned device memory (n_elements x 64 fp64; plus n_nodes x 8 fp64 of
 * contribution space).  Asynchronous.  Errors: HF_E_STATE (as hf_apply_impl), HF_E_OOM. */
hf_status hf_ablation_prepare(hf_ctx *ctx, double aK, double aM);

/* Jacobi diagonal diag_i = sum_{e ni i} (aK k_e K_ref[l,l] + aM c_e M_ref[l,l]) (P:117,
 * Jacobi_A P:659-662); 1 on Dirichlet rows (reading R3).  diag: n_nodes fp64. */
hf_status hf_diag(hf_ctx *ctx, double aK, double aM, double *diag);

/* Solve (P_F A P_F + P_D) x = b by Jacobi PCG, Algorithm 1, A = aK K + aM M.
 * b must already carry the Dirichlet lift (b_D = g_D); x: in initial guess, out solution
 * (x_D is set to b_D).  opts NULL -> defaults.  info may be NULL.  Synchronises.
 * Returns HF_OK, HF_E_NOCONV (x = last iterate) or HF_E_BREAKDOWN. */
hf_status hf_cg(hf_ctx *ctx, double aK, double aM, const double *b, double *x,
                const hf_cg_opts *opts, hf_cg_info *info);

/* theta-scheme time loop: for n = 0..nsteps-1 solve
 *   [M + theta dt K] u^{n+1} = [M - (1-theta) dt K] u^n + dt F   (readings R7, R8)
 * with Dirichlet lift (R3) and guess x0 = u^0 at n = 0, else 2 u^n - u^{n-1} (u0_update,
 * P:575-589, reading R9).  u: in u^0 (Dirichlet nodes are overwritten with g), out u^nsteps.
 * F: n_nodes (the flux load, NOT pre-multiplied by dt) or NULL (= 0).
 * snap: NULL, or nsteps x n_plane fp64 receiving plane z = snap_plane (0 = front face) of
 * u^{n+1} after every step.  Synchronises once at the end.  Returns the first failing
 * step's status (HF_E_NOCONV / HF_E_BREAKDOWN) with stats->first_failed_step set, u then
 * holding that step's last iterate. */
hf_status hf_simulate(hf_ctx *ctx, double theta, double dt, int32_t nsteps, const double *F,
                      double *u, int64_t snap_plane, double *snap, const hf_cg_opts *opts,
                      hf_sim_stats *stats);

/* Checkpoint / resume of the time loop (the stepper state is (u^n, u^{n-1}, n)): same as
 * hf_simulate without snapshots, but the guess of the first step is 2 u - u_prev when
 * step0 > 0 (u_prev required then).  On return u = u^{n+nsteps} and, if u_prev is non-NULL,
 * u_prev = u^{n+nsteps-1}, ready for the next call. */
hf_status hf_simulate_resume(hf_ctx *ctx, double theta, double dt, int32_t nsteps, const double *F,
                             double *u, double *u_prev, int64_t step0, const hf_cg_opts *opts,
                             hf_sim_stats *stats);

/* B independent forward simulations on the context's grid (P:345-365 inverse problem; the
 * paper's "rapid successive solutions").  k_batch: B x n_elements; c_batch: B x n_elements
 * or NULL (= the context's c for every system); F: n_nodes shared load; u_batch: B x n_nodes
 * (in u^0, out u^nsteps); front_out: NULL or B x n_plane receiving plane snap_plane of
 * u^nsteps per system (a failed system: its last iterate); stats: B entries (may be NULL).
 * Systems are independent: each has its own PCG (Alg. 1) scalars, its own stop test
 * ||r_j|| <= rtol ||b_j||, iteration counts and failure status.  Groups of systems (below 16M
 * stacked nodes, at most 64 systems) run as one grid: the systems are stacked along z with a
 * coefficient-free element layer between them, each kernel block works inside one system and
 * a converged system stops while the others iterate on.  Dirichlet faces apply per system.
 * Systems are grouped into stacks by a model of the GPU's CTA slots.
 * With hf_set_mixed on, each step's solves run as fp32 correction + fp64 finish per stack.
 * B = 0 is a no-op (the arrays may then be NULL).
 * Returns the first failing status (the other systems run on and are returned). */
hf_status hf_simulate_batched(hf_ctx *ctx, int32_t B, const double *k_batch,
                              const double *c_batch, double theta, double dt, int32_t nsteps,
                              const double *F, double *u_batch, int64_t snap_plane,
                              double *front_out, const hf_cg_opts *opts, hf_sim_stats *stats);

/* ---- multi-GPU z-slabs (§4.4, generalised to R ranks) ---------- */

/* Owned node planes [z_lo, z_hi) of rank `rank` out of `nranks` for a grid with nz1 node
 * planes: contiguous, sizes differ by at most one.  Pure host function (no device).
 * Errors: HF_E_PARTITION if nz1 < 2 * nranks, HF_E_ARG otherwise-bad input. */
hf_status hf_slab_plan(int64_t nz1, int32_t rank, int32_t nranks, int64_t *z_lo, int64_t *z_hi);

/* 128-byte NCCL unique id for hf_create_slab (call on one rank, broadcast the bytes).
 * Loads libnccl.so.2 at run time.  Errors: HF_E_NCCL. */
hf_status hf_nccl_unique_id(uint8_t id[128]);

/* Slab context of rank `rank` of `nranks` for the GLOBAL grid g (z-slabs, the paper's split of
 * the domain between GPUs generalised to R ranks).  Vectors passed to a slab context
 * cover the rank's LOCAL planes: owned planes [z_lo, z_hi) plus one ghost plane on each interior
 * side (hf_slab_range).  Ghost entries of outputs are kept consistent by the library; dot products
 * run over owned nodes only.  Every rank must make the same sequence of hf_cg /
 * hf_simulate* calls.  transport:
 *   0 = NCCL (one process per GPU; id = 128 bytes from hf_nccl_unique_id).  Ghost planes and the
 *       sums of each reduction go through ncclSend/Recv and ncclAllReduce between the kernels,
 *       driven by the host loop (the baseline transport).
 *   1 = peer memory, every rank in THIS process (one host thread per rank, any devices; id = the
 *       hf_local_group of the ranks cast to uint8_t*).  The call blocks until every rank joined.
 *   2 = peer memory, one process per rank (id ignored, may be NULL): each rank then calls
 *       hf_peer_export, all-gathers the blobs (e.g. torch.distributed) and calls hf_peer_connect.
 * With peer memory (1, 2) the kernels exchange everything themselves (heatfem kernels store the
 * boundary planes of P^{-1} r into the neighbours' ghost buffers and publish their reduction sums
 * into every rank's mailbox over NVLink; a consumer kernel waits for every rank's flag): the
 * whole slab solve runs in the device-side step graph with no host step and no NCCL call.  A
 * rank that stops making progress makes the others fail (device trap after 30 s) instead of
 * hanging.  At most 8 ranks (one node).  Errors: HF_E_ARG, HF_E_PARTITION, HF_E_NCCL, HF_E_CUDA. */
hf_status hf_create_slab(const hf_grid *g, int32_t rank, int32_t nranks, const uint8_t *id,
                         int32_t transport, int device, void *cuda_stream, hf_ctx **out);

/* In-process transport group for `nranks` ranks (transport 1 of hf_create_slab). */
typedef struct hf_local_group hf_local_group;
hf_status hf_local_group_create(int32_t nranks, hf_local_group **out);
void hf_local_group_destroy(hf_local_group *grp);

/* Transport 2: this rank's connection blob (its mailbox as a CUDA IPC handle, its GPU's PCI bus
 * id, its rank).  blob: HF_PEER_BLOB_BYTES bytes, written.  Errors: HF_E_ARG (not a transport-2
 * context), HF_E_CUDA. */
#define HF_PEER_BLOB_BYTES 256
hf_status hf_peer_export(hf_ctx *ctx, uint8_t blob[HF_PEER_BLOB_BYTES]);

/* Transport 2: connect to every rank.  blobs: nranks x HF_PEER_BLOB_BYTES, rank order (the
 * all-gathered hf_peer_export blobs, this rank's included).  Maps the peers' mailboxes (IPC).
 * hf_cg / hf_simulate* on a transport-2 context fail with HF_E_STATE before this call.
 * Errors: HF_E_ARG (blob of another group), HF_E_STATE (connected already), HF_E_CUDA. */
hf_status hf_peer_connect(hf_ctx *ctx, const uint8_t *blobs);

/* Global node planes [z_lo, z_hi) owned by this context, and the local plane count
 * (owned + ghosts) and the global index of local plane 0. */
hf_status hf_slab_range(const hf_ctx *ctx, int64_t *z_lo, int64_t *z_hi, int64_t *local_planes,
                        int64_t *local_z0);

/* ---- introspection used by tests and bench.py ----------------------------------------- */

/* Number of this library's kernels launched on the context so far (device counter). */
hf_status hf_get_launch_count(hf_ctx *ctx, int64_t *count);

/* Per-kernel-class timing (CUDA events around each launch; slows the loop slightly).
 * enable = 1 turns it on and clears totals.  Classes: 0 apply/stencil CG kernel A,
 * 1 pointwise kernel B, 2 residual kernel, 3 rhs, 4 other.  ms[c] total ms, n[c] launches. */
hf_status hf_profile(hf_ctx *ctx, int32_t enable);
hf_status hf_profile_read(hf_ctx *ctx, double ms[5], int64_t n[5]);

/* Instrumentation: average duration of PCG kernel A (the dominant kernel, Alg. 1 lines 6-7)
 * replayed `reps` times back to back on the context stream, bracketed by one pair of CUDA
 * events (no per-launch event overhead).  Uses the operator (theta dt, 1) of the last
 * hf_simulate* call and the primary system's current vectors; the replay runs the init kernel
 * first so that every replayed launch computes PCG iteration 0 (d = s, q = A d, d.q), which costs
 * the same as any other iteration.  Leaves the primary system's PCG state undefined (the next
 * hf_cg / hf_simulate* call resets it).  Errors: HF_E_STATE (no previous simulation). */
hf_status hf_time_kernel_a(hf_ctx *ctx, int32_t reps, double *ms_per_launch);

/* The same kernel A launch replayed as a CUDA graph of `reps` nodes joined by the PCG loop
 * body's programmatic edges (each launch's prologue overlaps the previous one's tail, as behind
 * kernel B in the loop); ms per launch from one timed graph launch after a warm-up launch.
 * Errors: HF_E_ARG, HF_E_STATE (no previous simulation), HF_E_CUDA. */
hf_status hf_time_kernel_a_graph(hf_ctx *ctx, int32_t reps, double *ms_per_launch);

/* Loop driver: 0 = CUDA graph with device-side WHILE loop (default), 1 = host loop.
 * Profiling (hf_profile) and the NCCL slab transport always use the host loop. */
hf_status hf_set_driver(hf_ctx *ctx, int32_t driver);

/* Mixed precision (NEXT row f3 at the fp64 bar): enable = 1 gives this fp64 context an fp32
 * shadow (same grid, coefficients, Dirichlet faces, element; every later setter is forwarded).
 * hf_simulate* then solves each time step in two stages on the device: the fp32 PCG (fp32
 * storage, fp64 reductions) from the extrapolated guess to rtol_lo (or the call's rtol if larger),
 * and the fp64 PCG from the fp32 iterate to the call's rtol.  The fp64 residual of the fp64
 * operator decides convergence (defect correction), so results have the fp64 path's accuracy
 * (reading R18); the fp32 stage carries most of the error reduction at half the bytes.  Call
 * before the coefficients; enable = 0 removes the shadow.  Graph driver only (the host-loop
 * driver runs plain fp64).  hf_simulate_batched on a mixed context runs every stack the same
 * way (each stack gets its own fp32 shadow with per-system fp32 PCG; a system that failed in an
 * earlier step gets no correction).  Errors: HF_E_ARG, HF_E_STATE (fp32 / slab context, or
 * coefficients already set), HF_E_CUDA. */
hf_status hf_set_mixed(hf_ctx *ctx, int32_t enable, double rtol_lo);

/* PCG iterations of the fp32 stage since hf_set_mixed (device counter; synchronises). */
hf_status hf_mixed_iters(hf_ctx *ctx, int64_t *lo_iters);

/* Tuning knobs of a context (performance only: every setting computes the same operator and
 * PCG; results agree to rounding order).  Keys and values:
 *   "tile_r"         0 = default (R = 2 below 16M local nodes, else 4; tets always 2), 2 or 4:
 *                    node rows per thread of the stencil tiles (a CTA owns 31 x (8 R - 1) nodes)
 *   "zchunk"         0 = sized to fill the SMs, else z planes per stencil CTA
 *   "unroll"         0 = by grid size, else 1..50 PCG iterations per WHILE-body launch
 *   "pdl"            1 (default) / 0: programmatic-launch edges between the loop kernels
 *   "fuse_ab"        0 (default) / 1: kernels A and B of an iteration in one launch (grid barrier)
 *   "check_every"    host-loop driver: iterations per asynchronous state check (default 8)
 *   "tm_fence"       0 (default) / 1: acquire the TMA descriptors in every launch
 *   "batch_group"    0 = modelled, else systems per stack of hf_simulate_batched
 *   "comm_timeout_s" host-loop slab transports: fail (HF_E_NCCL) after this many seconds
 *                    without progress (default 120)
 * Changing a knob rebuilds the context's cached graphs at the next call.  The environment
 * variables HF_TILE_R, HF_ZCHUNK, HF_UNROLL, HF_PDL, HF_FUSE_AB, HF_CHECK_EVERY, HF_TM_FENCE,
 * HF_BATCH_GROUP, HF_COMM_TIMEOUT_S (and HF_DRIVER, HF_RESIDENT: hf_set_driver,
 * hf_set_resident) give the defaults of a context when it is created; nothing reads them later.
 * Errors: HF_E_ARG (NULL, unknown key, value out of range), HF_E_CUDA. */
hf_status hf_set_tuning(hf_ctx *ctx, const char *key, int64_t value);

/* The current value of a tuning knob ("tile_r" reports the tile height in use).
 * Errors: HF_E_ARG. */
hf_status hf_get_tuning(const hf_ctx *ctx, const char *key, int64_t *value);

/* PCG arrangement of hf_simulate* (hf_set_cg_variant).  variant 0 (default): Alg. 1 as printed
 * (P:93-113), two streaming kernels per iteration (A: d = s + beta d, q = A d, d^T q; B: x, r, s
 * updates, r^T s, r^T r).  variant 1: the single-reduction (Chronopoulos-Gear) arrangement of the
 * same Jacobi PCG -- w = A u and s = A p are carried by recurrence, so alpha_i and beta_i follow
 * from one set of sums (r^T u, w^T u) and each iteration is ONE stencil kernel that also performs
 * the vector updates; identical iterates in exact arithmetic, the same residual replacement every
 * 50 iterations (Alg. 1 line 10: r = b - A x, then w = A P^-1 r) and the same stop test (R4).
 * Used when eligible: fp64 Q1 elements ((k, c) pairs or material ids), one system, no slab
 * transport, not mixed / on-chip; otherwise variant 0 runs.  DESIGN.md section 7b.
 * Errors: HF_E_ARG. */
hf_status hf_set_cg_variant(hf_ctx *ctx, int32_t variant);

/* out[0] = the variant set by hf_set_cg_variant, out[1] = 1 if the last hf_simulate* ran the
 * single-reduction PCG.  Errors: HF_E_ARG. */
hf_status hf_cg_variant(hf_ctx *ctx, int32_t out[2]);

/* On-chip PCG (opt-in, hf_set_resident): hf_simulate* runs each time step's whole PCG solve
 * (Alg. 1) in ONE cooperative launch whose CTAs (one per SM) keep d (+ a one-node
 * halo), r, q/s and the material ids of their brick of the grid in shared memory (x in the
 * L2-resident output vector); the Alg. 1 reductions ride on two grid barriers per iteration.  Same operator,
 * readings (R3-R6) and stop test as the streaming kernels; results agree to rounding order.
 * Eligible: fp64 Q1 with materials by id (hf_set_material_ids), one system, no slab transport,
 * graph driver, and a grid whose brick partition fits (<= 31 x 25 x 16 nodes per brick, one brick
 * per SM: about 1.1M nodes on 148 SMs).  mode 0 = never (streaming kernels, the default), 1 = when
 * eligible.  Measured slower than the streaming kernels at C3.
 * Errors: HF_E_ARG. */
hf_status hf_set_resident(hf_ctx *ctx, int32_t mode);

/* The on-chip PCG's plan for the current context: out[0] eligible, out[1..3] bricks per axis,
 * out[4..6] largest brick (nodes), out[7] plane capacity BZ, out[8] shared memory KB per CTA,
 * out[9] 1 if the last hf_simulate* used it.  When not eligible hf_last_error() says why.
 * Errors: HF_E_ARG, HF_E_CUDA. */
hf_status hf_resident_plan(hf_ctx *ctx, int32_t out[10]);

/* Instrumentation of the on-chip PCG: enable = 1 (re)starts per-phase timers of CTA 0 (the next
 * hf_simulate* rebuilds its graph with them), 0 stops them.  out (may be NULL) receives the totals
 * since the last start of CTA 0 in out[0..11] and the largest over the CTAs in out[12..23]: us in
 * [0] d update, [1] stencil (kernel A), [2] grid reduction of d^T q, [3] kernel B, [4] grid
 * reduction of r^T s, r^T r (and residual replacements), [5] init, [6] PCG iterations, and inside
 * the reductions [7] fence + arrival, [8] waiting for the other CTAs, [9] reading the partials.
 * Errors: HF_E_ARG, HF_E_CUDA. */
hf_status hf_resident_profile(hf_ctx *ctx, int32_t enable, double out[24]);

/* Enqueue a 512 MiB memset on the context stream (evicts the 126 MB L2; bench timing rule). */
hf_status hf_flush_l2(hf_ctx *ctx);

/* Benchmark mode of hf_simulate*: enable = 1 flushes L2 (as hf_flush_l2) before every time
 * step and times every step alone with CUDA events (hf_sim_stats.ms_steps), all enqueued
 * asynchronously; enable = 2 times every step without the flush; enable = 0 restores normal
 * operation.  Errors: HF_E_ARG. */
hf_status hf_set_step_flush(hf_ctx *ctx, int32_t enable);

#ifdef __cplusplus
}
#endif
#endif /* HEATFEM_H */
