/*
 * heat_oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 1905.07622 (assembly-free FEM for transient heat flow).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The CUDA product path
 * (paper_1905_07622_b200/, include/heatfem.h) shares no code, header, table or
 * constant generator with this file, and neither side includes or links the other.
 *
 * What it computes, each step cited to PAPER.md (P:line) and the DESIGN.md readings:
 *   - Q1 (trilinear hexahedron) reference matrices K_e, M_e by 2x2x2 Gauss-Legendre
 *     quadrature of the shape functions  (P:53 matrices M, K; P:59-61 elemental M_e,
 *     "material property coefficients ... constant over each element"; reading R1).
 *   - Explicit assembly of the global sparse K = A_e k_e K_e and M = A_e c_e M_e by
 *     scatter-add over elements into CSR  (assembly operator).
 *   - y = (aK K + aM M) u by CSR SpMV; the same by an element-by-element loop
 *     (Eq. (1)) and by per-node row sums for sampled rows.
 *   - Flux load F_i = int_face f phi_i ds, 2x2 Gauss per boundary quad.
 *   - Dirichlet faces (extension, reading R3) by symmetric elimination.
 *   - PCG exactly in the order of Algorithm 1 with readings R4-R6, R10.
 *   - theta-scheme time loop  [M + theta dt K] U^i = [M - (1-theta) dt K] U^{i-1} + dt F
 *      with the extrapolated guess of u0_update (reading R9).
 * All arithmetic is fp64.  Parallel with OpenMP (static schedules) in a way that leaves every
 * result independent of the thread count: a row sum (SpMV, diagonal) is one thread's sequential
 * left-to-right sum; a dot product is a sum of fixed 4096-node chunks (each chunk summed left to
 * right, the chunk sums added left to right in chunk order: reading R15); pointwise
 * vector updates are per-node.  Element scatter-add assembly stays sequential.
 * or_num_threads() reports the OpenMP thread count (OMP_NUM_THREADS, default all host cores).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_E_ARG (-1)
#define OR_E_NOCONV (-3)
#define OR_E_BREAKDOWN (-4)
#define OR_E_OOM (-8)

#define OR_CHUNK 4096      /* nodes per partial sum of a dot product (fixed: thread-count independent) */

int or_num_threads(void) { return omp_get_max_threads(); }

typedef struct {
    int64_t ne[3];         /* elements per axis */
    int64_t nn[3];         /* nodes per axis = ne + 1 */
    double h[3];
    double origin[3];
    int64_t nnodes, nelems;
    int elem;              /* 0: trilinear hexahedron (R1), 1: 6 P1 tets per voxel (f1),          */
                           /* 2: 6 P1 tets, each with its own coefficient (vertex averages) */
    double Ke[64], Me[64]; /* voxel element matrices (unit k, unit c) */
    double *k, *c;         /* per-element coefficients (copies) */
    double *kt, *ct;       /* elem 2: per-tet coefficients, 6 per voxel */
    double Kt[6][16], Mt[6][16];   /* elem 2: unit-coefficient tet matrices, local order of tloc */
    int tloc[6][4];        /* elem 2: voxel-local nodes of each tet */
    /* CSR of K and M (same pattern) */
    int has_csr;
    int64_t *rowptr;
    int64_t *col;
    double *Kv, *Mv;
    int64_t nnz;
    /* Dirichlet (reading R3) */
    unsigned bits;
    double gval[6];
    unsigned char *isD;    /* 1 on Dirichlet nodes */
    double *g;             /* Dirichlet value per node (0 on free nodes) */
} or_ctx;

/* ------------------------------------------------------------------------------------------ */
/* Reference element matrices by quadrature.                                   */
/* Local node l = bx + 2 by + 4 bz sits at (bx hx, by hy, bz hz).                               */
/* N_l(x) = prod_d phi_{b_d}(x_d), phi_0(t) = 1 - t/h, phi_1(t) = t/h.                          */

static double phi1d(int b, double t, double h) { return b ? t / h : 1.0 - t / h; }
static double dphi1d(int b, double h) { return b ? 1.0 / h : -1.0 / h; }

void or_element_matrices(const double h[3], double Ke[64], double Me[64])
{
    const double gp[2] = {0.5 * (1.0 - 1.0 / sqrt(3.0)), 0.5 * (1.0 + 1.0 / sqrt(3.0))};
    for (int i = 0; i < 64; i++) { Ke[i] = 0.0; Me[i] = 0.0; }
    for (int qz = 0; qz < 2; qz++)
    for (int qy = 0; qy < 2; qy++)
    for (int qx = 0; qx < 2; qx++) {
        double x[3] = {gp[qx] * h[0], gp[qy] * h[1], gp[qz] * h[2]};
        double w = (h[0] / 2.0) * (h[1] / 2.0) * (h[2] / 2.0);  /* weights 1 on [-1,1] -> h/2 */
        double N[8], G[8][3];
        for (int l = 0; l < 8; l++) {
            int b[3] = {l & 1, (l >> 1) & 1, (l >> 2) & 1};
            double p[3], dp[3];
            for (int d = 0; d < 3; d++) { p[d] = phi1d(b[d], x[d], h[d]); dp[d] = dphi1d(b[d], h[d]); }
            N[l] = p[0] * p[1] * p[2];
            G[l][0] = dp[0] * p[1] * p[2];
            G[l][1] = p[0] * dp[1] * p[2];
            G[l][2] = p[0] * p[1] * dp[2];
        }
        for (int a = 0; a < 8; a++)
            for (int b = 0; b < 8; b++) {
                Me[a * 8 + b] += w * N[a] * N[b];
                Ke[a * 8 + b] += w * (G[a][0] * G[b][0] + G[a][1] * G[b][1] + G[a][2] * G[b][2]);
            }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Paper's element (NEXT row f1): each voxel split into 6 linear tetrahedra (Fig. 2)  */
/* along the diagonal from local node 0 (0,0,0) to local node 7 (1,1,1): tet number t follows    */
/* the lattice path 0 -> e_a -> e_a + e_b -> 7 for the t-th permutation (a, b, c) of the axes.    */
/* P1 matrices from vertex coordinates: J = [p1-p0, p2-p0, p3-p0], V = |det J| / 6,              */
/* grad(lambda_i) = row i of J^{-1} (i = 1..3), grad(lambda_0) = -sum; K_ij = V g_i . g_j,        */
/* M_ij = V (1 + delta_ij) / 20.  Each tet carries its voxel's (k_e, c_e) (reading R1b), so the   */
/* voxel's element matrices are the assembly of its 6 tets into the 8 voxel nodes.        */

static const int tet_perm[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};

void or_tet_vertices(int t, int local[4])
{
    int b[3] = {0, 0, 0};
    local[0] = 0;
    for (int s = 0; s < 3; s++) {
        b[tet_perm[t][s]] = 1;
        local[s + 1] = b[0] + 2 * b[1] + 4 * b[2];
    }
}

void or_tet_matrices(const double p[4][3], double K[16], double M[16])
{
    double J[3][3];
    for (int r = 0; r < 3; r++)
        for (int c = 0; c < 3; c++) J[r][c] = p[c + 1][r] - p[0][r];   /* columns p_i - p_0 */
    double det = J[0][0] * (J[1][1] * J[2][2] - J[1][2] * J[2][1])
               - J[0][1] * (J[1][0] * J[2][2] - J[1][2] * J[2][0])
               + J[0][2] * (J[1][0] * J[2][1] - J[1][1] * J[2][0]);
    double inv[3][3];   /* inverse by cofactors */
    inv[0][0] = (J[1][1] * J[2][2] - J[1][2] * J[2][1]) / det;
    inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
    inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
    inv[1][0] = (J[1][2] * J[2][0] - J[1][0] * J[2][2]) / det;
    inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
    inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
    inv[2][0] = (J[1][0] * J[2][1] - J[1][1] * J[2][0]) / det;
    inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
    inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    double g[4][3];
    for (int d = 0; d < 3; d++) {
        g[1][d] = inv[0][d];
        g[2][d] = inv[1][d];
        g[3][d] = inv[2][d];
        g[0][d] = -(g[1][d] + g[2][d] + g[3][d]);
    }
    double V = fabs(det) / 6.0;
    for (int i = 0; i < 4; i++)
        for (int j = 0; j < 4; j++) {
            K[i * 4 + j] = V * (g[i][0] * g[j][0] + g[i][1] * g[j][1] + g[i][2] * g[j][2]);
            M[i * 4 + j] = V * (i == j ? 2.0 : 1.0) / 20.0;
        }
}

/* voxel matrices of the 6-tet split (sum of the tets' matrices over the voxel's 8 nodes) */
void or_tet_voxel_matrices(const double h[3], double Ke[64], double Me[64])
{
    for (int i = 0; i < 64; i++) { Ke[i] = 0.0; Me[i] = 0.0; }
    for (int t = 0; t < 6; t++) {
        int loc[4];
        or_tet_vertices(t, loc);
        double p[4][3], K[16], M[16];
        for (int v = 0; v < 4; v++)
            for (int d = 0; d < 3; d++) p[v][d] = ((loc[v] >> d) & 1) * h[d];
        or_tet_matrices(p, K, M);
        for (int a = 0; a < 4; a++)
            for (int b = 0; b < 4; b++) {
                Ke[loc[a] * 8 + loc[b]] += K[a * 4 + b];
                Me[loc[a] * 8 + loc[b]] += M[a * 4 + b];
            }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Index conventions: node (i,j,k) -> i + nnx (j + nny k), x fastest.        */

static int64_t node_id(const or_ctx *o, int64_t i, int64_t j, int64_t k)
{
    return i + o->nn[0] * (j + o->nn[1] * k);
}

static void elem_nodes(const or_ctx *o, int64_t e, int64_t nodes[8])
{
    int64_t ex = e % o->ne[0];
    int64_t ey = (e / o->ne[0]) % o->ne[1];
    int64_t ez = e / (o->ne[0] * o->ne[1]);
    for (int l = 0; l < 8; l++)
        nodes[l] = node_id(o, ex + (l & 1), ey + ((l >> 1) & 1), ez + ((l >> 2) & 1));
}

/* Coefficient-scaled matrices of voxel e in its 8 local nodes: k_e K_e, c_e M_e (elem 0, 1), or */
/* the sum over its 6 tets of k_t K_t, c_t M_t with per-tet coefficients (elem 2).              */
static void elem_scaled(const or_ctx *o, int64_t e, double Kel[64], double Mel[64])
{
    if (o->elem != 2) {
        for (int i = 0; i < 64; i++) { Kel[i] = o->k[e] * o->Ke[i]; Mel[i] = o->c[e] * o->Me[i]; }
        return;
    }
    for (int i = 0; i < 64; i++) { Kel[i] = 0.0; Mel[i] = 0.0; }
    for (int t = 0; t < 6; t++) {
        double kt = o->kt[6 * e + t], ct = o->ct[6 * e + t];
        for (int a = 0; a < 4; a++)
            for (int b = 0; b < 4; b++) {
                Kel[o->tloc[t][a] * 8 + o->tloc[t][b]] += kt * o->Kt[t][a * 4 + b];
                Mel[o->tloc[t][a] * 8 + o->tloc[t][b]] += ct * o->Mt[t][a * 4 + b];
            }
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Assembly: scatter-add every element matrix into 27 structured slots per row,      */
/* then compact to CSR (rows sorted, columns ascending).                                        */

static int assemble_csr(or_ctx *o)
{
    const int64_t N = o->nnodes;
    double *Ks = calloc((size_t)N * 27, sizeof(double));
    double *Ms = calloc((size_t)N * 27, sizeof(double));
    unsigned char *used = calloc((size_t)N * 27, 1);
    if (!Ks || !Ms || !used) { free(Ks); free(Ms); free(used); return OR_E_OOM; }
    for (int64_t e = 0; e < o->nelems; e++) {
        int64_t nodes[8];
        double Kel[64], Mel[64];
        elem_nodes(o, e, nodes);
        elem_scaled(o, e, Kel, Mel);
        for (int a = 0; a < 8; a++)
            for (int b = 0; b < 8; b++) {
                /* slot = offset of node b relative to node a, (dx,dy,dz) in {-1,0,1}^3 */
                int dx = (b & 1) - (a & 1), dy = ((b >> 1) & 1) - ((a >> 1) & 1), dz = ((b >> 2) & 1) - ((a >> 2) & 1);
                int slot = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
                size_t at = (size_t)nodes[a] * 27 + slot;
                Ks[at] += Kel[a * 8 + b];
                Ms[at] += Mel[a * 8 + b];
                used[at] = 1;
            }
    }
    int64_t nnz = 0;
    for (size_t t = 0; t < (size_t)N * 27; t++) nnz += used[t];
    o->rowptr = malloc(sizeof(int64_t) * (size_t)(N + 1));
    o->col = malloc(sizeof(int64_t) * (size_t)nnz);
    o->Kv = malloc(sizeof(double) * (size_t)nnz);
    o->Mv = malloc(sizeof(double) * (size_t)nnz);
    if (!o->rowptr || !o->col || !o->Kv || !o->Mv) { free(Ks); free(Ms); free(used); return OR_E_OOM; }
    int64_t p = 0;
    for (int64_t r = 0; r < N; r++) {
        o->rowptr[r] = p;
        int64_t i = r % o->nn[0], j = (r / o->nn[0]) % o->nn[1], k = r / (o->nn[0] * o->nn[1]);
        /* slots in ascending column order: dz outer, dy, dx inner */
        for (int slot = 0; slot < 27; slot++) {
            size_t at = (size_t)r * 27 + slot;
            if (!used[at]) continue;
            int dx = slot % 3 - 1, dy = (slot / 3) % 3 - 1, dz = slot / 9 - 1;
            o->col[p] = node_id(o, i + dx, j + dy, k + dz);
            o->Kv[p] = Ks[at];
            o->Mv[p] = Ms[at];
            p++;
        }
    }
    o->rowptr[N] = p;
    o->nnz = nnz;
    o->has_csr = 1;
    free(Ks); free(Ms); free(used);
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */

or_ctx *or_create(const int64_t ne[3], const double h[3], const double origin[3],
                  const double *k, const double *c, int assemble, int elem)
{
    or_ctx *o = calloc(1, sizeof(or_ctx));
    if (!o) return NULL;
    for (int d = 0; d < 3; d++) {
        o->ne[d] = ne[d]; o->nn[d] = ne[d] + 1; o->h[d] = h[d]; o->origin[d] = origin[d];
    }
    o->nnodes = o->nn[0] * o->nn[1] * o->nn[2];
    o->nelems = ne[0] * ne[1] * ne[2];
    o->elem = elem;
    if (elem == 1) or_tet_voxel_matrices(o->h, o->Ke, o->Me);
    else or_element_matrices(o->h, o->Ke, o->Me);
    o->k = malloc(sizeof(double) * (size_t)o->nelems);
    o->c = malloc(sizeof(double) * (size_t)o->nelems);
    o->isD = calloc((size_t)o->nnodes, 1);
    o->g = calloc((size_t)o->nnodes, sizeof(double));
    if (!o->k || !o->c || !o->isD || !o->g) return NULL;
    memcpy(o->k, k, sizeof(double) * (size_t)o->nelems);
    memcpy(o->c, c, sizeof(double) * (size_t)o->nelems);
    if (assemble && assemble_csr(o) != OR_OK) return NULL;
    return o;
}

/* Materials given per node (vertex values, "computed ... at each vertex and the values      */
/* averaged over each element", "averaged over the element"): elem 0 -> each voxel's        */
/* coefficient is the mean of its 8 corners; elem 1 -> each tet's coefficient is the mean of its 4 */
/* vertices (the oracle then runs in elem mode 2).                                                */
or_ctx *or_create_vertex(const int64_t ne[3], const double h[3], const double origin[3],
                         const double *kn, const double *cn, int assemble, int elem)
{
    const int64_t nx1 = ne[0] + 1, ny1 = ne[1] + 1, nel = ne[0] * ne[1] * ne[2];
    double *ke = malloc(sizeof(double) * (size_t)nel), *ce = malloc(sizeof(double) * (size_t)nel);
    if (!ke || !ce) { free(ke); free(ce); return NULL; }
    for (int64_t e = 0; e < nel; e++) {      /* per-voxel corner means (elem 0; placeholders for 1) */
        int64_t ex = e % ne[0], ey = (e / ne[0]) % ne[1], ez = e / (ne[0] * ne[1]);
        double sk = 0.0, sc = 0.0;
        for (int l = 0; l < 8; l++) {
            int64_t n = (ex + (l & 1)) + nx1 * ((ey + ((l >> 1) & 1)) + ny1 * (ez + ((l >> 2) & 1)));
            sk += kn[n];
            sc += cn[n];
        }
        ke[e] = sk / 8.0;
        ce[e] = sc / 8.0;
    }
    or_ctx *o = or_create(ne, h, origin, ke, ce, elem == 1 ? 0 : assemble, elem);
    free(ke);
    free(ce);
    if (!o || elem != 1) return o;
    o->elem = 2;
    o->kt = malloc(sizeof(double) * (size_t)nel * 6);
    o->ct = malloc(sizeof(double) * (size_t)nel * 6);
    if (!o->kt || !o->ct) return NULL;
    for (int t = 0; t < 6; t++) {
        or_tet_vertices(t, o->tloc[t]);
        double p[4][3];
        for (int v = 0; v < 4; v++)
            for (int d = 0; d < 3; d++) p[v][d] = ((o->tloc[t][v] >> d) & 1) * h[d];
        or_tet_matrices(p, o->Kt[t], o->Mt[t]);
    }
    for (int64_t e = 0; e < nel; e++) {
        int64_t nodes[8];
        elem_nodes(o, e, nodes);
        for (int t = 0; t < 6; t++) {
            double sk = 0.0, sc = 0.0;
            for (int v = 0; v < 4; v++) {
                sk += kn[nodes[o->tloc[t][v]]];
                sc += cn[nodes[o->tloc[t][v]]];
            }
            o->kt[6 * e + t] = sk / 4.0;
            o->ct[6 * e + t] = sc / 4.0;
        }
    }
    if (assemble && assemble_csr(o) != OR_OK) return NULL;
    return o;
}

void or_destroy(or_ctx *o)
{
    if (!o) return;
    free(o->k); free(o->c); free(o->kt); free(o->ct); free(o->rowptr); free(o->col); free(o->Kv); free(o->Mv);
    free(o->isD); free(o->g); free(o);
}

void or_get_element_matrices(const or_ctx *o, double Ke[64], double Me[64])
{
    memcpy(Ke, o->Ke, sizeof(o->Ke));
    memcpy(Me, o->Me, sizeof(o->Me));
}

int64_t or_nnz(const or_ctx *o) { return o->has_csr ? o->nnz : -1; }

int or_csr_copy(const or_ctx *o, int64_t *rowptr, int64_t *col, double *Kv, double *Mv)
{
    if (!o->has_csr) return OR_E_ARG;
    memcpy(rowptr, o->rowptr, sizeof(int64_t) * (size_t)(o->nnodes + 1));
    memcpy(col, o->col, sizeof(int64_t) * (size_t)o->nnz);
    memcpy(Kv, o->Kv, sizeof(double) * (size_t)o->nnz);
    memcpy(Mv, o->Mv, sizeof(double) * (size_t)o->nnz);
    return OR_OK;
}

/* y = (aK K + aM M) u, assembled CSR (the "explicit" reading of y = A x). */
int or_spmv(const or_ctx *o, double aK, double aM, const double *u, double *y)
{
    if (!o->has_csr) return OR_E_ARG;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < o->nnodes; r++) {
        double s = 0.0;
        for (int64_t p = o->rowptr[r]; p < o->rowptr[r + 1]; p++)
            s += (aK * o->Kv[p] + aM * o->Mv[p]) * u[o->col[p]];
        y[r] = s;
    }
    return OR_OK;
}

/* y = A_e (aK k_e K_e + aM c_e M_e) u_e, element by element (Eq. (1) left side). */
void or_apply_ebe(const or_ctx *o, double aK, double aM, const double *u, double *y)
{
    for (int64_t n = 0; n < o->nnodes; n++) y[n] = 0.0;
    for (int64_t e = 0; e < o->nelems; e++) {
        int64_t nodes[8];
        double Kel[64], Mel[64];
        elem_nodes(o, e, nodes);
        elem_scaled(o, e, Kel, Mel);
        for (int a = 0; a < 8; a++) {
            double s = 0.0;
            for (int b = 0; b < 8; b++)
                s += (aK * Kel[a * 8 + b] + aM * Mel[a * 8 + b]) * u[nodes[b]];
            y[nodes[a]] += s;
        }
    }
}

/* Sampled rows: y_i = sum_{e containing i} (A_e u_e)_{l(i,e)}  (Eq. (1) right side). */
void or_apply_rows(const or_ctx *o, double aK, double aM, const double *u,
                   const int64_t *rows, int64_t nrows, double *out)
{
    for (int64_t t = 0; t < nrows; t++) {
        int64_t r = rows[t];
        int64_t i = r % o->nn[0], j = (r / o->nn[0]) % o->nn[1], k = r / (o->nn[0] * o->nn[1]);
        double s = 0.0;
        for (int l = 0; l < 8; l++) {          /* node is local node l of element (i-bx, j-by, k-bz) */
            int64_t ex = i - (l & 1), ey = j - ((l >> 1) & 1), ez = k - ((l >> 2) & 1);
            if (ex < 0 || ey < 0 || ez < 0 || ex >= o->ne[0] || ey >= o->ne[1] || ez >= o->ne[2]) continue;
            int64_t e = ex + o->ne[0] * (ey + o->ne[1] * ez);
            int64_t nodes[8];
            double Kel[64], Mel[64];
            elem_nodes(o, e, nodes);
            elem_scaled(o, e, Kel, Mel);
            for (int b = 0; b < 8; b++)
                s += (aK * Kel[l * 8 + b] + aM * Mel[l * 8 + b]) * u[nodes[b]];
        }
        out[t] = s;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* Flux load F_i = int_face f phi_i ds, f = f_const + Gaussian beam (R12):    */
/*   beam(a,b) = P/(2 pi s^2) exp(-((a-ca)^2 + (b-cb)^2)/(2 s^2)),  (a, b) the in-plane        */
/*   coordinates of the face in increasing axis order.  2x2 Gauss per boundary quad.            */

static double beam_f(double f_const, const double *beam, double a, double b)
{
    double f = f_const;
    if (beam) {
        double P = beam[0], s = beam[1], ca = beam[2], cb = beam[3];
        f += P / (2.0 * M_PI * s * s) * exp(-((a - ca) * (a - ca) + (b - cb) * (b - cb)) / (2.0 * s * s));
    }
    return f;
}

/* Tet mesh: every boundary quad is two triangles {(0,0),(1,0),(1,1)} and {(0,0),(0,1),(1,1)}
 * in the face's (a, b) corner coordinates (the boundary faces of the Kuhn tets); P1 basis on
 * each triangle; 3-point quadrature (barycentric (2/3,1/6,1/6) and permutations, weight 1/3,
 * exact for quadratics). */
static int face_load_tets(const or_ctx *o, int face, double f_const, const double *beam, double *F)
{
    int nd = face / 2, ax = nd == 0 ? 1 : 0, bx = nd == 2 ? 1 : 2;
    int64_t plane = (face & 1) ? o->ne[nd] : 0;
    const int tri[2][3][2] = {{{0, 0}, {1, 0}, {1, 1}}, {{0, 0}, {0, 1}, {1, 1}}};
    const double bary[3][3] = {{2.0 / 3, 1.0 / 6, 1.0 / 6}, {1.0 / 6, 2.0 / 3, 1.0 / 6}, {1.0 / 6, 1.0 / 6, 2.0 / 3}};
    for (int64_t n = 0; n < o->nnodes; n++) F[n] = 0.0;
    double area = 0.5 * o->h[ax] * o->h[bx];
    for (int64_t qb = 0; qb < o->ne[bx]; qb++)
    for (int64_t qa = 0; qa < o->ne[ax]; qa++)
        for (int t = 0; t < 2; t++)
            for (int g = 0; g < 3; g++) {
                double a = o->origin[ax], b = o->origin[bx];
                for (int v = 0; v < 3; v++) {
                    a += bary[g][v] * (qa + tri[t][v][0]) * o->h[ax];
                    b += bary[g][v] * (qb + tri[t][v][1]) * o->h[bx];
                }
                double f = beam_f(f_const, beam, a, b);
                for (int v = 0; v < 3; v++) {
                    int64_t idx[3];
                    idx[nd] = plane; idx[ax] = qa + tri[t][v][0]; idx[bx] = qb + tri[t][v][1];
                    F[node_id(o, idx[0], idx[1], idx[2])] += (area / 3.0) * f * bary[g][v];
                }
            }
    return OR_OK;
}

int or_face_load(const or_ctx *o, int face, double f_const, const double *beam, double *F)
{
    if (o->elem >= 1) return (face < 0 || face > 5) ? OR_E_ARG : face_load_tets(o, face, f_const, beam, F);
    if (face < 0 || face > 5) return OR_E_ARG;
    int nd = face / 2;                       /* normal axis */
    int ax = nd == 0 ? 1 : 0;                /* first in-plane axis */
    int bx = nd == 2 ? 1 : 2;                /* second in-plane axis */
    int64_t plane = (face & 1) ? o->ne[nd] : 0;
    const double gp[2] = {0.5 * (1.0 - 1.0 / sqrt(3.0)), 0.5 * (1.0 + 1.0 / sqrt(3.0))};
    for (int64_t n = 0; n < o->nnodes; n++) F[n] = 0.0;
    for (int64_t qb = 0; qb < o->ne[bx]; qb++)
    for (int64_t qa = 0; qa < o->ne[ax]; qa++) {
        for (int gb = 0; gb < 2; gb++)
        for (int ga = 0; ga < 2; ga++) {
            double ta = gp[ga] * o->h[ax], tb = gp[gb] * o->h[bx];
            double a = o->origin[ax] + qa * o->h[ax] + ta;
            double b = o->origin[bx] + qb * o->h[bx] + tb;
            double f = f_const;
            if (beam) {
                double P = beam[0], s = beam[1], ca = beam[2], cb = beam[3];
                f += P / (2.0 * M_PI * s * s) * exp(-((a - ca) * (a - ca) + (b - cb) * (b - cb)) / (2.0 * s * s));
            }
            double w = (o->h[ax] / 2.0) * (o->h[bx] / 2.0);
            for (int cb2 = 0; cb2 < 2; cb2++)
            for (int ca2 = 0; ca2 < 2; ca2++) {
                double phi = phi1d(ca2, ta, o->h[ax]) * phi1d(cb2, tb, o->h[bx]);
                int64_t idx[3];
                idx[nd] = plane; idx[ax] = qa + ca2; idx[bx] = qb + cb2;
                F[node_id(o, idx[0], idx[1], idx[2])] += w * f * phi;
            }
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------ */
/* Dirichlet faces (extension, reading R3).  Node is Dirichlet if it lies on a flagged face;   */
/* its value is that of the lowest-numbered flagged face containing it.                          */

void or_set_dirichlet(or_ctx *o, unsigned bits, const double vals[6])
{
    o->bits = bits;
    for (int f = 0; f < 6; f++) o->gval[f] = vals ? vals[f] : 0.0;
    for (int64_t k = 0; k < o->nn[2]; k++)
    for (int64_t j = 0; j < o->nn[1]; j++)
    for (int64_t i = 0; i < o->nn[0]; i++) {
        int64_t n = node_id(o, i, j, k);
        int64_t idx[3] = {i, j, k};
        o->isD[n] = 0; o->g[n] = 0.0;
        for (int f = 0; f < 6; f++) {
            if (!(bits & (1u << f))) continue;
            int d = f / 2;
            int64_t at = (f & 1) ? o->ne[d] : 0;
            if (idx[d] == at) { o->isD[n] = 1; o->g[n] = o->gval[f]; break; }
        }
    }
}

int or_is_dirichlet(const or_ctx *o, unsigned char *mask)
{
    memcpy(mask, o->isD, (size_t)o->nnodes);
    return OR_OK;
}

/* diag(aK K + aM M), 1 on Dirichlet rows (P:117 Jacobi; reading R3). */
int or_diag(const or_ctx *o, double aK, double aM, double *diag)
{
    if (!o->has_csr) return OR_E_ARG;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < o->nnodes; r++) {
        double d = 0.0;
        for (int64_t p = o->rowptr[r]; p < o->rowptr[r + 1]; p++)
            if (o->col[p] == r) d = aK * o->Kv[p] + aM * o->Mv[p];
        diag[r] = o->isD[r] ? 1.0 : d;
    }
    return OR_OK;
}

/* Eliminated operator on free nodes: y_F = A_FF x_F, y_D = 0 (reading R3). */
static void spmv_free(const or_ctx *o, double aK, double aM, const double *x, double *y, double *tmp)
{
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < o->nnodes; n++) tmp[n] = o->isD[n] ? 0.0 : x[n];
    or_spmv(o, aK, aM, tmp, y);
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < o->nnodes; n++) if (o->isD[n]) y[n] = 0.0;
}

/* sum over free nodes of a_n b_n: chunks of OR_CHUNK nodes summed left to right, then the chunk
 * sums left to right (fixed order for any thread count) */
static double dot_free(const or_ctx *o, const double *a, const double *b)
{
    const int64_t N = o->nnodes, nch = (N + OR_CHUNK - 1) / OR_CHUNK;
    double *part = malloc(sizeof(double) * (size_t)(nch > 0 ? nch : 1));
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < nch; c++) {
        const int64_t n1 = (c + 1) * OR_CHUNK < N ? (c + 1) * OR_CHUNK : N;
        double s = 0.0;
        for (int64_t n = c * OR_CHUNK; n < n1; n++) if (!o->isD[n]) s += a[n] * b[n];
        part[c] = s;
    }
    double s = 0.0;
    for (int64_t c = 0; c < nch; c++) s += part[c];
    free(part);
    return s;
}

/*
 * PCG, Algorithm 1, on the eliminated system A_FF x_F = b_F; x_D = b_D.
 * Readings: R4 stop when ||r||_2 <= tol ||b_F||_2 (recurrence residual);
 *           R5 delta_old <- delta before recomputing delta;
 *           R6 residual replaced when i > 0 and i mod replace_every == 0;
 *           b_F = 0 -> x = 0 with 0 iterations;
 *           d^T q <= 0 or non-finite -> breakdown.
 * info[0] = iterations, info[1] = ||r||/||b||, info[2] = final delta.
 */
int or_pcg(const or_ctx *o, double aK, double aM, const double *b, double *x,
           double tol, int max_iter, int replace_every, double info[3])
{
    const int64_t N = o->nnodes;
    double *r = malloc(sizeof(double) * N), *s = malloc(sizeof(double) * N);
    double *d = malloc(sizeof(double) * N), *q = malloc(sizeof(double) * N);
    double *P = malloc(sizeof(double) * N), *tmp = malloc(sizeof(double) * N);
    if (!r || !s || !d || !q || !P || !tmp) return OR_E_OOM;
    or_diag(o, aK, aM, P);
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; n++) if (o->isD[n]) x[n] = b[n];
    double bnorm = sqrt(dot_free(o, b, b));
    int status = OR_OK, i = 0;
    double delta = 0.0, rr = 0.0;
    if (bnorm == 0.0) {
        for (int64_t n = 0; n < N; n++) if (!o->isD[n]) x[n] = 0.0;
        info[0] = 0; info[1] = 0.0; info[2] = 0.0;
        free(r); free(s); free(d); free(q); free(P); free(tmp);
        return OR_OK;
    }
    /* line 3: r <- b - A x */
    spmv_free(o, aK, aM, x, q, tmp);
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; n++) r[n] = o->isD[n] ? 0.0 : b[n] - q[n];
    /* line 4: d <- P^{-1} r ; line 5: delta <- r^T d */
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; n++) d[n] = r[n] / P[n];
    delta = dot_free(o, r, d);
    rr = dot_free(o, r, r);
    while (i < max_iter && sqrt(rr) > tol * bnorm) {
        spmv_free(o, aK, aM, d, q, tmp);                  /* line 7: q <- A d */
        double dq = dot_free(o, d, q);
        if (!(dq > 0.0) || !isfinite(dq)) { status = OR_E_BREAKDOWN; break; }
        double alpha = delta / dq;                        /* line 8 */
#pragma omp parallel for schedule(static)
        for (int64_t n = 0; n < N; n++) if (!o->isD[n]) x[n] += alpha * d[n];   /* line 9 */
        if (i > 0 && replace_every > 0 && i % replace_every == 0) {               /* line 10-11 */
            spmv_free(o, aK, aM, x, q, tmp);
#pragma omp parallel for schedule(static)
            for (int64_t n = 0; n < N; n++) r[n] = o->isD[n] ? 0.0 : b[n] - q[n];
        } else {
#pragma omp parallel for schedule(static)
            for (int64_t n = 0; n < N; n++) r[n] -= alpha * q[n];                 /* line 13 */
        }
#pragma omp parallel for schedule(static)
        for (int64_t n = 0; n < N; n++) s[n] = r[n] / P[n];                       /* line 15 */
        double delta_old = delta;                                                 /* R5 */
        delta = dot_free(o, r, s);                                                /* line 16 */
        rr = dot_free(o, r, r);
        double beta = delta / delta_old;                                          /* line 17 */
#pragma omp parallel for schedule(static)
        for (int64_t n = 0; n < N; n++) d[n] = s[n] + beta * d[n];                /* line 18 */
        i++;                                                                      /* line 19 */
    }
    if (status == OR_OK && sqrt(rr) > tol * bnorm) status = OR_E_NOCONV;
    info[0] = i; info[1] = sqrt(rr) / bnorm; info[2] = delta;
    free(r); free(s); free(d); free(q); free(P); free(tmp);
    return status;
}

/*
 * Right-hand side of one step (readings R7, R8, R3):
 *   b = L u^n + dt F,  L = M - (1-theta) dt K;  then the Dirichlet lift
 *   b_F -= (A g~)_F with A = M + theta dt K and g~ = g on D, 0 on F;  b_D = g_D.
 */
void or_rhs(const or_ctx *o, double theta, double dt, const double *F, const double *un, double *b)
{
    const int64_t N = o->nnodes;
    or_spmv(o, -(1.0 - theta) * dt, 1.0, un, b);
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < N; n++) b[n] += dt * F[n];
    if (o->bits) {
        double *Ag = malloc(sizeof(double) * N);
        or_spmv(o, theta * dt, 1.0, o->g, Ag);
        for (int64_t n = 0; n < N; n++) b[n] = o->isD[n] ? o->g[n] : b[n] - Ag[n];
        free(Ag);
    }
}

/*
 * theta-scheme time loop: for n = step0..step0+nsteps-1 solve A u^{n+1} = b(u^n).
 * Guess (reading R9): x0 = u^n at n = 0 of a run, else 2 u^n - u^{n-1}.
 * u: in u^{step0} (Dirichlet nodes are set to g first), out u^{step0+nsteps}.
 * uprev (may be NULL): in u^{step0-1} (used when step0 > 0: a resumed run), out the iterate
 * before the final one.  iters[n] receives the PCG iteration count of step n (may be NULL).
 * snap (may be NULL): after each step, the plane k = snap_plane of u is appended.
 */
int or_simulate_resume(const or_ctx *o, double theta, double dt, int nsteps, const double *F, double *u,
                       double *uprev_io, int64_t step0, double tol, int max_iter, int replace_every,
                       int32_t *iters, int64_t snap_plane, double *snap)
{
    const int64_t N = o->nnodes;
    const int64_t plane = o->nn[0] * o->nn[1];
    double *uprev = malloc(sizeof(double) * N), *b = malloc(sizeof(double) * N);
    double *x = malloc(sizeof(double) * N);
    if (!uprev || !b || !x) return OR_E_OOM;
    const int first = step0 <= 0 || !uprev_io;
    for (int64_t n = 0; n < N; n++) if (o->isD[n]) u[n] = o->g[n];
    if (first) memcpy(uprev, u, sizeof(double) * N);
    else {
        memcpy(uprev, uprev_io, sizeof(double) * N);
        for (int64_t n = 0; n < N; n++) if (o->isD[n]) uprev[n] = o->g[n];
    }
    int status = OR_OK;
    for (int step = 0; step < nsteps; step++) {
        or_rhs(o, theta, dt, F, u, b);
        const int guess_u = step == 0 && first;
#pragma omp parallel for schedule(static)
        for (int64_t n = 0; n < N; n++) x[n] = guess_u ? u[n] : 2.0 * u[n] - uprev[n];
        double info[3];
        status = or_pcg(o, theta * dt, 1.0, b, x, tol, max_iter, replace_every, info);
        if (iters) iters[step] = (int32_t)info[0];
        memcpy(uprev, u, sizeof(double) * N);
        memcpy(u, x, sizeof(double) * N);
        if (snap) memcpy(snap + (int64_t)step * plane, u + snap_plane * plane, sizeof(double) * plane);
        if (status != OR_OK) break;
    }
    if (uprev_io) memcpy(uprev_io, uprev, sizeof(double) * N);
    free(uprev); free(b); free(x);
    return status;
}

int or_simulate(const or_ctx *o, double theta, double dt, int nsteps, const double *F, double *u,
                double tol, int max_iter, int replace_every, int32_t *iters,
                int64_t snap_plane, double *snap)
{
    return or_simulate_resume(o, theta, dt, nsteps, F, u, NULL, 0, tol, max_iter, replace_every, iters,
                              snap_plane, snap);
}
