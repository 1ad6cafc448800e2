/*
 * ic_pcg.c -- the paper's stronger CPU comparison method (NEXT row f4): sparse-matrix PCG with an
 * incomplete Cholesky preconditioner of drop tolerance 1e-3 (§5.3 "Further CPU Comparison",
 * P:322-332, Table 3; "incomplete Cholesky factorization with drop tolerance of 10^-3 [golub]",
 * P:324), single core as in the paper.
 *
 * A COMPARISON PROGRAM, not the product and not the oracle: it takes an assembled CSR matrix
 * (tools/ic_comparator.py passes the oracle's assembly) and is only run by tools/ and tests/.
 *
 *   ic_factor   threshold incomplete Cholesky A ~ L L^T of the symmetrically scaled matrix
 *               S = D^{-1/2} A D^{-1/2} (unit diagonal; reading R19 in DESIGN.md: the drop test is
 *               then independent of the units of k and rho C), row by row (up-looking): for row i,
 *               G[i][j] = (s_ij - sum_{k<j} G[i][k] G[j][k]) / G[j][j] for the columns j < i that
 *               are nonzero after fill, in increasing j; an off-diagonal G[i][j] is dropped when
 *               |G[i][j]| < droptol * ||S(j:n, j)||_1 (the column-norm rule of the common ICT
 *               definition); G[i][i] = sqrt(s_ii - sum_j G[i][j]^2); L = D^{1/2} G.
 *               droptol = 0 keeps everything: the exact Cholesky factor (the pin).
 *   ic_pcg      textbook PCG with M = L L^T, stop ||r||_2 <= tol ||b||_2 (reading R4).
 *   ic_simulate the theta-scheme loop of P:55 with A = M + theta dt K (factorised once),
 *               b = (M - (1-theta) dt K) u^n + dt F and the guess 2u^n - u^{n-1} (reading R9).
 * fp64, sequential sums, one thread.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define IC_OK 0
#define IC_E_ARG (-1)
#define IC_E_NOCONV (-3)
#define IC_E_BREAKDOWN (-4)
#define IC_E_OOM (-8)

typedef struct {
    int64_t n, nnz;
    int64_t *rp, *ci;      /* CSR rows of L; within a row columns ascend, the diagonal is last */
    double *v;
} ic_L;

typedef struct {           /* column j of L below the diagonal, rows ascending (grows row by row) */
    int64_t *r;
    double *v;
    int64_t len, cap;
} col_list;

/* binary min-heap of column indices */
static void heap_push(int64_t *h, int64_t *n, int64_t x)
{
    int64_t i = (*n)++;
    h[i] = x;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h[p] <= h[i]) break;
        int64_t t = h[p]; h[p] = h[i]; h[i] = t;
        i = p;
    }
}

static int64_t heap_pop(int64_t *h, int64_t *n)
{
    int64_t top = h[0];
    h[0] = h[--(*n)];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && h[l] < h[m]) m = l;
        if (r < *n && h[r] < h[m]) m = r;
        if (m == i) break;
        int64_t t = h[m]; h[m] = h[i]; h[i] = t;
        i = m;
    }
    return top;
}

void ic_free(ic_L *L)
{
    if (!L) return;
    free(L->rp); free(L->ci); free(L->v);
    free(L);
}

int64_t ic_nnz(const ic_L *L) { return L ? L->nnz : -1; }

int ic_factor(int64_t n, const int64_t *rp, const int64_t *col, const double *val, double droptol, ic_L **out)
{
    if (n <= 0 || !rp || !col || !val || !out || droptol < 0) return IC_E_ARG;
    int rc = IC_OK;
    double *cn = calloc((size_t)n, sizeof(double));         /* ||S(j:n, j)||_1 (A symmetric) */
    double *sc = malloc(sizeof(double) * (size_t)n);         /* a_jj^{-1/2} */
    double *w = calloc((size_t)n, sizeof(double));
    unsigned char *mk = calloc((size_t)n, 1);
    int64_t *heap = malloc(sizeof(int64_t) * (size_t)n);
    int64_t *rowj = malloc(sizeof(int64_t) * (size_t)n);
    double *rowv = malloc(sizeof(double) * (size_t)n);
    double *dg = malloc(sizeof(double) * (size_t)n);
    col_list *cl = calloc((size_t)n, sizeof(col_list));
    ic_L *L = calloc(1, sizeof(ic_L));
    int64_t cap = rp[n] + n;
    if (L) {
        L->rp = malloc(sizeof(int64_t) * (size_t)(n + 1));
        L->ci = malloc(sizeof(int64_t) * (size_t)cap);
        L->v = malloc(sizeof(double) * (size_t)cap);
    }
    if (!cn || !sc || !w || !mk || !heap || !rowj || !rowv || !dg || !cl || !L || !L->rp || !L->ci || !L->v) {
        rc = IC_E_OOM;
        goto done;
    }
    for (int64_t j = 0; j < n; j++) {
        sc[j] = 0.0;
        for (int64_t p = rp[j]; p < rp[j + 1]; p++)
            if (col[p] == j) sc[j] += val[p];
        if (!(sc[j] > 0.0)) { rc = IC_E_BREAKDOWN; goto done; }
        sc[j] = 1.0 / sqrt(sc[j]);
    }
    for (int64_t j = 0; j < n; j++)
        for (int64_t p = rp[j]; p < rp[j + 1]; p++)
            if (col[p] >= j) cn[j] += fabs(val[p] * sc[j] * sc[col[p]]);
    L->n = n;
    int64_t nz = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t hn = 0, nrow = 0;
        double d = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; p++) {
            const int64_t j = col[p];
            if (j < i) {
                if (!mk[j]) { mk[j] = 1; w[j] = 0.0; heap_push(heap, &hn, j); }
                w[j] += val[p] * sc[i] * sc[j];
            } else if (j == i) {
                d += val[p] * sc[i] * sc[i];
            }
        }
        while (hn > 0) {
            const int64_t j = heap_pop(heap, &hn);
            mk[j] = 0;
            const double lij = w[j] / dg[j];
            w[j] = 0.0;
            if (fabs(lij) < droptol * cn[j] || lij == 0.0) continue;      /* dropped */
            rowj[nrow] = j;
            rowv[nrow] = lij;
            nrow++;
            d -= lij * lij;
            const col_list *c = &cl[j];
            for (int64_t q = 0; q < c->len; q++) {                       /* rows m, j < m < i */
                const int64_t m = c->r[q];
                if (!mk[m]) { mk[m] = 1; w[m] = 0.0; heap_push(heap, &hn, m); }
                w[m] -= lij * c->v[q];
            }
        }
        if (!(d > 0.0)) { rc = IC_E_BREAKDOWN; goto done; }
        dg[i] = sqrt(d);
        if (nz + nrow + 1 > cap) {
            cap = 2 * cap + nrow + 1;
            int64_t *nc = realloc(L->ci, sizeof(int64_t) * (size_t)cap);
            double *nv = realloc(L->v, sizeof(double) * (size_t)cap);
            if (!nc || !nv) { if (nc) L->ci = nc; if (nv) L->v = nv; rc = IC_E_OOM; goto done; }
            L->ci = nc;
            L->v = nv;
        }
        L->rp[i] = nz;
        for (int64_t t = 0; t < nrow; t++) {
            L->ci[nz] = rowj[t];
            L->v[nz] = rowv[t];
            nz++;
            col_list *c = &cl[rowj[t]];
            if (c->len == c->cap) {
                int64_t nc2 = c->cap ? 2 * c->cap : 8;
                int64_t *r2 = realloc(c->r, sizeof(int64_t) * (size_t)nc2);
                double *v2 = realloc(c->v, sizeof(double) * (size_t)nc2);
                if (!r2 || !v2) { if (r2) c->r = r2; if (v2) c->v = v2; rc = IC_E_OOM; goto done; }
                c->r = r2; c->v = v2; c->cap = nc2;
            }
            c->r[c->len] = i;
            c->v[c->len] = rowv[t];
            c->len++;
        }
        L->ci[nz] = i;
        L->v[nz] = dg[i];
        nz++;
    }
    L->rp[n] = nz;
    L->nnz = nz;
    for (int64_t i = 0; i < n; i++)
        for (int64_t p = L->rp[i]; p < L->rp[i + 1]; p++) L->v[p] /= sc[i];
done:
    if (cl) for (int64_t j = 0; j < n; j++) { free(cl[j].r); free(cl[j].v); }
    free(cl); free(cn); free(sc); free(w); free(mk); free(heap); free(rowj); free(rowv); free(dg);
    if (rc != IC_OK) { ic_free(L); L = NULL; }
    *out = L;
    return rc;
}

/* L (dense, row-major n x n) for the small-case pins */
int ic_to_dense(const ic_L *L, double *D)
{
    if (!L || !D) return IC_E_ARG;
    memset(D, 0, sizeof(double) * (size_t)(L->n * L->n));
    for (int64_t i = 0; i < L->n; i++)
        for (int64_t p = L->rp[i]; p < L->rp[i + 1]; p++) D[i * L->n + L->ci[p]] = L->v[p];
    return IC_OK;
}

/* z = (L L^T)^{-1} r: forward L y = r (rows), backward L^T z = y (rows of L scattered) */
static void ic_solve(const ic_L *L, const double *r, double *z)
{
    const int64_t n = L->n;
    for (int64_t i = 0; i < n; i++) {
        double s = r[i];
        const int64_t e = L->rp[i + 1] - 1;                          /* diagonal */
        for (int64_t p = L->rp[i]; p < e; p++) s -= L->v[p] * z[L->ci[p]];
        z[i] = s / L->v[e];
    }
    for (int64_t i = n - 1; i >= 0; i--) {
        const int64_t e = L->rp[i + 1] - 1;
        z[i] /= L->v[e];
        const double zi = z[i];
        for (int64_t p = L->rp[i]; p < e; p++) z[L->ci[p]] -= L->v[p] * zi;
    }
}

static void spmv(int64_t n, const int64_t *rp, const int64_t *col, const double *val, const double *x, double *y)
{
    for (int64_t i = 0; i < n; i++) {
        double s = 0.0;
        for (int64_t p = rp[i]; p < rp[i + 1]; p++) s += val[p] * x[col[p]];
        y[i] = s;
    }
}

static double dot(int64_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* PCG with M = L L^T; x: in guess, out solution; *iters = iterations taken */
int ic_pcg(int64_t n, const int64_t *rp, const int64_t *col, const double *val, const ic_L *L, const double *b,
           double *x, double tol, int max_iter, int *iters)
{
    if (!L || L->n != n || !b || !x) return IC_E_ARG;
    double *r = malloc(sizeof(double) * (size_t)n), *z = malloc(sizeof(double) * (size_t)n);
    double *p = malloc(sizeof(double) * (size_t)n), *q = malloc(sizeof(double) * (size_t)n);
    if (!r || !z || !p || !q) { free(r); free(z); free(p); free(q); return IC_E_OOM; }
    int rc = IC_OK, it = 0;
    const double bn = sqrt(dot(n, b, b));
    spmv(n, rp, col, val, x, q);
    for (int64_t i = 0; i < n; i++) r[i] = b[i] - q[i];
    if (bn == 0.0) {
        for (int64_t i = 0; i < n; i++) x[i] = 0.0;
        goto out;
    }
    ic_solve(L, r, z);
    memcpy(p, z, sizeof(double) * (size_t)n);
    double rho = dot(n, r, z);
    while (sqrt(dot(n, r, r)) > tol * bn) {
        if (it >= max_iter) { rc = IC_E_NOCONV; break; }
        spmv(n, rp, col, val, p, q);
        const double pq = dot(n, p, q);
        if (!(pq > 0.0)) { rc = IC_E_BREAKDOWN; break; }
        const double alpha = rho / pq;
        for (int64_t i = 0; i < n; i++) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
        ic_solve(L, r, z);
        const double rho_new = dot(n, r, z);
        const double beta = rho_new / rho;
        rho = rho_new;
        for (int64_t i = 0; i < n; i++) p[i] = z[i] + beta * p[i];
        it++;
    }
out:
    if (iters) *iters = it;
    free(r); free(z); free(p); free(q);
    return rc;
}

/* theta-scheme loop: A (values aval) and the RHS operator (values lval) share the pattern rp/col.
 * u: in u^0, out u^nsteps.  iters: per-step iteration counts (nsteps ints). */
int ic_simulate(int64_t n, const int64_t *rp, const int64_t *col, const double *aval, const double *lval,
                const ic_L *L, const double *F, double dt, int nsteps, double *u, double tol, int max_iter,
                int *iters)
{
    double *b = malloc(sizeof(double) * (size_t)n), *x = malloc(sizeof(double) * (size_t)n);
    double *up = malloc(sizeof(double) * (size_t)n);
    if (!b || !x || !up) { free(b); free(x); free(up); return IC_E_OOM; }
    int rc = IC_OK;
    for (int s = 0; s < nsteps && rc == IC_OK; s++) {
        spmv(n, rp, col, lval, u, b);
        if (F) for (int64_t i = 0; i < n; i++) b[i] += dt * F[i];
        for (int64_t i = 0; i < n; i++) x[i] = s == 0 ? u[i] : 2.0 * u[i] - up[i];
        rc = ic_pcg(n, rp, col, aval, L, b, x, tol, max_iter, iters ? &iters[s] : NULL);
        memcpy(up, u, sizeof(double) * (size_t)n);
        memcpy(u, x, sizeof(double) * (size_t)n);
    }
    free(b); free(x); free(up);
    return rc;
}
