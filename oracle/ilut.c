/*
 * oracle/ilut.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Plain, slow, obviously-correct dual-threshold incomplete LU (ILUT) of a
 * complex128 CSR matrix, written from:
 *   PAPER.md sec. II (lines 94): "incomplete LU factorization with dual-threshold
 *   ... a drop tolerance d and allowed fill-in p are specified such that all
 *   fill-in smaller than d times the infinity-norm of a row are dropped, and at
 *   most only p*NNZ(L~) fill-in elements are allowed."
 * and the row-wise (IKJ) ILUT algorithm the paper cites as [saad:2003]
 * (Saad, Iterative Methods for Sparse Linear Systems, Alg. 10.6).
 *
 * Readings fixed in DESIGN.md sec. "Readings" (R4..R7):
 *  - tau_i = d * max_j |a_ij| (row infinity norm of the ORIGINAL row i);
 *    every magnitude test is done on squared moduli: drop  <=>  |z|^2 < tau_i^2.
 *  - multiplier:  w_k <- w_k * (1/u_kk) with 1/u = (ur/(ur^2+ui^2), -ui/(ur^2+ui^2));
 *    the multiplier itself is dropped if |w_k|^2 < tau_i^2 (no update then).
 *  - update:      w_j <- w_j - w_k*u_kj   (naive complex product, no FMA).
 *  - fill cap:    per row, each of the L part and the strict-U part keeps at
 *    most  lfil_i = floor(p * nnz(a_i) / 2)  entries, the largest |.|^2
 *    (ties: smaller column first); so NNZ(L)+NNZ(U) <= p*NNZ(A) + n.
 *  - the diagonal is never dropped; an exactly-zero pivot is replaced by tau_i
 *    (error if tau_i == 0).
 * L is unit lower triangular (unit diagonal NOT stored); U stores its diagonal
 * as the FIRST entry of each row, then the strict upper part, columns ascending.
 * L's rows are stored columns ascending.
 * Compile with -ffp-contract=off (no FMA contraction).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef struct { double re, im; } cplx;

static double mag2(cplx z) { return z.re * z.re + z.im * z.im; }

/* ---- tiny binary min-heap of int64 column indices ---- */
typedef struct { int64_t *a; int64_t n; } heap_t;
static void heap_push(heap_t *h, int64_t v) {
    int64_t i = h->n++;
    h->a[i] = v;
    while (i > 0) {
        int64_t p = (i - 1) / 2;
        if (h->a[p] <= h->a[i]) break;
        int64_t t = h->a[p]; h->a[p] = h->a[i]; h->a[i] = t; i = p;
    }
}
static int64_t heap_pop(heap_t *h) {
    int64_t top = h->a[0];
    h->a[0] = h->a[--h->n];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < h->n && h->a[l] < h->a[m]) m = l;
        if (r < h->n && h->a[r] < h->a[m]) m = r;
        if (m == i) break;
        int64_t t = h->a[m]; h->a[m] = h->a[i]; h->a[i] = t; i = m;
    }
    return top;
}

/* growable output arrays */
typedef struct { int64_t *ptr, *col; cplx *val; int64_t nnz, cap; } csr_out;
static int out_push(csr_out *o, int64_t j, cplx v) {
    if (o->nnz == o->cap) {
        int64_t nc = o->cap ? 2 * o->cap : 1024;
        int64_t *c2 = realloc(o->col, nc * sizeof(int64_t));
        if (!c2) return -1;
        o->col = c2;
        cplx *v2 = realloc(o->val, nc * sizeof(cplx));
        if (!v2) return -1;
        o->val = v2;
        o->cap = nc;
    }
    o->col[o->nnz] = j; o->val[o->nnz] = v; o->nnz++;
    return 0;
}

/* selection of the lfil largest entries: sort (col,val) by |val|^2 desc, col asc */
typedef struct { int64_t j; cplx v; double m; } ent;
static int ent_cmp_mag(const void *a, const void *b) {
    const ent *x = a, *y = b;
    if (x->m > y->m) return -1;
    if (x->m < y->m) return 1;
    return (x->j < y->j) ? -1 : (x->j > y->j);
}
static int ent_cmp_col(const void *a, const void *b) {
    const ent *x = a, *y = b;
    return (x->j < y->j) ? -1 : (x->j > y->j);
}

/* Returns 0 on success, -(i+1) on an unrecoverable zero pivot at row i, -1e9-ish on OOM. */
int oracle_ilut(int64_t n, const int64_t *rowptr, const int64_t *colidx, const double *vals,
                double drop_tol, double fill_factor,
                int64_t **Lp, int64_t **Lj, double **Lx, int64_t *Lnnz,
                int64_t **Up, int64_t **Uj, double **Ux, int64_t *Unnz)
{
    const cplx *a = (const cplx *)vals;
    cplx *w = calloc(n, sizeof(cplx));
    char *present = calloc(n, 1);
    int64_t *nzlist = malloc(n * sizeof(int64_t));
    heap_t heap = { malloc(n * sizeof(int64_t)), 0 };
    ent *buf = malloc(n * sizeof(ent));
    csr_out L = {0}, U = {0};
    L.ptr = malloc((n + 1) * sizeof(int64_t));
    U.ptr = malloc((n + 1) * sizeof(int64_t));
    int rc = 0;
    if (!w || !present || !nzlist || !heap.a || !buf || !L.ptr || !U.ptr) { rc = -2000000000; goto done; }
    L.ptr[0] = 0; U.ptr[0] = 0;

    for (int64_t i = 0; i < n; i++) {
        int64_t nnzrow = rowptr[i + 1] - rowptr[i];
        int64_t lfil = (int64_t)(fill_factor * (double)nnzrow / 2.0);
        double rowmax2 = 0.0;
        int64_t nz = 0;
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; q++) {
            int64_t j = colidx[q];
            double m = mag2(a[q]);
            if (m > rowmax2) rowmax2 = m;
            w[j] = a[q];
            present[j] = 1;
            nzlist[nz++] = j;
            if (j < i) heap_push(&heap, j);
        }
        if (!present[i]) { present[i] = 1; w[i].re = 0; w[i].im = 0; nzlist[nz++] = i; }
        double tau2 = drop_tol * drop_tol * rowmax2;

        /* eliminate in increasing k */
        while (heap.n > 0) {
            int64_t k = heap_pop(&heap);
            /* u_kk is the first entry of U row k */
            cplx ukk = U.val[U.ptr[k]];
            double d = ukk.re * ukk.re + ukk.im * ukk.im;
            cplx inv = { ukk.re / d, -ukk.im / d };
            cplx wk = { w[k].re * inv.re - w[k].im * inv.im, w[k].re * inv.im + w[k].im * inv.re };
            if (mag2(wk) < tau2) { w[k].re = 0; w[k].im = 0; continue; }
            w[k] = wk;
            for (int64_t q = U.ptr[k] + 1; q < U.ptr[k + 1]; q++) {
                int64_t j = U.col[q];
                cplx u = U.val[q];
                if (!present[j]) {
                    present[j] = 1; w[j].re = 0; w[j].im = 0; nzlist[nz++] = j;
                    if (j < i) heap_push(&heap, j);
                }
                cplx p = { wk.re * u.re - wk.im * u.im, wk.re * u.im + wk.im * u.re };
                w[j].re = w[j].re - p.re;
                w[j].im = w[j].im - p.im;
            }
        }

        /* split, drop, cap: L part */
        int64_t nb = 0;
        for (int64_t t = 0; t < nz; t++) {
            int64_t j = nzlist[t];
            if (j < i) {
                double m = mag2(w[j]);
                if (m != 0.0 && !(m < tau2)) { buf[nb].j = j; buf[nb].v = w[j]; buf[nb].m = m; nb++; }
            }
        }
        if (nb > lfil) { qsort(buf, nb, sizeof(ent), ent_cmp_mag); nb = lfil; }
        qsort(buf, nb, sizeof(ent), ent_cmp_col);
        for (int64_t t = 0; t < nb; t++) if (out_push(&L, buf[t].j, buf[t].v)) { rc = -2000000000; goto done; }
        L.ptr[i + 1] = L.nnz;

        /* diagonal */
        cplx di = w[i];
        if (di.re == 0.0 && di.im == 0.0) {
            if (tau2 == 0.0) { rc = -(int)(i + 1); goto done; }
            di.re = drop_tol * sqrt(rowmax2); di.im = 0.0;
        }
        if (out_push(&U, i, di)) { rc = -2000000000; goto done; }
        /* strict U part */
        nb = 0;
        for (int64_t t = 0; t < nz; t++) {
            int64_t j = nzlist[t];
            if (j > i) {
                double m = mag2(w[j]);
                if (m != 0.0 && !(m < tau2)) { buf[nb].j = j; buf[nb].v = w[j]; buf[nb].m = m; nb++; }
            }
        }
        if (nb > lfil) { qsort(buf, nb, sizeof(ent), ent_cmp_mag); nb = lfil; }
        qsort(buf, nb, sizeof(ent), ent_cmp_col);
        for (int64_t t = 0; t < nb; t++) if (out_push(&U, buf[t].j, buf[t].v)) { rc = -2000000000; goto done; }
        U.ptr[i + 1] = U.nnz;

        /* reset work row */
        for (int64_t t = 0; t < nz; t++) { int64_t j = nzlist[t]; present[j] = 0; w[j].re = 0; w[j].im = 0; }
    }
done:
    free(w); free(present); free(nzlist); free(heap.a); free(buf);
    if (rc) { free(L.ptr); free(L.col); free(L.val); free(U.ptr); free(U.col); free(U.val); return rc; }
    *Lp = L.ptr; *Lj = L.col; *Lx = (double *)L.val; *Lnnz = L.nnz;
    *Up = U.ptr; *Uj = U.col; *Ux = (double *)U.val; *Unnz = U.nnz;
    return 0;
}


/* ------------------------------------------------------------------------------------
 * ILUTP: ILUT with column pivoting -- the "dual-threshold and pivoting (iLUTP)" of
 * PAPER.md:94 (Saad, Iterative Methods for Sparse Linear Systems, sec. 10.4.4, ILUTP).
 * Rules of oracle_ilut (R4-R7) plus (reading R13 of DESIGN.md):
 *  - A Pi = L U with a column permutation Pi (perm[position] = original column).  Row i
 *    is assembled in POSITION space (position of original column c = iperm[c]).
 *  - after elimination, dropping and the fill cap, the U part of row i (positions >= i,
 *    the diagonal position i included even if zero) is searched for its largest entry
 *    |w_t|^2 (ties: smaller position); if permtol^2 |w_t|^2 > |w_i|^2 and t != i, the
 *    columns at positions i and t are exchanged for row i and all later rows (the old
 *    diagonal value moves to position t and stays in U if nonzero).
 *  - a zero pivot left after that is repaired as in oracle_ilut.
 *  - U rows are kept in ORIGINAL columns while factoring (later exchanges move
 *    positions > i) and converted to final positions at the end; L entries have
 *    positions < i, which never move again.
 * permtol = 0 never exchanges and reproduces oracle_ilut exactly.
 * ------------------------------------------------------------------------------------ */
static int ent_cmp_col_ent(const void *a, const void *b) { return ent_cmp_col(a, b); }

int oracle_ilutp(int64_t n, const int64_t *rowptr, const int64_t *colidx, const double *vals,
                 double drop_tol, double fill_factor, double permtol,
                 int64_t **Lp, int64_t **Lj, double **Lx, int64_t *Lnnz,
                 int64_t **Up, int64_t **Uj, double **Ux, int64_t *Unnz, int64_t **perm_out)
{
    const cplx *a = (const cplx *)vals;
    cplx *w = calloc(n, sizeof(cplx));
    char *present = calloc(n, 1);
    int64_t *nzlist = malloc(n * sizeof(int64_t));
    heap_t heap = { malloc(n * sizeof(int64_t)), 0 };
    ent *buf = malloc(n * sizeof(ent));
    int64_t *perm = malloc(n * sizeof(int64_t)), *iperm = malloc(n * sizeof(int64_t));
    csr_out L = {0}, U = {0};
    L.ptr = malloc((n + 1) * sizeof(int64_t));
    U.ptr = malloc((n + 1) * sizeof(int64_t));
    int rc = 0;
    if (!w || !present || !nzlist || !heap.a || !buf || !L.ptr || !U.ptr || !perm || !iperm) { rc = -2000000000; goto done; }
    for (int64_t c = 0; c < n; c++) { perm[c] = c; iperm[c] = c; }
    L.ptr[0] = 0; U.ptr[0] = 0;
    const double pt2 = permtol * permtol;

    for (int64_t i = 0; i < n; i++) {
        int64_t nnzrow = rowptr[i + 1] - rowptr[i];
        int64_t lfil = (int64_t)(fill_factor * (double)nnzrow / 2.0);
        double rowmax2 = 0.0;
        int64_t nz = 0;
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; q++) {
            int64_t j = iperm[colidx[q]];
            double m = mag2(a[q]);
            if (m > rowmax2) rowmax2 = m;
            w[j] = a[q];
            present[j] = 1;
            nzlist[nz++] = j;
            if (j < i) heap_push(&heap, j);
        }
        if (!present[i]) { present[i] = 1; w[i].re = 0; w[i].im = 0; nzlist[nz++] = i; }
        double tau2 = drop_tol * drop_tol * rowmax2;

        while (heap.n > 0) {
            int64_t k = heap_pop(&heap);
            cplx ukk = U.val[U.ptr[k]];
            double d = ukk.re * ukk.re + ukk.im * ukk.im;
            cplx inv = { ukk.re / d, -ukk.im / d };
            cplx wk = { w[k].re * inv.re - w[k].im * inv.im, w[k].re * inv.im + w[k].im * inv.re };
            if (mag2(wk) < tau2) { w[k].re = 0; w[k].im = 0; continue; }
            w[k] = wk;
            for (int64_t q = U.ptr[k] + 1; q < U.ptr[k + 1]; q++) {
                int64_t j = iperm[U.col[q]];
                cplx u = U.val[q];
                if (!present[j]) {
                    present[j] = 1; w[j].re = 0; w[j].im = 0; nzlist[nz++] = j;
                    if (j < i) heap_push(&heap, j);
                }
                cplx p = { wk.re * u.re - wk.im * u.im, wk.re * u.im + wk.im * u.re };
                w[j].re = w[j].re - p.re;
                w[j].im = w[j].im - p.im;
            }
        }

        /* L part (positions < i are final) */
        int64_t nb = 0;
        for (int64_t t = 0; t < nz; t++) {
            int64_t j = nzlist[t];
            if (j < i) {
                double m = mag2(w[j]);
                if (m != 0.0 && !(m < tau2)) { buf[nb].j = j; buf[nb].v = w[j]; buf[nb].m = m; nb++; }
            }
        }
        if (nb > lfil) { qsort(buf, nb, sizeof(ent), ent_cmp_mag); nb = lfil; }
        qsort(buf, nb, sizeof(ent), ent_cmp_col);
        for (int64_t t = 0; t < nb; t++) if (out_push(&L, buf[t].j, buf[t].v)) { rc = -2000000000; goto done; }
        L.ptr[i + 1] = L.nnz;

        /* U part: drop, cap */
        nb = 0;
        for (int64_t t = 0; t < nz; t++) {
            int64_t j = nzlist[t];
            if (j > i) {
                double m = mag2(w[j]);
                if (m != 0.0 && !(m < tau2)) { buf[nb].j = j; buf[nb].v = w[j]; buf[nb].m = m; nb++; }
            }
        }
        if (nb > lfil) { qsort(buf, nb, sizeof(ent), ent_cmp_mag); nb = lfil; }
        /* pivot: largest kept entry (ties: smaller position) against the diagonal */
        cplx di = w[i];
        int64_t tbest = -1; double mbest = -1.0;
        for (int64_t t = 0; t < nb; t++)
            if (buf[t].m > mbest || (buf[t].m == mbest && buf[t].j < buf[tbest].j)) { mbest = buf[t].m; tbest = t; }
        if (tbest >= 0 && pt2 * buf[tbest].m > mag2(di)) {
            int64_t tpos = buf[tbest].j;
            cplx old = di;
            di = buf[tbest].v;
            /* exchange the columns at positions i and tpos */
            int64_t ci = perm[i], ct = perm[tpos];
            perm[i] = ct; perm[tpos] = ci; iperm[ct] = i; iperm[ci] = tpos;
            if (old.re != 0.0 || old.im != 0.0) { buf[tbest].v = old; buf[tbest].m = mag2(old); }
            else { buf[tbest] = buf[nb - 1]; nb--; }
        }
        if (di.re == 0.0 && di.im == 0.0) {
            if (tau2 == 0.0) { rc = -(int)(i + 1); goto done; }
            di.re = drop_tol * sqrt(rowmax2); di.im = 0.0;
        }
        qsort(buf, nb, sizeof(ent), ent_cmp_col_ent);
        /* store in ORIGINAL columns (positions > i may still be exchanged) */
        if (out_push(&U, perm[i], di)) { rc = -2000000000; goto done; }
        for (int64_t t = 0; t < nb; t++) if (out_push(&U, perm[buf[t].j], buf[t].v)) { rc = -2000000000; goto done; }
        U.ptr[i + 1] = U.nnz;

        for (int64_t t = 0; t < nz; t++) { int64_t j = nzlist[t]; present[j] = 0; w[j].re = 0; w[j].im = 0; }
    }
    /* U to final positions, strict part re-sorted by position */
    for (int64_t i = 0; i < n; i++) {
        int64_t q0 = U.ptr[i], q1 = U.ptr[i + 1];
        U.col[q0] = iperm[U.col[q0]];
        int64_t m = 0;
        for (int64_t q = q0 + 1; q < q1; q++) { buf[m].j = iperm[U.col[q]]; buf[m].v = U.val[q]; m++; }
        qsort(buf, m, sizeof(ent), ent_cmp_col_ent);
        for (int64_t t = 0; t < m; t++) { U.col[q0 + 1 + t] = buf[t].j; U.val[q0 + 1 + t] = buf[t].v; }
    }
done:
    free(w); free(present); free(nzlist); free(heap.a); free(buf); free(iperm);
    if (rc) { free(perm); free(L.ptr); free(L.col); free(L.val); free(U.ptr); free(U.col); free(U.val); return rc; }
    *Lp = L.ptr; *Lj = L.col; *Lx = (double *)L.val; *Lnnz = L.nnz;
    *Up = U.ptr; *Uj = U.col; *Ux = (double *)U.val; *Unnz = U.nnz;
    *perm_out = perm;
    return 0;
}

void oracle_free(void *p) { free(p); }
