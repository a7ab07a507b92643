/*
 * oracle/oracle.c -- the CPU ORACLE for the SpTRSV hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or helper with the CUDA library
 * (paper_1710_04985_b200/csrc) and never calls it.
 *
 * Plain, slow, obviously correct: sequential loops written in the paper's
 * order and notation, fp64 (plus an fp32 variant, reading Q21), compiled with
 * -O2 -ffp-contract=off so every a*b-c is two roundings (reading Q8).
 *
 * Paper: R. Li, "On Parallel Solution of Sparse Triangular Linear Systems in
 * CUDA", arXiv 1710.04985.  Readings of silent/ambiguous points
 * are the Q-numbers of SURVEY.md §8c, restated in DESIGN.md.
 *
 *   oracle_select     O-1/O-2  triangle selection, validation, dp counts
 *   oracle_levels_row O-3      lev(i) = 1 + max lev(j), row-wise
 *   oracle_levels_col A7       the column-wise loop
 *   oracle_schedule   O-4      nlev, ilev, jlev (stable)
 *   oracle_solve_f64  O-5      row-wise substitution
 *   oracle_solve_f32  O-5      same, float storage + accumulation (REAL)
 *   oracle_solve_col_f64       column-wise sweep over the CSC
 *   oracle_kahn       A18      Kahn topological sort by rounds
 *   oracle_backward_error      pin helper: componentwise backward error
 *
 * Build: gcc -O2 -ffp-contract=off -shared -fPIC -o liboracle.so oracle.c
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* Status names follow include/sptrsv.h's; the numbers are restated here (no
 * shared header): 0 SUCCESS, 1 INVALID_VALUE, 2 INVALID_MATRIX, 3 ZERO_PIVOT. */
#define OR_SUCCESS 0
#define OR_INVALID_VALUE 1
#define OR_INVALID_MATRIX 2
#define OR_ZERO_PIVOT 3
#define OR_ALLOC 4

#define OR_LOWER 0
#define OR_UPPER 1
#define OR_NON_UNIT 0
#define OR_UNIT 1

/* Is column j a dependency (off-diagonal entry of the selected triangle) of row i?
 * Eq. (1): L strictly lower, U strictly upper. */
static int in_triangle(int32_t i, int32_t j, int uplo) {
    return uplo == OR_LOWER ? (j < i) : (j > i);
}

/*
 * O-1 / O-2.  Validates the CSR (rules of include/sptrsv.h), selects the
 * `uplo` triangle (entries of the other triangle are ignored and counted,
 * reading Q2), locates the diagonal (reading Q1/Q3) and counts dependencies
 * dp[i] = #E_i ("counting the number of nonzeros per row" P:743).
 *
 * Row i is MALFORMED iff rowptr[i] < 0, rowptr[i+1] < rowptr[i],
 * rowptr[i+1] > rowptr[n], (i == 0 and rowptr[0] != 0), or -- when its
 * pointers are sound -- a column lies outside [0, n) or the columns of the
 * row are not strictly increasing.
 * Precedence: INVALID_VALUE, then INVALID_MATRIX (smallest malformed row in
 * *bad_row), then ZERO_PIVOT (NON_UNIT only; smallest row without a stored
 * diagonal or with a zero diagonal, in *zero_pivot_row).
 * Outputs (each may be NULL): dp[n], diagk[n] (index of the stored diagonal
 * entry or -1), *ignored (entries not referenced: other triangle, plus stored
 * diagonals when UNIT), *nnz_used (referenced off-diagonal entries).
 */
int oracle_select(int32_t n, const int32_t *rowptr, const int32_t *colidx, const double *vals,
                  int uplo, int diag, int32_t *dp, int32_t *diagk, int64_t *ignored,
                  int64_t *nnz_used, int32_t *bad_row, int32_t *zero_pivot_row) {
    if (bad_row) *bad_row = -1;
    if (zero_pivot_row) *zero_pivot_row = -1;
    if (ignored) *ignored = 0;
    if (nnz_used) *nnz_used = 0;
    if (n < 0) return OR_INVALID_VALUE;
    if (uplo != OR_LOWER && uplo != OR_UPPER) return OR_INVALID_VALUE;
    if (diag != OR_NON_UNIT && diag != OR_UNIT) return OR_INVALID_VALUE;
    if (n == 0) return OR_SUCCESS;
    if (!rowptr || !colidx || (!vals && diag == OR_NON_UNIT)) return OR_INVALID_VALUE;

    int32_t nnz = rowptr[n];
    /* malformed rows: scan all rows, keep the smallest */
    for (int32_t i = 0; i < n; ++i) {
        int32_t p = rowptr[i], q = rowptr[i + 1];
        int bad = 0;
        if (p < 0 || q < p || q > nnz || (i == 0 && p != 0)) bad = 1;
        else {
            for (int32_t k = p; k < q; ++k) {
                if (colidx[k] < 0 || colidx[k] >= n) { bad = 1; break; }
                if (k > p && colidx[k] <= colidx[k - 1]) { bad = 1; break; }
            }
        }
        if (bad) {
            if (bad_row) *bad_row = i;
            return OR_INVALID_MATRIX;
        }
    }
    int64_t ign = 0, used = 0;
    int32_t zp = -1;
    for (int32_t i = 0; i < n; ++i) {
        int32_t cnt = 0, dk = -1;
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
            int32_t j = colidx[k];
            if (j == i) dk = k;
            else if (in_triangle(i, j, uplo)) ++cnt;
            else ++ign;
        }
        if (dk >= 0 && diag == OR_UNIT) ++ign;       /* stored diagonal not referenced */
        if (dp) dp[i] = cnt;
        if (diagk) diagk[i] = dk;
        used += cnt;
        if (diag == OR_NON_UNIT && zp < 0 && (dk < 0 || vals[dk] == 0.0)) zp = i;
    }
    if (ignored) *ignored = ign;
    if (nnz_used) *nnz_used = used;
    if (zp >= 0) {
        if (zero_pivot_row) *zero_pivot_row = zp;
        return OR_ZERO_PIVOT;
    }
    return OR_SUCCESS;
}

/*
 * O-3.  Row-wise level recurrence with 0-based levels (reading
 * Q4): lev(i) = 0 if row i has no dependency, else 1 + max{lev(j) : j in E_i}.
 * LOWER sweeps i = 0..n-1; UPPER reverses the order (reading Q6).
 * Returns nlev = 1 + max lev (0 when n == 0).  Input must be valid.
 */
int32_t oracle_levels_row(int32_t n, const int32_t *rowptr, const int32_t *colidx, int uplo,
                          int32_t *lev) {
    int32_t nlev = 0;
    for (int32_t t = 0; t < n; ++t) {
        int32_t i = (uplo == OR_LOWER) ? t : n - 1 - t;
        int32_t l = 0;
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
            int32_t j = colidx[k];
            if (in_triangle(i, j, uplo) && lev[j] + 1 > l) l = lev[j] + 1;
        }
        lev[i] = l;
        if (l + 1 > nlev) nlev = l + 1;
    }
    return nlev;
}

/*
 * A7.  Column-wise level loop: lev initialised to zeros, then for
 * each column j in order, lev(i) = max{lev(j)+1, lev(i)} for every i with
 * T_ij != 0.  The columns come from this oracle's own transpose of the
 * selected strict triangle (TRANS).  Must equal the row-wise loop
 * (P:261-262).  Returns nlev, or -1 on allocation failure.
 */
int32_t oracle_levels_col(int32_t n, const int32_t *rowptr, const int32_t *colidx, int uplo,
                          int32_t *lev) {
    if (n == 0) return 0;
    int32_t *cp = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    if (!cp) return -1;
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (in_triangle(i, colidx[k], uplo)) cp[colidx[k] + 1]++;
    for (int32_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
    int32_t *ri = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cp[n] > 0 ? cp[n] : 1));
    int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!ri || !fill) { free(cp); free(ri); free(fill); return -1; }
    memcpy(fill, cp, sizeof(int32_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (in_triangle(i, colidx[k], uplo)) ri[fill[colidx[k]]++] = i;
    for (int32_t i = 0; i < n; ++i) lev[i] = 0;
    int32_t nlev = 0;
    for (int32_t t = 0; t < n; ++t) {
        int32_t j = (uplo == OR_LOWER) ? t : n - 1 - t;
        for (int32_t k = cp[j]; k < cp[j + 1]; ++k) {
            int32_t i = ri[k];
            if (lev[j] + 1 > lev[i]) lev[i] = lev[j] + 1;
        }
        if (lev[j] + 1 > nlev) nlev = lev[j] + 1;
    }
    free(cp); free(ri); free(fill);
    return nlev;
}

/*
 * O-4.  The level schedule: jlev lists the unknowns in
 * nondecreasing level order -- ascending unknown index within a level
 * (stable counting sort, reading Q5) -- and ilev[l] points at level l's first
 * entry; ilev[nlev] = n.
 */
void oracle_schedule(int32_t n, const int32_t *lev, int32_t nlev, int32_t *ilev, int32_t *jlev) {
    for (int32_t l = 0; l <= nlev; ++l) ilev[l] = 0;
    for (int32_t i = 0; i < n; ++i) ilev[lev[i] + 1]++;
    for (int32_t l = 0; l < nlev; ++l) ilev[l + 1] += ilev[l];
    int32_t *next = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nlev > 0 ? nlev : 1));
    for (int32_t l = 0; l < nlev; ++l) next[l] = ilev[l];
    for (int32_t i = 0; i < n; ++i) jlev[next[lev[i]]++] = i;
    free(next);
}

/*
 * O-5.  Row-wise substitution (backward: outer loop reversed,
 * P:202-205), one right-hand-side column at a time, row-major n x nrhs
 * (element (i, r) at i*nrhs + r, reading Q20).  For each row the running value
 * starts at f(i) and subtracts a(k)*x(ja(k)) term by term in storage order
 * (two roundings each), then divides by d(i) (reading Q7) unless UNIT.
 * x may alias b.  Returns the oracle_select status.
 */
int oracle_solve_f64(int32_t n, const int32_t *rowptr, const int32_t *colidx, const double *vals,
                     int uplo, int diag, int32_t nrhs, const double *b, double *x) {
    if (nrhs < 1) return OR_INVALID_VALUE;
    int32_t *diagk = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!diagk) return OR_ALLOC;
    int st = oracle_select(n, rowptr, colidx, vals, uplo, diag, NULL, diagk, NULL, NULL, NULL, NULL);
    if (st != OR_SUCCESS) { free(diagk); return st; }
    for (int32_t r = 0; r < nrhs; ++r) {
        for (int32_t t = 0; t < n; ++t) {
            int32_t i = (uplo == OR_LOWER) ? t : n - 1 - t;
            double s = b[(int64_t)i * nrhs + r];
            for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                int32_t j = colidx[k];
                if (in_triangle(i, j, uplo)) {
                    double p = vals[k] * x[(int64_t)j * nrhs + r];
                    s = s - p;
                }
            }
            x[(int64_t)i * nrhs + r] = (diag == OR_UNIT) ? s : s / vals[diagk[i]];
        }
    }
    free(diagk);
    return OR_SUCCESS;
}

/*
 * Column-wise sweep (Section "Column-wise SpTrSv"): x := f, then
 * for i = 1..n (upper: n..1) x(i) := x(i)/d(i) and every entry b(j) of
 * column i updates x(jb(j)) := x(jb(j)) - b(j)*x(i).  The CSC (ib, jb, b) of
 * the referenced strict triangle is built here by counting, entries of a
 * column in increasing row order.  The reference for the column-wise GPU
 * solves (SLFC / LEVC); same result as O-5 up to rounding order.
 */
int oracle_solve_col_f64(int32_t n, const int32_t *rowptr, const int32_t *colidx, const double *vals,
                         int uplo, int diag, const double *f, double *x) {
    int32_t *diagk = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *ib = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    if (!diagk || !ib) { free(diagk); free(ib); return OR_ALLOC; }
    int st = oracle_select(n, rowptr, colidx, vals, uplo, diag, NULL, diagk, NULL, NULL, NULL, NULL);
    if (st != OR_SUCCESS) { free(diagk); free(ib); return st; }
    for (int32_t r = 0; r < n; ++r)                       /* column counts */
        for (int32_t k = rowptr[r]; k < rowptr[r + 1]; ++k)
            if (in_triangle(r, colidx[k], uplo)) ib[colidx[k] + 1]++;
    for (int32_t i = 0; i < n; ++i) ib[i + 1] += ib[i];
    int32_t nnz = ib[n];
    int32_t *jb = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1));
    double *bv = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    int32_t *fill = (int32_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int32_t));
    if (!jb || !bv || !fill) { free(diagk); free(ib); free(jb); free(bv); free(fill); return OR_ALLOC; }
    for (int32_t r = 0; r < n; ++r)                       /* rows ascending: column entries by row */
        for (int32_t k = rowptr[r]; k < rowptr[r + 1]; ++k) {
            int32_t c = colidx[k];
            if (in_triangle(r, c, uplo)) {
                int32_t q = ib[c] + fill[c]++;
                jb[q] = r;
                bv[q] = vals[k];
            }
        }
    for (int32_t i = 0; i < n; ++i) x[i] = f[i];          /* x := f */
    for (int32_t t = 0; t < n; ++t) {
        int32_t i = (uplo == OR_LOWER) ? t : n - 1 - t;
        if (diag != OR_UNIT) x[i] = x[i] / vals[diagk[i]];
        for (int32_t j = ib[i]; j < ib[i + 1]; ++j) {
            double p = bv[j] * x[i];
            x[jb[j]] = x[jb[j]] - p;
        }
    }
    free(diagk); free(ib); free(jb); free(bv); free(fill);
    return OR_SUCCESS;
}

/* O-5 in single precision: float values, float accumulation (reading Q21). */
int oracle_solve_f32(int32_t n, const int32_t *rowptr, const int32_t *colidx, const float *vals,
                     int uplo, int diag, int32_t nrhs, const float *b, float *x) {
    if (nrhs < 1) return OR_INVALID_VALUE;
    if (n < 0) return OR_INVALID_VALUE;
    /* validation needs double values only for the zero test; build them */
    int64_t nnz = (n > 0 && rowptr) ? rowptr[n] : 0;
    double *dv = (double *)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
    int32_t *diagk = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!dv || !diagk) { free(dv); free(diagk); return OR_ALLOC; }
    for (int64_t k = 0; k < nnz && vals; ++k) dv[k] = (double)vals[k];
    int st = oracle_select(n, rowptr, colidx, vals ? dv : NULL, uplo, diag, NULL, diagk, NULL, NULL,
                           NULL, NULL);
    free(dv);
    if (st != OR_SUCCESS) { free(diagk); return st; }
    for (int32_t r = 0; r < nrhs; ++r) {
        for (int32_t t = 0; t < n; ++t) {
            int32_t i = (uplo == OR_LOWER) ? t : n - 1 - t;
            float s = b[(int64_t)i * nrhs + r];
            for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                int32_t j = colidx[k];
                if (in_triangle(i, j, uplo)) {
                    float p = vals[k] * x[(int64_t)j * nrhs + r];
                    s = s - p;
                }
            }
            x[(int64_t)i * nrhs + r] = (diag == OR_UNIT) ? s : s / vals[diagk[i]];
        }
    }
    free(diagk);
    return OR_SUCCESS;
}

/*
 * A18.  Kahn's algorithm by rounds, written sequentially: the
 * roots (dp == 0) form level 0 (FIND_LEVEL0); each round removes
 * the current level's vertices and their outgoing edges, and the vertices
 * whose counter reaches zero form the next level (FIND_LEVEL).
 * Bookkeeping follows reading Q9: level l = jlev[ilev[l] .. ilev[l+1]).
 * Within a round, vertices are emitted in the order the decrements reach
 * zero when the level is scanned in order -- the paper's atomic order is
 * nondeterministic, so only the SETS per level are compared.
 * lev_out[i] receives the round of vertex i.  Returns nlev, or -1 on a cycle
 * (impossible for triangular input) / allocation failure.
 */
int32_t oracle_kahn(int32_t n, const int32_t *rowptr, const int32_t *colidx, int uplo,
                    int32_t *ilev, int32_t *jlev, int32_t *lev_out) {
    if (n == 0) { ilev[0] = 0; return 0; }
    int32_t *dp = (int32_t *)calloc((size_t)n, sizeof(int32_t));
    int32_t *cp = (int32_t *)calloc((size_t)n + 1, sizeof(int32_t));
    if (!dp || !cp) { free(dp); free(cp); return -1; }
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (in_triangle(i, colidx[k], uplo)) { dp[i]++; cp[colidx[k] + 1]++; }
    for (int32_t j = 0; j < n; ++j) cp[j + 1] += cp[j];
    int32_t *out = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cp[n] > 0 ? cp[n] : 1));
    int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!out || !fill) { free(dp); free(cp); free(out); free(fill); return -1; }
    memcpy(fill, cp, sizeof(int32_t) * (size_t)n);
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (in_triangle(i, colidx[k], uplo)) out[fill[colidx[k]]++] = i;   /* edge j -> i */
    int32_t last = 0;
    for (int32_t i = 0; i < n; ++i) if (dp[i] == 0) jlev[last++] = i;     /* FIND_LEVEL0 */
    int32_t nlev = 0, first = 0;
    ilev[0] = 0;
    while (first < last) {
        int32_t end = last;
        for (int32_t t = first; t < end; ++t) lev_out[jlev[t]] = nlev;
        for (int32_t t = first; t < end; ++t) {                             /* FIND_LEVEL */
            int32_t j = jlev[t];
            for (int32_t k = cp[j]; k < cp[j + 1]; ++k)
                if (--dp[out[k]] == 0) jlev[last++] = out[k];
        }
        first = end;
        ilev[++nlev] = first;
    }
    free(dp); free(cp); free(out); free(fill);
    return (last == n) ? nlev : -1;
}

/*
 * Pin helper (not the solve): the componentwise backward error of a computed
 * x for the selected triangular system, in long double:
 *   max_i |b_i - (T x)_i| / (|T| |x|)_i        (Higham, Thm 8.5, with the
 * diagonal taken as 1 for UNIT).  Rows with a zero denominator and a zero
 * residual contribute 0.  Returns the max over all rows and columns.
 */
double oracle_backward_error(int32_t n, const int32_t *rowptr, const int32_t *colidx,
                             const double *vals, int uplo, int diag, int32_t nrhs,
                             const double *b, const double *x) {
    long double worst = 0.0L;
    for (int32_t r = 0; r < nrhs; ++r)
        for (int32_t i = 0; i < n; ++i) {
            long double xi = (long double)x[(int64_t)i * nrhs + r];
            long double acc = 0.0L, mag = 0.0L;
            int have_diag = 0;
            for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                int32_t j = colidx[k];
                long double xj = (long double)x[(int64_t)j * nrhs + r];
                if (j == i) {
                    if (diag == OR_NON_UNIT) {
                        acc += (long double)vals[k] * xi;
                        mag += fabsl((long double)vals[k] * xi);
                        have_diag = 1;
                    }
                } else if (in_triangle(i, j, uplo)) {
                    acc += (long double)vals[k] * xj;
                    mag += fabsl((long double)vals[k] * xj);
                }
            }
            if (diag == OR_UNIT) { acc += xi; mag += fabsl(xi); have_diag = 1; }
            (void)have_diag;
            long double res = fabsl((long double)b[(int64_t)i * nrhs + r] - acc);
            long double ratio = (mag > 0.0L) ? res / mag : (res > 0.0L ? INFINITY : 0.0L);
            if (ratio > worst) worst = ratio;
        }
    return (double)worst;
}

/* b = T x in long double, rounded once to double (constructing b from x_true). */
void oracle_matvec_ld(int32_t n, const int32_t *rowptr, const int32_t *colidx, const double *vals,
                      int uplo, int diag, int32_t nrhs, const double *x, double *b) {
    for (int32_t r = 0; r < nrhs; ++r)
        for (int32_t i = 0; i < n; ++i) {
            long double acc = 0.0L;
            for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
                int32_t j = colidx[k];
                if (j == i) {
                    if (diag == OR_NON_UNIT) acc += (long double)vals[k] * (long double)x[(int64_t)i * nrhs + r];
                } else if (in_triangle(i, j, uplo)) {
                    acc += (long double)vals[k] * (long double)x[(int64_t)j * nrhs + r];
                }
            }
            if (diag == OR_UNIT) acc += (long double)x[(int64_t)i * nrhs + r];
            b[(int64_t)i * nrhs + r] = (double)acc;
        }
}
