/*
 * workloads/gen.c -- seeded synthetic input generators shared by tests, bench
 * and smoke.  This module holds NONE of the triangular-solve arithmetic: it
 * only builds matrices (CSR, 0-based, strictly increasing columns per row)
 * shaped like the paper's workloads.  Neither the oracle nor the CUDA library
 * includes or links this file; the Python side passes its arrays to both.
 *
 * Recipes:
 *   - Laplacians (§5.1): lexicographic grid ordering with
 *     x fastest (reading Q17), off-diagonal -1, a Dirichlet constant diagonal
 *     (reading Q16), 5/9-point in 2-D and 7/27-point in 3-D (Moore
 *     neighbourhood for 9/27, reading Q18).
 *   - ILU(0) by the IKJ variant (Saad, "Iterative Methods", Alg. 10.4) on a
 *     Laplacian: the factors keep A's pattern.
 *   - cfg4 power-law generator with explicit levels.
 *
 * Build: gcc -O2 -shared -fPIC -o libworkloads.so gen.c
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ---------------------------------------------------------------- RNG ---- */
/* splitmix64: a counter-based generator, enough for seeded synthetic inputs */
static uint64_t sm64_next(uint64_t *s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* uniform in [0,1) with 53 random bits */
static double sm64_unif(uint64_t *s) {
    return (double)(sm64_next(s) >> 11) * (1.0 / 9007199254740992.0);
}

/* ---------------------------------------------------------- stencils ---- */
/*
 * gen_stencil: matrix of order nx*ny*nz for a 2-D (nz==1) or 3-D stencil.
 *   stencil: 5 or 9 (2-D; requires nz==1), 7 or 27 (3-D)
 *   part:    0 = full A, 1 = lower triangle incl. diagonal (L+D),
 *            2 = upper triangle incl. diagonal (U+D)
 *   dval:    the diagonal value (Dirichlet: 4/8/6/26; integer pins use 8)
 *   offval:  the off-diagonal value (-1)
 * Two-pass: call with rowptr only (colidx == NULL) to size, then again.
 * Returns nnz, or -1 on bad arguments.
 */
int64_t gen_stencil(int32_t nx, int32_t ny, int32_t nz, int32_t stencil, int32_t part,
                    double dval, double offval,
                    int32_t *rowptr, int32_t *colidx, double *vals) {
    if (nx < 1 || ny < 1 || nz < 1) return -1;
    int moore;
    if (stencil == 5 || stencil == 9) { if (nz != 1) return -1; moore = (stencil == 9); }
    else if (stencil == 7 || stencil == 27) { moore = (stencil == 27); }
    else return -1;
    int dzlo = (nz == 1) ? 0 : -1, dzhi = (nz == 1) ? 0 : 1;
    int64_t n = (int64_t)nx * ny * nz;
    if (n > INT32_MAX) return -1;
    int64_t nnz = 0;
    if (rowptr) rowptr[0] = 0;
    for (int32_t z = 0; z < nz; ++z)
    for (int32_t y = 0; y < ny; ++y)
    for (int32_t x = 0; x < nx; ++x) {
        int64_t i = x + (int64_t)nx * (y + (int64_t)ny * z);
        /* dz, dy, dx ascending => column index ascending (x fastest) */
        for (int dz = dzlo; dz <= dzhi; ++dz)
        for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
            int nzero = (dx != 0) + (dy != 0) + (dz != 0);
            if (!moore && nzero > 1) continue;
            int32_t xx = x + dx, yy = y + dy, zz = z + dz;
            if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz) continue;
            int64_t j = xx + (int64_t)nx * (yy + (int64_t)ny * zz);
            if (part == 1 && j > i) continue;
            if (part == 2 && j < i) continue;
            if (colidx) {
                colidx[nnz] = (int32_t)j;
                vals[nnz] = (j == i) ? dval : offval;
            }
            ++nnz;
        }
        if (rowptr) rowptr[i + 1] = (int32_t)nnz;
    }
    return nnz;
}

/* ------------------------------------------------------------- ILU(0) ---- */
/*
 * In-place ILU(0), IKJ variant (Saad Alg. 10.4) on a CSR matrix with sorted
 * columns and a stored nonzero diagonal in every row.  On exit the strict
 * lower part holds L (unit diagonal implied) and the diagonal + strict upper
 * part hold U.  Returns 0, or -(i+1) if row i has no diagonal / zero pivot.
 */
int32_t gen_ilu0(int32_t n, const int32_t *rowptr, const int32_t *colidx, double *vals) {
    int32_t *diagpos = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *where = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    if (!diagpos || !where) { free(diagpos); free(where); return -1; }
    for (int32_t i = 0; i < n; ++i) { where[i] = -1; diagpos[i] = -1; }
    for (int32_t i = 0; i < n; ++i)
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
            if (colidx[k] == i) diagpos[i] = k;
    int32_t rc = 0;
    for (int32_t i = 0; i < n && rc == 0; ++i) {
        if (diagpos[i] < 0) { rc = -(i + 1); break; }
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) where[colidx[k]] = k;
        for (int32_t kk = rowptr[i]; kk < rowptr[i + 1]; ++kk) {
            int32_t k = colidx[kk];
            if (k >= i) break;
            double piv = vals[diagpos[k]];
            if (piv == 0.0) { rc = -(k + 1); break; }
            vals[kk] /= piv;                       /* a_ik := a_ik / a_kk */
            double lik = vals[kk];
            for (int32_t jj = diagpos[k] + 1; jj < rowptr[k + 1]; ++jj) {
                int32_t w = where[colidx[jj]];     /* (i, j) in pattern? */
                if (w >= 0) vals[w] -= lik * vals[jj];
            }
        }
        for (int32_t k = rowptr[i]; k < rowptr[i + 1]; ++k) where[colidx[k]] = -1;
        if (rc == 0 && vals[diagpos[i]] == 0.0) rc = -(i + 1);
    }
    free(diagpos); free(where);
    return rc;
}

/* ---------------------------------------------------- power-law (cfg4) ---- */
/*
 * gen_powerlaw: lower triangular L+D of order n with explicit levels
 * (SURVEY.md §8d, cfg4).  Row i gets a base level floor(i*L/n); 30% of rows
 * step down by a Geometric(0.5) count (>=1) of levels.  A row of level l>0
 * takes one "critical" dependency among the 64 most recent rows of level
 * l-1 (so its level is exactly l), plus further dependencies at levels < l
 * found by a locality-biased search (geometric distance, mean `locality`).
 * Strict row length ~ floor(4*U^(-1/1.5)) (Pareto), capped at
 * min(maxlen, i) and >= 1 for rows of level > 0.  Off-diagonals U[-1,1),
 * diagonal 1 + 2*sum|a_ij| (strictly diagonally dominant).
 *
 * Outputs are malloc'ed by the generator (sizes unknown in advance) and must
 * be released with gen_free.  lev_out[i] is the intended (0-based) level.
 * Returns nnz or -1.
 */
void gen_free(void *p) { free(p); }

int64_t gen_powerlaw(int32_t n, int32_t L, int32_t maxlen, int32_t locality, uint64_t seed,
                     int32_t **rowptr_out, int32_t **colidx_out, double **vals_out,
                     int32_t **lev_out) {
    if (n < 1 || L < 1 || L > n || maxlen < 1 || locality < 1) return -1;
    const int R = 64;                               /* ring of recent rows per level */
    int32_t *lev = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    int32_t *ring = (int32_t *)malloc(sizeof(int32_t) * (size_t)L * R);
    int32_t *ringcnt = (int32_t *)calloc((size_t)L, sizeof(int32_t));
    int32_t *rowptr = (int32_t *)malloc(sizeof(int32_t) * ((size_t)n + 1));
    size_t cap = (size_t)n * 12 + 1024, nnz = 0;
    int32_t *colidx = (int32_t *)malloc(sizeof(int32_t) * cap);
    double *vals = (double *)malloc(sizeof(double) * cap);
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * ((size_t)maxlen + 1));
    if (!lev || !ring || !ringcnt || !rowptr || !colidx || !vals || !tmp) goto fail;
    uint64_t s = seed * 0x2545F4914F6CDD1DULL + 0x1234567ULL;
    double ploc = 1.0 / (double)locality;            /* geometric success prob. */
    rowptr[0] = 0;
    for (int32_t i = 0; i < n; ++i) {
        int32_t l = (int32_t)(((int64_t)i * L) / n);
        if (sm64_unif(&s) < 0.3) {                     /* jitter down */
            int32_t g = 1;
            while (sm64_unif(&s) < 0.5) ++g;
            l = (l - g > 0) ? l - g : 0;
        }
        while (l > 0 && ringcnt[l - 1] == 0) --l;        /* need a level l-1 row */
        int32_t len = 0;
        if (l > 0) {
            double u = sm64_unif(&s);
            if (u < 1e-300) u = 1e-300;
            double want = floor(4.0 * pow(u, -1.0 / 1.5));
            int32_t cap_i = (maxlen < i) ? maxlen : i;
            len = (want > (double)cap_i) ? cap_i : (int32_t)want;
            if (len < 1) len = 1;
            int32_t m = ringcnt[l - 1] < R ? ringcnt[l - 1] : R;
            int32_t pick = (int32_t)(sm64_next(&s) % (uint64_t)m);
            tmp[0] = ring[(size_t)(l - 1) * R + pick];   /* critical dependency */
            int32_t got = 1, tries = 0;
            while (got < len && tries < 8 * len) {
                ++tries;
                double uu = sm64_unif(&s);
                if (uu < 1e-300) uu = 1e-300;
                int64_t d = 1 + (int64_t)floor(log(uu) / log(1.0 - ploc));
                int64_t j = (int64_t)i - d;
                if (j < 0) j = (int64_t)(sm64_next(&s) % (uint64_t)i);
                if (lev[j] >= l) continue;
                tmp[got++] = (int32_t)j;
            }
            /* sort + unique (insertion sort is fine: rows are short on average) */
            for (int32_t a = 1; a < got; ++a) {
                int32_t v = tmp[a], b = a - 1;
                while (b >= 0 && tmp[b] > v) { tmp[b + 1] = tmp[b]; --b; }
                tmp[b + 1] = v;
            }
            int32_t u2 = 0;
            for (int32_t a = 0; a < got; ++a)
                if (u2 == 0 || tmp[u2 - 1] != tmp[a]) tmp[u2++] = tmp[a];
            len = u2;
        }
        if (nnz + (size_t)len + 1 > cap) {
            cap = cap * 3 / 2 + (size_t)len + 1;
            int32_t *c2 = (int32_t *)realloc(colidx, sizeof(int32_t) * cap);
            if (!c2) goto fail;
            colidx = c2;
            double *v2 = (double *)realloc(vals, sizeof(double) * cap);
            if (!v2) goto fail;
            vals = v2;
        }
        double asum = 0.0;
        for (int32_t a = 0; a < len; ++a) {
            double v = 2.0 * sm64_unif(&s) - 1.0;
            colidx[nnz] = tmp[a];
            vals[nnz] = v;
            asum += fabs(v);
            ++nnz;
        }
        colidx[nnz] = i;
        vals[nnz] = 1.0 + 2.0 * asum;
        ++nnz;
        rowptr[i + 1] = (int32_t)nnz;
        lev[i] = l;
        ring[(size_t)l * R + (ringcnt[l] % R)] = i;
        ringcnt[l]++;
    }
    free(ring); free(ringcnt); free(tmp);
    *rowptr_out = rowptr; *colidx_out = colidx; *vals_out = vals; *lev_out = lev;
    return (int64_t)nnz;
fail:
    free(lev); free(ring); free(ringcnt); free(rowptr); free(colidx); free(vals); free(tmp);
    return -1;
}
