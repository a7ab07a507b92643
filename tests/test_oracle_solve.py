"""Pins for the oracle's substitution (O-5), pair solve (O-6), validation (O-1)
and the ILU(0) generator -- CPU only.

Pins: dense triangular solves (LAPACK trtrs via scipy) on tiny systems, exact
integer solutions, the componentwise backward-error bound (Higham, Accuracy
and Stability, Thm 8.5), SPEC's worked examples, and the Eq. (3) pair solve.
"""
import numpy as np
import pytest
import scipy.linalg

import oracle
import workloads
from workloads import CSR

from test_oracle_levels import chain, random_triangular


def dense_triangle(m, uplo, diag):
    a = m.to_dense()
    t = np.tril(a, -1) if uplo == "lower" else np.triu(a, 1)
    d = np.ones(m.n) if diag == "unit" else np.diag(a)
    return t + np.diag(d)


@pytest.mark.parametrize("seed", range(30))
def test_solve_matches_dense_trtrs(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 200))
    uplo = ("lower", "upper")[seed % 2]
    diag = ("non_unit", "unit")[(seed // 2) % 2]
    m = random_triangular(n, float(rng.uniform(0.01, 0.2)), seed, uplo, extra_other=0.05)
    if diag == "unit":   # keep unit systems well conditioned
        m.vals[m.colidx != np.repeat(np.arange(n), np.diff(m.rowptr))] *= 0.3 / max(1, n ** 0.5)
    nrhs = int(rng.integers(1, 4))
    b = rng.uniform(-1, 1, size=(n, nrhs))
    x = oracle.solve(m, b, uplo, diag)
    ref = scipy.linalg.solve_triangular(dense_triangle(m, uplo, diag), b, lower=(uplo == "lower"))
    err = np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300)
    assert err <= 1e-12, err


def test_solve_columns_are_independent():
    m = random_triangular(80, 0.1, 7, "lower")
    b = np.random.default_rng(1).uniform(-1, 1, size=(80, 5))
    x = oracle.solve(m, b)
    for r in range(5):
        assert np.array_equal(x[:, r], oracle.solve(m, b[:, r]))


def test_solve_in_place_alias_semantics():
    # x := f, then the sweep: the oracle's result does not depend
    # on whether b and x share storage -- checked by solving twice
    m = random_triangular(40, 0.2, 3, "upper")
    b = np.random.default_rng(2).uniform(-1, 1, size=40)
    assert np.array_equal(oracle.solve(m, b, "upper"), oracle.solve(m, b.copy(), "upper"))


# ------------------------------------------------------------ exact pins
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", ["cfg1", "7pt_d8", "7pt_upper_d8"])
def test_integer_exact_solution(case, dtype):
    # integer T with a power-of-two diagonal and x_true in {+-1..+-4}: b = T x
    # is exact and every substitution step is exact, so x == x_true bit for bit
    if case == "cfg1":
        m, uplo = workloads.stencil((32, 32), 5, "lower"), "lower"          # d = 4
    elif case == "7pt_d8":
        m, uplo = workloads.stencil((12, 10, 9), 7, "lower", diag=8.0), "lower"
    else:
        m, uplo = workloads.stencil((12, 10, 9), 7, "upper", diag=8.0), "upper"
    xt = workloads.integer_xtrue(m.n, 2, seed=101)
    b = oracle.matvec(m, xt, uplo)
    assert np.array_equal(b, np.round(b))
    x = oracle.solve(m, b.astype(dtype), uplo, dtype=dtype)
    assert np.array_equal(x.astype(np.float64), xt)


def test_spec_chain_example():
    # lower chain, diag 1, subdiagonal 1, f = [1,1,1] -> x = [1,0,1]
    m = chain(3, sub=1.0, d=1.0)
    assert list(oracle.solve(m, np.ones(3))) == [1.0, 0.0, 1.0]


def test_spec_diagonal_example():
    # diag = [2,2], f = [4,6] -> x = [2,3]  (x = f / d)
    m = CSR(2, np.array([0, 1, 2], dtype=np.int32), np.array([0, 1], dtype=np.int32),
            np.array([2.0, 2.0]))
    for uplo in ("lower", "upper"):
        assert list(oracle.solve(m, np.array([4.0, 6.0]), uplo)) == [2.0, 3.0]


def test_spec_pair_2I():
    # A = 2I, x = [2,4] -> y = (U+D)^-1 (L+D)^-1 x = [0.5, 1]
    m = CSR(2, np.array([0, 1, 2], dtype=np.int32), np.array([0, 1], dtype=np.int32),
            np.array([2.0, 2.0]))
    z = oracle.solve(m, np.array([2.0, 4.0]), "lower")
    assert list(oracle.solve(m, z, "upper")) == [0.5, 1.0]


def test_eq3_pair_solve_recovers_ones():
    # S:283 / Eq. (3): on the 5-point 32x32 operator with
    # x = (L+D)(U+D) 1, y = (U+D)^-1 (L+D)^-1 x = 1 within 1e-12
    a = workloads.stencil((32, 32), 5, "full")
    ones = np.ones(a.n)
    x = oracle.matvec(a, oracle.matvec(a, ones, "upper"), "lower")
    y = oracle.solve(a, oracle.solve(a, x, "lower"), "upper")
    assert np.abs(y - 1).max() <= 1e-12


# ------------------------------------------------------- error bounds
def gamma(k, u=2.0 ** -53):
    return k * u / (1 - k * u)


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_backward_error_bound(cfg):
    # |b - T x^| <= gamma_{k+2} |T||x^| componentwise (Higham Thm 8.5), k = max deps
    m, p = workloads.config(cfg, scale=0.125 if cfg != 1 else 1.0)
    b = workloads.rhs(m.n, 1, seed=p["seed"])
    x = oracle.solve(m, b, "lower")
    k = int(oracle.select(m)["dp"].max())
    be = oracle.backward_error(m, b, x, "lower")
    assert be <= gamma(k + 2), (be, gamma(k + 2))


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_forward_error_vs_xtrue(cfg):
    # diagonally dominant generated factors: ||x - x_true|| / ||x_true|| <= 1e-10
    m, _ = workloads.config(cfg, scale=0.125 if cfg != 1 else 1.0)
    xt = workloads.rhs(m.n, 1, seed=77)
    b = oracle.matvec(m, xt)
    x = oracle.solve(m, b)
    assert np.abs(x - xt).max() / np.abs(xt).max() <= 1e-10


def test_fp32_forward_error():
    m, _ = workloads.config(2, scale=0.125)
    xt = workloads.rhs(m.n, 1, seed=78)
    b = oracle.matvec(m, xt)
    x = oracle.solve(m.astype(np.float32), b.astype(np.float32), dtype=np.float32)
    assert np.abs(x - xt).max() / np.abs(xt).max() <= 1e-4


# ------------------------------------------------------------ ILU(0) / cfg3
def test_ilu0_generator_reproduces_a_on_pattern():
    # (L U)_ij = A_ij for (i,j) in pattern(A) (the defining property of ILU(0))
    a = workloads.stencil((4, 3, 3), 27, "full")
    f = workloads.ilu0(a)
    F = f.to_dense()
    L = np.tril(F, -1) + np.eye(a.n)
    U = np.triu(F)
    A = a.to_dense()
    mask = A != 0
    assert np.abs((L @ U - A)[mask]).max() <= 1e-12
    assert np.diag(U).min() > 0
    # symmetric A: U = diag(U) L^T (IC(0) up to scaling, reading Q19)
    assert np.abs(U - np.diag(np.diag(U)) @ L.T).max() <= 1e-12


def test_pair_solve_ilu0_against_dense():
    a = workloads.stencil((5, 4, 3), 27, "full")
    f = workloads.ilu0(a)
    F = f.to_dense()
    L = np.tril(F, -1) + np.eye(a.n)
    U = np.triu(F)
    b = workloads.rhs(a.n, 2, seed=3)
    y = oracle.pair_solve(f, b)
    ref = scipy.linalg.solve_triangular(U, scipy.linalg.solve_triangular(L, b, lower=True), lower=False)
    assert np.abs(y - ref).max() / np.abs(ref).max() <= 1e-12
    sel = oracle.select(f, "lower", "unit")
    # unit lower: the stored diagonal and the strict upper part are not referenced
    assert sel["ignored"] == f.nnz - sel["nnz_used"]


# ------------------------------------------------------------- O-1 status
def csr(n, rows, vals=None):
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    colidx = np.array([c for r in rows for c in r], dtype=np.int32)
    v = np.ones(colidx.size) if vals is None else np.array(vals, dtype=np.float64)
    return CSR(n, rowptr, colidx, v)


def test_status_invalid_matrix_cases():
    ok = csr(3, [[0], [0, 1], [1, 2]])
    assert oracle.select(ok)["status"] == "SUCCESS"
    bad_order = csr(3, [[0], [1, 0], [1, 2]])
    s = oracle.select(bad_order)
    assert s["status"] == "INVALID_MATRIX" and s["bad_row"] == 1
    dup = csr(3, [[0], [0, 1], [2, 2]])
    s = oracle.select(dup)
    assert s["status"] == "INVALID_MATRIX" and s["bad_row"] == 2
    oob = csr(3, [[0], [0, 1], [1, 3]])
    s = oracle.select(oob)
    assert s["status"] == "INVALID_MATRIX" and s["bad_row"] == 2
    neg = csr(3, [[0], [-1, 1], [2]])
    assert oracle.select(neg)["bad_row"] == 1
    m = csr(3, [[0], [0, 1], [1, 2]])
    m.rowptr = m.rowptr.copy()
    m.rowptr[0] = 1
    s = oracle.select(m)
    assert s["status"] == "INVALID_MATRIX" and s["bad_row"] == 0
    m2 = csr(3, [[0], [0, 1], [1, 2]])
    m2.rowptr = np.array([0, 1, 0, 5], dtype=np.int32)      # decreasing at row 1
    assert oracle.select(m2)["bad_row"] == 1


def test_status_zero_pivot_and_unit():
    missing = csr(3, [[0], [0], [1, 2]])                      # row 1 has no diagonal
    s = oracle.select(missing)
    assert s["status"] == "ZERO_PIVOT" and s["zero_pivot_row"] == 1
    s = oracle.select(missing, "lower", "unit")
    assert s["status"] == "SUCCESS"
    zero = csr(3, [[0], [0, 1], [1, 2]], vals=[1, 1, 1, 1, 0.0])
    s = oracle.select(zero)
    assert s["status"] == "ZERO_PIVOT" and s["zero_pivot_row"] == 2
    # malformed takes precedence over zero pivot
    both = csr(3, [[0], [0], [2, 1]])
    assert oracle.select(both)["status"] == "INVALID_MATRIX"


def test_ignored_entries_counted():
    a = workloads.stencil((6, 5), 5, "full")
    s = oracle.select(a, "lower")
    lo = workloads.stencil((6, 5), 5, "lower")
    assert s["nnz_used"] == lo.nnz - a.n
    assert s["ignored"] == a.nnz - lo.nnz
    # solving with the full A and uplo=lower equals solving with L+D
    b = workloads.rhs(a.n, 1, 5)
    assert np.array_equal(oracle.solve(a, b, "lower"), oracle.solve(lo, b, "lower"))


# ------------------------------------------------ column-wise sweep, reference of SLFC / LEVC
@pytest.mark.parametrize("seed", range(20))
def test_solve_col_matches_dense_trtrs(seed):
    """Pinned to LAPACK trtrs on the dense triangle (not to the row oracle)."""
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(1, 200))
    uplo = ("lower", "upper")[seed % 2]
    diag = ("non_unit", "unit")[(seed // 2) % 2]
    m = random_triangular(n, float(rng.uniform(0.01, 0.2)), seed, uplo, extra_other=0.05)
    if diag == "unit":
        m.vals[m.colidx != np.repeat(np.arange(n), np.diff(m.rowptr))] *= 0.3 / max(1, n ** 0.5)
    b = rng.uniform(-1, 1, size=n)
    x = oracle.solve_col(m, b, uplo, diag)
    ref = scipy.linalg.solve_triangular(dense_triangle(m, uplo, diag), b, lower=(uplo == "lower"))
    assert np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300) <= 1e-12


@pytest.mark.parametrize("uplo", ["lower", "upper"])
def test_solve_col_integer_exact(uplo):
    m = workloads.stencil((12, 10, 9), 7, uplo, diag=8.0)
    xt = workloads.integer_xtrue(m.n, 1, seed=103)[:, 0]
    b = oracle.matvec(m, xt, uplo)
    assert np.array_equal(oracle.solve_col(m, b, uplo), xt)


def test_solve_col_hand_example():
    """3x3 lower, by hand: L = [[2,0,0],[1,4,0],[3,-2,8]], f = [2,9,17]
    column 1: x1 = 2/2 = 1; x2 = 9-1 = 8, x3 = 17-3 = 14
    column 2: x2 = 8/4 = 2; x3 = 14+4 = 18;  column 3: x3 = 18/8 = 2.25"""
    m = CSR(3, np.array([0, 1, 3, 6], dtype=np.int32), np.array([0, 0, 1, 0, 1, 2], dtype=np.int32),
            np.array([2.0, 1.0, 4.0, 3.0, -2.0, 8.0]))
    assert np.array_equal(oracle.solve_col(m, np.array([2.0, 9.0, 17.0])), np.array([1.0, 2.0, 2.25]))
    # unit diagonal ignores the stored 2, 4, 8; the upper part is not referenced
    assert np.array_equal(oracle.solve_col(m, np.array([2.0, 9.0, 17.0]), "lower", "unit"),
                          np.array([2.0, 7.0, 25.0]))


def test_solve_col_zero_pivot_status():
    m = CSR(2, np.array([0, 1, 2], dtype=np.int32), np.array([0, 0], dtype=np.int32), np.array([1.0, 1.0]))
    with pytest.raises(oracle.OracleError):
        oracle.solve_col(m, np.ones(2))


# ---- two-sided pins of the backward-error helper (it was only
# ever asserted from above).  Reference: the definition evaluated densely in
# numpy long double, max_i |b - T x|_i / (|T| |x|)_i (Higham, Thm 8.5).
def _dense_backward_error(m, b, x, uplo, diag):
    n = m.n
    T = np.zeros((n, n), dtype=np.longdouble)
    for i in range(n):
        for k in range(m.rowptr[i], m.rowptr[i + 1]):
            j = int(m.colidx[k])
            if (j < i and uplo == "lower") or (j > i and uplo == "upper"):
                T[i, j] = m.vals[k]
            elif j == i and diag == "non_unit":
                T[i, j] = m.vals[k]
    if diag == "unit":
        T[np.arange(n), np.arange(n)] = 1
    xl = np.asarray(x, dtype=np.longdouble).reshape(n, -1)
    bl = np.asarray(b, dtype=np.longdouble).reshape(n, -1)
    res = np.abs(bl - T @ xl)
    mag = np.abs(T) @ np.abs(xl)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.where(mag > 0, res / np.where(mag > 0, mag, 1), np.where(res > 0, np.inf, 0))
    return float(ratio.max())


@pytest.mark.parametrize("uplo,diag", [("lower", "non_unit"), ("upper", "non_unit"), ("lower", "unit"),
                                       ("upper", "unit")])
def test_backward_error_two_sided(uplo, diag):
    # integer system: the exact x has backward error exactly 0
    m = workloads.stencil((9, 7, 5), 7, uplo, diag=8.0)
    xt = workloads.integer_xtrue(m.n, 1, seed=5)[:, 0]
    b = oracle.matvec(m, xt, uplo, diag)
    assert oracle.backward_error(m, b, xt, uplo, diag) == 0.0
    # one entry perturbed up / down, several entries of mixed sign: equals the
    # dense long-double definition (a dropped fabs, a dropped term or a
    # constant return fails one of these)
    rng = np.random.default_rng(3)
    for delta_idx, delta in ((m.n // 2, 1e-6), (m.n // 3, -3e-7), (0, 2e-5)):
        x = xt.astype(np.float64).copy()
        x[delta_idx] += delta
        be = oracle.backward_error(m, b, x, uplo, diag)
        ref = _dense_backward_error(m, b, x, uplo, diag)
        assert be > 0 and abs(be - ref) <= 1e-12 * ref, (be, ref)
    x = xt + rng.uniform(-1e-4, 1e-4, size=m.n)
    be = oracle.backward_error(m, b, x, uplo, diag)
    ref = _dense_backward_error(m, b, x, uplo, diag)
    assert abs(be - ref) <= 1e-12 * ref, (be, ref)
    # multi-column: the max over columns
    X = np.stack([xt.astype(np.float64), x], axis=1)
    B = np.stack([b, b], axis=1)
    assert abs(oracle.backward_error(m, B, X, uplo, diag) - ref) <= 1e-12 * ref


def test_backward_error_zero_denominator_and_negative_residual():
    # x = 0: |T||x| = 0 in every row; row 0 has a zero residual (contributes 0),
    # row 1 a nonzero one -> infinite backward error
    m = csr(2, [[0], [0, 1]], vals=[2.0, 1.0, 4.0])
    assert oracle.backward_error(m, np.array([0.0, 3.0]), np.array([0.0, 0.0])) > 1e300
    assert oracle.backward_error(m, np.array([0.0, 0.0]), np.array([0.0, 0.0])) == 0.0
    # a residual of either sign counts by magnitude: b - T x = -0.5 in row 0
    be = oracle.backward_error(m, np.array([1.5, 1.0]), np.array([1.0, 0.0]))
    assert abs(be - 0.5 / 2.0) <= 1e-15
