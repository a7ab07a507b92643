"""Pins for the oracle's level analysis (O-2, O-3, O-4, A7, A18) -- CPU only.

Each pin comes from the paper or the mathematics, not from the oracle itself:
closed forms (P:319-323 and derived), Fig. 1's worked example,
the extremes, the row/column loop identity, brute-force
longest paths, and the power-law generator's levels-by-construction.
"""
import os
from math import comb

import numpy as np
import pytest

import oracle
import workloads
from workloads import CSR

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def grid_coords(dims):
    nx, ny, nz = (tuple(dims) + (1, 1))[:3]
    i = np.arange(nx * ny * nz)
    return i % nx, (i // nx) % ny, i // (nx * ny)


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("nx,ny", [(1, 1), (5, 5), (7, 3), (32, 32), (3, 11)])
def test_2d_5pt_levels_closed_form(nx, ny):
    # nlev = nx + ny - 1 for the lower part of the 5-point operator
    m = workloads.stencil((nx, ny), 5, "lower")
    lev, nlev = oracle.levels(m, "lower")
    x, y, _ = grid_coords((nx, ny))
    assert nlev == nx + ny - 1
    assert np.array_equal(lev, x + y)


@pytest.mark.parametrize("d", [(2, 2, 2), (5, 4, 3), (16, 16, 16), (3, 9, 2)])
def test_3d_7pt_levels_closed_form(d):
    # nlev = nx + ny + nz - 2 for the 7-point operator
    m = workloads.stencil(d, 7, "lower")
    lev, nlev = oracle.levels(m, "lower")
    x, y, z = grid_coords(d)
    assert nlev == sum(d) - 2
    assert np.array_equal(lev, x + y + z)
    # backward sweep: the upper part mirrors the grid
    mu = workloads.stencil(d, 7, "upper")
    levu, nlevu = oracle.levels(mu, "upper")
    assert nlevu == sum(d) - 2
    assert np.array_equal(levu, (d[0] - 1 - x) + (d[1] - 1 - y) + (d[2] - 1 - z))


@pytest.mark.parametrize("nx,ny", [(2, 2), (5, 5), (6, 3)])
def test_2d_9pt_levels_closed_form(nx, ny):
    # derived: the NE-SW diagonal neighbour (x+1, y-1) forces lev = x + 2y
    m = workloads.stencil((nx, ny), 9, "lower")
    lev, nlev = oracle.levels(m, "lower")
    x, y, _ = grid_coords((nx, ny))
    assert np.array_equal(lev, x + 2 * y)
    assert nlev == nx + 2 * ny - 2


@pytest.mark.parametrize("d", [(2, 2, 2), (4, 3, 3), (6, 6, 6)])
def test_3d_27pt_levels_closed_form(d):
    # derived: lev = x + 2y + 4z for the Moore neighbourhood (nx >= 2)
    m = workloads.stencil(d, 27, "lower")
    lev, nlev = oracle.levels(m, "lower")
    x, y, z = grid_coords(d)
    assert np.array_equal(lev, x + 2 * y + 4 * z)
    assert nlev == d[0] + 2 * d[1] + 4 * d[2] - 6


def test_3d_7pt_level_widths_inclusion_exclusion():
    # width of level m on an N^3 cube = #{x+y+z=m, 0<=x,y,z<N}:
    # C(m+2,2) - 3C(m-N+2,2) + 3C(m-2N+2,2) - C(m-3N+2,2); max 12288 at N=128
    N = 128
    def c2(k):
        return comb(k, 2) if k >= 2 else 0
    widths = [c2(m + 2) - 3 * c2(m - N + 2) + 3 * c2(m - 2 * N + 2) - c2(m - 3 * N + 2)
              for m in range(3 * N - 2)]
    m = workloads.stencil((N, N, N), 7, "lower")
    lev, nlev = oracle.levels(m, "lower")
    ilev, jlev = oracle.schedule(lev, nlev)
    assert nlev == 382
    assert np.array_equal(np.diff(ilev), widths)
    assert max(widths) == 12288


# --------------------------------------------------------------- Fig. 1 pin
def _read_fig1():
    levels, deps, nlev = {}, {}, None
    with open(os.path.join(GOLDEN, "fig1_5x5_levels.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("nlev"):
                nlev = int(line.split()[1])
            elif line.startswith("level"):
                head, nodes = line.split(":")
                levels[int(head.split()[1])] = [int(t) for t in nodes.split()]
            elif line.startswith("deps"):
                head, nodes = line.split(":")
                deps[int(head.split()[1])] = [int(t) for t in nodes.split()]
    return nlev, levels, deps


def test_fig1_worked_example():
    nlev_g, levels_g, deps_g = _read_fig1()
    m = workloads.stencil((5, 5), 5, "lower")
    lev, nlev = oracle.levels(m, "lower")
    assert nlev == nlev_g == 9
    ilev, jlev = oracle.schedule(lev, nlev)
    for L, nodes in levels_g.items():           # 1-based in the paper
        got = jlev[ilev[L - 1]:ilev[L]] + 1
        assert list(got) == nodes
    for node, dep in deps_g.items():
        i = node - 1
        cols = m.colidx[m.rowptr[i]:m.rowptr[i + 1]]
        assert sorted(int(c) + 1 for c in cols if c < i) == dep


# ------------------------------------------------------------- extremes
def test_diagonal_matrix_one_level():
    # diagonal matrices have nlev = 1
    n = 17
    m = CSR(n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.full(n, 2.0))
    for uplo in ("lower", "upper"):
        lev, nlev = oracle.levels(m, uplo)
        assert nlev == 1 and not lev.any()
        assert np.array_equal(oracle.select(m, uplo)["dp"], np.zeros(n))


def chain(n, sub=1.0, d=1.0):
    rowptr = np.zeros(n + 1, dtype=np.int32)
    cols, vals = [], []
    for i in range(n):
        if i > 0:
            cols.append(i - 1); vals.append(sub)
        cols.append(i); vals.append(d)
        rowptr[i + 1] = len(cols)
    return CSR(n, rowptr, np.array(cols, dtype=np.int32), np.array(vals))


def test_chain_n_levels():
    # a chain has nlev = n (fully sequential)
    m = chain(50)
    lev, nlev = oracle.levels(m, "lower")
    assert nlev == 50 and np.array_equal(lev, np.arange(50))
    ilev, jlev = oracle.schedule(lev, nlev)
    assert np.array_equal(ilev, np.arange(51)) and np.array_equal(jlev, np.arange(50))
    assert np.array_equal(oracle.select(m)["dp"], [0] + [1] * 49)


def test_empty_matrix():
    m = CSR(0, np.zeros(1, dtype=np.int32), np.zeros(0, dtype=np.int32), np.zeros(0))
    lev, nlev = oracle.levels(m)
    assert nlev == 0 and lev.size == 0
    a = oracle.analyze(m)
    assert a["status"] == "SUCCESS" and a["nlev"] == 0


def test_dependency_counts_5pt():
    # corner node 0 has 0 dependencies, an interior node has 2
    m = workloads.stencil((5, 5), 5, "lower")
    dp = oracle.select(m)["dp"]
    assert dp[0] == 0 and dp[12] == 2 and dp[1] == 1 and dp[5] == 1
    assert dp.sum() == 40          # nnz(L strict) = 40 on 5x5


# ------------------------------------------------- random DAGs, brute force
def random_triangular(n, density, seed, uplo="lower", extra_other=0.0, unit_diag_stored=True):
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        cols = set()
        for j in range(n):
            if j == i:
                if unit_diag_stored:
                    cols.add(j)
            elif (j < i) == (uplo == "lower"):
                if rng.random() < density:
                    cols.add(j)
            elif rng.random() < extra_other:
                cols.add(j)
        rows.append(sorted(cols))
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    colidx = np.array([c for r in rows for c in r], dtype=np.int32)
    vals = rng.uniform(-1, 1, size=colidx.size)
    for i, r in enumerate(rows):
        for k, c in enumerate(r):
            if c == i:
                vals[rowptr[i] + k] = rng.uniform(1, 2) * (1 if rng.random() < 0.5 else -1) * (1 + len(r))
    return CSR(n, rowptr, colidx, vals)


def longest_path_levels(m, uplo):
    """Brute force: lev(i) = length of the longest dependency path ending at i (DFS)."""
    n = m.n
    memo = {}

    def deps(i):
        cols = m.colidx[m.rowptr[i]:m.rowptr[i + 1]]
        return [int(c) for c in cols if (c < i if uplo == "lower" else c > i)]

    def lp(i):
        if i not in memo:
            ds = deps(i)
            memo[i] = 0 if not ds else 1 + max(lp(j) for j in ds)
        return memo[i]
    return np.array([lp(i) for i in range(n)], dtype=np.int32)


@pytest.mark.parametrize("seed", range(40))
def test_levels_row_col_dfs_agree(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    uplo = "lower" if seed % 2 == 0 else "upper"
    m = random_triangular(n, float(rng.uniform(0.02, 0.3)), seed, uplo, extra_other=0.1)
    lr, nr = oracle.levels(m, uplo, "row")
    lc, nc = oracle.levels(m, uplo, "col")
    ld = longest_path_levels(m, uplo)
    assert np.array_equal(lr, ld) and np.array_equal(lc, ld)
    assert nr == nc == (int(ld.max()) + 1 if n else 0)
    # O-4: stable order == sort by (lev, row id)
    ilev, jlev = oracle.schedule(lr, nr)
    ref = sorted(range(n), key=lambda i: (int(lr[i]), i))
    assert list(jlev) == ref
    assert np.array_equal(ilev, np.searchsorted(np.sort(lr), np.arange(nr + 1)))
    # A18 Kahn rounds give the same per-unknown levels and the same level sets
    ik, jk, lk, nk = oracle.kahn(m, uplo)
    assert nk == nr and np.array_equal(lk, lr) and np.array_equal(ik, ilev)
    for L in range(nr):
        assert sorted(jk[ik[L]:ik[L + 1]]) == list(jlev[ilev[L]:ilev[L + 1]])


def test_cfg1_schedule_pins():
    # SURVEY §8c (derived from lev = x + y on 32x32 and the stable order)
    m, _ = workloads.config(1)
    a = oracle.analyze(m)
    assert a["nlev"] == 63 and a["max_level_width"] == 32
    assert list(a["jlev"][:10]) == [0, 1, 32, 2, 33, 64, 3, 34, 65, 96]
    assert list(a["ilev"][:6]) == [0, 1, 3, 6, 10, 15]
    assert list(a["jlev"][-3:]) == [991, 1022, 1023]
    assert a["nnz_used"] == 3008 - 1024


@pytest.mark.parametrize("n,L,seed", [(5000, 97, 4), (20000, 300, 11), (3000, 3000, 2)])
def test_powerlaw_levels_by_construction(n, L, seed):
    # the generator places a critical dependency at level l-1 and the others
    # below l, so the oracle must reproduce its intended levels exactly
    m, lev_true = workloads.powerlaw(n, L, seed=seed)
    lev, nlev = oracle.levels(m, "lower")
    assert np.array_equal(lev, lev_true)
    assert nlev == int(lev_true.max()) + 1
    sel = oracle.select(m)
    assert sel["status"] == "SUCCESS" and sel["ignored"] == 0
