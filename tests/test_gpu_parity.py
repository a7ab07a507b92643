"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Analysis outputs (dp, lev, nlev, ilev, jlev) must match bit for bit; solutions
within the north-star tolerance: ||x - x_ref||_inf / ||x_ref||_inf <= 1e-10
(fp64), 1e-4 (fp32); integer-exact systems bit for bit.  Inputs are seeded
and synthetic (workloads/), at the five BASELINE.json configurations'
full sizes plus small cases that span several chunks and ragged tails.
"""
import numpy as np
import pytest
import torch

import oracle
import workloads
from workloads import CSR

from test_oracle_levels import chain, random_triangular

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

TOL = {np.float64: 1e-10, np.float32: 1e-4}
ALGOS = ["self", "level", "block", "auto"]


@pytest.fixture(scope="module")
def S():
    from paper_1710_04985_b200 import sptrsv
    return sptrsv


def relerr(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.abs(ref).max() if ref.size else 1.0
    return float(np.abs(x - ref).max() / den) if ref.size else 0.0


def avg_deps(m, uplo="lower"):
    rows = np.repeat(np.arange(m.n), np.diff(m.rowptr))
    strict = (m.colidx < rows) if uplo == "lower" else (m.colidx > rows)
    return strict.sum() / max(m.n, 1)


def gpu_solve(S, m, b, uplo="lower", diag="non_unit", dtype=np.float64, algo="self", solver=None):
    solver = solver or S.from_csr(m, uplo, diag, dtype, algo)
    bt = torch.from_numpy(np.ascontiguousarray(b, dtype=dtype)).cuda()
    x = solver.solve(bt)
    # every solve must complete: BLOCK's per-solve watchdog never fires on valid input
    assert solver.solve_status() == "SUCCESS"
    return x.cpu().numpy(), solver


def check_analysis(S, m, uplo, diag):
    ref = oracle.analyze(m, uplo, diag)
    assert ref["status"] == "SUCCESS"
    sv = S.from_csr(m, uplo, diag)
    lev, ilev, jlev, nlev = sv.levels()
    info = sv.info()
    assert nlev == ref["nlev"]
    assert np.array_equal(sv.dep_counts(), ref["dp"])
    assert np.array_equal(lev, ref["lev"])
    assert np.array_equal(ilev, ref["ilev"])
    assert np.array_equal(jlev, ref["jlev"])
    assert info["nnz_used"] == ref["nnz_used"]
    assert info["ignored_entries"] == ref["ignored"]
    assert info["max_level_width"] == ref["max_level_width"]
    assert info["max_row_deps"] == (int(ref["dp"].max()) if m.n else 0)
    return sv


# ------------------------------------------------------------ analysis
@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_analysis_bit_exact_full_configs(S, cfg):
    m, p = workloads.config(cfg)
    check_analysis(S, m, p["uplo"], p["diag"])


def test_analysis_bit_exact_cfg3_both_factors(S):
    m, _ = workloads.config(3)
    check_analysis(S, m, "lower", "unit")
    check_analysis(S, m, "upper", "non_unit")


@pytest.mark.parametrize("seed", range(12))
def test_analysis_random_small(S, seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    uplo = ("lower", "upper")[seed % 2]
    m = random_triangular_fast(n, float(rng.uniform(1, 40)), seed, uplo)
    check_analysis(S, m, uplo, "non_unit")


def random_triangular_fast(n, avg_deps, seed, uplo, other=0.5, long_frac=0.02):
    """Random triangle with a stored diagonal, some opposite-triangle entries,
    and a few long rows (> 16 deps -> warp-per-row)."""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        lo, hi = (0, i) if uplo == "lower" else (i + 1, n)
        span = hi - lo
        k = min(span, int(rng.poisson(avg_deps)) if rng.random() > long_frac else int(rng.integers(17, 200)))
        deps = rng.choice(span, size=k, replace=False) + lo if k > 0 else np.zeros(0, dtype=np.int64)
        olo, ohi = (i + 1, n) if uplo == "lower" else (0, i)
        no = min(ohi - olo, int(rng.poisson(other)))
        oth = rng.choice(ohi - olo, size=no, replace=False) + olo if no > 0 else np.zeros(0, dtype=np.int64)
        rows.append(np.unique(np.concatenate([deps, oth, [i]]).astype(np.int64)))
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum([len(r) for r in rows])
    colidx = np.concatenate(rows).astype(np.int32) if n else np.zeros(0, dtype=np.int32)
    vals = rng.uniform(-1, 1, size=colidx.size)
    for i in range(n):
        a, b = rowptr[i], rowptr[i + 1]
        k = a + int(np.searchsorted(colidx[a:b], i))
        vals[k] = (1.0 + np.abs(vals[a:b]).sum()) * (1 if rng.random() < 0.5 else -1)
    return CSR(n, rowptr, colidx, vals)


# ------------------------------------------------------------ solves
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_solve_full_configs(S, cfg, algo):
    m, p = workloads.config(cfg)
    if algo == "block" and cfg == 4:      # natural partition, 10.8 deps per row: refused (see sptrsv.h)
        with pytest.raises(S.SptrsvError) as e:
            S.from_csr(m, p["uplo"], p["diag"], algo=algo)
        assert e.value.name == "NOT_SUPPORTED"
        return
    b = workloads.rhs(m.n, 1, seed=p["seed"])[:, 0]
    ref = oracle.solve(m, b, p["uplo"], p["diag"])
    x, sv = gpu_solve(S, m, b, p["uplo"], p["diag"], algo=algo)
    assert relerr(x, ref) <= TOL[np.float64]
    # run-to-run bitwise reproducible
    x2, _ = gpu_solve(S, m, b, solver=sv)
    assert np.array_equal(x, x2)


@pytest.mark.parametrize("algo", ALGOS)
def test_cfg3_pair_solve_full(S, algo):
    m, p = workloads.config(3)
    b = workloads.rhs(m.n, 1, seed=p["seed"])[:, 0]
    ref = oracle.pair_solve(m, b)
    lo = S.from_csr(m, "lower", "unit", algo=algo)
    up = S.from_csr(m, "upper", "non_unit", algo=algo)
    bt = torch.from_numpy(b).cuda()
    y = up.solve(lo.solve(bt))
    assert relerr(y.cpu().numpy(), ref) <= TOL[np.float64]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("uplo,diag", [("lower", "non_unit"), ("upper", "non_unit"), ("lower", "unit"),
                                       ("upper", "unit")])
def test_solve_random_small(S, uplo, diag, dtype, algo):
    for seed in range(4):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(1, 2500))
        m = random_triangular_fast(n, float(rng.uniform(1, 20)), 10 * seed + 1, uplo)
        if diag == "unit":
            off = m.colidx != np.repeat(np.arange(n), np.diff(m.rowptr))
            m.vals[off] *= 0.5 / max(1.0, np.diff(m.rowptr).max())
        b = workloads.rhs(n, 1, seed=seed)[:, 0]
        ref = oracle.solve(m.astype(dtype), b.astype(dtype), uplo, diag, dtype=dtype)
        if algo == "block" and avg_deps(m, uplo) > 3:
            # BLOCK refuses natural partitions with > 3 dependencies per row on average
            with pytest.raises(S.SptrsvError) as e:
                S.from_csr(m, uplo, diag, dtype, algo)
            assert e.value.name == "NOT_SUPPORTED"
            continue
        x, _ = gpu_solve(S, m, b, uplo, diag, dtype, algo)
        assert relerr(x, ref) <= TOL[dtype], (seed, n)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", ["cfg1", "7pt_d8", "7pt_upper_d8"])
def test_integer_exact_bitwise(S, case, dtype, algo):
    if case == "cfg1":
        m, uplo = workloads.stencil((32, 32), 5, "lower"), "lower"
    elif case == "7pt_d8":
        m, uplo = workloads.stencil((40, 30, 20), 7, "lower", diag=8.0), "lower"
    else:
        m, uplo = workloads.stencil((40, 30, 20), 7, "upper", diag=8.0), "upper"
    xt = workloads.integer_xtrue(m.n, 1, seed=101)[:, 0]
    b = oracle.matvec(m, xt, uplo)
    x, _ = gpu_solve(S, m, b, uplo, dtype=dtype, algo=algo)
    assert np.array_equal(x.astype(np.float64), xt)


@pytest.mark.parametrize("algo", ALGOS)
def test_backward_error_bound_gpu(S, algo):
    m, p = workloads.config(2, scale=0.5)
    b = workloads.rhs(m.n, 1, seed=9)[:, 0]
    x, _ = gpu_solve(S, m, b, algo=algo)
    k = 3
    u = 2.0 ** -53
    assert oracle.backward_error(m, b, x) <= (k + 2) * u / (1 - (k + 2) * u)


@pytest.mark.parametrize("algo", ALGOS)
def test_chain_progress(S, algo):
    # P:315-316 worst case nlev = n: one long dependency chain
    n = 100000
    m = chain(n, sub=-0.5, d=1.0)
    b = workloads.rhs(n, 1, seed=4)[:, 0]
    x, _ = gpu_solve(S, m, b, algo=algo)
    assert relerr(x, oracle.solve(m, b)) <= 1e-10


@pytest.mark.parametrize("algo", ALGOS)
def test_diagonal_and_tiny(S, algo):
    for n in (1, 2, 31, 32, 33, 1000):
        m = CSR(n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
                np.linspace(1, 2, n))
        b = workloads.rhs(n, 1, seed=n)[:, 0]
        x, _ = gpu_solve(S, m, b, algo=algo)
        assert relerr(x, b / m.vals) <= 1e-15


def test_in_place_solve(S):
    m, _ = workloads.config(2, scale=0.25)
    b = workloads.rhs(m.n, 1, seed=3)[:, 0]
    ref = oracle.solve(m, b)
    for algo in ALGOS:
        sv = S.from_csr(m, algo=algo)
        bt = torch.from_numpy(b.copy()).cuda()
        sv.solve(bt, x=bt)
        assert relerr(bt.cpu().numpy(), ref) <= 1e-10


def test_solve_host_matches(S):
    m, _ = workloads.config(2, scale=0.25)
    b = workloads.rhs(m.n, 2, seed=3)
    sv = S.from_csr(m)
    x = sv.solve_host(b)
    assert relerr(x, oracle.solve(m, b)) <= 1e-10
    x1 = sv.solve_host(np.ascontiguousarray(b[:, 0]))
    assert relerr(x1, oracle.solve(m, b[:, 0])) <= 1e-10


# ------------------------------------------------------------ multi-RHS
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("nrhs", [2, 3, 33, 64, 100])
def test_multi_rhs_small(S, nrhs, algo):
    for uplo in ("lower", "upper"):
        m = (random_triangular_fast(3000, 6.0, 5, uplo) if algo != "block"
             else random_triangular_fast(3000, 1.5, 5, uplo, long_frac=0.004))
        b = workloads.rhs(m.n, nrhs, seed=nrhs)
        x, _ = gpu_solve(S, m, b, uplo=uplo, algo=algo)
        assert relerr(x, oracle.solve(m, b, uplo)) <= 1e-10


@pytest.mark.parametrize("nrhs", [2, 17, 64, 100])
@pytest.mark.parametrize("case", ["7pt_lower", "7pt_upper", "27pt_lower_unit", "5pt_2d"])
def test_multi_rhs_grids_block(S, case, nrhs):
    # BLOCK on detected grids: multi-RHS solves (column blocks, ragged widths)
    if case == "7pt_lower":
        m, uplo, diag = workloads.stencil((24, 20, 12), 7, "lower"), "lower", "non_unit"
    elif case == "7pt_upper":
        m, uplo, diag = workloads.stencil((24, 20, 12), 7, "upper"), "upper", "non_unit"
    elif case == "27pt_lower_unit":
        m, uplo, diag = workloads.ilu0(workloads.stencil((12, 10, 8), 27)), "lower", "unit"
    else:
        m, uplo, diag = workloads.stencil((64, 48), 5, "lower"), "lower", "non_unit"
    b = workloads.rhs(m.n, nrhs, seed=nrhs + 7)
    x, sv = gpu_solve(S, m, b, uplo=uplo, diag=diag, algo="block")
    assert sv.info()["nblocks"] > 0
    assert relerr(x, oracle.solve(m, b, uplo, diag)) <= 1e-10


@pytest.mark.parametrize("algo", ["self", "level", "block"])
def test_cfg5_full_64_rhs_and_partition_bitwise(S, algo):
    # cfg5: 64 RHS on the 128^3 factor; column blocks (G = 2, 4, 8) must equal
    # the G = 1 columns bit for bit, and match the oracle
    m, _ = workloads.config(5)
    b = workloads.rhs_columns(m.n, range(64))
    sv = S.from_csr(m, algo=algo)
    x_all = sv.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    cols = [0, 17, 40, 63]
    ref = oracle.solve(m, np.ascontiguousarray(b[:, cols]))
    assert relerr(x_all[:, cols], ref) <= 1e-10
    from paper_1710_04985_b200 import partition
    for G in (2, 4, 8):
        for r in range(G):
            a, e = partition.block_range(64, G, r)
            xb = sv.solve(torch.from_numpy(np.ascontiguousarray(b[:, a:e])).cuda()).cpu().numpy()
            assert np.array_equal(xb, x_all[:, a:e])


def test_multi_rhs_columns_equal_single_rhs_self(S):
    # TPR rows use the same per-(row, column) arithmetic in k_self and k_mrhs
    m, _ = workloads.config(2, scale=0.25)
    b = workloads.rhs(m.n, 4, seed=8)
    sv = S.from_csr(m)
    xm = sv.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    for r in range(4):
        xs = sv.solve(torch.from_numpy(np.ascontiguousarray(b[:, r])).cuda()).cpu().numpy()
        assert np.array_equal(xs, xm[:, r])


# ------------------------------------------------------------ status codes
def _upload(m):
    rp = torch.from_numpy(np.ascontiguousarray(m.rowptr, dtype=np.int32)).cuda()
    ci = torch.from_numpy(np.ascontiguousarray(m.colidx, dtype=np.int32)).cuda()
    va = torch.from_numpy(np.ascontiguousarray(m.vals, dtype=np.float64)).cuda()
    return rp, ci, va


def test_status_codes_match_oracle(S):
    from test_oracle_solve import csr
    cases = [
        (csr(3, [[0], [1, 0], [1, 2]]), "lower", "non_unit"),
        (csr(3, [[0], [0, 1], [1, 3]]), "lower", "non_unit"),
        (csr(3, [[0], [0], [1, 2]]), "lower", "non_unit"),
        (csr(3, [[0], [0], [1, 2]]), "lower", "unit"),
        (csr(3, [[0], [0, 1], [1, 2]], vals=[1, 1, 1, 1, 0.0]), "lower", "non_unit"),
        (csr(3, [[0], [0], [2, 1]]), "upper", "non_unit"),
    ]
    for m, uplo, diag in cases:
        ref = oracle.select(m, uplo, diag)
        rp, ci, va = _upload(m)
        if ref["status"] == "SUCCESS":
            S.TriangularSolver(m.n, rp, ci, va, uplo, diag).close()
            continue
        with pytest.raises(S.SptrsvError) as e:
            S.TriangularSolver(m.n, rp, ci, va, uplo, diag)
        assert e.value.name == ref["status"]
        assert e.value.info["bad_row"] == ref["bad_row"]
        assert e.value.info["zero_pivot_row"] == ref["zero_pivot_row"]
    # bad rowptr[0]
    m = csr(3, [[0], [0, 1], [1, 2]])
    m.rowptr = m.rowptr.copy()
    m.rowptr[0] = 1
    rp, ci, va = _upload(m)
    with pytest.raises(S.SptrsvError) as e:
        S.TriangularSolver(3, rp, ci, va)
    assert e.value.name == "INVALID_MATRIX" and e.value.info["bad_row"] == 0


def test_invalid_value_and_empty(S):
    m = CSR(0, np.zeros(1, dtype=np.int32), np.zeros(0, dtype=np.int32), np.zeros(0))
    rp, ci, va = _upload(m)
    sv = S.TriangularSolver(0, rp, ci, va)
    assert sv.info()["nlev"] == 0
    assert sv.solve(torch.zeros(0, dtype=torch.float64, device="cuda")).numel() == 0
    m2, _ = workloads.config(1)
    sv2 = S.from_csr(m2)
    b = torch.zeros(m2.n, dtype=torch.float64, device="cuda")
    assert S.sptrsv_solve(sv2.handle, S._dptr(b), S._dptr(b), 0, None) == 1   # nrhs < 1
    assert S.sptrsv_set_algo(sv2.handle, 9) == 1


# ------------------------------------------------------------ BLOCK (warp tiles)
GRID_CASES = [((32, 32), 5, "lower"), ((64, 48), 5, "upper"), ((16, 16, 16), 7, "lower"),
              ((40, 30, 20), 7, "lower"), ((40, 30, 20), 7, "upper"), ((128, 128, 128), 7, "lower"),
              ((97, 45, 13), 7, "lower"), ((33, 65), 9, "lower"), ((24, 20, 12), 27, "lower")]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("dims,pts,uplo", GRID_CASES)
def test_block_grids(S, dims, pts, uplo, dtype):
    """Detected grids (tiles), ragged tile edges, 9- and 27-point rows (more
    than 3 terms: overflow lists); oracle tolerance, run-to-run bitwise, and
    bitwise equal to the storage-order multi-RHS kernels column by column."""
    m = workloads.stencil(dims, pts, uplo)
    b = workloads.rhs(m.n, 1, seed=len(dims) * 10 + pts + 1)[:, 0]
    ref = oracle.solve(m.astype(dtype), b.astype(dtype), uplo, dtype=dtype)
    x, sv = gpu_solve(S, m, b, uplo, dtype=dtype, algo="block")
    assert sv.info()["algo"] == 2 and sv.info()["nblocks"] > 0
    assert relerr(x, ref) <= TOL[dtype]
    x2, _ = gpu_solve(S, m, b, uplo, dtype=dtype, solver=sv)
    assert np.array_equal(x, x2)
    if m.n <= 200000:                    # storage-order FMA: equal to the multi-RHS columns
        B2 = np.ascontiguousarray(np.stack([b, b], axis=1)).astype(dtype)
        X2 = sv.solve(torch.from_numpy(B2).cuda()).cpu().numpy()
        assert np.array_equal(X2[:, 1], x)


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("uplo,diag", [("lower", "non_unit"), ("upper", "unit")])
def test_block_natural_partition_and_integer(S, seed, uplo, diag):
    """Natural-order partition (no grid): SHFL / SMEM / GLOB / overflow terms
    of every kind; integer-exact grids bitwise, also in place."""
    m = random_triangular_fast(2500 + 611 * seed, 0.8 + 0.25 * seed, seed, uplo, long_frac=0.004)
    assert avg_deps(m, uplo) <= 3
    b = workloads.rhs(m.n, 1, seed=seed)[:, 0]
    ref = oracle.solve(m, b, uplo, diag)
    x, sv = gpu_solve(S, m, b, uplo, diag, algo="block")
    assert sv.info()["algo"] == 2
    assert relerr(x, ref) <= 1e-10
    g = workloads.stencil((40, 30, 20), 7, uplo, diag=8.0)
    xt = workloads.integer_xtrue(g.n, 1, seed=101 + seed)[:, 0]
    bb = oracle.matvec(g, xt, uplo)
    xg, sv = gpu_solve(S, g, bb, uplo, algo="block")
    assert np.array_equal(xg, xt)
    bt = torch.from_numpy(bb).cuda()                    # in place
    sv.solve(bt, x=bt)
    assert sv.solve_status() == "SUCCESS"
    assert np.array_equal(bt.cpu().numpy(), xt)


def random_lower_vec(n, avg_deps, seed, window=None):
    """Vectorised random lower triangle (diagonally dominant): Poisson(avg)
    dependencies per row, uniform over [0, i) or over the last `window` rows."""
    rng = np.random.default_rng(seed)
    cnt = np.minimum(rng.poisson(avg_deps, size=n), np.arange(n))
    rows = np.repeat(np.arange(n), cnt)
    lo = np.zeros(rows.size, dtype=np.int64) if window is None else np.maximum(0, rows - window)
    cols = lo + (rng.random(rows.size) * (rows - lo)).astype(np.int64)
    key = np.unique(rows.astype(np.int64) * n + cols)          # sorted, deduplicated (row, col)
    rows, cols = key // n, key % n
    allr = np.concatenate([rows, np.arange(n)])
    allc = np.concatenate([cols, np.arange(n)])
    o = np.lexsort((allc, allr))
    allr, allc = allr[o], allc[o]
    vals = rng.uniform(-1, 1, size=allr.size)
    diag = allr == allc
    absum = np.bincount(allr[~diag], weights=np.abs(vals[~diag]), minlength=n)
    vals[diag] = 1.0 + absum
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum(np.bincount(allr, minlength=n))
    return CSR(n, rowptr, allc.astype(np.int32), vals)


@pytest.mark.parametrize("n,window,dtype", [(60000, 300, np.float32), (200000, None, np.float64)])
def test_block_natural_partition_multi_cta(S, n, window, dtype):
    """Natural partitions over several CTAs (8192 rows each): cross-CTA values
    through mailboxes and fetcher warps when every CTA's shared slots fit
    (fp32, dependencies within 300 rows), or -- fp64, dependencies anywhere
    below, too many values to stage in shared memory -- the GL instance,
    whose consumers poll the mailboxes themselves."""
    m = random_lower_vec(n, 2.0, 17, window)
    b = workloads.rhs(m.n, 1, seed=5)[:, 0]
    ref = oracle.solve(m.astype(dtype), b.astype(dtype), dtype=dtype)
    x, sv = gpu_solve(S, m, b, dtype=dtype, algo="block")
    assert sv.info()["nblocks"] > 1
    import ctypes
    lib = ctypes.CDLL(S.LIB_PATH)
    lib.sptrsv_dbg_block_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    plan = (ctypes.c_longlong * 13)()
    assert lib.sptrsv_dbg_block_plan(ctypes.c_void_p(sv.handle), plan) == 0
    assert plan[12] == (1 if window is None else 0)          # GL instance only when slots cannot fit
    assert relerr(x, ref) <= (1e-10 if dtype == np.float64 else 1e-4)
    x2, _ = gpu_solve(S, m, b, dtype=dtype, solver=sv)
    assert np.array_equal(x, x2)


def test_block_refuses_dense_natural_partition(S):
    m, p = workloads.config(4, scale=1 / 64)
    with pytest.raises(S.SptrsvError) as e:
        S.from_csr(m, p["uplo"], p["diag"], algo="block")
    assert e.value.name == "NOT_SUPPORTED"
    assert S.from_csr(m, p["uplo"], p["diag"], algo="auto").info()["algo"] == 0


def test_block_watchdog_timeout_then_clean(S):
    """A BLOCK solve that gives up a spin wait reports TIMEOUT through
    sptrsv_get_solve_status (per handle, per solve); the next solve is clean."""
    import ctypes
    lib = ctypes.CDLL(S.LIB_PATH)
    lib.sptrsv_dbg_set_timeout_ns.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong]
    m = workloads.stencil((64, 64, 48), 7, "lower")     # many warps: downstream ones wait from the start
    b = workloads.rhs(m.n, 1, seed=4)[:, 0]
    sv = S.from_csr(m, algo="block")
    bt = torch.from_numpy(b).cuda()
    assert lib.sptrsv_dbg_set_timeout_ns(ctypes.c_void_p(sv.handle), 0) == 0
    sv.solve(bt)
    assert sv.solve_status() == "TIMEOUT"
    assert S.sptrsv_get_solve_status(sv.handle) == 7
    other = S.from_csr(m, algo="block")                  # another handle is unaffected
    x, _ = gpu_solve(S, m, b, solver=other)
    assert lib.sptrsv_dbg_set_timeout_ns(ctypes.c_void_p(sv.handle), 4_000_000_000) == 0
    x2 = sv.solve(bt)
    assert sv.solve_status() == "SUCCESS"
    ref = oracle.solve(m, b)
    assert relerr(x2.cpu().numpy(), ref) <= 1e-10 and relerr(x, ref) <= 1e-10


# ------------------------------------------------------------ column-wise SLFC / LEVC (NEXT-1)
COL_ALGOS = ["slfc", "levc"]


@pytest.mark.parametrize("algo", COL_ALGOS)
@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_column_full_configs(S, cfg, algo):
    """Alg. SLFC / LEVC at the full BASELINE sizes:
    atomics accumulate in arrival order, so parity is by the north-star tolerance."""
    m, p = workloads.config(cfg)
    b = workloads.rhs(m.n, 1, seed=p["seed"])[:, 0]
    ref = oracle.solve(m, b, p["uplo"], p["diag"])
    x, sv = gpu_solve(S, m, b, p["uplo"], p["diag"], algo=algo)
    assert sv.info()["algo"] == {"slfc": 5, "levc": 6}[algo]
    assert relerr(x, ref) <= 1e-10


@pytest.mark.parametrize("algo", COL_ALGOS)
def test_column_cfg3_pair(S, algo):
    m, p = workloads.config(3)
    b = workloads.rhs(m.n, 1, seed=p["seed"])[:, 0]
    y = oracle.solve(m, b, "lower", "unit")
    ref = oracle.solve(m, y, "upper", "non_unit")
    lo = S.from_csr(m, "lower", "unit", algo=algo)
    up = S.from_csr(m, "upper", "non_unit", algo=algo)
    bt = torch.from_numpy(b).cuda()
    x = up.solve(lo.solve(bt))
    torch.cuda.synchronize()
    assert relerr(x.cpu().numpy(), ref) <= 1e-10


@pytest.mark.parametrize("algo", COL_ALGOS)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("uplo,diag", [("lower", "non_unit"), ("upper", "non_unit"), ("lower", "unit"),
                                       ("upper", "unit")])
def test_column_random_small(S, uplo, diag, dtype, algo):
    for seed in range(3):
        m = random_triangular_fast(3000 + 517 * seed, 3.0 + 2 * seed, seed, uplo)
        b = workloads.rhs(m.n, 1, seed=seed)[:, 0]
        ref = oracle.solve(m.astype(dtype), b.astype(dtype), uplo, diag, dtype=dtype)
        x, _ = gpu_solve(S, m, b, uplo, diag, dtype=dtype, algo=algo)
        assert relerr(x, ref) <= TOL[dtype]
        if dtype == np.float64:                        # and the column-wise sweep
            assert relerr(x, oracle.solve_col(m, b, uplo, diag)) <= 1e-10


@pytest.mark.parametrize("algo", COL_ALGOS)
@pytest.mark.parametrize("uplo", ["lower", "upper"])
def test_column_integer_exact_in_place_and_repeat(S, uplo, algo):
    """Integer systems with power-of-two diagonals are exact in any summation
    order: atomics included, the result is bitwise x_true, every solve."""
    m = workloads.stencil((40, 30, 20), 7, uplo, diag=8.0)
    xt = workloads.integer_xtrue(m.n, 1, seed=101)[:, 0]
    b = oracle.matvec(m, xt, uplo)
    x, sv = gpu_solve(S, m, b, uplo, algo=algo)
    assert np.array_equal(x, xt)
    for _ in range(3):                                 # counters / barrier state carried across solves
        x2, _ = gpu_solve(S, m, b, uplo, solver=sv)
        assert np.array_equal(x2, xt)
    bt = torch.from_numpy(b).cuda()
    sv.solve(bt, x=bt)
    torch.cuda.synchronize()
    assert np.array_equal(bt.cpu().numpy(), xt)


@pytest.mark.parametrize("algo", COL_ALGOS)
def test_column_multi_rhs_and_degenerate(S, algo):
    """nrhs > 1 runs the row kernels; diagonal-only and 1x1 systems."""
    m = random_triangular_fast(2000, 4.0, 7, "lower")
    B = workloads.rhs(m.n, 5, seed=7)
    ref = oracle.solve(m, B, "lower")
    sv = S.from_csr(m, algo=algo)
    X = sv.solve(torch.from_numpy(B).cuda()).cpu().numpy()
    assert relerr(X, ref) <= 1e-10
    for n in (1, 37):
        d = CSR(n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), np.full(n, 4.0))
        bb = np.arange(1, n + 1, dtype=np.float64)
        x, _ = gpu_solve(S, d, bb, algo=algo)
        assert np.array_equal(x, bb / 4.0)


def test_auto_selection_rule(S):
    """AUTO: BLOCK on detected grids with <= 3 dependencies per row (5-/7-point
    factors); else SMALL when the level-ordered triangle fits one CTA's shared
    memory; else SELF (27-point ILU, general matrices)."""
    m7 = workloads.stencil((24, 20, 16), 7, "lower")
    assert S.from_csr(m7, algo="auto").info()["algo"] == 2
    m5 = workloads.stencil((40, 30), 5, "upper")
    assert S.from_csr(m5, "upper", algo="auto").info()["algo"] == 2
    for dims, want in (((8, 6, 5), 7), ((24, 20, 16), 0)):
        m27 = workloads.ilu0(workloads.stencil(dims, 27, "full"))
        for uplo, diag in (("lower", "unit"), ("upper", "non_unit")):
            sv = S.from_csr(m27, uplo, diag, algo="auto")
            assert sv.info()["algo"] == want
            b = workloads.rhs(m27.n, 1, seed=9)[:, 0]
            x, _ = gpu_solve(S, m27, b, uplo, diag, solver=sv)
            assert relerr(x, oracle.solve(m27, b, uplo, diag)) <= 1e-10


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", ["cfg1", "5pt_upper_unit", "random_wpr", "chain", "27pt_ilu"])
def test_small_single_cta(S, case, dtype):
    """SMALL (one CTA, triangle in shared memory): oracle tolerance, bitwise
    equal to SELF and LEVEL (same per-row sequences), integer-exact cfg1."""
    uplo, diag = "lower", "non_unit"
    if case == "cfg1":
        m, _ = workloads.config(1)
    elif case == "5pt_upper_unit":
        m, uplo, diag = workloads.stencil((40, 30), 5, "upper"), "upper", "unit"
    elif case == "random_wpr":
        m = random_triangular_fast(800, 2.0, 21, "lower", long_frac=0.02)       # some rows > 16 deps (WPR)
    elif case == "chain":
        m = chain(300)
    else:
        m, uplo, diag = workloads.ilu0(workloads.stencil((8, 6, 5), 27, "full")), "upper", "non_unit"
    b = workloads.rhs(m.n, 1, seed=4)[:, 0]
    sv = S.from_csr(m, uplo, diag, dtype, "small")
    assert sv.info()["algo"] == 7
    x, _ = gpu_solve(S, m, b, uplo, diag, dtype, solver=sv)
    ref = oracle.solve(m.astype(dtype), b.astype(dtype), uplo, diag, dtype=dtype)
    assert relerr(x, ref) <= TOL[dtype]
    for other in ("self", "level"):
        xo, _ = gpu_solve(S, m, b, uplo, diag, dtype, algo=other)
        assert np.array_equal(x, xo), other
    if case == "cfg1":
        xt = workloads.integer_xtrue(m.n, 1, 5)[:, 0]
        rows = np.repeat(np.arange(m.n), np.diff(m.rowptr))
        bi = np.zeros(m.n)
        np.add.at(bi, rows, m.vals * xt[m.colidx])
        xi, _ = gpu_solve(S, m, bi, dtype=dtype, solver=sv)
        assert np.array_equal(xi, xt.astype(dtype))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("uplo,diag", [("lower", "non_unit"), ("upper", "unit")])
@pytest.mark.parametrize("nrhs", [2, 5, 8, 16])
def test_multi_rhs_value_as_flag(S, nrhs, uplo, diag, dtype):
    """k_mrhs_vf (nrhs <= 16, per-column value-as-flag): oracle tolerance,
    bitwise equal to the level-scheduled multi-RHS kernel column by column,
    run-to-run bitwise, and in place."""
    m = random_triangular_fast(3000, 5.0, nrhs, uplo)
    B = workloads.rhs(m.n, nrhs, seed=nrhs)
    ref = oracle.solve(m.astype(dtype), B.astype(dtype), uplo, diag, dtype=dtype)
    Bt = torch.from_numpy(B.astype(dtype)).cuda()
    sv = S.from_csr(m, uplo, diag, dtype, algo="self")
    X = sv.solve(Bt).cpu().numpy()
    assert relerr(X, ref) <= TOL[dtype]
    assert np.array_equal(X, sv.solve(Bt).cpu().numpy())
    lv = S.from_csr(m, uplo, diag, dtype, algo="level")
    assert np.array_equal(X, lv.solve(Bt).cpu().numpy())
    Bi = Bt.clone()
    sv.solve(Bi, x=Bi)
    torch.cuda.synchronize()
    assert np.array_equal(Bi.cpu().numpy(), X)


@pytest.mark.parametrize("uplo", ["lower", "upper"])
def test_levels_kahn_and_syncfree_agree(S, uplo):
    """All three level computations (Kahn by rounds in one cooperative launch,
    default; the sync-free kernel; the paper's host loop with one launch per
    level) give the oracle's levels bit for bit."""
    import ctypes
    lib = ctypes.CDLL(S.LIB_PATH)
    m = random_triangular_fast(20000, 6.0, 11, uplo)
    ref = oracle.analyze(m, uplo, "non_unit")
    try:
        for mode in (0, 1, 2):
            assert lib.sptrsv_dbg_levels_mode(mode) == 0
            lev, ilev, jlev, nlev = S.from_csr(m, uplo).levels()
            assert nlev == ref["nlev"]
            assert np.array_equal(lev, ref["lev"]) and np.array_equal(jlev, ref["jlev"])
            assert np.array_equal(ilev, ref["ilev"])
    finally:
        lib.sptrsv_dbg_levels_mode(0)


# ------------------------------------------------------------ multi-RHS tile kernel (mrt.cu)
def random_lowdeg(n, seed, uplo, maxdeg=4, window=3000):
    """Triangle with 0..maxdeg dependencies per row (uniform), at distances
    1..window (a few per row much farther), diagonally dominant."""
    rng = np.random.default_rng(seed)
    rows, cols = [np.arange(n)], [np.arange(n)]
    deg = rng.integers(0, maxdeg + 1, size=n)
    for k in range(maxdeg):
        i = np.nonzero(deg > k)[0]
        far = rng.random(i.size) < 0.05
        dist = np.where(far, rng.integers(1, n + 1, size=i.size), rng.integers(1, window + 1, size=i.size))
        j = i - dist
        ok = j >= 0
        rows.append(i[ok])
        cols.append(j[ok])
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    key = np.unique(r.astype(np.int64) * n + c)
    r, c = (key // n).astype(np.int64), (key % n).astype(np.int64)
    if uplo == "upper":
        r, c = n - 1 - r, n - 1 - c
        o = np.lexsort((c, r))
        r, c = r[o], c[o]
    vals = rng.uniform(-1, 1, size=r.size)
    diag = r == c
    absum = np.bincount(r[~diag], weights=np.abs(vals[~diag]), minlength=n)
    vals[diag] = 1.0 + absum[r[diag]]
    rowptr = np.zeros(n + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum(np.bincount(r, minlength=n))
    return CSR(n, rowptr, c.astype(np.int32), vals)


def _mrhs_old_path(S, sv):
    import ctypes
    lib = ctypes.CDLL(S.LIB_PATH)
    lib.sptrsv_dbg_mrhs_path.argtypes = [ctypes.c_void_p, ctypes.c_int]
    assert lib.sptrsv_dbg_mrhs_path(ctypes.c_void_p(sv.handle), 1) == 0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", ["7pt_lower", "7pt_upper_unit", "5pt_2d", "natural_lower", "natural_upper"])
@pytest.mark.parametrize("nrhs", [18, 24, 33, 64, 100])
def test_mrhs_tile_kernel(S, case, nrhs, dtype):
    """Multi-RHS tile kernel (factors with <= 4 dependencies per row, grid tile
    or natural partitions, column blocks of 64): oracle tolerance, bitwise
    equal to the other multi-RHS kernels (same per-(row, column) arithmetic),
    run-to-run bitwise, in place, and the solve completes (watchdog quiet)."""
    algo = "auto"
    if case == "7pt_lower":
        m, uplo, diag = workloads.stencil((40, 24, 12), 7, "lower"), "lower", "non_unit"
    elif case == "7pt_upper_unit":
        m, uplo, diag = workloads.stencil((24, 40, 10), 7, "upper"), "upper", "unit"
    elif case == "5pt_2d":
        m, uplo, diag = workloads.stencil((96, 64), 5, "lower"), "lower", "non_unit"
    else:
        uplo = "lower" if case == "natural_lower" else "upper"
        m, diag, algo = random_lowdeg(30000, 7, uplo), "non_unit", "self"
    deps = np.diff(m.rowptr) - 1
    assert deps.max() <= 4
    B = workloads.rhs(m.n, nrhs, seed=nrhs + 3)
    ref = oracle.solve(m.astype(dtype), B.astype(dtype), uplo, diag, dtype=dtype)
    Bt = torch.from_numpy(B.astype(dtype)).cuda()
    sv = S.from_csr(m, uplo, diag, dtype, algo=algo)
    X = sv.solve(Bt).cpu().numpy()
    assert sv.solve_status() == "SUCCESS"
    assert relerr(X, ref) <= TOL[dtype]
    assert np.array_equal(X, sv.solve(Bt).cpu().numpy())
    Bi = Bt.clone()
    sv.solve(Bi, x=Bi)
    torch.cuda.synchronize()
    assert np.array_equal(Bi.cpu().numpy(), X)
    old = S.from_csr(m, uplo, diag, dtype, algo=algo)
    _mrhs_old_path(S, old)
    assert np.array_equal(old.solve(Bt).cpu().numpy(), X)


def test_mrhs_tile_kernel_timeout_then_clean(S):
    """A wait of the tile kernel that exceeds the watchdog is reported as
    TIMEOUT by sptrsv_get_solve_status; the next solve is clean."""
    import ctypes
    m = workloads.stencil((64, 64, 32), 7, "lower")
    B = torch.from_numpy(workloads.rhs(m.n, 32, seed=1)).cuda()
    sv = S.from_csr(m, algo="auto")
    X = sv.solve(B).cpu().numpy()
    assert sv.solve_status() == "SUCCESS"
    lib = ctypes.CDLL(S.LIB_PATH)
    lib.sptrsv_dbg_set_timeout_ns.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong]
    lib.sptrsv_dbg_set_timeout_ns(ctypes.c_void_p(sv.handle), 1)
    sv.solve(B)
    assert sv.solve_status() == "TIMEOUT"
    lib.sptrsv_dbg_set_timeout_ns(ctypes.c_void_p(sv.handle), 4_000_000_000)
    X2 = sv.solve(B).cpu().numpy()
    assert sv.solve_status() == "SUCCESS"
    assert np.array_equal(X, X2)


# ------------------------------------------------------------ value update (NEXT-2)
def _dev(m, dtype):
    rp = torch.from_numpy(np.ascontiguousarray(m.rowptr, dtype=np.int32)).cuda()
    ci = torch.from_numpy(np.ascontiguousarray(m.colidx, dtype=np.int32)).cuda()
    va = torch.from_numpy(np.ascontiguousarray(m.vals, dtype=dtype)).cuda()
    return rp, ci, va


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("case", ["7pt_lower", "27pt_ilu_upper", "random_unit_lower"])
def test_update_values_equals_fresh_analysis(S, case, dtype):
    """sptrsv_update_values on a handle that has built every layout (level
    rows, BLOCK records, multi-RHS tile / value-as-flag / level, CSC): every
    algorithm then gives bit for bit the result of a fresh analysis of the new
    values, and matches the oracle."""
    rng = np.random.default_rng(11)
    if case == "7pt_lower":
        m, uplo, diag = workloads.stencil((32, 24, 16), 7, "lower"), "lower", "non_unit"
    elif case == "27pt_ilu_upper":
        m, uplo, diag = workloads.ilu0(workloads.stencil((14, 12, 10), 27)), "upper", "non_unit"
    else:
        m, uplo, diag = random_lowdeg(20000, 5, "lower"), "lower", "unit"
    m2 = workloads.CSR(m.n, m.rowptr, m.colidx, m.vals * rng.uniform(0.5, 1.5, size=m.vals.size))
    b1 = workloads.rhs(m.n, 1, seed=3)[:, 0].astype(dtype)
    B = workloads.rhs(m.n, 32, seed=4).astype(dtype)
    rp, ci, va = _dev(m, dtype)
    _, _, va2 = _dev(m2, dtype)
    sv = S.TriangularSolver(m.n, rp, ci, va, uplo, diag, "auto")
    algos = ["self", "level", "block", "slfc", "levc", "auto"]
    if case == "27pt_ilu_upper":
        algos.remove("block")                      # refused on natural partitions with > 3 deps per row
    bt, Bt = torch.from_numpy(b1).cuda(), torch.from_numpy(B).cuda()
    for algo in algos:                             # build every layout on the old values
        sv.set_algo(algo)
        sv.solve(bt)
        sv.solve(Bt)
    sv.update_values(rp, ci, va2)
    fresh = S.TriangularSolver(m.n, rp, ci, va2, uplo, diag, "self")
    ref = oracle.solve(m2.astype(dtype), b1, uplo, diag, dtype=dtype)
    for algo in algos:
        sv.set_algo(algo)
        fresh.set_algo(algo)
        x = sv.solve(bt).cpu().numpy()
        assert sv.solve_status() == "SUCCESS"
        assert relerr(x, ref) <= TOL[dtype], algo
        if algo not in ("slfc", "levc"):          # atomics: order varies run to run
            assert np.array_equal(x, fresh.solve(bt).cpu().numpy()), algo
            assert np.array_equal(sv.solve(Bt).cpu().numpy(), fresh.solve(Bt).cpu().numpy()), algo


def test_update_values_rejects_other_pattern_and_keeps_values(S):
    m = workloads.stencil((16, 16, 8), 7, "lower")
    rp, ci, va = _dev(m, np.float64)
    sv = S.TriangularSolver(m.n, rp, ci, va, "lower", "non_unit", "auto")
    b = torch.from_numpy(workloads.rhs(m.n, 1, seed=1)[:, 0]).cuda()
    x0 = sv.solve(b).cpu().numpy()
    # another pattern: drop the last off-diagonal entry of row 100 (moved into the upper part)
    ci2 = ci.clone()
    k = int(m.rowptr[101]) - 2                      # an off-diagonal of row 100 (diagonal last)
    ci2[k] = 100 + 1
    ci_sorted = ci2.cpu().numpy()
    row = ci_sorted[m.rowptr[100]:m.rowptr[101]]
    ci_sorted[m.rowptr[100]:m.rowptr[101]] = np.sort(row)
    with pytest.raises(S.SptrsvError) as e:
        sv.update_values(rp, torch.from_numpy(ci_sorted).cuda(), va)
    assert e.value.name == "INVALID_VALUE"
    # a zero pivot: ZERO_PIVOT, values kept
    va0 = va.clone()
    va0[int(m.rowptr[7]) + (int(m.rowptr[8]) - int(m.rowptr[7])) - 1] = 0.0   # diagonal of row 7 (last in its row)
    with pytest.raises(S.SptrsvError) as e:
        sv.update_values(rp, ci, va0)
    assert e.value.name == "ZERO_PIVOT"
    assert np.array_equal(sv.solve(b).cpu().numpy(), x0)


def test_stream_batch_equals_sequential(S):
    """NEXT-4 on one GPU: independent factor pairs issued concurrently on a
    stream pool (StreamBatch) give the sequential results bit for bit."""
    blocks, p = workloads.config(6, scale=0.25)
    chains, xs, ref = [], [], []
    for i, b in enumerate(blocks[:6]):
        hl = S.from_csr(b, "lower", "unit", algo="auto")
        hu = S.from_csr(b, "upper", "non_unit", algo="auto")
        r = torch.from_numpy(workloads.rhs(b.n, 1, seed=p["seed"] + i)[:, 0]).cuda()
        y, x = torch.empty_like(r), torch.empty_like(r)
        chains.append([(hl, r, y), (hu, y, x)])
        xs.append(x)
        ref.append(hu.solve(hl.solve(r)).cpu().numpy())
    S.StreamBatch(3).run(chains)
    torch.cuda.synchronize()
    for x, r in zip(xs, ref):
        assert np.array_equal(x.cpu().numpy(), r)
