"""Seeded synthetic workloads for the SpTRSV path (inputs only -- no solve arithmetic).

Shared by ``tests/``, ``bench.py`` and ``__graft_entry__.smoke()``.  Neither the
oracle (``oracle/``) nor the CUDA library (``paper_1710_04985_b200``) imports
this module; callers hand its numpy arrays to both sides.

Recipes follow SURVEY.md §8c O-7 / §8d and are restated in DESIGN.md
("Input recipe"):

* ``stencil``   -- 2-D 5/9-point and 3-D 7/27-point Laplacians (§5.1,
  P:872-884), lexicographic with x fastest, off-diagonal -1, Dirichlet diagonal.
* ``ilu0``      -- ILU(0) (IKJ) factors sharing A's pattern.
* ``powerlaw``  -- generated lower factor with power-law row lengths and explicit
  levels (stand-in for the paper's SuiteSparse set).
* ``rhs``       -- x_true ~ U[-1,1) (numpy PCG64), and the integer variant.
* ``config(k)`` -- the five BASELINE.json configurations.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libworkloads.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile gen.c into libworkloads.so (host C, no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32p = ctypes.POINTER(ctypes.c_int32)
        f64p = ctypes.POINTER(ctypes.c_double)
        lib.gen_stencil.restype = ctypes.c_int64
        lib.gen_stencil.argtypes = [ctypes.c_int32] * 5 + [ctypes.c_double, ctypes.c_double,
                                                          ctypes.c_void_p, ctypes.c_void_p,
                                                          ctypes.c_void_p]
        lib.gen_ilu0.restype = ctypes.c_int32
        lib.gen_ilu0.argtypes = [ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.gen_powerlaw.restype = ctypes.c_int64
        lib.gen_powerlaw.argtypes = [ctypes.c_int32] * 4 + [ctypes.c_uint64,
                                                           ctypes.POINTER(i32p), ctypes.POINTER(i32p),
                                                           ctypes.POINTER(f64p), ctypes.POINTER(i32p)]
        lib.gen_free.restype = None
        lib.gen_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class CSR:
    """A square CSR matrix: 0-based int32 indices, strictly increasing columns per row."""
    n: int
    rowptr: np.ndarray
    colidx: np.ndarray
    vals: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def astype(self, dtype) -> "CSR":
        return CSR(self.n, self.rowptr, self.colidx, self.vals.astype(dtype), dict(self.meta))

    def to_dense(self) -> np.ndarray:
        a = np.zeros((self.n, self.n), dtype=self.vals.dtype)
        for i in range(self.n):
            for k in range(self.rowptr[i], self.rowptr[i + 1]):
                a[i, self.colidx[k]] = self.vals[k]
        return a


_STENCIL_DIAG = {5: 4.0, 9: 8.0, 7: 6.0, 27: 26.0}
_PART = {"full": 0, "lower": 1, "upper": 2}


def stencil(dims, points: int, part: str = "full", diag: float | None = None,
            off: float = -1.0) -> CSR:
    """Laplacian on an nx x ny (x nz) grid; ``part`` in {full, lower, upper}.

    The diagonal defaults to the Dirichlet constant 4/8/6/26 (reading Q16);
    ``lower``/``upper`` keep the diagonal (L+D / U+D of Eq. (2)).
    """
    dims = tuple(int(d) for d in dims)
    nx, ny, nz = (dims + (1, 1))[:3]
    dval = _STENCIL_DIAG[points] if diag is None else float(diag)
    lib = _load()
    n = nx * ny * nz
    rowptr = np.zeros(n + 1, dtype=np.int32)
    nnz = lib.gen_stencil(nx, ny, nz, points, _PART[part], dval, off, _ptr(rowptr), None, None)
    if nnz < 0:
        raise ValueError(f"bad stencil arguments {dims} {points}")
    colidx = np.empty(nnz, dtype=np.int32)
    vals = np.empty(nnz, dtype=np.float64)
    lib.gen_stencil(nx, ny, nz, points, _PART[part], dval, off, _ptr(rowptr), _ptr(colidx), _ptr(vals))
    return CSR(n, rowptr, colidx, vals, {"kind": "stencil", "dims": (nx, ny, nz), "points": points,
                                          "part": part, "diag": dval})


def ilu0(a: CSR) -> CSR:
    """ILU(0) of ``a`` (IKJ, Saad Alg. 10.4), returned as ONE combined CSR:
    strict lower = L (unit diagonal implied), diagonal + strict upper = U."""
    vals = np.array(a.vals, dtype=np.float64, copy=True)
    rc = _load().gen_ilu0(a.n, _ptr(a.rowptr), _ptr(a.colidx), _ptr(vals))
    if rc != 0:
        raise ValueError(f"ILU(0) breakdown at row {-rc - 1}")
    meta = dict(a.meta)
    meta["kind"] = "ilu0"
    return CSR(a.n, a.rowptr, a.colidx, vals, meta)


def powerlaw(n: int, nlev: int, seed: int, maxlen: int = 4096, locality: int = 512):
    """cfg4 generator.  Returns (CSR of L+D, intended 0-based levels)."""
    lib = _load()
    rp = ctypes.POINTER(ctypes.c_int32)()
    ci = ctypes.POINTER(ctypes.c_int32)()
    va = ctypes.POINTER(ctypes.c_double)()
    lv = ctypes.POINTER(ctypes.c_int32)()
    nnz = lib.gen_powerlaw(n, nlev, maxlen, locality, seed, ctypes.byref(rp), ctypes.byref(ci),
                           ctypes.byref(va), ctypes.byref(lv))
    if nnz < 0:
        raise ValueError("powerlaw generator failed")
    try:
        rowptr = np.ctypeslib.as_array(rp, shape=(n + 1,)).copy()
        colidx = np.ctypeslib.as_array(ci, shape=(nnz,)).copy()
        vals = np.ctypeslib.as_array(va, shape=(nnz,)).copy()
        lev = np.ctypeslib.as_array(lv, shape=(n,)).copy()
    finally:
        for p in (rp, ci, va, lv):
            lib.gen_free(ctypes.cast(p, ctypes.c_void_p))
    return CSR(n, rowptr, colidx, vals, {"kind": "powerlaw", "nlev": nlev, "seed": seed}), lev


def rhs(n: int, nrhs: int, seed: int, dtype=np.float64) -> np.ndarray:
    """Row-major (n, nrhs) right-hand side, U[-1,1) from numpy PCG64 (reading Q15)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(n, nrhs)).astype(dtype)


def rhs_columns(n: int, cols, base_seed: int = 1000, dtype=np.float64) -> np.ndarray:
    """cfg5: column r drawn from seed base_seed + r, so any column block of the 64
    RHS is reproducible on any rank without generating the others."""
    cols = list(cols)
    out = np.empty((n, len(cols)), dtype=dtype)
    for c, r in enumerate(cols):
        out[:, c] = np.random.default_rng(base_seed + r).uniform(-1.0, 1.0, size=n)
    return out


def integer_xtrue(n: int, nrhs: int, seed: int) -> np.ndarray:
    """x_true with entries in {+-1..+-4} for the integer-exact pin."""
    rng = np.random.default_rng(seed)
    mag = rng.integers(1, 5, size=(n, nrhs))
    sgn = np.where(rng.integers(0, 2, size=(n, nrhs)) == 0, -1, 1)
    return (mag * sgn).astype(np.float64)


# ------------------------------------------------------------------ configs
CONFIGS = {
    1: "lower triangle of 2D 5-point Laplacian 32x32 (n=1024), fp64, single RHS",
    2: "lower triangle of 3D 7-point Laplacian 128^3 (n=2097152), fp64",
    3: "ILU(0) L and U of 3D 27-point 96^3, forward+backward",
    4: "generated power-law lower triangular, n=4194304, nlev=12288, fp64",
    5: "64 independent RHS on the 3D 7-point 128^3 factor",
}

SEEDS = {1: 1, 2: 2, 3: 3, 4: 4, 5: 1000}


def slab_thicknesses(nz: int, nblocks: int, seed: int) -> list[int]:
    """Thicknesses (>= 1) of ``nblocks`` z-slabs summing to ``nz``: a seeded
    random composition (uneven subdomains, so the batch partition matters)."""
    rng = np.random.default_rng(seed)
    w = rng.uniform(0.5, 1.5, size=nblocks)
    t = np.maximum(1, np.floor(w / w.sum() * nz).astype(int))
    t[int(np.argmax(t))] += nz - int(t.sum())
    assert t.min() >= 1 and int(t.sum()) == nz
    return [int(v) for v in t]


def block_jacobi_ilu0(dims=(128, 128, 128), points: int = 27, nblocks: int = 16, seed: int = 6) -> list:
    """NEXT-4 workload: a block-Jacobi preconditioner of the ``points``-point
    Laplacian on ``dims``, split into ``nblocks`` z-slabs (couplings between
    slabs dropped); each block's ILU(0) (IKJ, reading Q19) as one combined CSR
    -- independent factors, each solved as the Eq. (3) pair (unit L, then U)."""
    nx, ny, nz = dims
    return [ilu0(stencil((nx, ny, t), points, "full")) for t in slab_thicknesses(nz, nblocks, seed)]


def config(k: int, scale: float = 1.0):
    """Matrix for configuration ``k``.  ``scale`` < 1 shrinks the grid / n for
    fast tests (same recipe).  Returns (CSR, dict of solve parameters)."""
    if k == 1:
        g = max(2, int(round(32 * scale)))
        m = stencil((g, g), 5, "lower")
        return m, {"uplo": "lower", "diag": "non_unit", "nrhs": 1, "seed": 1}
    if k in (2, 5):
        g = max(2, int(round(128 * scale)))
        m = stencil((g, g, g), 7, "lower")
        return m, {"uplo": "lower", "diag": "non_unit", "nrhs": 1 if k == 2 else 64,
                   "seed": SEEDS[k]}
    if k == 3:
        g = max(2, int(round(96 * scale)))
        m = ilu0(stencil((g, g, g), 27, "full"))
        return m, {"pair": True, "seed": 3}
    if k == 4:
        n = max(1024, int(4194304 * scale))
        nlev = max(4, int(12288 * scale))
        m, lev = powerlaw(n, nlev, seed=4)
        m.meta["lev"] = lev
        return m, {"uplo": "lower", "diag": "non_unit", "nrhs": 1, "seed": 5}
    if k == 6:
        g = max(4, int(round(128 * scale)))
        blocks = block_jacobi_ilu0((g, g, g), 27, 16, seed=6)
        return blocks, {"pair": True, "seed": 7, "blocks": True}
    raise KeyError(k)
