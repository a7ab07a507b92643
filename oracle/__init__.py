"""CPU ORACLE for the SpTRSV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_1710_04985_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle.c`` (plain sequential C, fp64, built with
``-ffp-contract=off``); this file only marshals numpy arrays through ctypes.
Every function cites the PAPER.md passage it follows; readings of the paper
(Q1..Q21) are listed in DESIGN.md.

Parity status: every oracle function below is pinned by ``tests/test_oracle_*.py``
(closed forms, the paper's Fig. 1 example, brute-force dense solves, DFS longest
paths, integer-exact solutions, backward-error bounds).  None is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

STATUS = {0: "SUCCESS", 1: "INVALID_VALUE", 2: "INVALID_MATRIX", 3: "ZERO_PIVOT", 4: "ALLOC"}
_UPLO = {"lower": 0, "upper": 1}
_DIAG = {"non_unit": 0, "unit": 1}


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-shared", "-fPIC", "-o", tmp,
                               _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        lib.oracle_select.restype = ctypes.c_int
        lib.oracle_select.argtypes = [i32, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, vp]
        lib.oracle_levels_row.restype = i32
        lib.oracle_levels_row.argtypes = [i32, vp, vp, ctypes.c_int, vp]
        lib.oracle_levels_col.restype = i32
        lib.oracle_levels_col.argtypes = [i32, vp, vp, ctypes.c_int, vp]
        lib.oracle_schedule.restype = None
        lib.oracle_schedule.argtypes = [i32, vp, i32, vp, vp]
        for name in ("oracle_solve_f64", "oracle_solve_f32"):
            f = getattr(lib, name)
            f.restype = ctypes.c_int
            f.argtypes = [i32, vp, vp, vp, ctypes.c_int, ctypes.c_int, i32, vp, vp]
        lib.oracle_solve_col_f64.restype = ctypes.c_int
        lib.oracle_solve_col_f64.argtypes = [i32, vp, vp, vp, ctypes.c_int, ctypes.c_int, vp, vp]
        lib.oracle_kahn.restype = i32
        lib.oracle_kahn.argtypes = [i32, vp, vp, ctypes.c_int, vp, vp, vp]
        lib.oracle_backward_error.restype = ctypes.c_double
        lib.oracle_backward_error.argtypes = [i32, vp, vp, vp, ctypes.c_int, ctypes.c_int, i32, vp, vp]
        lib.oracle_matvec_ld.restype = None
        lib.oracle_matvec_ld.argtypes = [i32, vp, vp, vp, ctypes.c_int, ctypes.c_int, i32, vp, vp]
        _ = i64
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _csr(m):
    rowptr = np.ascontiguousarray(m.rowptr, dtype=np.int32)
    colidx = np.ascontiguousarray(m.colidx, dtype=np.int32)
    return rowptr, colidx


class OracleError(RuntimeError):
    def __init__(self, status, info=None):
        super().__init__(f"oracle: {status} {info or ''}")
        self.status = status
        self.info = info or {}


def select(m, uplo="lower", diag="non_unit"):
    """O-1/O-2: status name + dp counts + diagnostics."""
    rowptr, colidx = _csr(m)
    vals = np.ascontiguousarray(m.vals, dtype=np.float64)
    n = m.n
    dp = np.zeros(max(n, 1), dtype=np.int32)
    dk = np.zeros(max(n, 1), dtype=np.int32)
    ign = ctypes.c_int64(0)
    used = ctypes.c_int64(0)
    bad = ctypes.c_int32(-1)
    zp = ctypes.c_int32(-1)
    st = _load().oracle_select(n, _p(rowptr), _p(colidx), _p(vals), _UPLO[uplo], _DIAG[diag],
                               _p(dp), _p(dk), ctypes.byref(ign), ctypes.byref(used),
                               ctypes.byref(bad), ctypes.byref(zp))
    return {"status": STATUS[st], "dp": dp[:n], "diagk": dk[:n], "ignored": ign.value,
            "nnz_used": used.value, "bad_row": bad.value, "zero_pivot_row": zp.value}


def levels(m, uplo="lower", method="row"):
    """O-3 levels (0-based, reading Q4): ``row`` = P:240-249, ``col`` = P:250-258."""
    rowptr, colidx = _csr(m)
    lev = np.zeros(max(m.n, 1), dtype=np.int32)
    fn = _load().oracle_levels_row if method == "row" else _load().oracle_levels_col
    nlev = fn(m.n, _p(rowptr), _p(colidx), _UPLO[uplo], _p(lev))
    if nlev < 0:
        raise MemoryError
    return lev[:m.n], int(nlev)


def schedule(lev, nlev):
    """O-4: ilev[nlev+1], jlev[n] by stable counting sort."""
    lev = np.ascontiguousarray(lev, dtype=np.int32)
    n = lev.shape[0]
    ilev = np.zeros(nlev + 1, dtype=np.int32)
    jlev = np.zeros(max(n, 1), dtype=np.int32)
    _load().oracle_schedule(n, _p(lev), nlev, _p(ilev), _p(jlev))
    return ilev, jlev[:n]


def analyze(m, uplo="lower", diag="non_unit"):
    """O-1..O-4 in one call: what sptrsv_analyze must reproduce bit-exactly."""
    sel = select(m, uplo, diag)
    if sel["status"] != "SUCCESS":
        return sel
    lev, nlev = levels(m, uplo, "row")
    ilev, jlev = schedule(lev, nlev)
    widths = np.diff(ilev) if nlev > 0 else np.zeros(0, dtype=np.int32)
    sel.update({"lev": lev, "nlev": nlev, "ilev": ilev, "jlev": jlev,
                "max_level_width": int(widths.max()) if nlev > 0 else 0})
    return sel


def solve(m, b, uplo="lower", diag="non_unit", dtype=np.float64):
    """O-5: x = T^{-1} b, b row-major (n,) or (n, nrhs)."""
    rowptr, colidx = _csr(m)
    b = np.asarray(b)
    squeeze = b.ndim == 1
    b2 = np.ascontiguousarray(b.reshape(m.n, -1), dtype=dtype)
    nrhs = b2.shape[1] if m.n > 0 else (b.shape[1] if b.ndim == 2 else 1)
    x = np.zeros_like(b2)
    vals = np.ascontiguousarray(m.vals, dtype=dtype)
    fn = _load().oracle_solve_f64 if dtype == np.float64 else _load().oracle_solve_f32
    st = fn(m.n, _p(rowptr), _p(colidx), _p(vals), _UPLO[uplo], _DIAG[diag], max(nrhs, 1),
            _p(b2), _p(x))
    if st != 0:
        raise OracleError(STATUS[st])
    return x.reshape(-1) if squeeze else x


def solve_col(m, b, uplo="lower", diag="non_unit"):
    """Column-wise sweep over the CSC of the referenced strict
    triangle: x := f; x(i) /= d(i); x(jb) -= b x(i).  One fp64 RHS."""
    rowptr, colidx = _csr(m)
    f = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(-1))
    x = np.zeros_like(f)
    vals = np.ascontiguousarray(m.vals, dtype=np.float64)
    st = _load().oracle_solve_col_f64(m.n, _p(rowptr), _p(colidx), _p(vals), _UPLO[uplo], _DIAG[diag],
                                      _p(f), _p(x))
    if st != 0:
        raise OracleError(STATUS[st])
    return x


def pair_solve(m, b, dtype=np.float64):
    """O-6, Eq. (3) on a combined ILU(0) CSR: y = U^{-1} (L^{-1} b) with
    L unit lower (strict part of m) and U = diagonal + strict upper part of m."""
    z = solve(m, b, "lower", "unit", dtype)
    return solve(m, z, "upper", "non_unit", dtype)


def kahn(m, uplo="lower"):
    """A18 Kahn rounds: (ilev, jlev, lev, nlev); sets per level are unique."""
    rowptr, colidx = _csr(m)
    n = m.n
    ilev = np.zeros(n + 1, dtype=np.int32)
    jlev = np.zeros(max(n, 1), dtype=np.int32)
    lev = np.zeros(max(n, 1), dtype=np.int32)
    nlev = _load().oracle_kahn(n, _p(rowptr), _p(colidx), _UPLO[uplo], _p(ilev), _p(jlev), _p(lev))
    if nlev < 0:
        raise OracleError("CYCLE")
    return ilev[:nlev + 1], jlev[:n], lev[:n], int(nlev)


def backward_error(m, b, x, uplo="lower", diag="non_unit"):
    """max_i |b - T x|_i / (|T||x|)_i in long double (pin helper, Higham Thm 8.5)."""
    rowptr, colidx = _csr(m)
    b2 = np.ascontiguousarray(np.asarray(b, dtype=np.float64).reshape(m.n, -1))
    x2 = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(m.n, -1))
    vals = np.ascontiguousarray(m.vals, dtype=np.float64)
    return float(_load().oracle_backward_error(m.n, _p(rowptr), _p(colidx), _p(vals), _UPLO[uplo],
                                               _DIAG[diag], b2.shape[1], _p(b2), _p(x2)))


def matvec(m, x, uplo="lower", diag="non_unit"):
    """b = T x accumulated in long double (builds b from a known x_true)."""
    rowptr, colidx = _csr(m)
    x2 = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(m.n, -1))
    b = np.zeros_like(x2)
    vals = np.ascontiguousarray(m.vals, dtype=np.float64)
    _load().oracle_matvec_ld(m.n, _p(rowptr), _p(colidx), _p(vals), _UPLO[uplo], _DIAG[diag],
                             x2.shape[1], _p(x2), _p(b))
    return b.reshape(np.asarray(x).shape)
