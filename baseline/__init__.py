"""Context baselines for bench.py (not the product): cuSPARSE SpSV and SpSM."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "cusparse_spsv.cu")
LIB = os.path.join(HERE, "libspsv_cusparse.so")
_lib = None


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    nvcc = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-Xcompiler", "-fPIC",
                           "-shared", "-o", tmp, SRC, "-lcusparse"])
    os.replace(tmp, LIB)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(LIB)
        vp = ctypes.c_void_p
        lib.spsv_create.restype = ctypes.c_int
        lib.spsv_create.argtypes = [ctypes.c_int, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, vp, vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_float)]
        lib.spsv_solve.restype = ctypes.c_int
        lib.spsv_solve.argtypes = [vp, vp]
        lib.spsv_destroy.restype = None
        lib.spsv_destroy.argtypes = [vp]
        lib.spsm_create.restype = ctypes.c_int
        lib.spsm_create.argtypes = [ctypes.c_int, ctypes.c_int64, vp, vp, vp, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, vp, vp, ctypes.POINTER(vp),
                                    ctypes.POINTER(ctypes.c_float)]
        lib.spsm_solve.restype = ctypes.c_int
        lib.spsm_solve.argtypes = [vp, vp]
        lib.spsm_destroy.restype = None
        lib.spsm_destroy.argtypes = [vp]
        _lib = lib
    return _lib


def triangle(m, uplo: str, keep_diag: bool):
    """CSR (numpy) of the referenced triangle of m (diagonal kept if keep_diag)."""
    n = m.n
    rows = np.repeat(np.arange(n), np.diff(m.rowptr))
    c = m.colidx
    keep = (c < rows) if uplo == "lower" else (c > rows)
    if keep_diag:
        keep |= c == rows
    rp = np.zeros(n + 1, dtype=np.int32)
    np.cumsum(np.bincount(rows[keep], minlength=n), out=rp[1:])
    return rp, c[keep].astype(np.int32), m.vals[keep]


class CusparseSpSV:
    """cuSPARSE SpSV on one triangle: x = T^{-1} b, b / x torch CUDA tensors."""

    def __init__(self, m, uplo, diag, b, x, dtype=np.float64):
        import torch
        rp, ci, va = triangle(m, uplo, keep_diag=True)
        self._keep = [torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                      torch.from_numpy(va.astype(dtype)).cuda(), b, x]
        out = ctypes.c_void_p()
        an = ctypes.c_float(0.0)
        st = _load().spsv_create(m.n, int(ci.size), self._keep[0].data_ptr(), self._keep[1].data_ptr(),
                                 self._keep[2].data_ptr(), int(uplo == "upper"), int(diag == "unit"),
                                 int(dtype == np.float32), b.data_ptr(), x.data_ptr(), ctypes.byref(out),
                                 ctypes.byref(an))
        self.analysis_ms = float(an.value)      # cusparseSpSV_analysis alone (CUDA events)
        if st != 0:
            raise RuntimeError(f"cuSPARSE SpSV setup failed ({st})")
        self.ctx = out

    def solve(self, stream_ptr: int):
        st = _load().spsv_solve(self.ctx, ctypes.c_void_p(stream_ptr))
        if st != 0:
            raise RuntimeError(f"cuSPARSE SpSV solve failed ({st})")

    def __del__(self):
        try:
            _load().spsv_destroy(self.ctx)
        except Exception:
            pass


class CusparseSpSM:
    """cuSPARSE SpSM on one triangle: X = T^{-1} B, B / X row-major (n, nrhs) torch CUDA tensors."""

    def __init__(self, m, uplo, diag, b, x, dtype=np.float64):
        import torch
        rp, ci, va = triangle(m, uplo, keep_diag=True)
        self._keep = [torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda(),
                      torch.from_numpy(va.astype(dtype)).cuda(), b, x]
        out = ctypes.c_void_p()
        an = ctypes.c_float(0.0)
        st = _load().spsm_create(m.n, int(ci.size), self._keep[0].data_ptr(), self._keep[1].data_ptr(),
                                 self._keep[2].data_ptr(), int(uplo == "upper"), int(diag == "unit"),
                                 int(dtype == np.float32), int(b.shape[1]), b.data_ptr(), x.data_ptr(),
                                 ctypes.byref(out), ctypes.byref(an))
        self.analysis_ms = float(an.value)      # cusparseSpSM_analysis alone (CUDA events)
        if st != 0:
            raise RuntimeError(f"cuSPARSE SpSM setup failed ({st})")
        self.ctx = out

    def solve(self, stream_ptr: int):
        st = _load().spsm_solve(self.ctx, ctypes.c_void_p(stream_ptr))
        if st != 0:
            raise RuntimeError(f"cuSPARSE SpSM solve failed ({st})")

    def __del__(self):
        try:
            _load().spsm_destroy(self.ctx)
        except Exception:
            pass
