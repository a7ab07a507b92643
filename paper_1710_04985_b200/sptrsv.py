"""Thin ctypes binding of include/sptrsv.h -- argument marshalling only.

Every step of the path runs in libsptrsv.so (hand-written sm_100a kernels).
There is no fallback: if the library is missing or fails to load, importing
this module raises.  torch supplies device memory and streams only.

Low-level functions keep the C names (``sptrsv_analyze`` ... ``sptrsv_status_string``);
``TriangularSolver`` wraps a handle for tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import build as _build

# SPTRSV_DEV_LIB: a development variant of the library (tools/build_variant.py)
LIB_PATH = os.environ.get("SPTRSV_DEV_LIB") or _build.LIB

LOWER, UPPER = 0, 1
NON_UNIT, UNIT = 0, 1
F64, F32 = 0, 1
ALGO_SELF, ALGO_LEVEL, ALGO_BLOCK, ALGO_AUTO, ALGO_SLFC, ALGO_LEVC, ALGO_SMALL = 0, 1, 2, 3, 5, 6, 7
ALGOS = {"self": ALGO_SELF, "level": ALGO_LEVEL, "block": ALGO_BLOCK, "auto": ALGO_AUTO,
         "slfc": ALGO_SLFC, "levc": ALGO_LEVC, "small": ALGO_SMALL}
UPLO = {"lower": LOWER, "upper": UPPER}
DIAG = {"non_unit": NON_UNIT, "unit": UNIT}

STATUS_NAMES = {0: "SUCCESS", 1: "INVALID_VALUE", 2: "INVALID_MATRIX", 3: "ZERO_PIVOT", 4: "ALLOC",
                5: "CUDA", 6: "NOT_SUPPORTED", 7: "TIMEOUT"}


class sptrsv_info_t(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32), ("nlev", ctypes.c_int32), ("max_level_width", ctypes.c_int32),
        ("zero_pivot_row", ctypes.c_int32), ("bad_row", ctypes.c_int32),
        ("uplo", ctypes.c_int32), ("diag", ctypes.c_int32), ("dtype", ctypes.c_int32),
        ("algo", ctypes.c_int32), ("max_row_deps", ctypes.c_int32),
        ("nnz_input", ctypes.c_int64), ("nnz_used", ctypes.c_int64), ("ignored_entries", ctypes.c_int64),
        ("status", ctypes.c_int32), ("nblocks", ctypes.c_int32),
        ("analysis_ms", ctypes.c_double), ("device_bytes", ctypes.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libsptrsv.so not built at {LIB_PATH}: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i32 = ctypes.c_void_p, ctypes.c_int32
    lib.sptrsv_analyze.restype = ctypes.c_int
    lib.sptrsv_analyze.argtypes = [i32, vp, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                   ctypes.POINTER(vp)]
    lib.sptrsv_solve.restype = ctypes.c_int
    lib.sptrsv_solve.argtypes = [vp, vp, vp, i32, vp]
    lib.sptrsv_solve_host.restype = ctypes.c_int
    lib.sptrsv_solve_host.argtypes = [vp, vp, vp, i32, vp]
    lib.sptrsv_destroy.restype = ctypes.c_int
    lib.sptrsv_destroy.argtypes = [vp]
    lib.sptrsv_update_values.restype = ctypes.c_int
    lib.sptrsv_update_values.argtypes = [vp, vp, vp, vp, vp]
    lib.sptrsv_set_algo.restype = ctypes.c_int
    lib.sptrsv_set_algo.argtypes = [vp, ctypes.c_int]
    lib.sptrsv_get_info.restype = ctypes.c_int
    lib.sptrsv_get_info.argtypes = [vp, ctypes.POINTER(sptrsv_info_t)]
    lib.sptrsv_get_levels.restype = ctypes.c_int
    lib.sptrsv_get_levels.argtypes = [vp, vp, vp, vp]
    lib.sptrsv_get_dep_counts.restype = ctypes.c_int
    lib.sptrsv_get_dep_counts.argtypes = [vp, vp]
    lib.sptrsv_get_solve_status.restype = ctypes.c_int
    lib.sptrsv_get_solve_status.argtypes = [vp]
    lib.sptrsv_status_string.restype = ctypes.c_char_p
    lib.sptrsv_status_string.argtypes = [ctypes.c_int]
    lib.sptrsv_last_cuda_error.restype = ctypes.c_char_p
    lib.sptrsv_last_cuda_error.argtypes = []
    return lib


_lib = _load()


class SptrsvError(RuntimeError):
    def __init__(self, status: int, where: str, info: dict | None = None):
        name = STATUS_NAMES.get(status, str(status))
        extra = ""
        if status == 5:
            extra = " (" + _lib.sptrsv_last_cuda_error().decode() + ")"
        super().__init__(f"{where}: {name}{extra}")
        self.status = status
        self.name = name
        self.info = info or {}


# ----------------------------------------------------------- C-named calls
def sptrsv_status_string(status: int) -> str:
    return _lib.sptrsv_status_string(status).decode()


def sptrsv_analyze(n, rowptr_ptr, colidx_ptr, vals_ptr, uplo, diag, dtype, stream_ptr):
    """Returns (status, handle or None) exactly as the C call does."""
    h = ctypes.c_void_p()
    st = _lib.sptrsv_analyze(int(n), rowptr_ptr, colidx_ptr, vals_ptr, int(uplo), int(diag), int(dtype),
                             stream_ptr, ctypes.byref(h))
    return st, (h.value if h.value else None)


def sptrsv_solve(handle, b_ptr, x_ptr, nrhs, stream_ptr) -> int:
    return _lib.sptrsv_solve(handle, b_ptr, x_ptr, int(nrhs), stream_ptr)


def sptrsv_solve_host(handle, b_ptr, x_ptr, nrhs, stream_ptr) -> int:
    return _lib.sptrsv_solve_host(handle, b_ptr, x_ptr, int(nrhs), stream_ptr)


def sptrsv_destroy(handle) -> int:
    return _lib.sptrsv_destroy(handle)


def sptrsv_update_values(handle, rowptr_ptr, colidx_ptr, vals_ptr, stream_ptr) -> int:
    return _lib.sptrsv_update_values(handle, rowptr_ptr, colidx_ptr, vals_ptr, stream_ptr)


def sptrsv_set_algo(handle, algo) -> int:
    return _lib.sptrsv_set_algo(handle, int(algo))


def sptrsv_get_info(handle):
    info = sptrsv_info_t()
    st = _lib.sptrsv_get_info(handle, ctypes.byref(info))
    return st, info


def sptrsv_get_levels(handle, lev_ptr, ilev_ptr, jlev_ptr) -> int:
    return _lib.sptrsv_get_levels(handle, lev_ptr, ilev_ptr, jlev_ptr)


def sptrsv_get_dep_counts(handle, dp_ptr) -> int:
    return _lib.sptrsv_get_dep_counts(handle, dp_ptr)


def sptrsv_get_solve_status(handle) -> int:
    return _lib.sptrsv_get_solve_status(handle)


# ------------------------------------------------------------- wrapper
def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else None


class TriangularSolver:
    """Analyzed triangular factor on the current CUDA device.

    rowptr/colidx: int32 CUDA tensors; vals: float64/float32 CUDA tensor (the
    value dtype selects the solve precision).  The inputs may be freed after
    construction (the handle copies what it needs).
    """

    def __init__(self, n, rowptr, colidx, vals, uplo="lower", diag="non_unit", algo="self", stream=None):
        import torch
        dtype = F64 if vals is None or vals.dtype == torch.float64 else F32
        if vals is not None and vals.dtype not in (torch.float64, torch.float32):
            raise TypeError("vals must be float64 or float32")
        self.torch_dtype = torch.float64 if dtype == F64 else torch.float32
        self.n = int(n)
        for t in (rowptr, colidx):
            if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
                raise TypeError("rowptr/colidx must be contiguous int32 CUDA tensors")
        if rowptr.numel() != self.n + 1:
            raise ValueError(f"rowptr must have n + 1 = {self.n + 1} entries")
        nnz = int(rowptr[-1].item()) if self.n > 0 else 0
        if colidx.numel() < nnz:
            raise ValueError(f"colidx has {colidx.numel()} entries, rowptr[n] = {nnz}")
        if vals is not None:
            if not vals.is_cuda or not vals.is_contiguous() or vals.numel() < nnz:
                raise ValueError(f"vals must be a contiguous CUDA tensor of >= rowptr[n] = {nnz} values")
        st, h = sptrsv_analyze(self.n, _dptr(rowptr), _dptr(colidx), _dptr(vals), UPLO[uplo], DIAG[diag],
                               dtype, _stream_ptr(stream))
        self.handle = h
        if st != 0:
            info = self.info() if h else {}
            if h:
                sptrsv_destroy(h)
                self.handle = None
            raise SptrsvError(st, "sptrsv_analyze", info)
        if algo != "self":
            self.set_algo(algo)

    def update_values(self, rowptr, colidx, vals, stream=None):
        """New values for the analyzed pattern (same rowptr / colidx CUDA tensors'
        contents); raises SptrsvError (INVALID_VALUE: another pattern) and keeps
        the old values on failure."""
        import torch
        for t in (rowptr, colidx):
            if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
                raise TypeError("rowptr/colidx must be contiguous int32 CUDA tensors")
        if rowptr.numel() != self.n + 1:
            raise ValueError(f"rowptr must have n + 1 = {self.n + 1} entries")
        if vals is not None and (vals.dtype != self.torch_dtype or not vals.is_cuda or not vals.is_contiguous()):
            raise TypeError("vals must be a contiguous CUDA tensor of the handle's dtype")
        st = sptrsv_update_values(self.handle, _dptr(rowptr), _dptr(colidx), _dptr(vals), _stream_ptr(stream))
        if st != 0:
            raise SptrsvError(st, "sptrsv_update_values")

    def set_algo(self, algo: str):
        st = sptrsv_set_algo(self.handle, ALGOS[algo])
        if st != 0:
            raise SptrsvError(st, "sptrsv_set_algo")

    def info(self) -> dict:
        st, info = sptrsv_get_info(self.handle)
        if st != 0:
            raise SptrsvError(st, "sptrsv_get_info")
        return info.as_dict()

    def levels(self):
        info = self.info()
        lev = np.zeros(max(self.n, 1), dtype=np.int32)
        ilev = np.zeros(info["nlev"] + 1, dtype=np.int32)
        jlev = np.zeros(max(self.n, 1), dtype=np.int32)
        st = sptrsv_get_levels(self.handle, lev.ctypes.data_as(ctypes.c_void_p),
                               ilev.ctypes.data_as(ctypes.c_void_p), jlev.ctypes.data_as(ctypes.c_void_p))
        if st != 0:
            raise SptrsvError(st, "sptrsv_get_levels")
        return lev[:self.n], ilev, jlev[:self.n], info["nlev"]

    def dep_counts(self):
        dp = np.zeros(max(self.n, 1), dtype=np.int32)
        st = sptrsv_get_dep_counts(self.handle, dp.ctypes.data_as(ctypes.c_void_p))
        if st != 0:
            raise SptrsvError(st, "sptrsv_get_dep_counts")
        return dp[:self.n]

    def solve(self, b, x=None, stream=None):
        """x = T^{-1} b for a CUDA tensor b of shape (n,) or (n, nrhs), row-major."""
        import torch
        if b.dtype != self.torch_dtype or not b.is_cuda or not b.is_contiguous():
            raise TypeError(f"b must be a contiguous {self.torch_dtype} CUDA tensor")
        if b.dim() not in (1, 2) or b.shape[0] != self.n:
            raise ValueError(f"b must have shape ({self.n},) or ({self.n}, nrhs), got {tuple(b.shape)}")
        nrhs = 1 if b.dim() == 1 else b.shape[1]
        if x is None:
            x = torch.empty_like(b)
        elif (x.shape != b.shape or x.dtype != b.dtype or x.device != b.device or not x.is_contiguous()):
            raise TypeError("x must be a contiguous tensor with b's shape, dtype and device")
        st = sptrsv_solve(self.handle, _dptr(b), _dptr(x), nrhs, _stream_ptr(stream))
        if st != 0:
            raise SptrsvError(st, "sptrsv_solve")
        return x

    def solve_status(self) -> str:
        """Synchronizes; "SUCCESS", or "TIMEOUT" if the last (BLOCK) solve gave up a spin wait."""
        return STATUS_NAMES.get(sptrsv_get_solve_status(self.handle), "UNKNOWN")

    def solve_host(self, b, x=None, stream=None):
        """The same solve on HOST arrays (numpy or CPU tensors); copies are inside the call."""
        want = np.float64 if self.torch_dtype.is_floating_point and self.torch_dtype.itemsize == 8 else np.float32
        for name, a in (("b", b), ("x", x)):
            if a is None:
                continue
            arr = a if isinstance(a, np.ndarray) else a.numpy()
            if arr.dtype != want or not arr.flags["C_CONTIGUOUS"]:
                raise TypeError(f"{name} must be a C-contiguous {np.dtype(want).name} host array")
        if b.ndim not in (1, 2) or b.shape[0] != self.n:
            raise ValueError(f"b must have shape ({self.n},) or ({self.n}, nrhs), got {tuple(b.shape)}")
        nrhs = 1 if b.ndim == 1 else b.shape[1]
        if x is None:
            x = np.empty_like(b) if isinstance(b, np.ndarray) else b.new_empty(b.shape)
        elif tuple(x.shape) != tuple(b.shape):
            raise ValueError("x must have b's shape")
        bp = b.ctypes.data_as(ctypes.c_void_p) if isinstance(b, np.ndarray) else ctypes.c_void_p(b.data_ptr())
        xp = x.ctypes.data_as(ctypes.c_void_p) if isinstance(x, np.ndarray) else ctypes.c_void_p(x.data_ptr())
        st = sptrsv_solve_host(self.handle, bp, xp, nrhs, _stream_ptr(stream))
        if st != 0:
            raise SptrsvError(st, "sptrsv_solve_host")
        return x

    def close(self):
        if getattr(self, "handle", None):
            sptrsv_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StreamBatch:
    """Independent solves (NEXT-4: independent factors, or several RHS sets)
    issued concurrently: chain i (a list of (solver, b, x) solves run in
    order, e.g. an Eq. (3) pair) goes to stream i % nstreams of a small pool
    forked from and joined back into the caller's stream.  Latency-bound
    persistent solve kernels of independent handles then share the SMs.
    Marshalling only: each solve is an ordinary sptrsv_solve."""

    def __init__(self, nstreams: int = 4):
        import torch
        self.streams = [torch.cuda.Stream() for _ in range(max(1, int(nstreams)))]

    def run(self, chains, stream=None):
        import torch
        caller = stream or torch.cuda.current_stream()
        start = torch.cuda.Event()
        start.record(caller)
        for s in self.streams:
            s.wait_event(start)
        for i, chain in enumerate(chains):
            s = self.streams[i % len(self.streams)]
            for solver, b, x in chain:
                solver.solve(b, x, stream=s)
        for s in self.streams:
            done = torch.cuda.Event()
            done.record(s)
            caller.wait_event(done)


def from_csr(m, uplo="lower", diag="non_unit", dtype=None, algo="self", device="cuda"):
    """Upload a host CSR (workloads.CSR-like: n, rowptr, colidx, vals) and analyze it."""
    import torch
    dt = torch.float64 if dtype in (None, np.float64, torch.float64) else torch.float32
    rp = torch.from_numpy(np.ascontiguousarray(m.rowptr, dtype=np.int32)).to(device)
    ci = torch.from_numpy(np.ascontiguousarray(m.colidx, dtype=np.int32)).to(device)
    va = torch.from_numpy(np.ascontiguousarray(m.vals)).to(device=device, dtype=dt)
    return TriangularSolver(m.n, rp, ci, va, uplo, diag, algo)
