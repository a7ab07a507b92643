"""BLOCK development check: parity + timing on a set of grids, with the
per-warp step trace (sptrsv_dbg_block_trace) summarised.

python tools/block_dev.py [cfg2|one|all] [--trace]
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: parity of the dev runs)
import workloads  # noqa: E402
from paper_1710_04985_b200 import sptrsv as S  # noqa: E402

lib = ctypes.CDLL(S.LIB_PATH)
lib.sptrsv_dbg_block_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
lib.sptrsv_dbg_block_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p]

flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def timed(sv, b, x, reps=20, do_flush=True):
    ts = []
    for _ in range(3):
        sv.solve(b, x)
    torch.cuda.synchronize()
    for _ in range(reps):
        if do_flush:
            flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sv.solve(b, x)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts)), float(np.min(ts))


def plan(sv):
    out = (ctypes.c_longlong * 13)()
    lib.sptrsv_dbg_block_plan(ctypes.c_void_p(sv.handle), out)
    return dict(zip(["K", "wpc", "nsteps", "G", "nslots", "smem", "rec", "tw", "th", "cs", "csx", "items", "gl"], list(out)))


def run(name, m, uplo="lower", dtype=np.float64, trace=False, check=True):
    t0 = time.time()
    sv = S.from_csr(m, uplo, "non_unit", dtype, "block")
    ta = time.time() - t0
    info = sv.info()
    b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0].astype(dtype)).cuda()
    x = torch.empty_like(b)
    sv.solve(b, x)
    st = sv.solve_status()
    err = -1.0
    if check:
        ref = oracle.solve(m.astype(dtype), b.cpu().numpy(), uplo, dtype=dtype)
        xx = x.cpu().numpy()
        err = float(np.abs(xx - ref).max() / np.abs(ref).max())
    med, mn = timed(sv, b, x)
    es = 8 if dtype == np.float64 else 4
    nnz = info["nnz_used"] + m.n
    byts = 4 * (m.n + 1) + (4 + es) * nnz + 2 * es * m.n
    gbs = byts / (med * 1e-6) / 1e9
    p = plan(sv)
    print(f"{name:28s} n={m.n:8d} nlev={info['nlev']:5d} plan={p} analysis+build {ta*1e3:7.1f} ms | "
          f"status {st} err {err:.2e} | solve med {med:8.1f} us min {mn:8.1f} us | {gbs:7.1f} GB/s "
          f"({gbs/6526.8:.4f}) | {med*1e3/info['nlev']:6.1f} ns/level", flush=True)
    if trace:
        U = p["K"] * p["wpc"]
        cap = 4096
        buf = torch.zeros(U * cap, dtype=torch.int64, device="cuda")
        lib.sptrsv_dbg_block_trace(ctypes.c_void_p(sv.handle), ctypes.c_void_p(buf.data_ptr()), cap)
        sv.solve(b, x)
        torch.cuda.synchronize()
        lib.sptrsv_dbg_block_trace(ctypes.c_void_p(sv.handle), None, 0)
        tr = buf.view(U, cap).cpu().numpy().astype(np.float64)
        t0 = tr[tr > 0].min()
        starts = tr[:, 0] - t0
        ends = tr[:, cap - 1] - t0
        # per-warp step rate over the steps it recorded (every UB=4 steps)
        rates = []
        for u in range(U):
            r = tr[u, :cap - 1]
            idx = np.nonzero(r)[0]
            if len(idx) > 8:
                rates.append((r[idx[-1]] - r[idx[0]]) / (idx[-1] - idx[0]))
        rates = np.array(rates)
        print(f"   trace: start first {starts.min():.0f} ns last {starts.max():.0f} ns; end max {ends.max():.0f} ns; "
              f"ns/step per warp: min {rates.min():.1f} med {np.median(rates):.1f} max {rates.max():.1f}")
        order = np.argsort(starts)
        for u in list(order[:3]) + list(order[-3:]):
            print(f"     warp {u:4d} start {starts[u]:9.0f} end {ends[u]:9.0f}")
    return med


if __name__ == "__main__":
    which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    trace = "--trace" in sys.argv
    if which in ("one", "all"):
        for nz in (512, 2048):
            run(f"one tile 8x4x{nz}", workloads.stencil((8, 4, nz), 7, "lower"), trace=trace)
        run("one CTA 16x8x1024", workloads.stencil((16, 8, 1024), 7, "lower"), trace=trace)
        run("2 CTAs 32x8x1024", workloads.stencil((32, 8, 1024), 7, "lower"), trace=trace)
    if which in ("cfg2", "all"):
        m, _ = workloads.config(2)
        run("cfg2 f64", m, trace=trace)
        run("cfg2 f32", m, dtype=np.float32, trace=False)
    if which == "all":
        m, _ = workloads.config(1)
        run("cfg1", m, trace=trace)
        run("7pt upper 40x30x20", workloads.stencil((40, 30, 20), 7, "upper"), uplo="upper")
        run("27pt 24x20x12", workloads.ilu0(workloads.stencil((24, 20, 12), 27)), check=True)
