"""Where BLOCK's cfg2 time goes: the 128^3 7-point L+D solved with the
couplings across warp-tile / CTA / cluster boundaries dropped (the partition
stays the same, so each variant removes one class of hand-off).

  none     the real cfg2 factor
  cluster  no edges between clusters      (only warp, CTA and DSMEM hand-offs)
  cta      no edges between CTAs          (only in-CTA hand-offs)
  warp     no edges between warp tiles    (every warp independent: step time
                                            with all 512 warps streaming at once)

usage: python tools/decouple.py [N=128] [reps=20] [none|cluster|cta|warp]
"""
import os
import sys

import ctypes

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_1710_04985_b200 import sptrsv as S  # noqa: E402


def plan_of(sv):
    lib = ctypes.CDLL(S.LIB_PATH)
    lib.sptrsv_dbg_block_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    out = (ctypes.c_longlong * 13)()
    lib.sptrsv_dbg_block_plan(ctypes.c_void_p(sv.handle), out)
    return list(out)


def drop(m, nx, ny, ex, ey):
    """CSR with every off-diagonal entry crossing an x boundary (multiple of ex)
    or a y boundary (multiple of ey) removed."""
    rows = np.repeat(np.arange(m.n), np.diff(m.rowptr))
    c = m.colidx.astype(np.int64)
    xr, yr = rows % nx, (rows // nx) % ny
    xc, yc = c % nx, (c // nx) % ny
    keep = (rows == c) | ((xr // ex == xc // ex) & (yr // ey == yc // ey))
    rp = np.zeros(m.n + 1, dtype=np.int32)
    np.add.at(rp, rows[keep] + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    return workloads.CSR(m.n, rp, m.colidx[keep].copy(), m.vals[keep].copy(), dict(m.meta))


def timeit(sv, b, x, reps):
    for _ in range(3):
        sv.solve(b, x)
    torch.cuda.synchronize()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sv.solve(b, x)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts)), float(np.min(ts))


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    only = sys.argv[3] if len(sys.argv) > 3 else None     # run one variant only (for ncu)
    m = workloads.stencil((N, N, N), 7, "lower")
    b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
    x = torch.empty_like(b)
    sv = S.from_csr(m, algo="block")
    plan = plan_of(sv)
    print("plan", plan, "nlev", sv.info()["nlev"])
    tw, th = int(plan[7]), int(plan[8])
    cs, csx = int(plan[9]), int(plan[10])
    cx, cy = 2 * tw, 2 * th                      # CTA = 2 x 2 warp tiles on cfg2
    kx, ky = csx, max(1, cs // max(csx, 1))
    res = {"none": timeit(sv, b, x, reps)} if only in (None, "none") else {}
    sv.close()
    for name, ex, ey in (("cluster", cx * kx, cy * ky), ("cta", cx, cy), ("warp", tw, th)):
        if only not in (None, name):
            continue
        md = drop(m, N, N, ex, ey)
        svd = S.from_csr(md, algo="block")
        p = plan_of(svd)
        assert tuple(p[:2]) == tuple(plan[:2]) and p[7] == tw and p[8] == th, (name, p)
        res[name] = timeit(svd, b, x, reps)
        lev = svd.info()["nlev"]
        svd.close()
        print(f"{name:8s} edges kept inside {ex}x{ey}: nlev {lev}")
    for k, (med, mn) in res.items():
        print(f"{k:8s} median {med:8.1f} us  min {mn:8.1f} us")


if __name__ == "__main__":
    main()
