"""NEXT-3 (Table 2 / Eq. (5)): the solve pair of Eq. (3) -- (L+D) then
(U+D) of the Laplacian A = L + D + U -- on the paper's regular grids with
growing aspect ratios, 5/9-point (2-D) and 7/27-point (3-D) stencils, fp64 and
fp32.  GFLOP/s by Eq. (4) (2 nnz(A) per pair), effective GB/s
(compulsory bytes of both solves), nlev of the lower factor, AUTO
algorithm, L2 flushed before every timed pair (median of 10).  Prints markdown."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_1710_04985_b200 import sptrsv as S  # noqa: E402

GRIDS2 = [(1024, 1024), (512, 2048), (256, 4096), (128, 8192), (64, 16384)]
GRIDS3 = [(128, 128, 128), (64, 128, 256), (64, 64, 512), (32, 64, 1024), (32, 32, 2048)]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
which = sys.argv[1] if len(sys.argv) > 1 else "all"
dtypes = [np.float64, np.float32]
print("| grid | rho | stencil | dtype | n | nnz(A) | nlev | algo (L/U) | pair us | GFLOP/s (Eq. 4) | GB/s | frac of HBM |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for dims, pts_list, grids in (("2d", (5, 9), GRIDS2), ("3d", (7, 27), GRIDS3)):
    if which not in ("all", dims):
        continue
    for g in grids:
        rho = (g[1] // g[0]) if dims == "2d" else (g[2] // g[0])
        for pts in pts_list:
            full = workloads.stencil(g, pts, "full")
            lo = workloads.stencil(g, pts, "lower")
            up = workloads.stencil(g, pts, "upper")
            nnz_a = int(full.rowptr[-1])
            for dt in dtypes:
                es = 8 if dt == np.float64 else 4
                tdt = torch.float64 if dt == np.float64 else torch.float32
                hl = S.from_csr(lo, "lower", "non_unit", dt, "auto")
                hu = S.from_csr(up, "upper", "non_unit", dt, "auto")
                il, iu = hl.info(), hu.info()
                b = torch.from_numpy(workloads.rhs(full.n, 1, seed=5)[:, 0].astype(dt)).cuda()
                y, x = torch.empty_like(b), torch.empty_like(b)
                for _ in range(3):
                    hl.solve(b, y)
                    hu.solve(y, x)
                ts = []
                for _ in range(10):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    hl.solve(b, y)
                    hu.solve(y, x)
                    e1.record()
                    e1.synchronize()
                    ts.append(e0.elapsed_time(e1) * 1e-3)
                t = float(np.median(ts))
                n = full.n
                byts = sum(4 * (n + 1) + (4 + es) * (i["nnz_used"] + n) + 2 * es * n for i in (il, iu))
                gf = 2 * nnz_a / t / 1e9
                gbs = byts / t / 1e9
                names = {0: "self", 1: "level", 2: "block"}
                print(f"| {'x'.join(map(str, g))} | {rho} | {pts}-pt | {'f64' if es == 8 else 'f32'} | {n} | {nnz_a} | "
                      f"{il['nlev']} | {names.get(il['algo'])}/{names.get(iu['algo'])} | {t * 1e6:.1f} | {gf:.1f} | "
                      f"{gbs:.1f} | {gbs / 6453.1:.3f} |", flush=True)
                del hl, hu
