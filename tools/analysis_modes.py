"""Setup-phase study (NEXT-2; Tables 4-6): analysis time of every
configuration with each level computation -- Kahn by rounds in one
cooperative launch (default), the sync-free kernel, and the paper's host loop
with one launch per level (FIND_LEVEL) -- beside cuSPARSE SpSV's
analysis (warm context; CUDA events), all on device-resident CSR.
Prints a markdown table."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_1710_04985_b200 import sptrsv as S  # noqa: E402

lib = ctypes.CDLL(S.LIB_PATH)
cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4]
w, wp = workloads.config(1)
S.from_csr(w, wp["uplo"], wp["diag"])
try:
    import baseline
    bw = torch.ones(w.n, dtype=torch.float64, device="cuda")
    baseline.CusparseSpSV(w, "lower", "non_unit", bw, torch.empty_like(bw), np.float64)
except Exception as e:                     # context only
    baseline = None
    print("cuSPARSE unavailable:", e)
torch.cuda.synchronize()
names = {0: "Kahn rounds, 1 launch", 1: "sync-free", 2: "1 launch per level"}
print("| cfg | factor | nlev | " + " | ".join(names[m] + " ms" for m in (0, 1, 2)) + " | cuSPARSE SpSV analysis ms |")
print("|---|---|---|---|---|---|---|")
for cfg in cfgs:
    m, p = workloads.config(cfg)
    solves = [("lower", "unit"), ("upper", "non_unit")] if cfg == 3 else [(p["uplo"], p["diag"])]
    rp = torch.from_numpy(np.ascontiguousarray(m.rowptr, dtype=np.int32)).cuda()
    ci = torch.from_numpy(np.ascontiguousarray(m.colidx, dtype=np.int32)).cuda()
    va = torch.from_numpy(np.ascontiguousarray(m.vals)).cuda()
    for uplo, diag in solves:
        row = []
        nlev = None
        for mode in (0, 1, 2):
            lib.sptrsv_dbg_levels_mode(mode)
            ts = []
            for _ in range(3):
                sv = S.TriangularSolver(m.n, rp, ci, va, uplo, diag, "self")
                torch.cuda.synchronize()
                ts.append(sv.info()["analysis_ms"])
                nlev = sv.info()["nlev"]
                del sv
            row.append(float(np.median(ts)))
        lib.sptrsv_dbg_levels_mode(0)
        cs = None
        if baseline is not None:
            b = torch.ones(m.n, dtype=torch.float64, device="cuda")
            x = torch.empty_like(b)
            ts = []
            for _ in range(3):
                c = baseline.CusparseSpSV(m, uplo, diag, b, x, np.float64)
                ts.append(c.analysis_ms)
                del c
            cs = float(np.median(ts))
        print(f"| {cfg} | {uplo} {diag} | {nlev} | " + " | ".join(f"{t:.1f}" for t in row) +
              f" | {cs:.1f} |" if cs is not None else " | n/a |", flush=True)
