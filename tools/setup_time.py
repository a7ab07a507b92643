"""Setup (analysis) cost per configuration, warm process: the CSR is uploaded
once, then sptrsv_analyze (+ the algorithm's build, set_algo) is timed on the
host clock over a few repetitions.  Usage: python tools/setup_time.py [cfg ...]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_1710_04985_b200 import sptrsv as S  # noqa: E402

cfgs = [int(c) for c in sys.argv[1:]] or [1, 2, 3, 4]
w, wp = workloads.config(1)
S.from_csr(w, wp["uplo"], wp["diag"], algo="auto")          # context + module load
torch.cuda.synchronize()
for cfg in cfgs:
    m, p = workloads.config(cfg)
    solves = [("lower", "unit"), ("upper", "non_unit")] if cfg == 3 else [(p["uplo"], p["diag"])]
    rp = torch.from_numpy(np.ascontiguousarray(m.rowptr, dtype=np.int32)).cuda()
    ci = torch.from_numpy(np.ascontiguousarray(m.colidx, dtype=np.int32)).cuda()
    va = torch.from_numpy(np.ascontiguousarray(m.vals)).cuda()
    torch.cuda.synchronize()
    for uplo, diag in solves:
        for algo in ("self", "auto"):
            tot, an = [], []
            for _ in range(5):
                t0 = time.perf_counter()
                sv = S.TriangularSolver(m.n, rp, ci, va, uplo, diag, algo)
                torch.cuda.synchronize()
                tot.append(1e3 * (time.perf_counter() - t0))
                an.append(sv.info()["analysis_ms"])
                used = sv.info()["algo"]
                del sv
            print(f"cfg{cfg} {uplo:5s} {algo:4s} (algo {used}): analyze {np.median(an):7.2f} ms, "
                  f"analyze + build {np.median(tot):7.2f} ms (median of 5; all {[round(t, 1) for t in tot]})", flush=True)
