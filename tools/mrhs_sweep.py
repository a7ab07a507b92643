"""Per-rank cfg5 work on one GPU: the cfg2 factor with nrhs = 64/G right-hand
sides (G = 1, 2, 4, 8), per multi-RHS kernel.  usage: python tools/mrhs_sweep.py"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

m, p = workloads.config(2)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for nrhs in (64, 32, 16, 8):
    B = torch.from_numpy(workloads.rhs(m.n, nrhs, seed=1000)).cuda()
    X = torch.empty_like(B)
    res = {}
    for algo, env in (("auto", None), ("self", None), ("vf", "1")):
        os.environ.pop("SPTRSV_MRHS_VF", None)
        if env:
            os.environ["SPTRSV_MRHS_VF"] = env
            if nrhs > 32:
                continue
        sv = S.from_csr(m, algo="self" if algo == "vf" else algo)
        for _ in range(3):
            sv.solve(B, X)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); sv.solve(B, X); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[algo] = round(float(np.median(ts)), 3)
        del sv
    print(f"nrhs={nrhs} (G={64 // nrhs}) ms:", res, flush=True)
