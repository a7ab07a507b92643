"""Small BLOCK solves (debugging aid): 2-D 32x32 and 3-D 16^3 stencils vs the oracle."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, workloads
from paper_1710_04985_b200 import sptrsv as S

for dims, pts in [((32, 32), 5), ((16, 16, 16), 7), ((40, 30, 20), 7)]:
    m = workloads.stencil(dims, pts, "lower")
    b = workloads.rhs(m.n, 1, seed=1)[:, 0]
    sv = S.from_csr(m, algo="block")
    x = sv.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    ref = oracle.solve(m, b)
    print(dims, sv.info()["nblocks"], float(np.abs(x - ref).max() / np.abs(ref).max()), flush=True)
