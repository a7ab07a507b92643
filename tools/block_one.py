"""One BLOCK solve of a single-warp-tile 7-point grid (8 x 4 x nz): the
intrinsic per-step cost, for ncu source-level stall sampling."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

nz = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dims = (8, 4, nz) if len(sys.argv) <= 2 else tuple(int(v) for v in sys.argv[2].split("x"))
m = workloads.stencil(dims, 7, "lower")
sv = S.from_csr(m, algo="block")
b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
x = torch.empty_like(b)
for _ in range(3):
    sv.solve(b, x)
torch.cuda.synchronize()
print("ok", sv.solve_status())
