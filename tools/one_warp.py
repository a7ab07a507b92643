"""Intrinsic BLOCK step cost: a 7-point grid of one warp tile (8 x 4 columns,
nz levels deep) -> one warp, one CTA; time per level = solve time / nlev."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

nz = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
m = workloads.stencil((8, 4, nz), 7, "lower")
sv = S.from_csr(m, algo="block")
info = sv.info()
b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
x = torch.empty_like(b)
for _ in range(3):
    sv.solve(b, x)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sv.solve(b, x); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
t = float(np.median(ts))
print(f"one-warp: n={m.n} nlev={info['nlev']} blocks={info['nblocks']} solve {t:.1f} us -> {t * 1e3 / info['nlev']:.1f} ns/level")
