"""Intrinsic per-level cost of a single-CTA tile solve: 7-point grid of one
CTA tile (dims from argv, default 16 x 8 x 2048), algo from argv."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

algo = sys.argv[1] if len(sys.argv) > 1 else "tile"
dims = tuple(int(v) for v in sys.argv[2].split("x")) if len(sys.argv) > 2 else (16, 8, 2048)
m = workloads.stencil(dims, 7, "lower")
sv = S.from_csr(m, algo=algo)
info = sv.info()
b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
x = torch.empty_like(b)
for _ in range(3):
    sv.solve(b, x)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sv.solve(b, x); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
t = float(np.median(ts))
print(f"{algo} {dims}: nlev={info['nlev']} ctas={info['nblocks']} solve {t:.1f} us -> {t * 1e3 / info['nlev']:.1f} ns/level")
