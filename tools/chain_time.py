"""BLOCK on a long dependency chain (bidiagonal, natural partition): CUDA-event
time of a solve after an L2 flush, for A/B runs of the prologue stagger."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S
tag = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
rp = np.arange(0, 2 * n, 2, dtype=np.int32); rp = np.concatenate([[0], np.minimum(np.arange(1, n + 1) * 2 - 1, 2 * n - 1)]).astype(np.int32)
ci = np.empty(rp[-1], dtype=np.int32); va = np.empty(rp[-1])
for i in range(n):
    a, b_ = rp[i], rp[i + 1]
    if b_ - a == 2: ci[a], va[a], ci[a + 1], va[a + 1] = i - 1, -0.5, i, 2.0
    else: ci[a], va[a] = i, 2.0
m = workloads.CSR(n, rp, ci, va, {})
sv = S.from_csr(m, algo="block")
b = torch.ones(n, dtype=torch.float64, device="cuda"); x = torch.empty_like(b)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(2): sv.solve(b, x)
torch.cuda.synchronize(); ts = []
for _ in range(5):
    flush.fill_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sv.solve(b, x); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1))
inf = sv.info()
print(f"{tag:8s} chain n={n}: {np.median(ts):.2f} ms  {sv.solve_status()}  algo {inf['algo']} blocks {inf['nblocks']} nlev {inf['nlev']}")
