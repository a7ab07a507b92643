"""CUDA-event time of BLOCK solves (L2 flushed before each) on 7-point grids, for A/B runs of
development variants (SPTRSV_DEV_LIB).  usage: python tools/variant_time.py TAG [DIMS ...]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
import oracle
from paper_1710_04985_b200 import sptrsv as S

tag = sys.argv[1]
specs = sys.argv[2:] or ["128x128x128"]
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for spec in specs:
    dims = tuple(int(v) for v in spec.split("x"))
    m = workloads.stencil(dims, 7, "lower")
    sv = S.from_csr(m, algo="block")
    bn = workloads.rhs(m.n, 1, seed=2)[:, 0]
    b = torch.from_numpy(bn).cuda()
    x = torch.empty_like(b)
    for _ in range(3):
        sv.solve(b, x)
    torch.cuda.synchronize()
    def loop(with_solve, k=20):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(k):
            flush.fill_(1.0)
            if with_solve:
                sv.solve(b, x)
        e1.record(); e1.synchronize()
        return e0.elapsed_time(e1) * 1e3 / k
    ts = []
    for _ in range(7):      # (flush + solve) - flush, 20 of each per sample: below the event granularity
        ts.append(loop(True) - loop(False))
    ok = sv.solve_status()
    ref = oracle.solve(m, bn) if m.n <= 300000 else None
    err = float(np.abs(x.cpu().numpy() - ref).max() / np.abs(ref).max()) if ref is not None else float("nan")
    print(f"{tag:12s} {spec:14s} median {np.median(ts):7.1f} us  p10 {np.percentile(ts, 10):7.1f}  min {min(ts):7.1f}  {ok} err {err:.1e}")
    sv.close()
