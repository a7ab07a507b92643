"""Hop cost of SPTRSV_ALGO_BLOCK: a 7-point grid of T warp tiles along x
(8T x 4 x nz), tiles grouped WX per CTA (env SPTRSV_BLOCK_WX/WY set by the
caller).  time(T) ~ nlev * t_step + (T - 1) * t_hop."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

nz = 1024
out = {}
for T in (1, 2, 4, 8, 16):
    m = workloads.stencil((8 * T, 4, nz), 7, "lower")
    sv = S.from_csr(m, algo="block")
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
    out[T] = {"us": round(t, 1), "nlev": info["nlev"], "ctas": info["nblocks"], "ns_per_level": round(t * 1e3 / info["nlev"], 1)}
    sv.close()
print(json.dumps({"WX": os.environ.get("SPTRSV_BLOCK_WX"), "res": out}))
