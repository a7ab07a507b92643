"""Launch / fixed cost of a BLOCK solve: CUDA-event time of one solve after an L2 flush,
one solve right after another, and the mean of 20 back-to-back solves.
usage: python tools/launch_oh.py DIMS [DIMS ...]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
small = torch.empty(1024, dtype=torch.float32, device="cuda")


def ev(fn, pre=None, reps=10):
    ts = []
    for _ in range(reps):
        if pre is not None:
            pre()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


for spec in sys.argv[1:]:
    dims = tuple(int(v) for v in spec.split("x"))
    m = workloads.stencil(dims, 7, "lower")
    sv = S.from_csr(m, algo="block")
    b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
    x = torch.empty_like(b)
    for _ in range(3):
        sv.solve(b, x)
    torch.cuda.synchronize()
    one = lambda: sv.solve(b, x)
    r_flush = ev(one, lambda: flush.fill_(1.0))
    r_small = ev(one, lambda: small.fill_(1.0))
    r_prev = ev(one, one)
    r_20 = ev(lambda: [sv.solve(b, x) for _ in range(20)], reps=5) / 20
    e_fill = ev(lambda: small.fill_(1.0))
    print(f"{spec}: nlev {sv.info()['nlev']}: after flush {r_flush:.1f} us, after tiny kernel {r_small:.1f} us, "
          f"after a solve {r_prev:.1f} us, 20 back-to-back {r_20:.1f} us/solve; tiny fill kernel alone {e_fill:.1f} us")
    sv.close()
