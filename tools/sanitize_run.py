"""Small solves of every spin-wait kernel, for compute-sanitizer runs
(memcheck / racecheck / synccheck; scripts/gpu_sanitize.sh): cfg1 (2-D 5-point
32x32) with SELF, LEVEL, BLOCK, SLFC, LEVC; the value-as-flag multi-RHS kernel
(8 RHS) and the multi-RHS tile kernel (64 RHS) on a 7-point 16^3 grid.  Each
result is checked against the exact solution of an integer-exact system
(power-of-two diagonal, x_true in +-{1..4}: any summation order is exact)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402
from paper_1710_04985_b200 import sptrsv as S  # noqa: E402


def exact_system(m, nrhs, seed):
    """b = T x_true for an integer T (the CSR as given), by a plain sparse product."""
    xt = workloads.integer_xtrue(m.n, nrhs, seed)
    rows = np.repeat(np.arange(m.n), np.diff(m.rowptr))
    b = np.zeros((m.n, nrhs))
    np.add.at(b, rows, m.vals[:, None] * xt[m.colidx])
    return b, xt


which = sys.argv[1] if len(sys.argv) > 1 else "all"
ok = True
m1 = workloads.stencil((32, 32), 5, "lower", diag=4.0)
m3 = workloads.stencil((16, 16, 16), 7, "lower", diag=8.0)
cases = [("self", m1, 1), ("level", m1, 1), ("block", m1, 1), ("slfc", m1, 1), ("levc", m1, 1),
         ("vf8", m3, 8), ("mrt64", m3, 64), ("block3d", m3, 1)]
for name, m, nrhs in cases:
    if which not in ("all", name):
        continue
    algo = {"vf8": "self", "mrt64": "auto", "block3d": "block"}.get(name, name)
    b, xt = exact_system(m, nrhs, 7)
    sv = S.from_csr(m, algo=algo)
    bt = torch.from_numpy(b[:, 0] if nrhs == 1 else b).cuda()
    x = sv.solve(bt).cpu().numpy()
    st = sv.solve_status()
    good = st == "SUCCESS" and np.array_equal(x.reshape(m.n, -1), xt)
    ok &= good
    print(f"{name:8s} nrhs {nrhs:3d} status {st} exact {good}", flush=True)
print("ALL OK" if ok else "MISMATCH")
