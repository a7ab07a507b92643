"""Multi-RHS development check: parity vs the oracle (sampled columns) and
timing of the tile kernel vs the other multi-RHS kernels on cfg5 (64 RHS on
the 128^3 7-point factor) and its per-rank widths 32 / 16 / 8."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (dev parity check)
import workloads  # noqa: E402
from paper_1710_04985_b200 import sptrsv as S  # noqa: E402

lib = ctypes.CDLL(S.LIB_PATH)
lib.sptrsv_dbg_mrhs_path.argtypes = [ctypes.c_void_p, ctypes.c_int]
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
m, _ = workloads.config(5)
es = 8
nnz = 8339456
for nrhs in [int(a) for a in (sys.argv[1:] or ["64", "32", "16", "8"])]:
    B = workloads.rhs_columns(m.n, range(nrhs))
    Bt = torch.from_numpy(B).cuda()
    for path in (0, 1):
        sv = S.from_csr(m, algo="auto")
        lib.sptrsv_dbg_mrhs_path(ctypes.c_void_p(sv.handle), path)
        X = sv.solve(Bt)
        st = sv.solve_status()
        cols = [0, nrhs - 1]
        ref = oracle.solve(m, np.ascontiguousarray(B[:, cols]))
        err = np.abs(X.cpu().numpy()[:, cols] - ref).max() / np.abs(ref).max()
        ts = []
        for _ in range(3):
            sv.solve(Bt, X)
        for _ in range(10):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sv.solve(Bt, X)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        med = float(np.median(ts))
        byts = 4 * (m.n + 1) + (4 + es) * nnz + 2 * es * m.n * nrhs
        print(f"nrhs {nrhs:3d} path {'tile' if path == 0 else 'old '} status {st} err {err:.1e} "
              f"median {med:8.1f} us  {byts / med / 1e3:7.1f} GB/s ({byts / med / 1e3 / 6453.1:.3f})", flush=True)
