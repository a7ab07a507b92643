"""Per-CTA group timeline of the multi-RHS tile kernel on cfg5 (64 RHS):
barrier times and producer-ready times per group, summarised."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S
lib = ctypes.CDLL(S.LIB_PATH)
lib.sptrsv_dbg_mrt_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m, _ = workloads.config(5)
B = torch.from_numpy(workloads.rhs_columns(m.n, range(nrhs))).cuda()
sv = S.from_csr(m, algo="auto")
X = sv.solve(B)
torch.cuda.synchronize()
K = ctypes.c_int(0)
cap = 512
lib.sptrsv_dbg_mrt_trace(ctypes.c_void_p(sv.handle), None, 0, ctypes.byref(K))
K = K.value
buf = torch.zeros(K * cap * 2, dtype=torch.int64, device="cuda")
lib.sptrsv_dbg_mrt_trace(ctypes.c_void_p(sv.handle), ctypes.c_void_p(buf.data_ptr()), cap, None)
sv.solve(B, X)
torch.cuda.synchronize()
lib.sptrsv_dbg_mrt_trace(ctypes.c_void_p(sv.handle), None, 0, None)
tr = buf.view(K, cap, 2).cpu().numpy().astype(np.float64)
t0 = tr[tr > 0].min()
bar = np.where(tr[:, :, 0] > 0, tr[:, :, 0] - t0, np.nan)
rdy = np.where(tr[:, :, 1] > 0, tr[:, :, 1] - t0, np.nan)
print("K", K, "end", np.nanmax(bar))
for c in [0, 1, 8, K // 2, K - 1]:
    b_ = bar[c][~np.isnan(bar[c])]
    r_ = rdy[c][~np.isnan(rdy[c])]
    d = np.diff(b_)
    print(f"CTA {c:3d}: groups {len(b_)} first {b_[0]:8.0f} last {b_[-1]:8.0f} per-group ns p10 {np.percentile(d,10):.0f} p50 {np.median(d):.0f} p90 {np.percentile(d,90):.0f}")
    n = min(len(b_), len(r_))
    w = r_[:n] - b_[:n]
    print(f"          group start -> next group prepared (producers ready, halo issued): p50 {np.median(w):.0f} p90 {np.percentile(w,90):.0f}")


