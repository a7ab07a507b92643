import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import workloads, oracle
from paper_1710_04985_b200 import sptrsv as S
from test_oracle_levels import chain
lib = ctypes.CDLL(S.LIB_PATH)
lib.sptrsv_dbg_set_timeout_ns.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong]
lib.sptrsv_dbg_block_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
m = chain(200000, sub=-0.5, d=1.0)
b = workloads.rhs(m.n, 1, seed=4)[:, 0]
sv = S.from_csr(m, algo="block")
out = (ctypes.c_longlong * 13)(); lib.sptrsv_dbg_block_plan(ctypes.c_void_p(sv.handle), out); print("plan", list(out))
bt = torch.from_numpy(b).cuda()
for tmo in (4_000_000_000, 0, 1000, 0, 4_000_000_000):
    lib.sptrsv_dbg_set_timeout_ns(ctypes.c_void_p(sv.handle), tmo)
    torch.cuda.synchronize(); t0 = time.time()
    x = sv.solve(bt)
    st = sv.solve_status(); dt = time.time() - t0
    err = np.abs(x.cpu().numpy() - oracle.solve(m, b)).max()
    print("timeout", tmo, "status", st, "time %.1f ms" % (dt * 1e3), "err", err)
