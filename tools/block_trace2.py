"""Dump the per-warp BLOCK step trace of one cfg2-like solve to gpurun_out/trace_<tag>.npz
(timestamps of every 4th step per warp, plan summary) for offline analysis."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

tag = sys.argv[1] if len(sys.argv) > 1 else "x"
g = int(sys.argv[2]) if len(sys.argv) > 2 else 128
lib = ctypes.CDLL(S.LIB_PATH)
lib.sptrsv_dbg_block_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
lib.sptrsv_dbg_block_plan.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.sptrsv_dbg_block_ftrace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.sptrsv_dbg_block_items.argtypes = [ctypes.c_void_p] * 4
lib.sptrsv_dbg_block_ptrace.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
m = workloads.stencil((g, g, g), 7, "lower")
sv = S.from_csr(m, algo="block")
out = (ctypes.c_longlong * 13)()
lib.sptrsv_dbg_block_plan(ctypes.c_void_p(sv.handle), out)
K, wpc = out[0], out[1]
U = K * wpc
cap = 1024
b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
x = torch.empty_like(b)
for _ in range(3):
    sv.solve(b, x)
buf = torch.zeros(U * cap, dtype=torch.int64, device="cuda")
nit = int(out[11])
fbuf = torch.zeros(max(nit, 1), dtype=torch.int64, device="cuda")
lib.sptrsv_dbg_block_trace(ctypes.c_void_p(sv.handle), ctypes.c_void_p(buf.data_ptr()), cap)
lib.sptrsv_dbg_block_ftrace(ctypes.c_void_p(sv.handle), ctypes.c_void_p(fbuf.data_ptr()))
pbuf = torch.zeros(max(int(out[3]), 1), dtype=torch.int64, device="cuda")
lib.sptrsv_dbg_block_ptrace(ctypes.c_void_p(sv.handle), ctypes.c_void_p(pbuf.data_ptr()))
sv.solve(b, x)
torch.cuda.synchronize()
lib.sptrsv_dbg_block_trace(ctypes.c_void_p(sv.handle), None, 0)
lib.sptrsv_dbg_block_ftrace(ctypes.c_void_p(sv.handle), None)
lib.sptrsv_dbg_block_ptrace(ctypes.c_void_p(sv.handle), None)
items = np.zeros((max(nit, 1), 2), dtype=np.int32)
fptr = np.zeros(U + 1, dtype=np.int32)
keys = np.zeros(max(nit, 1), dtype=np.uint32)
lib.sptrsv_dbg_block_items(ctypes.c_void_p(sv.handle), items.ctypes.data_as(ctypes.c_void_p),
                           fptr.ctypes.data_as(ctypes.c_void_p), keys.ctypes.data_as(ctypes.c_void_p))
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed(f"gpurun_out/trace_{tag}.npz", tr=buf.view(U, cap).cpu().numpy(), plan=np.array(list(out)), g=g,
                    ftr=fbuf.cpu().numpy(), ptr=pbuf.cpu().numpy(), items=items, fptr=fptr, keys=keys, nlev=sv.info()["nlev"])
print("saved", U, "warps", sv.solve_status())
