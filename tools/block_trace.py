"""Per-CTA timelines of one SPTRSV_ALGO_BLOCK solve (debug hook), summarised."""
import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
m, p = workloads.config(cfg)
uplo, diag = ("lower", "unit") if cfg == 3 else (p["uplo"], p["diag"])
sv = S.from_csr(m, uplo, diag, algo="block")
info = sv.info()
K = info["nblocks"] * 8          # >= warps (wpc <= 8)
cap = 4096
buf = torch.zeros(K * cap, dtype=torch.int64, device="cuda")
lib = ctypes.CDLL(S.LIB_PATH)
b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
for _ in range(3):
    sv.solve(b)
torch.cuda.synchronize()
assert lib.sptrsv_dbg_block_trace(ctypes.c_void_p(buf.data_ptr()), cap) == 0
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda"); flush.zero_()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ph = torch.zeros(6 * 128, dtype=torch.int64, device="cuda")
lib.sptrsv_dbg_block_phase(ctypes.c_void_p(ph.data_ptr()))
ev0.record(); sv.solve(b); ev1.record(); torch.cuda.synchronize()
lib.sptrsv_dbg_block_trace(None, 0)
lib.sptrsv_dbg_block_phase(None)
P = ph.view(128, 6).cpu().numpy().astype(np.int64)
d = np.diff(P, axis=1)
print("warp0 cycles, median steps 8..120: cp.async wait | compute+stores+syncwarp | issue+wait(s+PB) | cp.async+wait(s+1) | load fields:",
      np.median(d[8:120], axis=0).tolist(), " loop gap:", float(np.median(P[9:120, 0] - P[8:119, 5])))


t = buf.view(K, cap).cpu().numpy()
os.makedirs("gpurun_out", exist_ok=True)
np.savez_compressed(f"gpurun_out/trace_cfg{cfg}.npz", t=t, info=json.dumps(info))
t0 = t[t > 0].min()
out = {"solve_us": ev0.elapsed_time(ev1) * 1e3, "K": K, "ctas": []}
durs = []
for k in range(K):
    row = t[k]
    nz = np.nonzero(row)[0]
    if len(nz) < 2:
        continue
    ts = row[nz] - t0
    d = np.diff(ts) / np.maximum(1, np.diff(nz))     # entries may be per block of steps
    durs.append(d)
    out["ctas"].append({"warp": k, "start_us": ts[0] / 1e3, "end_us": ts[-1] / 1e3, "steps": int(nz[-1]),
                        "step_med_ns": float(np.median(d)), "step_p90_ns": float(np.percentile(d, 90))})
alld = np.concatenate(durs)
out["step_ns_median"] = float(np.median(alld)); out["step_ns_p90"] = float(np.percentile(alld, 90))
out["step_ns_mean"] = float(alld.mean())
ends = [c["end_us"] for c in out["ctas"]]; starts = [c["start_us"] for c in out["ctas"]]
out["first_start_us"] = min(starts); out["last_start_us"] = max(starts); out["last_end_us"] = max(ends)
print(json.dumps({k: v for k, v in out.items() if k != "ctas"}))
sel = sorted(out["ctas"], key=lambda c: c["warp"])
for c in sel[:: max(1, len(sel) // 12)]:
    print(json.dumps(c))
