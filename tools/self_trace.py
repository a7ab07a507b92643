"""Where does a SELF solve spend its time?  Publication time of every row
(debug hook sptrsv_dbg_self_trace) -> per row: ready time (latest publication
of its dependencies) and delay (own publication - ready).  Summarised by row
class (TPR <= 16 deps, WPR longer) and along the critical path.
usage: python tools/self_trace.py [cfg=4] [scale=1.0]"""
import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
m, p = workloads.config(cfg, scale)
if p.get("pair"):                      # cfg3: the forward (unit lower) solve
    p = dict(p, uplo="lower", diag="unit")
sv = S.from_csr(m, p["uplo"], p["diag"], algo="self")
n = m.n
b = torch.from_numpy(workloads.rhs(n, 1, seed=2)[:, 0]).cuda()
for _ in range(3):
    sv.solve(b)
torch.cuda.synchronize()
buf = torch.zeros(n, dtype=torch.int64, device="cuda")
lib = ctypes.CDLL(S.LIB_PATH)
assert lib.sptrsv_dbg_self_trace(ctypes.c_void_p(buf.data_ptr())) == 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); sv.solve(b); e1.record(); torch.cuda.synchronize()
lib.sptrsv_dbg_self_trace(None)
tp = buf.cpu().numpy().astype(np.int64)
assert (tp > 0).all(), "rows without a publication stamp"
tp = (tp - tp.min()) / 1e3          # us
lev, _, _, nlev = sv.levels()
# strict lower part of the matrix: dependencies
rp, ci = m.rowptr.astype(np.int64), m.colidx.astype(np.int64)
row_of = np.repeat(np.arange(n), np.diff(rp))
strict = (ci < row_of) if p["uplo"] == "lower" else (ci > row_of)
deps_row, deps_col = row_of[strict], ci[strict]
ndeps = np.bincount(deps_row, minlength=n)
ready = np.full(n, 0.0)
np.maximum.at(ready, deps_row, tp[deps_col])
delay = tp - ready
# critical predecessor of every row (latest dependency)
crit = np.full(n, -1, dtype=np.int64)
order = np.lexsort((tp[deps_col], deps_row))
last = np.r_[deps_row[order][1:] != deps_row[order][:-1], True]
crit[deps_row[order][last]] = deps_col[order][last]
end = int(np.argmax(tp))
path = [end]
while crit[path[-1]] >= 0:
    path.append(int(crit[path[-1]]))
path = np.array(path[::-1])
wpr = ndeps > 16


def summ(mask):
    d = delay[mask]
    return {"rows": int(mask.sum()), "delay_us_median": round(float(np.median(d)), 3) if d.size else None,
            "p90": round(float(np.percentile(d, 90)), 3) if d.size else None,
            "mean": round(float(d.mean()), 3) if d.size else None}


out = {"cfg": cfg, "n": n, "nlev": int(nlev), "solve_us": round(e0.elapsed_time(e1) * 1e3, 1),
       "last_pub_us": round(float(tp.max()), 1),
       "tpr": summ(~wpr & (ndeps > 0)), "wpr": summ(wpr), "level0": summ(ndeps == 0),
       "critical_path": {"hops": int(len(path) - 1), "us_per_hop": round(float(tp.max() / max(1, len(path) - 1)), 3),
                         "delay_tpr_sum_us": round(float(delay[path][~wpr[path]].sum()), 1),
                         "delay_wpr_sum_us": round(float(delay[path][wpr[path]].sum()), 1),
                         "wpr_hops": int(wpr[path].sum()),
                         "ndeps_median_on_path": float(np.median(ndeps[path]))}}
for lo, hi in ((17, 64), (65, 256), (257, 1024), (1025, 5000)):
    out[f"wpr_{lo}_{hi}"] = summ((ndeps >= lo) & (ndeps <= hi))
print(json.dumps(out))
