"""Wavefront timeline of one BLOCK solve on a 3-D 7-point grid (debug hook):
where does the time go -- tile start lags (hand-offs between tiles) or the
tiles' own step rate?  usage: python tools/wave_trace.py [nx ny nz]"""
import ctypes, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads
from paper_1710_04985_b200 import sptrsv as S

dims = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (128, 128, 128)
TW, TH = int(os.environ.get("SPTRSV_BLOCK_TW", 8)), 4
WX, WY = int(os.environ.get("SPTRSV_BLOCK_WX", 2)), int(os.environ.get("SPTRSV_BLOCK_WY", 2))
m = workloads.stencil(dims, 7, "lower")
sv = S.from_csr(m, algo="block")
info = sv.info()
wpc = WX * WY
U = info["nblocks"] * wpc
cap = 1024
buf = torch.zeros(U * cap, dtype=torch.int64, device="cuda")
lib = ctypes.CDLL(S.LIB_PATH)
b = torch.from_numpy(workloads.rhs(m.n, 1, seed=2)[:, 0]).cuda()
for _ in range(3):
    sv.solve(b)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(); sv.solve(b); ev1.record(); torch.cuda.synchronize()
t_plain = ev0.elapsed_time(ev1) * 1e3
assert lib.sptrsv_dbg_block_trace(ctypes.c_void_p(buf.data_ptr()), cap) == 0
ev0.record(); sv.solve(b); ev1.record(); torch.cuda.synchronize()
lib.sptrsv_dbg_block_trace(None, 0)
t = buf.view(U, cap).cpu().numpy().astype(np.int64)
t0 = t[:, :cap - 16][t[:, :cap - 16] > 0].min()
ntx = (dims[0] + TW - 1) // TW
cxn = (ntx + WX - 1) // WX
rows = []
for u in range(U):
    r = t[u]
    nz = np.nonzero(r[:cap - 16])[0]
    if len(nz) < 2 or r[cap - 1] == 0:
        continue
    cta, w = divmod(u, wpc)
    tx = (cta % cxn) * WX + w % WX
    ty = (cta // cxn) * WY + w // WX
    st = (r[nz] - t0) / 1e3
    steps = nz[-1]
    rows.append(dict(u=u, cta=cta, tx=tx, ty=ty, off=tx * TW + ty * TH, start=st[0], end=(r[cap - 1] - t0) / 1e3,
                     slow_cyc_per_step=float(r[cap - 2]) / max(1, steps), bw_cyc_per_step=float(r[cap - 3]) / max(1, steps),
                     slow_frac=float(r[cap - 4]) / max(1, steps),
                     dbg=[int(v) for v in r[cap - 16:cap - 8]],
                     mid_step_ns=float(np.median(np.diff(st) / np.diff(nz)) * 1e3), steps=int(steps)))
off = np.array([r["off"] for r in rows]); start = np.array([r["start"] for r in rows])
end = np.array([r["end"] for r in rows])
A = np.vstack([off, np.ones_like(off)]).T
slope = np.linalg.lstsq(A, start, rcond=None)[0][0]
byxy = {(r["tx"], r["ty"]): r for r in rows}
lag = {"x_same": [], "x_cross": [], "y_same": [], "y_cross": []}
for (tx, ty), r in byxy.items():
    for dx, dy, key, span in ((1, 0, "x", TW), (0, 1, "y", TH)):
        q = byxy.get((tx - dx, ty - dy))
        if q is None:
            continue
        kind = "same" if q["cta"] == r["cta"] else "cross"
        lag[f"{key}_{kind}"].append((r["start"] - q["start"]) * 1e3)
out = {"dims": dims, "solve_us_plain": round(t_plain, 1), "tiles": len(rows), "last_end_us": float(end.max()),
       "start_ns_per_offset_level": round(slope * 1e3, 1),
       "median_tile_step_ns": float(np.median([r["mid_step_ns"] for r in rows])),
       "median_tile_duration_us": float(np.median(end - start)),
       "median_slow_cyc_per_step": float(np.median([r["slow_cyc_per_step"] for r in rows])),
       "median_bw_cyc_per_step": float(np.median([r["bw_cyc_per_step"] for r in rows])),
       "median_slow_frac": float(np.median([r["slow_frac"] for r in rows])),
       "dbg_median_per_step [start, glob_slow, n_glob_slow, smem_slow, block_work, -, -, n_smem_slow]":
           [round(float(np.median([r["dbg"][i] / r["steps"] for r in rows])), 2) for i in range(8)],
       "start_lag_ns": {k: (round(float(np.median(v)), 1) if v else None) for k, v in lag.items()}}
print(json.dumps(out))
# global fit: time a tile reaches its block k vs the level it is at (off + UB k)
pts = []
for u_ in range(U):
    r = t[u_]
    nz = np.nonzero(r[:cap - 16])[0]
    cta, w = divmod(u_, wpc)
    tx = (cta % cxn) * WX + w % WX
    ty = (cta // cxn) * WY + w // WX
    for i in nz[1:]:
        pts.append((tx * TW + ty * TH + i, (r[i] - t0) / 1e3))
P = np.array(pts)
A = np.vstack([P[:, 0], np.ones(len(P))]).T
fit = np.linalg.lstsq(A, P[:, 1], rcond=None)[0]
print(json.dumps({"level_fit_ns_per_level": round(fit[0] * 1e3, 1), "fit_t0_us": round(fit[1], 2)}))
diag = [byxy[(i, 2 * i)] for i in range(0, min(ntx, 16), 3) if (i, 2 * i) in byxy]
print(json.dumps([{k: (round(v, 1) if isinstance(v, float) else v) for k, v in d.items()} for d in diag]))
last = max(rows, key=lambda r: r["end"])
print(json.dumps({"last_tile": last}))
