"""Where BLOCK's cfg2 critical path waits, from a block_trace2 dump taken with
the per-step trace (trc[t] = %globaltimer when step t's inputs were present)
and the mailbox publication trace (ptrace)."""
import sys
import numpy as np
d = np.load(sys.argv[1])
tr = d["tr"].astype(np.float64)
nlev = int(d["nlev"])
plan = d["plan"]
K, wpc = int(plan[0]), int(plan[1])
ftr, ptr, items, keys = d["ftr"].astype(np.float64), d["ptr"].astype(np.float64), d["items"], d["keys"].astype(np.int64)
U, cap = tr.shape
t0 = tr[tr > 0].min()
# step intervals
dl = []
for u in range(U):
    r = tr[u, :cap - 1]
    idx = np.nonzero(r)[0]
    if len(idx) > 8:
        dl.append(np.diff(r[idx]))
dl = np.concatenate(dl)
print("step interval ns: p10 %.0f p50 %.0f p90 %.0f p99 %.0f; share of time in steps > 400 ns: %.2f" %
      (*np.percentile(dl, [10, 50, 90, 99]), dl[dl > 400].sum() / dl.sum()))
# publication -> fetched, and fetched/published -> first ready warp of the consumer CTA at that level
lat = ftr - ptr[items[:, 0]]
print("publish -> fetched ns: p10 %.0f p50 %.0f p90 %.0f" % tuple(np.percentile(lat, [10, 50, 90])))
# per warp: level of step t = first level + t; first level from the first nonzero? use lev keys: for CTA c, level L
# the warp's step index of level L is L - L0(u), L0(u) = min level of its rows: unknown here, estimate from items' keys
cta = keys // nlev        # consumer warp
lev = keys % nlev
res = []
for c in np.unique(cta):
    sel = np.nonzero(cta == c)[0]
    for L in np.unique(lev[sel]):
        s2 = sel[lev[sel] == L]
        res.append((c, L, ptr[items[s2, 0]].max(), ftr[s2].max()))
res = np.array(res)
print("(CTA, level) groups with inbound items:", len(res))
print("last publication -> last fetch of a group ns: p10 %.0f p50 %.0f p90 %.0f p99 %.0f" %
      tuple(np.percentile(res[:, 3] - res[:, 2], [10, 50, 90, 99])))
