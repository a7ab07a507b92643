"""Lag per tile crossing and per-warp step rate from a block_trace2 dump (7-point g^3 grid,
8x4 warp tiles, 2x2 tiles per CTA): T_u(level) per warp, then lags between neighbours."""
import sys
import numpy as np
d = np.load(sys.argv[1])
tr = d["tr"].astype(np.float64)
g = int(d["g"])
K, wpc = int(d["plan"][0]), int(d["plan"][1])
tw, th = int(d["plan"][7]), int(d["plan"][8])
ntx, nty = g // tw, g // th
wx = 2 if wpc >= 2 else 1
wy = wpc // wx
cxn = ntx // wx
cs, csx = (int(d["plan"][9]), int(d["plan"][10])) if len(d["plan"]) > 9 else (1, 1)
csy = cs // csx
t0 = tr[tr > 0].min()
U, cap = tr.shape
T = {}
for u in range(U):
    cta, w = divmod(u, wpc)
    cl, rk = divmod(cta, cs)
    ccx, ccy = cl % (cxn // csx), cl // (cxn // csx)
    cx, cy = ccx * csx + rk % csx, ccy * csy + rk // csx
    tx, ty = cx * wx + w % wx, cy * wy + w // wx
    T[(tx, ty)] = tr[u]
def at(tx, ty, lev):
    t = lev - (tx * tw + ty * th)
    r = T[(tx, ty)]
    if t < 0 or t >= cap - 1 or t % 4: return np.nan
    v = r[t]
    return v - t0 if v > 0 else np.nan
# per crossing lag at a mid level for the diagonal chain of tiles
print("tile grid", ntx, nty, "K", K, "wpc", wpc)
lags_x, lags_y = [], []
for tx in range(ntx - 1):
    for ty in range(nty):
        lev = tx * tw + ty * th + 64
        lev -= lev % 4
        a, b = at(tx, ty, lev), at(tx + 1, ty, lev + tw - (tw % 4))
        # compare at the same global level: b's level lev is at its t = lev - origin
        a = at(tx, ty, lev + tw); b = at(tx + 1, ty, lev + tw)
        if not np.isnan(a) and not np.isnan(b): lags_x.append((b - a, (tx % wx == wx - 1)))
for ty in range(nty - 1):
    for tx in range(ntx):
        lev = tx * tw + ty * th + 64 + th
        lev -= lev % 4
        a = at(tx, ty, lev); b = at(tx, ty + 1, lev)
        if not np.isnan(a) and not np.isnan(b): lags_y.append((b - a, (ty % wy == wy - 1)))
lx = np.array(lags_x); ly = np.array(lags_y)
for nm, l in (("x", lx), ("y", ly)):
    cross = l[l[:, 1] == 1, 0]; inner = l[l[:, 1] == 0, 0]
    print(f"lag {nm}: CTA crossing median {np.median(cross):.0f} ns (n={len(cross)}), in-CTA median {np.median(inner) if len(inner) else float('nan'):.0f} ns")
print("cluster", cs, "=", csx, "x", csy)
# crossings by kind along x / y: warp (in CTA), CTA (in cluster), cluster
for nm, dx, dy in (("x", 1, 0), ("y", 0, 1)):
    kinds = {"warp": [], "cta": [], "cluster": []}
    for (tx, ty) in T:
        if (tx + dx, ty + dy) not in T: continue
        lev = tx * tw + ty * th + 64 + (tw if dx else th); lev -= lev % 4
        a_, b_ = at(tx, ty, lev), at(tx + dx, ty + dy, lev)
        if np.isnan(a_) or np.isnan(b_): continue
        c1x, c1y = tx // wx, ty // wy
        c2x, c2y = (tx + dx) // wx, (ty + dy) // wy
        if (c1x, c1y) == (c2x, c2y): kinds["warp"].append(b_ - a_)
        elif (c1x // csx, c1y // csy) == (c2x // csx, c2y // csy): kinds["cta"].append(b_ - a_)
        else: kinds["cluster"].append(b_ - a_)
    print(nm, {k: (f"{np.median(v):.0f} ns", len(v)) for k, v in kinds.items() if v})
# step rate per warp (ns per step) over its middle
rates = []
for k, r in T.items():
    idx = np.nonzero(r[:cap - 1])[0]
    if len(idx) > 16:
        a, b = idx[len(idx) // 4], idx[3 * len(idx) // 4]
        rates.append((r[b] - r[a]) / (b - a))
rates = np.array(rates)
print(f"ns/step per warp (middle half): min {rates.min():.0f} med {np.median(rates):.0f} max {rates.max():.0f}")
ends = np.array([r[cap - 1] - t0 for r in T.values()])
print(f"end: max {ends.max():.0f} ns")
# arrival of level L at the far corner vs origin
for lev in (100, 200, 300):
    print("level", lev, "origin", at(0, 0, lev), "diag", [at(i, 2 * i, lev) for i in range(0, min(ntx, nty // 2), 3)])
