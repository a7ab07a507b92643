"""Per-level view of a BLOCK trace (tools/overhead.py dump, 3-D 7-point grid):
F(L) = time level L's last row became computable (max over warp tiles), the
origin tile's own pace, and the per-level growth of F split by what the
slowest tile at that level crossed.  usage: python tools/wave_levels.py gpurun_out/oh_128x128x128.npz"""
import sys
import numpy as np

d = np.load(sys.argv[1])
tr = d["tr"].astype(np.int64)
plan = d["plan"]
nx, ny, nz = (int(v) for v in d["dims"])
nlev = int(d["nlev"])
K, wpc, tw, th, cs, csx = (int(plan[i]) for i in (0, 1, 7, 8, 9, 10))
U, cap = tr.shape
csy = cs // csx
wx = wy = 2 if wpc == 4 else None
ntx, nty = nx // tw, ny // th
cxn = ntx // wx
# unit -> tile origin (k_part_tiles, lower)
L0 = np.full(U, -1)
TX = np.zeros(U, int); TY = np.zeros(U, int)
for tyi in range(nty):
    for txi in range(ntx):
        cx, cy = txi // wx, tyi // wy
        cta = ((cy // csy) * (cxn // csx) + cx // csx) * (csx * csy) + (cy % csy) * csx + cx % csx
        w = (tyi % wy) * wx + (txi % wx)
        u = cta * (wx * wy) + w
        L0[u] = txi * tw + tyi * th
        TX[u], TY[u] = txi, tyi
t0 = tr[:, :cap - 8][tr[:, :cap - 8] > 0].min()
T = (tr[:, :cap - 8] - t0) / 1e3        # us
nst = (tr[:, :cap - 8] > 0).sum(1)
F = np.zeros(nlev)
arg = np.zeros(nlev, int)
for L in range(nlev):
    best, bu = -1, -1
    for u in range(U):
        t = L - L0[u]
        if 0 <= t < nst[u] and tr[u, t] > 0:
            if T[u, t] > best:
                best, bu = T[u, t], u
    F[L], arg[L] = best, bu
o = np.argmin(L0)
print(f"origin tile pace: {np.median(np.diff(T[o, :130])) * 1e3:.0f} ns/step; first step at {T[o, 0]:.2f} us")
print(f"F(0) {F[0]:.2f}  F(nlev-1) {F[-1]:.2f} us")
for a, b in ((0, 50), (50, 100), (100, 150), (150, 200), (200, 250), (250, 300), (300, 350), (350, nlev - 1)):
    print(f"levels {a:3d}-{b:3d}: {(F[b] - F[a]) / (b - a) * 1e3:6.0f} ns/level")
# the slowest tile at level L: its (tx, ty); count level-to-level jumps where the argmax tile changes
chg = np.nonzero(arg[1:] != arg[:-1])[0]
print("argmax tile changes:", len(chg))
# back-trace the critical path: from the last level, walk back picking the predecessor (tile itself or x-/y-neighbour) with the latest time
u, L = arg[-1], nlev - 1
path = []
pos = {(TX[v], TY[v]): v for v in range(U)}
while L > 0:
    t = L - L0[u]
    cands = [u]
    if (TX[u] - 1, TY[u]) in pos: cands.append(pos[(TX[u] - 1, TY[u])])
    if (TX[u], TY[u] - 1) in pos: cands.append(pos[(TX[u], TY[u] - 1)])
    best, bv = -1, u
    for v in cands:
        tv = L - 1 - L0[v]
        if 0 <= tv < nst[v] and T[v, tv] > best:
            best, bv = T[v, tv], v
    path.append((L, u, T[u, t], bv != u, (u // wpc) // cs != (bv // wpc) // cs, u // wpc != bv // wpc))
    u, L = bv, L - 1
path = path[::-1]
steps = np.array([p[2] for p in path])
cross = np.array([p[3] for p in path]); ccl = np.array([p[4] for p in path]); ccta = np.array([p[5] for p in path])
dt = np.diff(steps)
print(f"critical path: {len(path)} levels, crossings {cross[1:].sum()} (cluster {ccl[1:].sum()}, CTA {ccta[1:].sum()})")
print(f"  time in own-tile steps {dt[~cross[1:]].sum():.1f} us ({np.median(dt[~cross[1:]]) * 1e3:.0f} ns median), "
      f"in warp crossings {dt[cross[1:] & ~ccta[1:]].sum():.1f} us, CTA crossings (same cluster) "
      f"{dt[ccta[1:] & ~ccl[1:]].sum():.1f} us, cluster crossings {dt[ccl[1:]].sum():.1f} us")
print(f"  per crossing: warp {np.mean(dt[cross[1:] & ~ccta[1:]]) * 1e3 if (cross[1:] & ~ccta[1:]).any() else 0:.0f} ns, "
      f"CTA {np.mean(dt[ccta[1:] & ~ccl[1:]]) * 1e3 if (ccta[1:] & ~ccl[1:]).any() else 0:.0f} ns, cluster "
      f"{np.mean(dt[ccl[1:]]) * 1e3 if ccl[1:].any() else 0:.0f} ns")
own = dt[~cross[1:]]
print("own-tile step ns on the path: p10 %.0f p50 %.0f p75 %.0f p90 %.0f p99 %.0f max %.0f" % tuple(np.percentile(own * 1e3, [10, 50, 75, 90, 99, 100])))
big = np.argsort(dt)[::-1][:15]
for i in big:
    L, u = path[i + 1][0], path[i + 1][1]
    print(f"  L {L:3d} tile ({TX[u]:2d},{TY[u]:2d}) cta {u // wpc:3d} step {L - L0[u]:3d}: {dt[i] * 1e3:6.0f} ns cross={cross[i + 1]}")
hist = np.zeros(nlev)
for i in range(len(dt)):
    hist[path[i + 1][0]] = dt[i]
for a in range(0, nlev, 25):
    seg = hist[a:a + 25]
    print(f"  levels {a:3d}+: mean {seg.mean() * 1e3:5.0f} ns")
# excess over the fast step, by whether the tile has an input across a cluster / CTA boundary
cx_ext = tw * 2 * csx                      # cluster extent in x (columns)
cy_ext = th * 2 * csy
def kind(u):
    x0, y0 = TX[u] * tw, TY[u] * th
    if (x0 % cx_ext == 0 and x0 > 0) or (y0 % cy_ext == 0 and y0 > 0):
        return "cluster-edge"
    if (x0 % (2 * tw) == 0 and x0 > 0) or (y0 % (2 * th) == 0 and y0 > 0):
        return "cta-edge"
    return "inner" if (x0 > 0 or y0 > 0) else "origin"
ex = {}
for i in range(len(dt)):
    if cross[i + 1]:
        continue
    k = kind(path[i + 1][1])
    e = ex.setdefault(k, [0, 0.0, 0.0])
    e[0] += 1; e[1] += dt[i]; e[2] += max(0.0, dt[i] - 0.192)
for k, (c, tot, exc) in ex.items():
    print(f"  own steps in {k:12s} tiles: {c:3d} steps, {tot:6.1f} us, excess over 192 ns {exc:6.1f} us")
