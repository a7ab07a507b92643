"""Critical-path model of blocked self-scheduling (global-level steps):
start(b,l) = max(end(b,l-1), max_{ext dep j of rows in (b,l)} end(blk(j),lev(j)) + t_cross)
end(b,l)   = start(b,l) + t_step(rows in (b,l))
Used to choose the row->CTA partition (D2)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads, oracle

def simulate(m, lev, nlev, blk, K, t_step=0.1, t_cross=0.3, t_row=0.0):
    n = m.n
    rows_by_lev = np.argsort(lev, kind="stable")
    ilev = np.searchsorted(lev[rows_by_lev], np.arange(nlev + 1))
    end = np.zeros((K, nlev))
    prev = np.zeros(K)
    rp, ci = m.rowptr, m.colidx
    deg = np.diff(rp)
    rowid = np.repeat(np.arange(n), deg)
    tri = ci < rowid
    dep_row, dep_col = rowid[tri], ci[tri]
    ext = blk[dep_row] != blk[dep_col]
    er, ec = dep_row[ext], dep_col[ext]
    order = np.argsort(lev[er], kind="stable")
    er, ec = er[order], ec[order]
    eb = np.searchsorted(lev[er], np.arange(nlev + 1))
    crossings = len(er)
    for l in range(nlev):
        rows = rows_by_lev[ilev[l]:ilev[l + 1]]
        cnt = np.bincount(blk[rows], minlength=K)
        start = prev.copy()
        a, b = eb[l], eb[l + 1]
        if b > a:
            ready = end[blk[ec[a:b]], lev[ec[a:b]]] + t_cross
            np.maximum.at(start, blk[er[a:b]], ready)
        e = np.where(cnt > 0, start + t_step + t_row * cnt, prev)
        end[:, l] = e
        prev = e
    return prev.max(), crossings

def main():
    g = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    m = workloads.stencil((g, g, g), 7, "lower")
    lev, nlev = oracle.levels(m)
    n = m.n
    ilev, jlev = oracle.schedule(lev, nlev)
    rank = np.empty(n, dtype=np.int64); rank[jlev] = np.arange(n)
    width = np.diff(ilev)
    frac = (rank - ilev[lev]) / width[lev]
    x = np.arange(n) % g; y = (np.arange(n) // g) % g; z = np.arange(n) // (g * g)
    for K in (16, 32, 64, 128, 148):
        parts = {
            "natural": (np.arange(n) * K) // n,
            "rank_in_level": np.minimum((frac * K).astype(np.int64), K - 1),
        }
        tx = int(round(np.sqrt(K)))
        if tx * tx == K:
            parts["xy_tiles"] = (x * tx // g) * tx + (y * tx // g)
        for name, blk in parts.items():
            T, c = simulate(m, lev, nlev, blk.astype(np.int64), K)
            print(f"K={K:4d} {name:14s} T={T:7.1f}us  ext_deps={c}")

if __name__ == "__main__":
    main()
