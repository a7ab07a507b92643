"""Per-SASS-instruction stall listing from an ncu report's source page."""
import csv, io, subprocess, sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    return rows[k], rows[k + 1:]


def main(rep, thresh=0.004, lo=None, hi=None):
    hdr, data = load(rep)
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    tot = sum(int(r[iss] or 0) for r in data) or 1
    print("total stall samples", tot, "instructions executed", sum(int(r[iex] or 0) for r in data))
    for r in data:
        s, e = int(r[iss] or 0), int(r[iex] or 0)
        a = int(r[ia], 16) & 0xFFFFF
        if lo is not None and not (lo <= a <= hi):
            continue
        if e == 0 and s == 0:
            continue
        if lo is None and s < tot * thresh:
            continue
        rs = sorted(((float(r[i] or 0), hdr[i][6:]) for i in sc), reverse=True)[:2]
        print(f"{a:05x} ex={e:7d} st={s:5d} {100*s/tot:5.1f}% {r[isrc][:64]:64s} "
              + ",".join(f"{n}:{v:.0f}" for v, n in rs if v > 0))


if __name__ == "__main__":
    rep = sys.argv[1]
    if len(sys.argv) > 3:
        main(rep, lo=int(sys.argv[2], 16), hi=int(sys.argv[3], 16))
    else:
        main(rep, float(sys.argv[2]) if len(sys.argv) > 2 else 0.004)
