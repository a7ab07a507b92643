"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per kernel name, launches and mean/total duration (cold-cache, serialised)."""
import csv
import sys
from collections import OrderedDict


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    agg = OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "").replace("sptrsv::<unnamed>::", "")
        unit = r[13]
        v = float(r[14].replace(",", "")) * (1e-3 if unit == "ns" else 1.0 if unit == "us" else 1e3)
        a = agg.setdefault(name, [0, 0.0, r[7], r[8]])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    lines = [f"# launch list: {path}", "", "| kernel | launches | mean us | total us | share | block | grid |",
             "|---|---|---|---|---|---|---|"]
    for k, (c, t, blk, grd) in agg.items():
        lines.append(f"| {k} | {c} | {t / c:.2f} | {t:.1f} | {t / tot:.1%} | {blk} | {grd} |")
    s = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(s)
    print(s)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
