"""Summarise ncu reports (--set full) into profiles/: duration, DRAM traffic,
L2 hit rate, occupancy, top stall reasons and the hottest SASS lines."""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS or (h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")):
            d[h] = (v, u)
    d["Kernel Name"] = (vals[hdr.index("Kernel Name")], "")
    return d


def hot(rep, top=12):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        try:
            data.append((int(r[iss] or 0), r[ia][-5:], r[isrc]))
        except Exception:
            pass
    tot = sum(d[0] for d in data) or 1
    return [f"{100 * s / tot:5.1f}%  {a}  {src}" for s, a, src in sorted(data, reverse=True)[:top]]


if __name__ == "__main__":
    rep, out = sys.argv[1], sys.argv[2]
    d = raw(rep)
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(v[0]) for k, v in d.items()
              if k.startswith("smsp__pcsamp") and v[0] not in ("", "0")}
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: {rep}\n\nkernel: {d['Kernel Name'][0]}\n\n")
        for k in KEYS:
            if k in d:
                f.write(f"- {k}: {d[k][0]} {d[k][1]}\n")
        f.write("\nwarp-stall samples (all):\n")
        for k, v in sorted(stalls.items(), key=lambda t: -t[1]):
            f.write(f"- {k}: {v}\n")
        f.write("\nhottest SASS (share of stall samples):\n```\n" + "\n".join(hot(rep)) + "\n```\n")
    print(open(out).read())
