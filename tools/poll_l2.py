"""L2 behaviour of the flag / value polls (north_star: "L2 hit rate on the
flag array") from one ncu --set full report.  The polls are the strong
gpu-scope loads (SASS LDG.E.*.STRONG.GPU: ld.relaxed.gpu / ld.acquire.gpu of
x values, mailboxes or counters); everything else the kernel reads from
global memory is the compulsory stream (matrix records, b).

SourceCounters give the L2 sectors every poll instruction requested; ncu does
not split L2 hits by address range, so the poll hit rate is bounded from the
DRAM side: every DRAM read byte is either the kernel's stream (the matrix or
its records, b -- STREAM_BYTES, given: read once per solve) or a poll miss, so

    poll misses <= max(0, DRAM read bytes - STREAM_BYTES) / 32
    poll L2 hit rate >= 1 - poll misses / poll sectors

(a lower bound: every other DRAM read is charged to the polls).

python tools/poll_l2.py REPORT.ncu-rep STREAM_BYTES [markdown out]"""
import csv
import io
import subprocess
import sys


def source_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    k = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    return rows[k], rows[k + 1:]


def raw(rep, keys):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k in keys:
        if k in hdr:
            v, u = vals[hdr.index(k)], units[hdr.index(k)]
            f = float(v.replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            d[k] = f * scale
    d["kernel"] = vals[hdr.index("Kernel Name")]
    return d


def main(rep, stream_bytes, out=None):
    hdr, data = source_rows(rep)
    isrc, isec = hdr.index("Source"), hdr.index("L2 Theoretical Sectors Global")
    iop = hdr.index("Access Operation") if "Access Operation" in hdr else None
    poll = stream_ld = 0
    for r in data:
        src = r[isrc]
        sec = float(r[isec] or 0)
        if sec == 0:
            continue
        op = src.split()[0] if not src.startswith("@") else src.split()[1]
        if op.startswith("LDG") and ".STRONG.GPU" in op:
            poll += sec
        elif op.startswith("LDG") or op.startswith("LDGSTS") or op.startswith("LD."):
            stream_ld += sec
    d = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct"])
    dram_rd_sec = d.get("dram__bytes_read.sum", 0) / 32
    misses_ub = max(0.0, dram_rd_sec - stream_bytes / 32)
    lb = 1 - min(1.0, misses_ub / poll) if poll else float("nan")
    lines = [f"# Poll L2 behaviour: {rep}", "", f"kernel: {d['kernel']}", "",
             f"- poll sectors requested (strong gpu-scope LDG): {poll:.0f}",
             f"- other global load sectors (LDG / LDGSTS): {stream_ld:.0f}",
             f"- DRAM read sectors: {dram_rd_sec:.0f} ({d.get('dram__bytes_read.sum', 0) / 1e6:.1f} MB)",
             f"- overall L2 sector hit rate: {d.get('lts__t_sector_hit_rate.pct', float('nan')):.1f} %",
             f"- compulsory stream (matrix / records + b, read once): {stream_bytes / 1e6:.1f} MB",
             f"- poll L2 hit rate >= {100 * lb:.1f} % (every DRAM read byte beyond the stream charged to the polls)"]
    txt = "\n".join(lines) + "\n"
    print(txt)
    if out:
        open(out, "w").write(txt)


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else None)
