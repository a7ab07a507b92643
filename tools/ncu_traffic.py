"""Record the DRAM traffic per launch of a kernel from an ncu --set full
report into profiles/ncu_traffic.json, tagged with the build digest (sha256 of
the library's sources and nvcc flags, build.source_digest) of the build the
report was taken on (bench.py only uses an entry whose digest matches the
library it runs).

python tools/ncu_traffic.py REPORT.ncu-rep KEY [KERNEL_REGEX]
  KEY e.g. cfg2_k_block_f64 (cfg<config>_<kernel>_<dtype>, as bench.py builds it)
"""
import csv
import hashlib
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rep, key = sys.argv[1], sys.argv[2]
    pat = re.compile(sys.argv[3] if len(sys.argv) > 3 else key.split("_", 1)[1].rsplit("_", 1)[0])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    kn, rd, wr = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = []
    for r in rows[2:]:
        if pat.search(r[kn]):
            vals.append(float(r[rd].replace(",", "")) * scale.get(units[rd], 1) +
                        float(r[wr].replace(",", "")) * scale.get(units[wr], 1))
    if not vals:
        sys.exit(f"no launch of {pat.pattern} in {rep}")
    sys.path.insert(0, ROOT)
    from paper_1710_04985_b200 import build as B
    digest = B.source_digest()
    with open(B.LIB, "rb") as f:
        sha = hashlib.sha256(f.read()).hexdigest()
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            db = json.load(f)
    except (OSError, ValueError):
        db = {}
    db = {k: v for k, v in db.items() if isinstance(v, dict)}      # drop round-1 unversioned entries
    db[key] = {"bytes": int(sum(vals) / len(vals)), "launches": len(vals), "build_digest": digest, "lib_sha256": sha,
               "source": f"ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum, {os.path.basename(rep)}"}
    with open(path, "w") as f:
        json.dump(db, f, indent=1, sort_keys=True)
    print(key, db[key])


if __name__ == "__main__":
    main()
