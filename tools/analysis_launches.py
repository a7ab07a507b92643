"""Analysis only (for an ncu launch list): build the handle of config k and exit."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import workloads
from paper_1710_04985_b200 import sptrsv as S

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
algo = sys.argv[2] if len(sys.argv) > 2 else "auto"
m, p = workloads.config(cfg)
uplo, diag = ("lower", "unit") if p.get("pair") else (p["uplo"], p["diag"])
torch.cuda.init()
w, wp = workloads.config(1)                     # warm-up: context + module load
S.from_csr(w, wp["uplo"], wp["diag"], algo=algo)
torch.cuda.synchronize()
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ts = []
for _ in range(reps):
    t0 = time.perf_counter()
    sv = S.from_csr(m, uplo, diag, algo=algo)
    torch.cuda.synchronize()
    ts.append(1e3 * (time.perf_counter() - t0))
    del sv
print(f"cfg{cfg} {algo} analysis ms", [round(t, 1) for t in ts])
