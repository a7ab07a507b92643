#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-tile}
timeout 300 compute-sanitizer --tool memcheck python -c "
import sys; sys.path.insert(0,'.')
import numpy as np, torch, oracle, workloads
from paper_1710_04985_b200 import sptrsv as S
for dims in [(32,32),(16,16,16),(40,30,20)]:
    m = workloads.stencil(dims, 5 if len(dims)==2 else 7, 'lower'); b = workloads.rhs(m.n,1,seed=1)[:,0]
    sv = S.from_csr(m, algo='tile'); x = sv.solve(torch.from_numpy(b).cuda()).cpu().numpy()
    print(dims, float(np.abs(x-oracle.solve(m,b)).max()/np.abs(x).max()))
" 2>&1 | tail -6
timeout 300 python bench.py --algo tile --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/b_$TAG.json; tail -3 gpurun_out/b_$TAG.err
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider -k "tile or auto" > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t_$TAG.log | cut -c1-300
