#!/bin/bash
# usage: scripts/gpu_ab_cfg.sh TAG CFG VAR1 VAR2 ... -- bench.py --config CFG with the release lib and variants
mkdir -p gpurun_out
TAG=$1; CFG=$2; shift 2
run() { python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu --no-e2e --no-cusparse 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$1', d['ms_per_step'], d['roofline']['frac'], d['roofline'].get('kernel'))"; }
run release > gpurun_out/abc_$TAG.txt 2>&1
for v in "$@"; do SPTRSV_DEV_LIB=paper_1710_04985_b200/lib/var_$v.so run $v >> gpurun_out/abc_$TAG.txt 2>&1; done
run release >> gpurun_out/abc_$TAG.txt 2>&1
