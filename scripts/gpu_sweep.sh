#!/bin/bash
# usage: scripts/gpu_sweep.sh TAG CFG "ENV1" "ENV2" ...   (each ENV a space-separated VAR=val list)
mkdir -p gpurun_out
TAG=$1; CFG=$2; shift 2
for e in "$@"; do
  r=$(env $e timeout 300 python bench.py --config $CFG --algo block --steps 20 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/sw_$TAG.err | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']*1e3, d['config']['median_us'], d['value'])" 2>&1)
  echo "[$e] us/median/GBs: $r" | tee -a gpurun_out/sweep_$TAG.txt
done
