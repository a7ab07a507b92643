#!/bin/bash
# usage: scripts/gpu_ncu_more.sh TAG -- ncu --set full of the dominant kernel of cfg3 (k_self), cfg4 (k_self), cfg5 (k_level_mrhs)
mkdir -p gpurun_out
TAG=${1:-r1}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_self -s 3 -c 1 -o gpurun_out/prof_self_cfg3_$TAG \
   python bench.py --config 3 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cusparse > gpurun_out/ncu_self3_$TAG.log 2>&1; echo "ncu self cfg3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_self -s 2 -c 1 -o gpurun_out/prof_self_cfg4_$TAG \
   python bench.py --config 4 --steps 1 --warmup 3 --no-cpu --no-e2e --no-cusparse > gpurun_out/ncu_self4_$TAG.log 2>&1; echo "ncu self cfg4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level_mrhs -s 3 -c 1 -o gpurun_out/prof_mrhs_cfg5_$TAG \
   python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cusparse > gpurun_out/ncu_mrhs5_$TAG.log 2>&1; echo "ncu mrhs cfg5 rc=$?"
