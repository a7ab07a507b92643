#!/bin/bash
# usage: scripts/gpu_lean_ncu.sh TAG -- ncu source-level capture of the lean BLOCK kernel (one warp tile, and cfg2)
mkdir -p gpurun_out
TAG=${1:-lean}
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_block1 -s 3 -c 1 -o gpurun_out/prof_ow_$TAG \
   python tools/one_warp.py 2048 5 > gpurun_out/ncu_ow_$TAG.log 2>&1; echo "ncu ow rc=$?"; tail -1 gpurun_out/ncu_ow_$TAG.log | cut -c1-200
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block1 -s 3 -c 1 -o gpurun_out/prof_c2_$TAG \
   python bench.py --algo block --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_c2_$TAG.log 2>&1; echo "ncu c2 rc=$?"; tail -1 gpurun_out/ncu_c2_$TAG.log | cut -c1-200
