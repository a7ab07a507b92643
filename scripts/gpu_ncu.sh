#!/bin/bash
# usage: scripts/gpu_ncu.sh <kernel-regex> <tag> [bench args...]
mkdir -p gpurun_out
K=$1; TAG=$2; shift 2
timeout 900 ncu --set full --warp-sampling-interval 2 --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_$TAG \
   python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e "$@" > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$TAG.log | cut -c1-300
