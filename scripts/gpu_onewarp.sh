#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-ow}
timeout 120 python tools/one_warp.py 2048 20 2>&1 | tail -1
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:k_block -s 2 -c 1 -o gpurun_out/prof_$TAG python tools/one_warp.py 4096 3 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"; tail -1 gpurun_out/ncu_$TAG.log
