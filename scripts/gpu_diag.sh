#!/bin/bash
# usage: scripts/gpu_diag.sh TAG -- latency microbench, BLOCK dev timings and the per-warp step trace of cfg2
mkdir -p gpurun_out
TAG=${1:-diag}
./tools/lat_bench > gpurun_out/lat_$TAG.txt 2>&1
timeout 600 python tools/block_dev.py all --trace > gpurun_out/block_dev_$TAG.txt 2>&1; echo "dev rc=$?"
timeout 300 python tools/block_trace2.py $TAG 128 > gpurun_out/trace2_$TAG.log 2>&1; echo "trace rc=$?"
timeout 300 python tools/trace_lag.py gpurun_out/trace_$TAG.npz > gpurun_out/lag_$TAG.txt 2>&1
cat gpurun_out/lat_$TAG.txt gpurun_out/lag_$TAG.txt
