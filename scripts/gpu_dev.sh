#!/bin/bash
# usage: scripts/gpu_dev.sh TAG [block_dev args] -- BLOCK dev timings + cfg2 step trace + lag summary
mkdir -p gpurun_out
TAG=${1:-dev}; shift
timeout 600 python tools/block_dev.py ${@:-cfg2} > gpurun_out/block_dev_$TAG.txt 2>&1; echo "dev rc=$?"
SPTRSV_DEV_LIB=$PWD/paper_1710_04985_b200/lib/var_trace.so timeout 300 python tools/block_trace2.py $TAG 128 > gpurun_out/trace2_$TAG.log 2>&1; echo "trace rc=$?"
timeout 300 python tools/trace_lag.py gpurun_out/trace_$TAG.npz > gpurun_out/lag_$TAG.txt 2>&1
cat gpurun_out/block_dev_$TAG.txt | grep -v "^ *warp" ; cat gpurun_out/lag_$TAG.txt
