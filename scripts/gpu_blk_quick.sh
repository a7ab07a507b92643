#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-blk}
timeout 120 python tools/one_warp.py 2048 20 2>&1 | tail -1
timeout 300 python tools/block_trace.py 2 > gpurun_out/trace_$TAG.txt 2>&1; echo "trace rc=$?"; head -3 gpurun_out/trace_$TAG.txt | cut -c1-400
timeout 300 python bench.py --algo block --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err; echo "bench rc=$?"; cut -c1-330 gpurun_out/b_$TAG.json; tail -3 gpurun_out/b_$TAG.err
timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider -k "block" > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t_$TAG.log | cut -c1-300
