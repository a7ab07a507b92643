#!/bin/bash
# quick BLOCK check: parity subset + bench cfg2 with auto + trace
mkdir -p gpurun_out
TAG=${1:-blk}
timeout 600 python -m pytest tests -m gpu -q -x --timeout 120 -p no:cacheprovider -k "block or auto" > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/t_$TAG.log | cut -c1-300
timeout 300 python bench.py --algo block --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/b_$TAG.json; tail -3 gpurun_out/b_$TAG.err
timeout 300 python tools/block_trace.py 2 > gpurun_out/trace_$TAG.txt 2>&1; echo "trace rc=$?"; head -20 gpurun_out/trace_$TAG.txt
