#!/bin/bash
# usage: scripts/gpu_lean.sh TAG -- lean vs helper BLOCK kernel: one-warp step cost, cfg2 bench, block parity tests
mkdir -p gpurun_out
TAG=${1:-lean}
timeout 120 python tools/one_warp.py 2048 20 2>&1 | tail -1
SPTRSV_BLOCK_LEAN=0 timeout 120 python tools/one_warp.py 2048 20 2>&1 | tail -1
timeout 300 python bench.py --algo block --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err; echo "bench rc=$?"; cut -c1-330 gpurun_out/b_$TAG.json; tail -3 gpurun_out/b_$TAG.err
SPTRSV_BLOCK_LEAN=0 timeout 300 python bench.py --algo block --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b0_$TAG.json 2> gpurun_out/b0_$TAG.err; echo "bench0 rc=$?"; cut -c1-330 gpurun_out/b0_$TAG.json
timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider -k "block or auto" > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t_$TAG.log | cut -c1-300
