#!/bin/bash
mkdir -p gpurun_out
TAG=${1:-blk}
timeout 900 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider -k "block" > gpurun_out/t_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/t_$TAG.log | cut -c1-300
timeout 300 python bench.py --algo block --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/b_$TAG.json; tail -3 gpurun_out/b_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_block -s 2 -c 1 -o gpurun_out/prof_$TAG \
   python bench.py --algo block --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_$TAG.log | cut -c1-300
