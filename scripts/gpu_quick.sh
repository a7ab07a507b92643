#!/bin/bash
# usage: scripts/gpu_quick.sh TAG -- smoke, pytest -m gpu, default bench line, cfg4/cfg5 lines
mkdir -p gpurun_out
TAG=${1:-q}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_$TAG.json
for c in 3 4 5; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_cfgs_$TAG.json 2>> gpurun_out/bench_cfgs_$TAG.err; echo "cfg$c rc=$?"; done
