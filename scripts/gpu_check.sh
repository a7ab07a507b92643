#!/bin/bash
# usage: scripts/gpu_check.sh [tests|notests] [extra bench args...]
mkdir -p gpurun_out
MODE=${1:-tests}; shift
if [ "$MODE" = "tests" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -8 gpurun_out/gpu_tests.log
fi
timeout 600 python bench.py --steps 30 --warmup 5 --extra "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
