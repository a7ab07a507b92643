#!/bin/bash
# usage: scripts/gpu_round.sh TAG  -- smoke, gpu tests, bench (all configs), ncu launch list + full capture
mkdir -p gpurun_out
TAG=${1:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke_$TAG.log
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py --steps 30 --warmup 5 --extra > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/bench_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
for c in 1 3 4 5; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --extra >> gpurun_out/bench_cfgs_$TAG.json 2>> gpurun_out/bench_cfgs_$TAG.err; echo "cfg$c rc=$?"; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block -s 3 -c 1 -o gpurun_out/prof_block_$TAG \
   python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_block_$TAG.log 2>&1; echo "ncu full rc=$?"
