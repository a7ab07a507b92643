#!/bin/bash
# usage: scripts/gpu_round2.sh TAG -- the round-2 evidence set: smoke, pytest -m gpu, bench lines of every
# config (+ f32 cfg2, the reference arm), an ncu launch list of the default bench and ncu --set full
# captures of the dominant kernels (k_block cfg2, k_self cfg4, k_mrt cfg5), setup timings
mkdir -p gpurun_out
TAG=${1:-r2}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gpu_tests_$TAG.log
timeout 900 python bench.py --steps 30 --warmup 5 --extra > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/bench_$TAG.json
for c in 1 3 4 5 6; do timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --extra >> gpurun_out/bench_cfgs_$TAG.json 2>> gpurun_out/bench_cfgs_$TAG.err; echo "cfg$c rc=$?"; done
timeout 600 python bench.py --dtype f32 --steps 20 --warmup 3 --no-cpu >> gpurun_out/bench_cfgs_$TAG.json 2>> gpurun_out/bench_cfgs_$TAG.err; echo "f32 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-cusparse > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k k_block -s 3 -c 1 -o gpurun_out/prof_block_$TAG \
   python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --no-cusparse > gpurun_out/ncu_block_$TAG.log 2>&1; echo "ncu block rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k k_self -s 3 -c 1 -o gpurun_out/prof_self4_$TAG \
   python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cusparse > gpurun_out/ncu_self4_$TAG.log 2>&1; echo "ncu self rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k k_mrt -s 3 -c 1 -o gpurun_out/prof_mrt5_$TAG \
   python bench.py --config 5 --steps 2 --warmup 3 --no-cpu --no-e2e --no-cusparse > gpurun_out/ncu_mrt5_$TAG.log 2>&1; echo "ncu mrt rc=$?"
timeout 600 python tools/setup_time.py 1 2 3 4 > gpurun_out/setup_$TAG.txt 2>&1; echo "setup rc=$?"
