#!/bin/bash
mkdir -p gpurun_out
timeout 120 ./tools/microbench > gpurun_out/microbench.json 2>&1; echo "mb rc=$?"; cat gpurun_out/microbench.json
# launch list of the bench command (cold-cache, serialized)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1a.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu list rc=$?"
# full capture of one k_self launch
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_self -s 3 -c 1 -o gpurun_out/prof_self_r1a \
   python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/ncu_self.log 2>&1; echo "ncu self rc=$?"; tail -3 gpurun_out/ncu_self.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level -s 3 -c 1 -o gpurun_out/prof_level_r1a \
   python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e --algo level > gpurun_out/ncu_level.log 2>&1; echo "ncu level rc=$?"; tail -3 gpurun_out/ncu_level.log
