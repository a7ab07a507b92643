#!/bin/bash
# usage: scripts/gpu_check_block.sh TAG -- the BLOCK tests, the smoke and the cfg2 bench on the bounds-checked
# development build (every record-driven shared-slot / mailbox / cluster-rank / row index asserted; a
# violation traps), standing in for compute-sanitizer where the tool is closed
mkdir -p gpurun_out
TAG=${1:-chk}
export SPTRSV_DEV_LIB=paper_1710_04985_b200/lib/var_check.so
timeout 900 python -m pytest tests -m gpu -q -k "block or auto or cfg2 or smoke or grid or watchdog or update" -p no:cacheprovider > gpurun_out/check_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/check_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/check_smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-cusparse > gpurun_out/check_bench_$TAG.json 2>&1; echo "bench rc=$?"
timeout 600 python tools/decouple.py 128 3 > gpurun_out/check_decouple_$TAG.txt 2>&1; echo "decouple rc=$?"
timeout 600 python tools/laplacian_sweep.py > gpurun_out/check_sweep_$TAG.txt 2>&1; echo "sweep rc=$?"
