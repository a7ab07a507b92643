#!/bin/bash
# usage: scripts/gpu_round2_final.sh TAG -- the end-of-round evidence set: scripts/gpu_round2.sh (smoke,
# pytest -m gpu, bench lines of every config, reference arm, ncu launch list, ncu --set full of k_block /
# k_self / k_mrt, setup timings), then compute-sanitizer on the BLOCK and tile kernels and the BLOCK
# decomposition runs (decoupled partitions, per-warp trace of the critical path)
TAG=${1:-r2k}
scripts/gpu_round2.sh $TAG
for tool in memcheck racecheck synccheck; do
  for c in block block3d mrt64 self; do
    echo "== $tool $c" >> gpurun_out/sanitize_$TAG.log
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py $c >> gpurun_out/sanitize_$TAG.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_$TAG.log
  done
done
echo "sanitize done"
timeout 300 python tools/decouple.py 128 20 > gpurun_out/decouple_$TAG.txt 2>&1; echo "decouple rc=$?"
python tools/build_variant.py trace -DSPTRSV_BLOCK_TRACE=1 > /dev/null 2>&1
SPTRSV_DEV_LIB=paper_1710_04985_b200/lib/var_trace.so timeout 300 python tools/overhead.py 128x128x128 > gpurun_out/overhead_$TAG.txt 2>&1
SPTRSV_DEV_LIB=paper_1710_04985_b200/lib/var_trace.so timeout 300 python tools/block_trace2.py $TAG 128 > gpurun_out/bt_$TAG.txt 2>&1; echo "trace rc=$?"
