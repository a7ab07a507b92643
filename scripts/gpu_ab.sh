#!/bin/bash
# usage: scripts/gpu_ab.sh TAG VAR1 VAR2 ... -- release lib + variants (paper_1710_04985_b200/lib/var_NAME.so) timed on cfg2-like grids
mkdir -p gpurun_out
TAG=$1; shift
DIMS=${DIMS:-"128x128x128 8x4x512 64x64x64"}
python tools/variant_time.py release $DIMS > gpurun_out/ab_$TAG.txt 2>&1
for v in "$@"; do SPTRSV_DEV_LIB=paper_1710_04985_b200/lib/var_$v.so python tools/variant_time.py $v $DIMS >> gpurun_out/ab_$TAG.txt 2>&1; done
python tools/variant_time.py release $DIMS >> gpurun_out/ab_$TAG.txt 2>&1
