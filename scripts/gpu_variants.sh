#!/bin/bash
# usage: scripts/gpu_variants.sh TAG -- cfg2 BLOCK timing of the default library and every lib/var_*.so
mkdir -p gpurun_out
TAG=${1:-var}
for lib in paper_1710_04985_b200/lib/libsptrsv.so paper_1710_04985_b200/lib/var_*.so; do
  echo "== $lib"
  SPTRSV_DEV_LIB=$PWD/$lib timeout 300 python tools/block_dev.py cfg2 2>&1 | grep "cfg2 f64" | sed 's/plan=.*| status/| status/'
done | tee gpurun_out/variants_$TAG.txt
