#!/bin/bash
# SELF poll back-off variants on cfg3 / cfg4 (bench lines, algo self)
for lib in paper_1710_04985_b200/lib/libsptrsv.so paper_1710_04985_b200/lib/var_*.so; do
  for c in 3 4; do
    r=$(SPTRSV_DEV_LIB=$PWD/$lib timeout 300 python bench.py --config $c --algo self --steps 10 --warmup 3 --no-cpu --no-e2e --no-cusparse 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
    echo "$lib cfg$c $r ms"
  done
done
