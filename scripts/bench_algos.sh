#!/bin/bash
# usage: scripts/bench_algos.sh "CFGS" "ALGOS" -- short bench per (config, algo): ms per solve and GB/s
for c in $1; do for a in $2; do
  timeout 600 python bench.py --config $c --algo $a --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg$c', '$a', d['ms_per_step'], 'ms', d['value'], 'GB/s')" \
   || echo "cfg$c $a failed"
done; done
