#!/bin/bash
# usage: scripts/gpu_sanitize.sh TAG -- compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py
mkdir -p gpurun_out
TAG=${1:-san}
for tool in memcheck racecheck synccheck; do
  for c in self level block slfc levc vf8 mrt64 block3d; do
    echo "== $tool $c" >> gpurun_out/sanitize_$TAG.log
    timeout 600 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_run.py $c >> gpurun_out/sanitize_$TAG.log 2>&1
    echo "rc=$?" >> gpurun_out/sanitize_$TAG.log
  done
done
grep -E "^== |rc=|ERROR SUMMARY|exact|Hazard|error" gpurun_out/sanitize_$TAG.log | head -120
