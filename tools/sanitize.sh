#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py; logs -> gpurun_out/sanitize_<tool>.log
# usage (on the GPU box): bash tools/sanitize.sh [scale]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
SCALE=${1:-1.0}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  # racecheck is by far the slowest: a smaller workload
  sc=$SCALE; [ "$tool" = racecheck ] && sc=$(python -c "print($SCALE*0.25)")
  echo "== $tool (scale $sc)"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_run.py $sc \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
