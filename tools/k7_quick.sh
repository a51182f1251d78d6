#!/bin/bash
# Quick K7 check on the GPU box: parity subset, phase profile, instruction count of one K7 launch.
# usage: tools/k7_quick.sh c2 c5f:100000000 ...
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for A in "$@"; do
  CFG=${A%%:*}; N=${A#*:}; NARG=""; [ "$N" != "$A" ] && NARG="--n $N"
  echo "== $A"
  python tools/k7_prof.py --config $CFG $NARG | head -9
  ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed.avg.per_cycle_active -k regex:k7_kernel -c 1 \
      python tools/prof_run.py --config $CFG $NARG --reps 1 2>&1 | grep -E "inst_executed|duration"
done
