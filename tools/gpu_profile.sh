#!/bin/bash
# One GPU profiling pass (run under gpurun): K7 phase cycles, launch list, ncu --set full of the
# top kernels for workload $1 (default c2). Outputs land in gpurun_out/prof_$1/.
set -x
CFG=${1:-c2}
N=${2:-}
O=gpurun_out/prof_${CFG}
mkdir -p $O
NARG=""; [ -n "$N" ] && NARG="--n $N"
python tools/k7_prof.py --config $CFG $NARG > $O/k7_phases.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python tools/prof_run.py --config $CFG $NARG --reps 2 > $O/ncu_launch.log 2>&1
for K in k7_kernel k_split_scatter k_split_count; do
  ncu --set full --import-source on --clock-control none -k regex:$K -s 1 -c 1 -o $O/$K -f \
      python tools/prof_run.py --config $CFG $NARG --reps 2 > $O/ncu_$K.log 2>&1
done
ls -la $O
