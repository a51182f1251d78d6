#!/bin/bash
# ncu --set full of one launch of kernel regex $2 (skipping $3 launches) for workload $1
CFG=${1:-c2}; K=${2:-k7_kernel}; SKIP=${3:-1}; N=${4:-}
NARG=""; [ -n "$N" ] && NARG="--n $N"
python tools/prof_run.py --config $CFG $NARG --reps 2 > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:$K -s $SKIP -c 1 -o gpurun_out/${K}_$CFG -f \
    python tools/prof_run.py --config $CFG $NARG --reps 2 > gpurun_out/ncu_${K}_$CFG.log 2>&1
