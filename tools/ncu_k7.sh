#!/bin/bash
# ncu --set full of one K7 launch (second sort) for workload $1 -> gpurun_out/k7_$1.ncu-rep
CFG=${1:-c2}
python tools/prof_run.py --config $CFG --reps 2 > gpurun_out/plain_$CFG.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:k7_kernel -s 1 -c 1 -o gpurun_out/k7_$CFG -f \
    python tools/prof_run.py --config $CFG --reps 2 > gpurun_out/ncu_k7_$CFG.log 2>&1
