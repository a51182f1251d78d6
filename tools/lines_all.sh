#!/bin/bash
# Full per-line instruction / stall table of one launch of kernel $2 on workload $1
# (every source line, for aggregation by region) -> gpurun_out/alllines_<kernel>_<cfg>.txt
CFG=${1:-c5f}; K=${2:-k7_kernel}; SKIP=${3:-0}
mkdir -p gpurun_out
bash tools/ncu_kernel.sh $CFG "$K" $SKIP
python tools/ncu_lines.py gpurun_out/${K}_$CFG.ncu-rep 100000 --by-instr > gpurun_out/alllines_${K}_$CFG.txt 2>&1
rm -f gpurun_out/${K}_$CFG.ncu-rep
