#!/bin/bash
# usage: bash tools/prof_lines.sh "cfg:kernel_regex:skip ..."  -> gpurun_out/lines_{instr,stall}_<kernel>_<cfg>.txt
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for spec in $1; do
  IFS=: read CFG K SKIP <<< "$spec"
  bash tools/ncu_kernel.sh $CFG "$K" ${SKIP:-1}
  python tools/ncu_lines.py gpurun_out/${K}_$CFG.ncu-rep 60 --by-instr > gpurun_out/lines_instr_${K}_$CFG.txt 2>&1
  python tools/ncu_lines.py gpurun_out/${K}_$CFG.ncu-rep 40 > gpurun_out/lines_stall_${K}_$CFG.txt 2>&1
  ncu -i gpurun_out/${K}_$CFG.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed.avg.per_cycle_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum > gpurun_out/raw_${K}_$CFG.csv 2>&1
  rm -f gpurun_out/${K}_$CFG.ncu-rep
done
