#!/bin/bash
# Round profiling pass (run under gpurun, one GPU): bench line, launch list of the
# bench command, ncu --set full captures of the top kernels.  -> gpurun_out/prof/
O=gpurun_out/prof; mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench_c2.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
for CFG in c2 c5f; do
  for K in k7_kernel k_split_scatter k_split_count; do
    ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -o $O/${K}_$CFG -f \
        python tools/prof_run.py --config $CFG --reps 1 > $O/ncu_${K}_$CFG.log 2>&1
  done
done
ls -la $O
