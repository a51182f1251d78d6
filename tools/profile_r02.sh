#!/bin/bash
# Round-2 profiling pass (one GPU): the bench line (c5f), the ncu launch list of the same
# bench command, and ncu --set full captures of the top kernels.  -> gpurun_out/prof2/
O=gpurun_out/prof2; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python bench.py > $O/bench_c5f.json 2> $O/bench_c5f.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file $O/launches_bench_c5f.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
cap() {   # cap CFG KERNEL_REGEX SKIP NAME
  ncu --set full --import-source on --clock-control none -k regex:$2 -s $3 -c 1 -o $O/$4 -f \
      python tools/prof_run.py --config $1 --reps 1 > $O/ncu_$4.log 2>&1
}
cap c5f k7_kernel 0 k7_kernel_c5f
cap c5f "k_split_count$" 0 k_split_count_r1_c5f
cap c5f k_split_count_tile 0 k_split_count_tile_r2_c5f
cap c5f k_split_scatter 0 k_split_scatter_r1_c5f
cap c5f k_split_scatter 1 k_split_scatter_r2_c5f
cap c2 k7_kernel 0 k7_kernel_c2
# the Standard-Sort radix rounds run inside CUDA-graph conditional nodes (not profiled per kernel); c4 launch list
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c4.csv \
    python tools/prof_run.py --config c4 --reps 1 > $O/ncu_launch_c4.log 2>&1
# summaries on the box (ncu -i), then drop the multi-MB reports (gpurun_out is capped at 64 MiB)
python tools/summarize_profiles.py $O $O/sum c5f > $O/sum.log 2>&1
rm -f $O/*.ncu-rep
ls -la $O $O/sum
