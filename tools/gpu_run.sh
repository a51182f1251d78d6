#!/bin/bash
# One GPU-box session: build, probe, GPU tests, bench (logs -> gpurun_out/<tag>_*)
# usage: bash tools/gpu_run.sh TAG [pytest-args...]
TAG=${1:-run}; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
[ -x tools/micro/graph_cond ] && timeout 60 tools/micro/graph_cond > gpurun_out/${TAG}_graph_cond.log 2>&1
timeout 1800 python -m pytest tests -x -q -m gpu --durations=20 "$@" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/${TAG}_bench.err
for cfg in ${BENCH_EXTRA:-}; do
  timeout 600 python bench.py --config $cfg --no-cpu-baseline > gpurun_out/${TAG}_bench_$cfg.json 2> gpurun_out/${TAG}_bench_$cfg.err; echo "bench $cfg rc=$?"
done
