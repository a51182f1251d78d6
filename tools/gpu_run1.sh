set -x
free -g; nproc; lscpu | head -20; nvidia-smi --query-gpu=name,memory.total,clocks.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python bench.py > gpurun_out/bench_c5f_v0.json 2> gpurun_out/bench_c5f_v0.err; echo bench rc=$?
timeout 2400 python -m pytest tests -x -q -m gpu --durations=15 > gpurun_out/pytest_gpu_v0.log 2>&1; echo pytest rc=$?
tail -25 gpurun_out/pytest_gpu_v0.log
