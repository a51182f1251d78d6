#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/san_build.log 2>&1 || exit 1
timeout 600 python -m pytest tests -x -q -m gpu -k "r6 or async or host_entry or repeated" > gpurun_out/san_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/san_pytest.log
bash tools/sanitize.sh 1.0
