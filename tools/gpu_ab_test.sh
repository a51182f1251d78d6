#!/bin/bash
# usage: bash tools/gpu_ab_test.sh TAG "configs" "pytest files" lib1.so lib2.so ...
# parity tests against the in-tree build, then an A/B of the listed builds -> gpurun_out/TAG_*
TAG=$1; shift; CFGS=$1; shift; TESTS=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
if [ -n "$TESTS" ]; then
  timeout 1200 python -m pytest $TESTS -x -q -m gpu > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
  tail -5 gpurun_out/${TAG}_pytest.log
fi
for rep in 1 2; do bash tools/ab.sh "$CFGS" "$@"; done 2>&1 | tee gpurun_out/${TAG}_ab.txt
