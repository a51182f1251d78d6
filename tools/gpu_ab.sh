#!/bin/bash
# usage: bash tools/gpu_ab.sh TAG "configs" lib1.so lib2.so ...  -> gpurun_out/TAG_ab.txt
TAG=$1; shift; CFGS=$1; shift
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for rep in 1 2; do bash tools/ab.sh "$CFGS" "$@"; done 2>&1 | tee gpurun_out/${TAG}_ab.txt
