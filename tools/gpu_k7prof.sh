#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in c2 c5f c5u c3; do python tools/k7_prof.py --config $c; done 2>&1 | tee gpurun_out/k7prof.txt
