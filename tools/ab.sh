#!/bin/bash
# A/B bench of library builds: tools/ab.sh "c2 c5f" lib1.so lib2.so ...  (ms_per_step and per-pass ms)
CFGS=$1; shift
for A in $CFGS; do
  for L in "$@"; do
    PCF_LIB=$L python bench.py --config $A --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$A', '$L'.split('/')[-1], round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['passes'].items()})"
  done
done
