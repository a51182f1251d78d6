#!/bin/bash
# A/B of environment settings on the in-tree build: tools/ab_env.sh "c2 c5f" "PCF_K7_VARIANT=512" "X=1" ...
# ("-" = no extra variable)
CFGS=$1; shift
for A in $CFGS; do
  for E in "$@"; do
    [ "$E" = "-" ] && E="PCF_NONE=0"
    env $E python bench.py --config $A --steps 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$A', '$E', round(d['ms_per_step'],3), {k:round(v['ms_per_step'],3) for k,v in d['passes'].items()})"
  done
done
