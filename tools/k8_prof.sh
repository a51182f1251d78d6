#!/bin/bash
# per-kernel time of the K8 fallback sort on a workload (ncu launch list)
CFG=${1:-c4}
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k8_ python tools/prof_run.py --config $CFG --reps 1 2>&1 | grep -E "^  [a-z]|duration" > gpurun_out/k8_$CFG.txt
python3 - $CFG <<'PY'
import sys
from collections import defaultdict
lines=open(f'gpurun_out/k8_{sys.argv[1]}.txt').read().splitlines()
agg=defaultdict(lambda:[0,0.0]); name=None
for l in lines:
    if 'duration' not in l: name=l.split('(')[0].strip()
    else:
        p=l.split(); v=float(p[-1].replace(',',''))*{'us':1e-3,'ms':1,'ns':1e-6}.get(p[-2],1); agg[name][0]+=1; agg[name][1]+=v
for k,(c,t) in agg.items(): print(f"{t:8.3f} ms x{c} {k}")
PY
