#!/bin/bash
# K7 instruction count / duration of build variants: tools/k7_variants.sh "cfg[:n] ..." lib1.so lib2.so ...
CFGS=$1; shift
for L in paper_2405_07122_b200/libpcfsort.so "$@"; do
  for A in $CFGS; do
    CFG=${A%%:*}; N=${A#*:}; NARG=""; [ "$N" != "$A" ] && NARG="--n $N"
    echo "== $L $A"
    PCF_LIB=$L python tools/k7_prof.py --config $CFG $NARG | head -1
    PCF_LIB=$L ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum -k regex:k7_kernel -c 1 \
        python tools/prof_run.py --config $CFG $NARG --reps 1 2>&1 | grep -E "inst_executed|duration"
  done
done
