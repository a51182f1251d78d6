#!/bin/bash
# K7 phase profile (PCF_FLAG_PROFILE) for the fallback-heavy configs
for c in ${@:-c4 c3}; do python tools/k7_prof.py --config $c; done
