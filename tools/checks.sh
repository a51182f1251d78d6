#!/bin/bash
# Debug bounds-check run (the compute-sanitizer substitute): the GPU
# parity suite against a -DPCF_CHECKS=1 build; any violated index bound makes the
# sort return PCF_ERR_INTERNAL, i.e. a failing test.  Log -> gpurun_out/checks_pytest.log
mkdir -p gpurun_out
python -c "
import sys; sys.path.insert(0, '.')
from paper_2405_07122_b200._build import build_variant
build_variant('build/checks.so', {'PCF_CHECKS': 1})" > gpurun_out/checks_build.log 2>&1
PCF_LIB=build/checks.so timeout 1500 python -m pytest tests -q -m gpu -k "not 1e9" "$@" > gpurun_out/checks_pytest.log 2>&1
echo "checks pytest rc=$?"; tail -3 gpurun_out/checks_pytest.log
