#!/bin/bash
# Bounds / protocol assertions of our own (TSDS_CHECK, -DTSDS_CHECKED) over the kernel families:
# build the checked library, run the sanitizer cases, the mode-forcing parity tests and the
# stress tests through it (run under gpurun; the library must have been built here first:
#   make -C paper_2307_05389_b200/csrc ../libtsds_checked.so VFLAGS=-DTSDS_CHECKED).
TAG=${1:-r02}
LIB=$PWD/paper_2307_05389_b200/libtsds_checked.so
[ -f "$LIB" ] || { echo "missing $LIB"; exit 1; }
mkdir -p gpurun_out
{
  echo "== TSDS_CHECKED build: tools/sanitize_cases.py"
  TSDS_LIB=$LIB timeout 900 python tools/sanitize_cases.py 2>&1 | tail -30
  echo "== TSDS_CHECKED build: pytest (mode-forcing parity, stress, configs C1-C3)"
  TSDS_LIB=$LIB timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -m gpu -q 2>&1 | tail -6
} > gpurun_out/${TAG}_checked.log 2>&1
tail -12 gpurun_out/${TAG}_checked.log
