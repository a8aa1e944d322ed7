#!/bin/bash
# Session 4: separable restriction forced onto cfg4's fine level (STGMG_RESTRICT_SEP=2) vs the gather form:
# per-level R+P and V-cycle times (CUDA events); V-cycle parity with the forced form.
mkdir -p gpurun_out
STGMG_SETUP_TIMES=2 timeout 300 python tools/setup_times.py 4 4 3 > gpurun_out/setup_host_s4.log 2>&1
( timeout 600 python tools/kernel_times.py --config 4; echo "=== STGMG_RESTRICT_SEP=2";
  STGMG_RESTRICT_SEP=2 timeout 600 python tools/kernel_times.py --config 4 ) > gpurun_out/k5_sep_cfg4_s4.log 2>&1
STGMG_RESTRICT_SEP=2 timeout 900 python -m pytest tests/test_gpu_transfer_sep.py tests/test_gpu_fullsize_ebe.py -q \
  -p no:cacheprovider > gpurun_out/pytest_k5_sep_s4.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_k5_sep_s4.log
