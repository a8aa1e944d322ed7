#!/bin/bash
# Session 4: K4 inverses on streams of their own (launch_inverse_async): setup time async vs serial
# (STGMG_SETUP_SERIAL=1), the bitwise async == serial test, parity suites fed by the inverses.
mkdir -p gpurun_out
( python tools/setup_times.py 4 4 3 3 2 2;
  STGMG_SETUP_SERIAL=1 python tools/setup_times.py 4 4 3 3 2 2 ) > gpurun_out/setup_async_s4.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_setup_async.py tests/test_gpu_parity.py tests/test_gpu_api.py \
  tests/test_gpu_multirank.py tests/test_gpu_lshape.py -q -p no:cacheprovider > gpurun_out/pytest_gpu_s4b.log 2>&1
echo "pytest rc $?" >> gpurun_out/pytest_gpu_s4b.log
