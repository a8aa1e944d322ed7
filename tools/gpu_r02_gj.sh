#!/bin/bash
# GJ panel (division-free rows x columns mapping) and trailing update (coalesced epilogue): setup times, GJ launch
# durations (ncu) during a cfg3 setup, and the parity suites whose inverses come from it.
mkdir -p gpurun_out
STGMG_SETUP_TIMES=1 timeout 300 python tools/setup_times.py 4 4 3 > gpurun_out/setup_gj9.log 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:gjb_ --csv --log-file gpurun_out/gj_launches9.csv python tools/setup_times.py 3 > gpurun_out/gj_ncu9.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lshape.py tests/test_gpu_api.py tests/test_gpu_k2_variants.py -x -q -p no:cacheprovider > gpurun_out/gj_tests9.log 2>&1; echo "rc $?" >> gpurun_out/gj_tests9.log
