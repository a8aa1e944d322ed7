#!/bin/bash
# Session-3 check: parity suites that run the cfg4 fine level (sum-factorised K1 on by default there), the bench line,
# and the setup-phase breakdown of cfg4 / cfg3.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_k1_fgemm.py tests/test_gpu_fullsize_ebe.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/s3_tests.log 2>&1; echo "rc $?" >> gpurun_out/s3_tests.log
timeout 900 python bench.py > gpurun_out/bench_s3.json 2> gpurun_out/bench_s3.err; echo "bench rc $?" >> gpurun_out/bench_s3.err
STGMG_SETUP_TIMES=1 timeout 300 python tools/setup_times.py 4 3 > gpurun_out/setup_s3.log 2>&1
