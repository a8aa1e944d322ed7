#!/bin/bash
# Interleaved patch results on the dense K2 levels: K3 / sweep times (cfg4, cfg3, cfg2; on and off), then the suites
# that run dense levels (parity, dense, overwrite smoother, K2 variants, multi-rank, full size).
mkdir -p gpurun_out
for c in 4 3 2; do
  timeout 600 python tools/kernel_times.py --config $c > gpurun_out/kt_cfg${c}_yil1.log 2>&1
  STGMG_Y_IL=0 timeout 600 python tools/kernel_times.py --config $c > gpurun_out/kt_cfg${c}_yil0.log 2>&1
done
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_overwrite.py tests/test_gpu_k2_variants.py tests/test_gpu_multirank.py tests/test_gpu_fullsize_ebe.py tests/test_gpu_api.py -x -q -p no:cacheprovider > gpurun_out/yil_tests.log 2>&1; echo "rc $?" >> gpurun_out/yil_tests.log
