#!/bin/bash
# K1 factored element GEMM: parity (new A/B test + the parity suites that use the element route), then per-level
# kernel times with the factored and the full route on cfg3 / cfg4 / cfg2.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_k1_fgemm.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/k1_tests.log 2>&1; echo "rc $?" >> gpurun_out/k1_tests.log
for c in 3 4 2; do
  for f in 1 0; do
    STGMG_K1_FGEMM=$f timeout 600 python tools/kernel_times.py --config $c > gpurun_out/kt_cfg${c}_fg$f.log 2>&1
  done
done
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:op_fgemm -s 0 -c 1 -o gpurun_out/full_cfg4_fgemm python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_fg.log 2>&1
python tools/ncu_summary.py gpurun_out/full_cfg4_fgemm.ncu-rep > gpurun_out/sum_cfg4_fgemm.txt 2>&1
ncu -i gpurun_out/full_cfg4_fgemm.ncu-rep --page source --csv > gpurun_out/src_cfg4_fgemm.csv 2>/dev/null
rm -f gpurun_out/full_cfg4_fgemm.ncu-rep
