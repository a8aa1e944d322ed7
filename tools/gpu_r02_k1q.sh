#!/bin/bash
# quick K1 iteration: A/B parity test and cfg4 / cfg3 per-level times, ncu of the fine-level factored GEMM
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_k1_fgemm.py -x -q -p no:cacheprovider > gpurun_out/k1q_tests.log 2>&1; echo "rc $?" >> gpurun_out/k1q_tests.log
for c in 4 3; do timeout 600 python tools/kernel_times.py --config $c > gpurun_out/ktq_cfg$c.log 2>&1; done
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:op_fgemm -s 0 -c 1 -o gpurun_out/fq python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_fq.log 2>&1
python tools/ncu_summary.py gpurun_out/fq.ncu-rep > gpurun_out/sum_fq.txt 2>&1
ncu -i gpurun_out/fq.ncu-rep --page source --csv > gpurun_out/src_fq.csv 2>/dev/null
rm -f gpurun_out/fq.ncu-rep
