#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_transfer_sep.py tests/test_gpu_k2_variants.py -x -q -p no:cacheprovider > gpurun_out/chk.log 2>&1; echo "rc $?" >> gpurun_out/chk.log
for c in 4 3 2; do timeout 400 python tools/kernel_times.py --config $c > gpurun_out/ktc_cfg$c.log 2>&1; done
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:patch_gemm_dense -s 0 -c 1 --csv python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/k2d_dram.csv 2>&1
