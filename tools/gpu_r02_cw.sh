#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transfer_sep.py tests/test_gpu_parity.py tests/test_gpu_multirank.py tests/test_gpu_multiproc.py tests/test_gpu_fold.py -x -q -p no:cacheprovider > gpurun_out/cw.log 2>&1; echo "rc $?" >> gpurun_out/cw.log
for c in 4 3 2 1; do timeout 400 python tools/kernel_times.py --config $c > gpurun_out/ktcw_cfg$c.log 2>&1; done
timeout 600 ncu --profile-from-start off --clock-control none --set full -k regex:restrict_cw -s 0 -c 1 -o gpurun_out/rc4 python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_rc4.log 2>&1
python tools/ncu_summary.py gpurun_out/rc4.ncu-rep > gpurun_out/sum_cfg4_restrict_cw.txt 2>&1; rm -f gpurun_out/rc4.ncu-rep
timeout 600 ncu --profile-from-start off --clock-control none --set full -k regex:prolong_cw -s 8 -c 1 -o gpurun_out/pc4 python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_pc4.log 2>&1
python tools/ncu_summary.py gpurun_out/pc4.ncu-rep > gpurun_out/sum_cfg4_prolong_cw.txt 2>&1; rm -f gpurun_out/pc4.ncu-rep
