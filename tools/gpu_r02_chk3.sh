#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_overwrite.py tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -x -q -p no:cacheprovider > gpurun_out/chk3.log 2>&1; echo "rc $?" >> gpurun_out/chk3.log
for c in 4 3 2; do timeout 400 python tools/kernel_times.py --config $c > gpurun_out/kt3_cfg$c.log 2>&1; done
timeout 600 ncu --profile-from-start off --clock-control none --set full -k regex:avg_nodal -s 0 -c 1 -o gpurun_out/av4 python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_av4.log 2>&1
python tools/ncu_summary.py gpurun_out/av4.ncu-rep > gpurun_out/sum_cfg4_avg_nodal_v2.txt 2>&1; rm -f gpurun_out/av4.ncu-rep
timeout 600 ncu --profile-from-start off --clock-control none --set full -k regex:avg_nodal -s 0 -c 1 -o gpurun_out/av3 python tools/profile_step.py --config 3 --warmup 1 > gpurun_out/ncu_av3.log 2>&1
python tools/ncu_summary.py gpurun_out/av3.ncu-rep > gpurun_out/sum_cfg3_avg_nodal_v2.txt 2>&1; rm -f gpurun_out/av3.ncu-rep
