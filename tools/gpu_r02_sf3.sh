#!/bin/bash
# SF v3 (pressure/mass warp) parity + K1 times; ncu launch durations of the GJ kernels during a cfg3 setup.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1_fgemm.py -x -q -p no:cacheprovider > gpurun_out/sf3_tests.log 2>&1; echo "rc $?" >> gpurun_out/sf3_tests.log
timeout 600 python tools/kernel_times.py --config 4 > gpurun_out/kt_cfg4_sf3v3.log 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -k regex:gjb_ --csv --log-file gpurun_out/gj_launches.csv python tools/setup_times.py 3 > gpurun_out/gj_ncu.log 2>&1
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:op_sf3 -s 0 -c 1 -o gpurun_out/full_cfg4_sf3 python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_sf.log 2>&1
python tools/ncu_summary.py gpurun_out/full_cfg4_sf3.ncu-rep > gpurun_out/sum_cfg4_sf3v3.txt 2>&1
rm -f gpurun_out/full_cfg4_sf3.ncu-rep
