#!/bin/bash
# K1 sum-factorised volume kernel (op_sf3.cu): route parity tests, per-level K1 times with SF on (3 or 2 CTAs/SM) and
# off (cfg4, cfg3), then one ncu --set full capture of op_sf3 at cfg4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_k1_fgemm.py -x -q -p no:cacheprovider > gpurun_out/sf_tests.log 2>&1; echo "rc $?" >> gpurun_out/sf_tests.log
for c in 4 3; do
  for m in 3 2; do
    STGMG_SF3_MINB=$m timeout 600 python tools/kernel_times.py --config $c > gpurun_out/kt_cfg${c}_sf1_m$m.log 2>&1
  done
  STGMG_K1_SF=0 timeout 600 python tools/kernel_times.py --config $c > gpurun_out/kt_cfg${c}_sf0.log 2>&1
done
if [ "${SF_NCU:-1}" = 1 ]; then
timeout 600 ncu --profile-from-start off --clock-control none --set full --import-source on -k regex:op_sf3 -s 0 -c 1 -o gpurun_out/full_cfg4_sf3 python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_sf.log 2>&1
python tools/ncu_summary.py gpurun_out/full_cfg4_sf3.ncu-rep > gpurun_out/sum_cfg4_sf3.txt 2>&1
ncu -i gpurun_out/full_cfg4_sf3.ncu-rep --page source --csv > gpurun_out/src_cfg4_sf3.csv 2>/dev/null
rm -f gpurun_out/full_cfg4_sf3.ncu-rep
fi
