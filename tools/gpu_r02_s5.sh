#!/bin/bash
# Session-5 closing evidence on one B200: bench lines of cfg1-3 at the final state, ncu launch list of one cfg4 slab
# step (profile_step.py, as the s3 list) and setup times of cfg2-4.
mkdir -p gpurun_out/s5
for c in 1 2 3; do
  timeout 900 python bench.py --config $c > gpurun_out/s5/bench_cfg$c.json 2> gpurun_out/s5/bench_cfg$c.err; echo "bench cfg$c rc $?" >> gpurun_out/s5/bench_cfg$c.err
done
timeout 600 python tools/setup_times.py 4 4 3 3 2 2 > gpurun_out/s5/setup_times.log 2>&1
P="ncu --profile-from-start off --clock-control none"
timeout 900 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/s5/launches_r02_cfg4_s5.csv \
  python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/s5/ncu_launches.log 2>&1
python tools/launch_summary.py gpurun_out/s5/launches_r02_cfg4_s5.csv > gpurun_out/s5/launches_r02_cfg4_s5.txt
rm -f gpurun_out/s5/launches_r02_cfg4_s5.csv
head -12 gpurun_out/s5/launches_r02_cfg4_s5.txt; tail -6 gpurun_out/s5/setup_times.log
