#!/bin/bash
# Round-2 evidence for the bench workload (cfg4): launch list of one slab step, ncu --set full of fine K1 / K2D.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_r02_cfg4.csv python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/prof_step.log 2>&1
python tools/launch_summary.py gpurun_out/launches_r02_cfg4.csv > gpurun_out/launches_r02_cfg4.txt
