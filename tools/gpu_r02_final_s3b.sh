#!/bin/bash
# Session-3 closing check on one B200: full -m gpu suite, smoke, default bench line (cfg4), ncu --set full of the
# fine-level K3 and gather after the predicated loads.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_s3b.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_s3b.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3b.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_s3b.log
timeout 900 python bench.py > gpurun_out/bench_s3b.json 2> gpurun_out/bench_s3b.err; echo "bench rc $?" >> gpurun_out/bench_s3b.err
P="ncu --profile-from-start off --clock-control none"
for k in avg_nodal gather_nodal; do
  timeout 600 $P --set full -k regex:$k -s 0 -c 1 -o gpurun_out/f4b_$k python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_f4b_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/f4b_$k.ncu-rep > gpurun_out/sum_cfg4_${k}_s3b.txt 2>&1
  rm -f gpurun_out/f4b_$k.ncu-rep
done
