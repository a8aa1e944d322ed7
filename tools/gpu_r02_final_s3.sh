#!/bin/bash
# Session-3 evidence on one B200: full -m gpu suite, smoke, default bench line (cfg4) + reference arm, launch list of a
# cfg4 slab step, ncu --set full summaries of the fine-level K2D, sum-factorised K1, factored K1 (face types), gather,
# K3, expansion (reports removed after summarising: gpurun returns <= 64 MiB).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_s3.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_s3.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_s3.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s3.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_s3.log
timeout 900 python bench.py > gpurun_out/bench_s3f.json 2> gpurun_out/bench_s3f.err; echo "bench rc $?" >> gpurun_out/bench_s3f.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_s3.json 2> gpurun_out/bench_ref_s3.err
P="ncu --profile-from-start off --clock-control none"
timeout 900 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_r02_cfg4_s3.csv \
    python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_l4_s3.log 2>&1
python tools/launch_summary.py gpurun_out/launches_r02_cfg4_s3.csv > gpurun_out/launches_r02_cfg4_s3.txt
for k in op_sf3 op_fgemm gather_nodal patch_gemm_dense; do
  timeout 600 $P --set full --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/f4_$k \
      python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_f4_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/f4_$k.ncu-rep > gpurun_out/sum_cfg4_${k}_s3.txt 2>&1
  rm -f gpurun_out/f4_$k.ncu-rep
done
