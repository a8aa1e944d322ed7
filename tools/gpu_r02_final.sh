#!/bin/bash
# Round-2 evidence on one B200: full -m gpu suite, smoke, default bench line (cfg4) + reference arm, launch list of a
# cfg4 slab step, ncu --set full summaries of the fine-level K2D, factored K1, gather, K3, expansion and the
# separable restriction (reports removed after summarising: gpurun returns <= 64 MiB).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
P="ncu --profile-from-start off --clock-control none"
timeout 900 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_r02_cfg4_final.csv \
    python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_l4.log 2>&1
python tools/launch_summary.py gpurun_out/launches_r02_cfg4_final.csv > gpurun_out/launches_r02_cfg4_final.txt
for k in patch_gemm_dense op_fgemm gather_nodal avg_nodal expand_pull restrict_pass; do
  timeout 600 $P --set full --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/f4_$k \
      python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_f4_$k.log 2>&1
  python tools/ncu_summary.py gpurun_out/f4_$k.ncu-rep > gpurun_out/sum_cfg4_$k.txt 2>&1
  rm -f gpurun_out/f4_$k.ncu-rep
done
for c in 2 3; do
  for k in restrict_pass avg_nodal; do
    timeout 600 $P --set full -k regex:$k -s 0 -c 1 -o gpurun_out/f${c}_$k python tools/profile_step.py --config $c --warmup 1 > gpurun_out/ncu_f${c}_$k.log 2>&1
    python tools/ncu_summary.py gpurun_out/f${c}_$k.ncu-rep > gpurun_out/sum_cfg${c}_$k.txt 2>&1
    rm -f gpurun_out/f${c}_$k.ncu-rep
  done
done
