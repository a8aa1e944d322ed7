#!/bin/bash
# Round-2 ncu evidence at BASELINE sizes: launch list of one cfg4 slab step, then ncu --set full of the fine-level
# instance of K1 (element GEMM + node gather), K3, the residual expansion, K5 restriction, the MGS pass and K2D on
# cfg4; K3/K5/gather at cfg2 and cfg3.  Reports land in gpurun_out/ (read back with ncu -i).
mkdir -p gpurun_out
P="ncu --profile-from-start off --clock-control none"
timeout 300 python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/plain4.log 2>&1; tail -1 gpurun_out/plain4.log
timeout 900 $P --metrics gpu__time_duration.sum --csv --log-file gpurun_out/launches_r02_cfg4.csv \
    python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_l4.log 2>&1; tail -1 gpurun_out/ncu_l4.log
for k in patch_gemm_kernel gather_nodal avg_nodal expand_pull restrict_nodal mgs_dot patch_gemm_dense; do
  timeout 600 $P --set full --import-source on -k regex:$k -s 0 -c 1 -o gpurun_out/full_cfg4_$k \
      python tools/profile_step.py --config 4 --warmup 1 > gpurun_out/ncu_f4_$k.log 2>&1; tail -1 gpurun_out/ncu_f4_$k.log
  python tools/ncu_summary.py gpurun_out/full_cfg4_$k.ncu-rep > gpurun_out/sum_cfg4_$k.txt 2>&1
done
for c in 2 3; do
  for k in gather_nodal avg_nodal restrict_nodal expand_pull; do
    timeout 600 $P --set full -k regex:$k -s 0 -c 1 -o gpurun_out/full_cfg${c}_$k \
        python tools/profile_step.py --config $c --warmup 1 > gpurun_out/ncu_f${c}_$k.log 2>&1; tail -1 gpurun_out/ncu_f${c}_$k.log
    python tools/ncu_summary.py gpurun_out/full_cfg${c}_$k.ncu-rep > gpurun_out/sum_cfg${c}_$k.txt 2>&1
  done
done
python tools/launch_summary.py gpurun_out/launches_r02_cfg4.csv > gpurun_out/launches_r02_cfg4.txt
# the reports exceed gpurun's 64 MiB return limit: keep the text summaries and the K1 / K3 reports only
for f in gpurun_out/full_*.ncu-rep; do
  case $f in *cfg4_patch_gemm_kernel*|*cfg4_avg_nodal*) ;; *) rm -f $f ;; esac
done
ls -la gpurun_out
