# Round evidence: bench line (cfg1, with CPU baseline), ncu launch list of one slab step, ncu --set full of the
# dominant kernel (dense K2 on the fine level) for cfg1 and cfg3.
mkdir -p gpurun_out
R=${1:-r01}
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; tail -2 gpurun_out/bench_$R.err; cat gpurun_out/bench_$R.json
timeout 300 python tools/profile_step.py > gpurun_out/plain.log 2>&1 && timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1; tail -1 gpurun_out/ncu1.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:patch_gemm_dense -s 0 -c 1 -o gpurun_out/k2d_cfg1_$R python tools/profile_step.py > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:patch_gemm_dense -s 0 -c 1 -o gpurun_out/k2d_cfg3_$R python tools/profile_step.py --config 3 --warmup 1 > gpurun_out/ncu3.log 2>&1; tail -1 gpurun_out/ncu3.log
