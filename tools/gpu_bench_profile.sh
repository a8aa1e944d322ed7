# Full bench line + ncu launch list + one ncu --set full capture of the dominant kernel (K2 fine level).
mkdir -p gpurun_out
R=${1:-r01}
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; tail -3 gpurun_out/bench_$R.err; cat gpurun_out/bench_$R.json
timeout 300 python tools/profile_step.py > gpurun_out/plain.log 2>&1 && timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:patch_gemm -s 0 -c 1 -o gpurun_out/k2_full_$R python tools/profile_step.py > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
