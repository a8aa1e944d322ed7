# Full GPU check: gpu tests, smoke, bench line, ncu launch list, one ncu --set full capture of K2 (fine level).
mkdir -p gpurun_out
R=${1:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_$R.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_$R.log 2>&1; tail -3 gpurun_out/pytest_gpu_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; tail -1 gpurun_out/smoke_$R.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; tail -3 gpurun_out/bench_$R.err; cat gpurun_out/bench_$R.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_bench_$R.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu0.log 2>&1; tail -1 gpurun_out/ncu0.log
timeout 300 python tools/profile_step.py > gpurun_out/plain.log 2>&1 && timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$R.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1; tail -1 gpurun_out/ncu1.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:patch_gemm -s 0 -c 1 -o gpurun_out/k2_full_$R python tools/profile_step.py > gpurun_out/ncu2.log 2>&1; tail -1 gpurun_out/ncu2.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:op2d_cell -s 0 -c 1 -o gpurun_out/k1_full_$R python tools/profile_step.py > gpurun_out/ncu3.log 2>&1; tail -1 gpurun_out/ncu3.log
