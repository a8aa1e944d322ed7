mkdir -p gpurun_out
timeout 300 python tools/kernel_times.py --config 1 2>&1 | tail -12
timeout 300 python tools/profile_step.py > gpurun_out/plain.log 2>&1 && timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:patch_gemm -s 0 -c 1 -o gpurun_out/k2_full python tools/profile_step.py > gpurun_out/ncu2.log 2>&1; tail -2 gpurun_out/ncu2.log
