mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 600 python tools/kernel_times.py --config 3 2>&1 | tail -9
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -2 gpurun_out/bench_c3.err
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print('cfg3', d['value'], 'ms/slab', d['ms_per_step'], 'its', d['config']['gmres_iterations_total'], 'setup', d['config']['setup_s'], 'vc', d['config']['vcycle_ms'], 'K2 frac', d['roofline']['frac'])"
