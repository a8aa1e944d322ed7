mkdir -p gpurun_out
for c in 2 3; do
  timeout 600 python tools/kernel_times.py --config $c 2>&1 | tail -12
  timeout 900 python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; tail -2 gpurun_out/bench_c$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print('cfg', $c, d['value'], 'ms/slab', d['ms_per_step'], 'its', d['config']['gmres_iterations_total'], 'setup', d['config']['setup_s'], 'vc', d['config']['vcycle_ms'], 'K2 frac', d['roofline']['frac'])"
done
