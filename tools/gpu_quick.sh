# Quick GPU iteration: all GPU tests, per-level kernel times (cfg1, optional extra configs), short bench line.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
for c in ${CFGS:-1}; do timeout 600 python tools/kernel_times.py --config $c 2>&1 | tail -9; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python -c "import json; d=json.load(open('gpurun_out/bench_q.json')); print('value', d['value'], 'ms/slab', d['ms_per_step'], 'vcycle_ms', d['config']['vcycle_ms'], 'K2 frac', d['roofline']['frac'])"
