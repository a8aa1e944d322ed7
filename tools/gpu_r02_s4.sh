#!/bin/bash
# Session-4 opening check on one B200 after the container rebuild: full -m gpu suite, smoke, default bench line (cfg4).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_s4.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_s4.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s4.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_s4.log
timeout 900 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; echo "bench rc $?" >> gpurun_out/bench_s4.err
