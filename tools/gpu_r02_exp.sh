#!/bin/bash
# expand_pull loads in flight per thread: 4 (default) / 8 / 16 — one sweep time on the dense fine levels
mkdir -p gpurun_out
cat > /tmp/sw.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch
from stgmg_inputs import config
from paper_2303_06742_b200 import Solver
for c in (4, 3, 2):
    s = Solver(config(c)); L = s.levels - 1
    print(c, "sweep_us %.1f" % (s.time_kernel(6, L, reps=10) * 1e3), flush=True); s.close()
PY
for p in 4 8 16; do echo "per $p" >> gpurun_out/exp.log; STGMG_EXPAND_PER=$p timeout 400 python /tmp/sw.py >> gpurun_out/exp.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_dense.py -x -q -p no:cacheprovider > gpurun_out/exp_t.log 2>&1; echo rc $? >> gpurun_out/exp_t.log
