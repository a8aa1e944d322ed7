"""One slab step of the hot path between cudaProfilerStart/Stop, for ncu (--profile-from-start off).

  python tools/profile_step.py [--config 1] [--warmup 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from stgmg_inputs import config, uniform_load  # noqa: E402
from paper_2303_06742_b200 import Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--warmup", type=int, default=2)
a = ap.parse_args()
cfg = config(a.config)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
s = Solver(cfg, stream=stream)
N = s.size()
Xp = torch.zeros(N, dtype=torch.float64, device="cuda")
rhs, x = torch.zeros_like(Xp), torch.zeros_like(Xp)
kind = {"manufactured": 0, "beam": 1}.get(cfg["load"])   # LOAD_MANUFACTURED / LOAD_BEAM_TRACTION, as bench.py
L = torch.as_tensor(uniform_load(N, cfg["seed"] or 1), device="cuda") if kind is None else torch.zeros_like(Xp)
if kind == 0:
    s.initial_state(0, 0.0, Xp)
n = [0]


def step():
    if kind is not None:
        s.slab_load(kind, n[0] * cfg["tau"], L)
    n[0] += 1
    s.slab_rhs(L, Xp, rhs)
    x.zero_()
    st = s.solve(rhs, x)
    Xp.copy_(x)
    return st


for _ in range(a.warmup):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
st = step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("profiled step:", st, "launches", s.launch_count())
s.close()
