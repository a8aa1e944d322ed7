"""Where the FGMRES solve's time goes beyond its V-cycles: device time of stgmg_solve (stats) vs the same number of
V-cycles + operator applies enqueued back to back without host synchronisation."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from stgmg_inputs import config, uniform_load  # noqa: E402
from paper_2303_06742_b200 import Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
a = ap.parse_args()
cfg = config(a.config)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
s = Solver(cfg, stream=st)
N = s.size()
b = torch.as_tensor(uniform_load(N, 1), device="cuda")
x = torch.zeros_like(b)
z = torch.zeros_like(b)
w = torch.zeros_like(b)
for _ in range(3):
    x.zero_()
    r = s.solve(b, x)
torch.cuda.synchronize()
secs = []
for _ in range(10):
    x.zero_()
    r = s.solve(b, x)
    secs.append(r["seconds"])
its = r["iterations"]
t_solve = sorted(secs)[len(secs) // 2] * 1e3
vc = s.time_kernel(3, reps=20)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
for _ in range(10):
    for i in range(its):
        s.vcycle(b, z)
        s.apply(z, w)
e1.record(st)
torch.cuda.synchronize()
t_seq = e0.elapsed_time(e1) / 10
print("config %s its %d: solve %.3f ms  vcycle %.3f ms  its x (vcycle + apply) no-sync %.3f ms  overhead %.3f ms"
      % (cfg["name"], its, t_solve, vc, t_seq, t_solve - t_seq))
s.close()
