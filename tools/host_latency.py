import sys, time, os
sys.path.insert(0, "/root/repo")
import torch
from stgmg_inputs import config, uniform_load
from paper_2303_06742_b200 import Solver
cfg = config(1)
st = torch.cuda.Stream(); torch.cuda.set_stream(st)
s = Solver(cfg, stream=st)
N = s.size()
b = torch.as_tensor(uniform_load(N, 1), device="cuda"); z = torch.zeros_like(b); w = torch.zeros_like(b)
for _ in range(5): s.vcycle(b, z)
torch.cuda.synchronize()
# host time of one vcycle enqueue when the GPU is idle (sync before each)
ts = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); s.vcycle(b, z); t1 = time.perf_counter(); ts.append(t1 - t0)
print("host enqueue of one V-cycle (memcpy + graph launch + memcpy): median %.1f us" % (sorted(ts)[25] * 1e6))
ts = []
for _ in range(50):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); s.apply(z, w); t1 = time.perf_counter(); ts.append(t1 - t0)
print("host enqueue of one apply: median %.1f us" % (sorted(ts)[25] * 1e6))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(30):
    torch.cuda.synchronize()
    e0.record(st); s.vcycle(b, z); e1.record(st); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("device time event->event around one V-cycle issued from idle: median %.3f ms" % sorted(ts)[15])
s.close()
