"""Per-level CUDA-event timings of the hot-path kernels (K2 patch GEMM, K1 apply, K3 average) and the V-cycle."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from stgmg_inputs import config  # noqa: E402
from paper_2303_06742_b200 import Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
a = ap.parse_args()
cfg = config(a.config)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
s = Solver(cfg, stream=st)
print("config", cfg["name"])
for l in range(s.levels - 1, -1, -1):
    line = "level %d N=%d" % (l, s.size(l))
    if l >= 1:
        w = s.level_work(l)
        t2 = s.time_kernel(0, l, reps=50)
        line += "  K2 %.2f us (%.2f TF/s)" % (t2 * 1e3, w["k2_flops"] / t2 / 1e9)
        line += "  K3 %.2f us" % (s.time_kernel(2, l, reps=50) * 1e3)
        line += "  sweep %.2f us  R+P %.2f us" % (s.time_kernel(6, l, reps=50) * 1e3, s.time_kernel(7, l, reps=50) * 1e3)
    line += "  K1 %.2f us" % (s.time_kernel(1, l, reps=50) * 1e3)
    print(line)
print("vcycle %.3f ms" % s.time_kernel(3, s.levels - 1, reps=20))
print("noop kernel (1 block) %.2f us, (148 blocks) %.2f us" % (s.time_kernel(4, 0, reps=50) * 1e3, s.time_kernel(5, 0, reps=50) * 1e3))
s.close()
