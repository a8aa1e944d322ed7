import sys, time
sys.path.insert(0, '.')
import torch
from stgmg_inputs import config
from paper_2303_06742_b200 import Solver
for c in (int(a) for a in sys.argv[1:]):
    t = time.perf_counter(); s = Solver(config(c)); torch.cuda.synchronize(); print("cfg", c, "setup", time.perf_counter() - t, flush=True); s.close()
