"""Table 4 rows of the L-shaped benchmark on the GPU: march I = (0, T] with tau = 0.01 and report the
average GMRES iterations and the ranges of the goal quantities (Eq:DefGQ).

  python tools/lshape_table4.py --ref 2 --k 1 --r 2 [--E 20000] [--tol 1e-8] [--abs] [--T 4]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2303_06742_b200 import LShapeSolver  # noqa: E402
from paper_2303_06742_b200.stgmg import LOAD_LSHAPE_TRACTION, TOL_ABS, TOL_REL  # noqa: E402


def params(r, E, nu=0.3):
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    return dict(rho=1.0, alpha=0.9, c0=0.01, lam=lam, mu=mu, K=[1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0],
                gamma_a=5e4 * r * (r + 1), gamma_b=0.5 * r * (r - 1))


ap = argparse.ArgumentParser()
ap.add_argument("--ref", type=int, default=2)
ap.add_argument("--coarse", type=int, default=1)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--r", type=int, default=2)
ap.add_argument("--E", type=float, default=20000.0)
ap.add_argument("--tol", type=float, default=1e-8)
ap.add_argument("--abs", action="store_true")
ap.add_argument("--T", type=float, default=4.0)
ap.add_argument("--hf", default="measure", choices=["measure", "edge", "dir_edge", "frozen", "u_meas_p_edge", "u_edge_p_meas", "face"])
a = ap.parse_args()
tau = 0.01
t0 = time.perf_counter()
s = LShapeSolver(a.ref, a.ref - a.coarse + 1, a.r, a.k, tau, params(a.r, a.E), hF_mode={"measure": 0, "edge": 1, "dir_edge": 2, "frozen": 3, "u_meas_p_edge": 4, "u_edge_p_meas": 5, "face": 6}[a.hf])
setup = time.perf_counter() - t0
N = s.size()
X = torch.zeros(N, dtype=torch.float64, device="cuda")
L, F, x = torch.zeros_like(X), torch.zeros_like(X), torch.zeros_like(X)
its, goal, secs, conv = [], [], [], []
nsl = int(round(a.T / tau))
for n in range(nsl):
    s.slab_load(LOAD_LSHAPE_TRACTION, n * tau, L)
    s.slab_rhs(L, X, F)
    x.zero_()
    st = s.solve(F, x, tol=a.tol, tol_mode=TOL_ABS if a.abs else TOL_REL, restart=30, maxit=300)
    its.append(st["iterations"])
    conv.append(st["converged"])
    secs.append(st["seconds"])
    X.copy_(x)
    goal.append(s.goal_quantities(X, 1))
g = np.array(goal)
# the dominant kernel: K2u (per-patch inverse GEMV) on the fine level, HBM-bound (MEASURED_PEAKS copy bandwidth)
lf = s.levels - 1
t2 = s.time_kernel(0, lf, reps=20)
fl2, by2 = s.kernel_work(0, lf)
tv = s.time_kernel(3, lf, reps=5)
k2u = dict(avg_launch_ms=t2, bytes=by2, hbm_gbs=by2 / (t2 * 1e-3) / 1e9, hbm_frac=by2 / (t2 * 1e-3) / 1e9 / 6550.7,
           vcycle_ms=tv)
print(json.dumps(dict(ref=a.ref, coarse=a.coarse, k=a.k, r=a.r, E=a.E, hF=a.hf, dofs=N, tol=a.tol, tol_mode="abs" if a.abs else "rel",
                      slabs=nsl, avg_its=float(np.mean(its)), min_its=int(min(its)), max_its=int(max(its)),
                      converged=int(sum(conv)), bu=[float(g[:, 0].min()), float(g[:, 0].max())],
                      bp=[float(g[:, 1].min()), float(g[:, 1].max())], s_per_slab=float(np.median(secs)),
                      setup_s=setup, k2u=k2u)))
s.close()
