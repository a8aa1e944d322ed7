"""GPU parity at BASELINE's full sizes (configs 2, 3, 4; -m gpu), in the launch configuration bench.py times.

The oracle cannot assemble these levels in seconds, so it is evaluated on samples (oracle/sampled.py, itself pinned
against the assembled definitions by tests/test_oracle_pins.py::test_sampled_helpers_match_global_definitions):
  * rows of A x on random vectors (corner, face and interior rows): 1e-13 relative;
  * one smoothing sweep of Algorithm 1 at sampled DoFs: 1e-9 relative (derivation in test_gpu_parity.py);
  * a full FGMRES-GMG slab solve: converged to the config's rtol, and the GPU's residual agrees with the oracle's
    rows of b - A x at sampled rows to 1e-10 ||b||_inf (a property that holds at any size).
"""
import numpy as np
import pytest

from stgmg_inputs import config, uniform_load, random_vector
from tests.gpu_common import to_gpu, to_np, oracle_params

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[2, 3, 4], ids=["cfg2", "cfg3", "cfg4"])
def full(request):
    import torch
    from paper_2303_06742_b200 import Solver
    from oracle.mesh import Level
    from oracle.sampled import LiteOperator
    cfg = config(request.param)
    s = Solver(cfg)
    d = cfg["dim"]
    lev = Level(d, cfg["cells"][:d], cfg["lo"][:d], cfg["hi"][:d], cfg["r"], cfg["k"], list(cfg["bc_u"][:2 * d]),
                list(cfg["bc_p"][:2 * d]))
    lite = LiteOperator(lev, oracle_params(cfg), cfg["tau"])
    cfg = dict(cfg, test_seed=cfg["seed"] if cfg["seed"] is not None else 100 + request.param)
    yield cfg, s, lev, lite
    s.close()
    torch.cuda.synchronize()


def sample_rows(lev, n, seed):
    rng = np.random.default_rng(seed)
    fixed = [0, lev.nq - 1, lev.R + lev.nq // 2, 2 * lev.R, lev.block - 1, lev.N - 1]   # corners, pressure, last
    return np.unique(np.concatenate([fixed, rng.choice(lev.N, n, replace=False)]))


def test_full_sizes(full):
    cfg, s, lev, lite = full
    assert s.size() == lev.N
    coarse = lev
    for l in range(cfg["levels"] - 1, -1, -1):
        assert s.size(l) == coarse.N
        if l:
            coarse = coarse.coarsen()


def test_full_operator_sampled_rows(full):
    import torch
    cfg, s, lev, lite = full
    x = random_vector(lev.N, 201)
    y = torch.zeros(lev.N, dtype=torch.float64, device="cuda")
    s.apply(to_gpu(x), y)
    torch.cuda.synchronize()
    yg = to_np(y)
    rows = sample_rows(lev, 40, 202)
    yo = lite.rows(x, rows)
    assert np.abs(yg[rows] - yo).max() <= 1e-13 * np.abs(yg).max()


def test_full_sweep_sampled(full):
    import torch
    cfg, s, lev, lite = full
    b, d0 = random_vector(lev.N, 203), random_vector(lev.N, 204, 1e-3)
    d = to_gpu(d0)
    s.smooth_sweep(to_gpu(b), d)
    torch.cuda.synchronize()
    dg = to_np(d)
    rng = np.random.default_rng(205)
    sample = np.concatenate([[0, lev.N - 1], rng.choice(lev.N, 3, replace=False)])
    do = lite.sampled_sweep(b, d0, sample)
    assert np.abs(dg[sample] - do).max() <= 1e-9 * np.abs(dg).max()


def test_full_solve_residual(full):
    import torch
    cfg, s, lev, lite = full
    b = uniform_load(lev.N, cfg["test_seed"])
    bt = to_gpu(b)
    x = torch.zeros(lev.N, dtype=torch.float64, device="cuda")
    st = s.solve(bt, x, tol=cfg["rtol"], restart=cfg["restart"])
    r = torch.zeros_like(x)
    s.residual(bt, x, r)
    torch.cuda.synchronize()
    assert st["converged"], st
    rg, xg = to_np(r), to_np(x)
    assert np.linalg.norm(rg) <= cfg["rtol"] * np.linalg.norm(b) * (1 + 1e-6)
    rows = sample_rows(lev, 30, 206)
    ro = b[rows] - lite.rows(xg, rows)
    assert np.abs(rg[rows] - ro).max() <= 1e-10 * np.abs(b).max()
    assert 1 <= st["iterations"] <= 60
