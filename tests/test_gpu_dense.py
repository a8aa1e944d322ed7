"""GPU parity of the dense K2 path (patch-expanded residual + bulk-copied B, warp-specialised pipeline) against the
oracle.  The dense path runs on levels with >= 2000 patches (the big / wide tile variants); here it is forced onto
the fine level of small configurations (STGMG_K2_VARIANT + STGMG_K2_DENSE=1, read at setup) so that the oracle finishes in seconds.
The full-size configurations exercise it without forcing in test_gpu_fullsize.py."""
import os

import numpy as np
import pytest

from stgmg_inputs import uniform_load, random_vector
from tests.gpu_common import small_config, oracle_hierarchy, cfg_key, to_gpu, to_np

pytestmark = pytest.mark.gpu

CASES = [("cfg1s_big", 1, 2), ("cfg1s_wide", 1, 6), ("cfg3s_big", 3, 2), ("cfg4s_wide", 4, 6)]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def pair(request):
    import torch
    from paper_2303_06742_b200 import Solver
    _, ci, var = request.param
    cfg = small_config(ci)
    saved = {k: os.environ.get(k) for k in ("STGMG_K2_VARIANT", "STGMG_K2_DENSE")}
    os.environ["STGMG_K2_VARIANT"] = str(var)
    os.environ["STGMG_K2_DENSE"] = "1"
    try:
        s = Solver(cfg)
    finally:
        for k, v in saved.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    H = oracle_hierarchy(cfg_key(cfg))
    yield cfg, s, H
    s.close()
    torch.cuda.synchronize()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_dense_sweep_fine(pair):
    import torch
    cfg, s, H = pair
    l = len(H.levels) - 1
    N = H.levels[l].N
    for zero in (False, True):
        b, d0 = random_vector(N, 241), (np.zeros(N) if zero else random_vector(N, 251, 1e-3))
        d = to_gpu(d0)
        s.smooth_sweep(to_gpu(b), d, level=l)
        torch.cuda.synchronize()
        do = H.smoothers[l].sweep(b, d0)
        assert rel(to_np(d), do) < 1e-9, rel(to_np(d), do)


def test_dense_vcycle_and_solve(pair):
    import torch
    from oracle.gmres import fgmres
    cfg, s, H = pair
    N = H.fine.N
    b = uniform_load(N, 25)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), x)
    torch.cuda.synchronize()
    assert rel(to_np(x), H.vcycle(b)) < 1e-8
    x.zero_()
    st = s.solve(to_gpu(b), x, tol=cfg["rtol"], restart=cfg["restart"])
    torch.cuda.synchronize()
    A = H.A[-1]
    xo, info = fgmres(lambda v: A @ v, b, H.vcycle, tol=cfg["rtol"], restart=cfg["restart"])
    assert st["converged"] and abs(st["iterations"] - info["iterations"]) <= 1
    assert rel(to_np(x), xo) <= 1e-8
