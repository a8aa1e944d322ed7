"""GPU parity of Alg. 1 without averaging (STGMG_SMOOTH_OVERWRITE: every DoF keeps the last
patch's update) against the oracle's ``sweep_overwrite`` (pinned by the literal patch loop and the fixed point).
Same tolerances as test_gpu_parity.py: sweep 1e-9, V-cycle 1e-8, solve per north_star."""
import numpy as np
import pytest

from stgmg_inputs import config, uniform_load, random_vector
from tests.gpu_common import small_config, oracle_params, to_gpu, to_np

pytestmark = pytest.mark.gpu

CASES = [("cfg0", config(0)), ("cfg1s", small_config(1)), ("cfg3s", small_config(3)), ("cfg4s", small_config(4))]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def pair(request):
    import torch
    from paper_2303_06742_b200 import Solver
    from paper_2303_06742_b200.stgmg import SMOOTH_OVERWRITE
    from oracle.mg import Hierarchy
    cfg = request.param[1]
    s = Solver(cfg, smoother=SMOOTH_OVERWRITE)
    d = cfg["dim"]
    H = Hierarchy(d, cfg["cells"][:d], cfg["lo"][:d], cfg["hi"][:d], cfg["r"], cfg["k"], cfg["levels"],
                  oracle_params(cfg), cfg["tau"], bc_u=list(cfg["bc_u"][:2 * d]), bc_p=list(cfg["bc_p"][:2 * d]),
                  overwrite=True)
    yield cfg, s, H
    s.close()
    torch.cuda.synchronize()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_overwrite_sweep(pair):
    import torch
    cfg, s, H = pair
    for l in range(1, len(H.levels)):
        N = H.levels[l].N
        b, d0 = random_vector(N, 641 + l), random_vector(N, 651 + l, 1e-3)
        d = to_gpu(d0)
        s.smooth_sweep(to_gpu(b), d, level=l)
        torch.cuda.synchronize()
        do = H.smoothers[l].sweep_overwrite(b, d0)
        assert rel(to_np(d), do) < 1e-9, (l, rel(to_np(d), do))


def test_overwrite_vcycle(pair):
    import torch
    cfg, s, H = pair
    N = H.fine.N
    b = uniform_load(N, 15)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), x)
    torch.cuda.synchronize()
    xo = H.vcycle(b)
    assert rel(to_np(x), xo) < 1e-8, rel(to_np(x), xo)


def test_overwrite_fgmres_solve(pair):
    import torch
    from oracle.gmres import fgmres
    cfg, s, H = pair
    N = H.fine.N
    b = uniform_load(N, cfg.get("seed") or 1)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    st = s.solve(to_gpu(b), x, tol=cfg["rtol"], restart=cfg["restart"])
    torch.cuda.synchronize()
    A = H.A[-1]
    xo, info = fgmres(lambda v: A @ v, b, H.vcycle, tol=cfg["rtol"], restart=cfg["restart"])
    xg = to_np(x)
    assert st["converged"] and info["converged"]
    assert abs(st["iterations"] - info["iterations"]) <= 1
    assert rel(xg, xo) <= 1e-8
    bn = np.linalg.norm(b)
    assert np.linalg.norm((b - A @ xg) - (b - A @ xo)) / bn <= 1e-10


def test_overwrite_rejects_multi_rank():
    from paper_2303_06742_b200 import Solver
    from paper_2303_06742_b200.stgmg import SMOOTH_OVERWRITE, StgmgError, loopback_hub, loopback_hub_destroy
    from paper_2303_06742_b200.stgmg import COMM_LOOPBACK
    hub = loopback_hub(2)
    try:
        with pytest.raises(StgmgError):
            Solver(small_config(1), rank=0, nranks=2, comm=hub, comm_kind=COMM_LOOPBACK, smoother=SMOOTH_OVERWRITE)
    finally:
        loopback_hub_destroy(hub)
