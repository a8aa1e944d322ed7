"""GPU parity of the Problem B.1 (DS) formulation (STGMG_FORM_DS) against the oracle, whose DS
operator / slab RHS are pinned in test_oracle_pins.py (DS = DSA on time-steady states, EOC ~2).  Tolerances as in
test_gpu_parity.py."""
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
    from paper_2303_06742_b200.stgmg import FORM_DS
    from oracle.mg import Hierarchy
    cfg = request.param[1]
    s = Solver(cfg, formulation=FORM_DS)
    d = cfg["dim"]
    H = Hierarchy(d, cfg["cells"][:d], cfg["lo"][:d], cfg["hi"][:d], cfg["r"], cfg["k"], cfg["levels"],
                  oracle_params(cfg), cfg["tau"], bc_u=list(cfg["bc_u"][:2 * d]), bc_p=list(cfg["bc_p"][:2 * d]),
                  ds=True)
    yield cfg, s, H
    s.close()
    torch.cuda.synchronize()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_ds_operator_all_levels(pair):
    import torch
    cfg, s, H = pair
    for l, lev in enumerate(H.levels):
        x = random_vector(lev.N, 300 + l)
        y = torch.zeros(lev.N, dtype=torch.float64, device="cuda")
        s.apply(to_gpu(x), y, level=l)
        torch.cuda.synchronize()
        assert rel(to_np(y), H.A[l] @ x) < 1e-13, (l, rel(to_np(y), H.A[l] @ x))


def test_ds_slab_rhs(pair):
    import torch
    from oracle.loads import slab_rhs, end_state
    cfg, s, H = pair
    lev, op = H.fine, H.ops[-1]
    S = op.assemble_spatial()
    Xp, L = random_vector(lev.N, 361), random_vector(lev.N, 362)
    U, V, P = end_state(lev, Xp)
    ro = slab_rhs(lev, S, op.chi_m1, op.th, U, V, P, None, None, ds=True) + L
    out = torch.zeros(lev.N, dtype=torch.float64, device="cuda")
    s.slab_rhs(to_gpu(L), to_gpu(Xp), out)
    torch.cuda.synchronize()
    assert rel(to_np(out), ro) < 1e-13


def test_ds_vcycle_and_solve(pair):
    import torch
    from oracle.gmres import fgmres
    cfg, s, H = pair
    N = H.fine.N
    b = uniform_load(N, 35)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), x)
    torch.cuda.synchronize()
    assert rel(to_np(x), H.vcycle(b)) < 1e-8
    x.zero_()
    st = s.solve(to_gpu(b), x, tol=cfg["rtol"], restart=cfg["restart"])
    torch.cuda.synchronize()
    A = H.A[-1]
    xo, info = fgmres(lambda v: A @ v, b, H.vcycle, tol=cfg["rtol"], restart=cfg["restart"])
    assert st["converged"] and info["converged"] and abs(st["iterations"] - info["iterations"]) <= 1
    assert rel(to_np(x), xo) <= 1e-8
    bn = np.linalg.norm(b)
    assert np.linalg.norm(A @ (to_np(x) - xo)) / bn <= 1e-10
