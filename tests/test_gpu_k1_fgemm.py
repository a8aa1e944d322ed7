"""K1 routes against each other and against the oracle (-m gpu): the full slab element matrices, the factored element
GEMMs (csrc/op_fgemm.cu) and, in 3D Q2, the sum-factorised kernel on the volume-only cell types (csrc/op_sf3.cu).
All compute y = A_l x of Problem 3.1 from the same element integrals (Def:ACB / Def:ab) and
differ in summation order only, so they agree to 1e-13 relative on every level of the shrunken 3D and 2D Q3
configurations (STGMG_K1_FGEMM=2 forces the factored form onto levels below its size threshold), and each matches
the oracle's assembled operator."""
import os

import numpy as np
import pytest

from stgmg_inputs import random_vector
from tests.gpu_common import small_config, oracle_hierarchy, cfg_key, to_gpu, to_np

pytestmark = pytest.mark.gpu


def _solver(cfg, fgemm, sf="2"):
    """fgemm: STGMG_K1_FGEMM ("0" full element matrices, "2" factored on every element-route level); sf:
    STGMG_K1_SF ("2": 3D Q2 volume-only cell types by sum factorisation, csrc/op_sf3.cu, on every factored level)."""
    from paper_2303_06742_b200 import Solver
    env = {"STGMG_K1_FGEMM": fgemm, "STGMG_K1_SF": sf}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return Solver(cfg)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("i", [2, 3, 4])
def test_factored_and_sumfact_equal_full_element_route_and_oracle(i):
    """Three GPU routes of y = A_l x on every level: full slab element matrices, factored element GEMMs on every
    cell type, and (3D) sum factorisation on the volume-only types + factored GEMMs on the Nitsche types."""
    import torch
    cfg = small_config(i)
    s0, s1, s2 = _solver(cfg, "0"), _solver(cfg, "2", "0"), _solver(cfg, "2", "2")
    H = oracle_hierarchy(cfg_key(cfg))
    for l in range(cfg["levels"]):
        n = s0.size(l)
        x = to_gpu(random_vector(n, 100 + l))
        ys = []
        for s in (s0, s1, s2):
            y = torch.zeros(n, dtype=torch.float64, device="cuda")
            s.apply(x, y, level=l)
            ys.append(y)
        torch.cuda.synchronize()
        b = to_np(ys[0])
        yo = H.A[l] @ to_np(x)
        for a in map(to_np, ys[1:]):
            assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b), l
            assert np.linalg.norm(a - yo) <= 1e-13 * np.linalg.norm(yo), l
    for s in (s0, s1, s2):
        s.close()


@pytest.mark.parametrize("i", [3, 4])
def test_sumfact_solve_matches_oracle(i):
    """FGMRES-GMG solve with the sum-factorised K1 forced on the fine level: iterations +-1 and solution 1e-8 against
    the oracle (north_star tolerances)."""
    import torch
    from oracle.gmres import fgmres
    from stgmg_inputs import uniform_load
    cfg = small_config(i)
    s = _solver(cfg, "2", "2")
    H = oracle_hierarchy(cfg_key(cfg))
    N = s.size()
    b = uniform_load(N, 7)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    st = s.solve(to_gpu(b), x, tol=cfg["rtol"], restart=cfg["restart"])
    torch.cuda.synchronize()
    xo, info = fgmres(lambda v: H.A[-1] @ v, b, H.vcycle, tol=cfg["rtol"], restart=cfg["restart"])
    assert st["converged"]
    assert abs(st["iterations"] - info["iterations"]) <= 1
    assert np.linalg.norm(to_np(x) - xo) <= 1e-8 * np.linalg.norm(xo)
    s.close()


@pytest.mark.parametrize("i", [3, 4])
def test_sumfact_slab_rhs_equals_warp_kernel(i):
    """K8 F_n = L_n + J X_{n-1}: theta = 0 leaves only mass terms, so the sum-factorised kernel runs on
    every cell type of the fine level; against the warp-per-cell kernel of the full element route (1e-13)."""
    import torch
    cfg = small_config(i)
    s0, s2 = _solver(cfg, "0"), _solver(cfg, "2", "2")
    n = s0.size()
    xp = to_gpu(random_vector(n, 31))
    load = to_gpu(random_vector(n, 32))
    outs = []
    for s in (s0, s2):
        rhs = torch.zeros(n, dtype=torch.float64, device="cuda")
        s.slab_rhs(load, xp, rhs)
        outs.append(to_np(rhs))
    torch.cuda.synchronize()
    assert np.linalg.norm(outs[1] - outs[0]) <= 1e-13 * np.linalg.norm(outs[0])
    for s in (s0, s2):
        s.close()
