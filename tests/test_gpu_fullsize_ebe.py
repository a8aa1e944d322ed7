"""Full-size parity of the whole solver at BASELINE sizes (configs 2, 3 and the bench workload 4; -m gpu), against the
element-by-element
oracle (oracle/ebe.py: the assembled oracle's definitions without a global matrix, pinned against it in
tests/test_oracle_ebe.py).  North-star tolerances, on the bench's launch configuration (single GPU, default kernels):
  * one V-cycle:     ||d_gpu - d_orc|| / ||d_orc|| <= 1e-8
  * FGMRES solve:    iterations +-1, ||x_gpu - x_orc|| / ||x_orc|| <= 1e-8,
                     ||r_gpu - r_orc|| / ||b|| <= 1e-10 with each side's own r = b - A x
Right-hand sides: the configs' slab-1 F_1 (cfg3: manufactured loads + interpolated initial data, assembled by the
oracle; cfg4: the beam traction (reading A23) from a zero state; the device's own F_1 is compared with both; cfg2: the
seed-2 U[-1,1) load, reading A21).
The oracle runs on the host's cores (minutes); one module-scoped oracle solve per config.  cfg4 (26.6M DoFs: one
oracle V-cycle takes over a minute, a whole oracle solve 5-7 minutes of the suite's 20-minute limit on the driver's
box) compares, by default, the V-cycle, the FIRST FGMRES iterate (both sides stopped by maxit = 1: Arnoldi step,
Givens, update at full size) and the converged GPU solution's residual evaluated by the oracle;
STGMG_FULLSIZE_ORACLE_SOLVE=1 runs the whole oracle solve for cfg4 too (iterations +-1, solution, residual: green in
profiles/r02/pytest_gpu_s5.log and the earlier sessions' logs).
"""
import os

import numpy as np
import pytest

from stgmg_inputs import config
from tests.gpu_common import to_gpu, to_np

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


# cfg4 (the bench workload, 26.6M DoFs) costs 2-6 minutes of host-side oracle work — more on a slow host — of the
# driver's 1200-s limit for the whole GPU suite: it runs when STGMG_FULLSIZE_CFG4=1 (V-cycle, first FGMRES iterate,
# oracle-evaluated residual) or STGMG_FULLSIZE_ORACLE_SOLVE=1 (whole oracle solve; green in
# profiles/r02/pytest_gpu_s5.log and the earlier sessions' logs).  tests/test_gpu_fullsize.py covers cfg4 at full
# size by sampled operator rows, sweep DoFs and residual rows in every run.
_CFG4 = os.environ.get("STGMG_FULLSIZE_CFG4") == "1" or os.environ.get("STGMG_FULLSIZE_ORACLE_SOLVE") == "1"
_CASES = [3, 2] + ([4] if _CFG4 else [])


@pytest.fixture(scope="module", params=_CASES, ids=["cfg%d" % c for c in _CASES])
def case(request):
    import torch
    from threadpoolctl import threadpool_limits
    import os
    from paper_2303_06742_b200 import Solver
    from oracle.ebe import EbeHierarchy, ebe_slab_rhs
    from oracle.gmres import fgmres
    cfg = config(request.param)
    one_step = request.param == 4 and os.environ.get("STGMG_FULLSIZE_ORACLE_SOLVE") != "1"
    with threadpool_limits(max(1, (os.cpu_count() or 2) // 2)):
        H = EbeHierarchy.from_config(cfg)
        b = ebe_slab_rhs(H, cfg, 0)
        d_orc = H.vcycle(b)
        x_orc, info = fgmres(H.fine_op.apply, b, H.vcycle, tol=cfg["rtol"], restart=cfg["restart"],
                             maxit=1 if one_step else 1000)
        r_orc = b - H.fine_op.apply(x_orc)
    s = Solver(cfg)
    yield dict(cfg=cfg, H=H, b=b, d_orc=d_orc, x_orc=x_orc, info=info, r_orc=r_orc, s=s, one_step=one_step)
    s.close()
    torch.cuda.synchronize()


def test_fullsize_rhs(case):
    """The device's slab-1 right-hand side (on-device loads + K8) equals the oracle's (cfg3, cfg4)."""
    import torch
    cfg, s, b = case["cfg"], case["s"], case["b"]
    if cfg["load"] not in ("manufactured", "beam"):
        pytest.skip("random load: the vector is an input")
    from paper_2303_06742_b200.stgmg import LOAD_MANUFACTURED, LOAD_BEAM_TRACTION
    kind = LOAD_MANUFACTURED if cfg["load"] == "manufactured" else LOAD_BEAM_TRACTION
    N = s.size()
    X0 = torch.zeros(N, dtype=torch.float64, device="cuda")
    L, F = torch.zeros_like(X0), torch.zeros_like(X0)
    if kind == LOAD_MANUFACTURED:
        s.initial_state(LOAD_MANUFACTURED, 0.0, X0)
    s.slab_load(kind, 0.0, L)
    s.slab_rhs(L, X0, F)
    torch.cuda.synchronize()
    assert rel(to_np(F), b) < 1e-12, rel(to_np(F), b)


def test_fullsize_vcycle(case):
    import torch
    s, b = case["s"], case["b"]
    d = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), d)
    torch.cuda.synchronize()
    e = rel(to_np(d), case["d_orc"])
    assert e <= 1e-8, e


def test_fullsize_solve(case):
    import torch
    cfg, s, b, H = case["cfg"], case["s"], case["b"], case["H"]
    x = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    nb = np.linalg.norm(b)
    if case["one_step"]:
        # first FGMRES iterate on both sides (maxit = 1), then the converged GPU solve checked by the oracle's operator
        st = s.solve(to_gpu(b), x, tol=cfg["rtol"], restart=cfg["restart"], maxit=1)
        r_gpu = torch.zeros_like(x)
        s.residual(to_gpu(b), x, r_gpu)
        torch.cuda.synchronize()
        assert st["iterations"] == 1 and case["info"]["iterations"] == 1 and not case["info"]["converged"]
        assert rel(to_np(x), case["x_orc"]) <= 1e-8, rel(to_np(x), case["x_orc"])
        assert np.linalg.norm(to_np(r_gpu) - case["r_orc"]) / nb <= 1e-10
        assert abs(st["rel_residual"] - case["info"]["rel_residual"]) <= 1e-10
        x.zero_()
        st = s.solve(to_gpu(b), x, tol=cfg["rtol"], restart=cfg["restart"])
        torch.cuda.synchronize()
        assert st["converged"] and 2 <= st["iterations"] <= 8, st
        assert np.linalg.norm(b - H.fine_op.apply(to_np(x))) <= 1.01 * cfg["rtol"] * nb
        return
    st = s.solve(to_gpu(b), x, tol=cfg["rtol"], restart=cfg["restart"])
    r_gpu = torch.zeros_like(x)
    s.residual(to_gpu(b), x, r_gpu)
    torch.cuda.synchronize()
    xg = to_np(x)
    assert st["converged"] and case["info"]["converged"]
    assert abs(st["iterations"] - case["info"]["iterations"]) <= 1, (st["iterations"], case["info"]["iterations"])
    assert rel(xg, case["x_orc"]) <= 1e-8, rel(xg, case["x_orc"])
    assert np.linalg.norm(to_np(r_gpu) - case["r_orc"]) / nb <= 1e-10
    # the GPU iterate's residual evaluated by the oracle meets the tolerance too
    assert np.linalg.norm(b - H.fine_op.apply(xg)) <= 1.01 * cfg["rtol"] * nb
