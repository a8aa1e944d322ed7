"""GPU parity of the L-shaped benchmark (stgmg_setup_lshape) against oracle/lshape.py (-m gpu).

Cases: ref_0 -> ref_1 (2 levels) for r = 2, k = 1 and r = 3, k = 0 (several patch sizes, ragged CSR rows), and the
Table 4 hierarchy ref_1 -> ref_2 (r = 2, k = 1, 25,836 DoFs per slab).  Per case: DoF counts, the operator on every
level (1e-13), transfers (1e-14), one Alg. 1 sweep (1e-9), the V-cycle (1e-8), slab load / RHS (1e-13), goal
quantities (1e-12), and a full FGMRES solve (iterations +-1, solution 1e-8, residual 1e-10 ||b||) — the
tolerances of DESIGN.md §4.  The Table 4 row itself (ref_2, k = 1, r = 2: 11 GMRES iterations per slab averaged over
the 400 slabs of I = (0, 4]) is checked in test_table4_ref2_iterations.
"""
import numpy as np
import pytest

from tests.gpu_common import to_gpu, to_np

pytestmark = pytest.mark.gpu

CASES = {"ref1_r2_k1": (1, 2, 2, 1), "ref1_r3_k0": (1, 2, 3, 0), "ref2_r2_k1": (2, 2, 2, 1)}


@pytest.fixture(scope="module", params=list(CASES))
def pair(request):
    import torch
    from oracle import lshape as LS
    from paper_2303_06742_b200 import LShapeSolver
    ref, levels, r, k = CASES[request.param]
    params = LS.lshape_params(r)
    H = LS.LHierarchy(ref - levels + 1, levels, r, k, 0.01, params=params)
    s = LShapeSolver(ref, levels, r, k, 0.01, params)
    yield H, s
    s.close()
    torch.cuda.synchronize()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_sizes(pair):
    H, s = pair
    for l, lv in enumerate(H.levels):
        assert s.size(l) == lv.N


def test_operator_every_level(pair):
    import torch
    H, s = pair
    rng = np.random.default_rng(11)
    for l, lv in enumerate(H.levels):
        x = rng.uniform(-1, 1, lv.N)
        y = torch.zeros(lv.N, dtype=torch.float64, device="cuda")
        s.apply(to_gpu(x), y, level=l)
        torch.cuda.synchronize()
        assert rel(to_np(y), H.A[l] @ x) <= 1e-13


def test_transfer(pair):
    import torch
    H, s = pair
    rng = np.random.default_rng(12)
    for l in range(1, len(H.levels)):
        rf = rng.uniform(-1, 1, H.levels[l].N)
        bc = torch.zeros(H.levels[l - 1].N, dtype=torch.float64, device="cuda")
        s.restrict(l, to_gpu(rf), bc)
        dc = rng.uniform(-1, 1, H.levels[l - 1].N)
        df0 = rng.uniform(-1, 1, H.levels[l].N)
        df = to_gpu(df0)
        s.prolong_add(l, to_gpu(dc), df)
        torch.cuda.synchronize()
        assert rel(to_np(bc), H.P[l].T @ rf) <= 1e-14
        assert rel(to_np(df), df0 + H.P[l] @ dc) <= 1e-14


def test_sweep(pair):
    import torch
    H, s = pair
    rng = np.random.default_rng(13)
    l = len(H.levels) - 1
    b = rng.uniform(-1, 1, H.levels[l].N)
    d0 = rng.uniform(-1, 1, H.levels[l].N)
    d = to_gpu(d0)
    s.smooth_sweep(to_gpu(b), d, level=l)
    torch.cuda.synchronize()
    assert rel(to_np(d), H.smoothers[l].sweep(b, d0)) <= 1e-9


def test_vcycle(pair):
    import torch
    H, s = pair
    rng = np.random.default_rng(14)
    b = rng.uniform(-1, 1, H.fine.N)
    x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), x)
    torch.cuda.synchronize()
    assert rel(to_np(x), H.vcycle(b)) <= 1e-8


def test_load_rhs_goal_and_solve(pair):
    import torch
    from oracle import lshape as LS
    from oracle.gmres import fgmres
    from paper_2303_06742_b200.stgmg import LOAD_LSHAPE_TRACTION
    H, s = pair
    N = H.fine.N
    rng = np.random.default_rng(15)
    t_prev = 0.07
    L = torch.zeros(N, dtype=torch.float64, device="cuda")
    s.slab_load(LOAD_LSHAPE_TRACTION, t_prev, L)
    Lo = LS.slab_load(H, t_prev)
    xp = rng.uniform(-1, 1, N)
    F = torch.zeros_like(L)
    s.slab_rhs(L, to_gpu(xp), F)
    Fo = LS.slab_rhs(H, Lo, xp)
    torch.cuda.synchronize()
    assert rel(to_np(L), Lo) <= 1e-13
    assert rel(to_np(F), Fo) <= 1e-13
    bu, bp = s.goal_quantities(to_gpu(xp), 1)
    bo = LS.goal_quantities(H.fine, xp)
    assert abs(bu - bo[0]) <= 1e-12 * max(abs(bo[0]), 1) and abs(bp - bo[1]) <= 1e-12 * max(abs(bo[1]), 1)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    st = s.solve(to_gpu(Fo), x, tol=1e-8, restart=30)
    xo, info = fgmres(lambda v: H.A[-1] @ v, Fo, H.vcycle, tol=1e-8, restart=30)
    xg = to_np(x)
    assert st["converged"] and info["converged"]
    assert abs(st["iterations"] - info["iterations"]) <= 1
    assert rel(xg, xo) <= 1e-8
    assert np.linalg.norm(H.A[-1] @ xg - Fo) <= 1.01e-8 * np.linalg.norm(Fo)
    assert all(v > 0 for v in st["level_seconds"][:len(H.levels)])


def test_table4_ref2_iterations():
    """Table 4, row k = 1, r = 2, ref_2: 25,836 DoFs per slab, coarse level ref_1, 11 GMRES iterations
    per time step on average over I = (0, 4] (tau = 0.01, 400 slabs).  The paper stops at an ABSOLUTE residual of
    1e-8; with the literal Sec. 5.2 data (traction 5e9, E = 20000) the right-hand sides here reach 1e6-1e7
    and an absolute 1e-8 lies below the fp64 rounding floor of ||b - A x|| (the oracle stalls at 2e-8 - 5e-8), so the
    march uses the relative rule (reading A3) at 1e-8.  Pinned: the average within 11 +- 2 and every slab converged."""
    import torch
    from oracle import lshape as LS
    from paper_2303_06742_b200 import LShapeSolver
    from paper_2303_06742_b200.stgmg import LOAD_LSHAPE_TRACTION
    s = LShapeSolver(2, 2, 2, 1, 0.01, LS.lshape_params(2))
    N = s.size()
    assert N == 25836
    X = torch.zeros(N, dtype=torch.float64, device="cuda")
    L, F, x = torch.zeros_like(X), torch.zeros_like(X), torch.zeros_like(X)
    its, goal = [], []
    for n in range(400):
        s.slab_load(LOAD_LSHAPE_TRACTION, n * 0.01, L)
        s.slab_rhs(L, X, F)
        x.zero_()
        st = s.solve(F, x, tol=1e-8, restart=30)
        assert st["converged"], (n, st)
        its.append(st["iterations"])
        X.copy_(x)
        goal.append(s.goal_quantities(X, 1))
    avg = float(np.mean(its))
    g = np.array(goal)
    print("Table 4 ref2 k=1 r=2: average GMRES iterations %.2f (paper 11); min/max its %d/%d; b_u in [%.4g, %.4g] "
          "(paper [-1.674e-2, 1.676e-2]); b_p in [%.4g, %.4g] (paper [-942.6, 945.2])"
          % (avg, min(its), max(its), g[:, 0].min(), g[:, 0].max(), g[:, 1].min(), g[:, 1].max()))
    assert abs(avg - 11.0) <= 2.0, its
    s.close()


@pytest.mark.parametrize("mode", [4, 5, 6])
def test_penalty_length_modes_operator_and_vcycle(mode):
    """The penalty-length experiment modes of DESIGN.md §7.6 (separate u-Nitsche / SIP lengths, face measure): the
    operator on every level (1e-13) and one V-cycle (1e-8) against the oracle with the same mode, ref_0 -> ref_1."""
    import torch
    from oracle import lshape as LS
    from paper_2303_06742_b200 import LShapeSolver
    params = dict(LS.lshape_params(2), hF_mode=mode)
    H = LS.LHierarchy(0, 2, 2, 1, 0.01, params=params)
    s = LShapeSolver(1, 2, 2, 1, 0.01, params, hF_mode=mode)
    rng = np.random.default_rng(40 + mode)
    for l, lv in enumerate(H.levels):
        x = rng.uniform(-1, 1, lv.N)
        y = torch.zeros(lv.N, dtype=torch.float64, device="cuda")
        s.apply(to_gpu(x), y, level=l)
        torch.cuda.synchronize()
        assert rel(to_np(y), H.A[l] @ x) <= 1e-13
    N = H.levels[-1].N
    b = rng.uniform(-1, 1, N)
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), x)
    torch.cuda.synchronize()
    assert rel(to_np(x), H.vcycle(b)) <= 1e-8
    s.close()
