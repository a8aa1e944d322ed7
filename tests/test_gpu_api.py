"""Boundary behaviour of stgmg_solve / stgmg_solve_host on the GPU (-m gpu): determinism (no atomics: repeated calls
are bitwise identical), host-buffer entry point = device entry point, absolute tolerance (STGMG_TOL_ABS),
restarts (reading A4) and maxit / STGMG_NOT_CONVERGED, each against the oracle's FGMRES where it applies."""
import numpy as np
import pytest

from stgmg_inputs import uniform_load, random_vector
from tests.gpu_common import small_config, oracle_hierarchy, cfg_key, to_gpu, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    import torch
    from paper_2303_06742_b200 import Solver
    cfg = small_config(1)
    s = Solver(cfg)
    H = oracle_hierarchy(cfg_key(cfg))
    yield cfg, s, H
    s.close()
    torch.cuda.synchronize()


def test_repeated_solves_are_bitwise_identical(pair):
    import torch
    cfg, s, H = pair
    b = to_gpu(uniform_load(H.fine.N, 91))
    xs, its = [], []
    for _ in range(3):
        x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
        st = s.solve(b, x, tol=cfg["rtol"], restart=cfg["restart"])
        torch.cuda.synchronize()
        xs.append(to_np(x))
        its.append(st["iterations"])
    assert its[0] == its[1] == its[2]
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[0], xs[2])
    v1 = torch.zeros_like(b)
    v2 = torch.zeros_like(b)
    s.vcycle(b, v1)
    s.vcycle(b, v2)
    torch.cuda.synchronize()
    assert torch.equal(v1, v2)


def test_solve_host_equals_solve(pair):
    import torch
    cfg, s, H = pair
    bn = uniform_load(H.fine.N, 92)
    x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
    st = s.solve(to_gpu(bn), x, tol=cfg["rtol"], restart=cfg["restart"])
    torch.cuda.synchronize()
    xh = np.zeros(H.fine.N)
    sth = s.solve_host(np.ascontiguousarray(bn), xh, tol=cfg["rtol"], restart=cfg["restart"])
    assert sth["iterations"] == st["iterations"]
    assert np.array_equal(xh, to_np(x))


def test_absolute_tolerance_and_restarts_match_oracle(pair):
    """TOL_ABS stops on ||r|| <= tol; restart m = 2 forces restarts from the true residual (A4).  Both against
    the oracle's FGMRES with the same settings: iterations +-1, solution 1e-8."""
    import torch
    from oracle.gmres import fgmres, TOL_ABS
    from paper_2303_06742_b200.stgmg import TOL_ABS as GPU_TOL_ABS
    cfg, s, H = pair
    bn = uniform_load(H.fine.N, 93)
    A = H.A[-1]
    tabs = 3e-9 * np.linalg.norm(bn)       # an absolute target that no relative setting of the same run reproduces
    for tol, mode, gmode, restart in [(tabs, TOL_ABS, GPU_TOL_ABS, 30), (1e-10, 0, 0, 2)]:
        x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
        st = s.solve(to_gpu(bn), x, tol=tol, tol_mode=gmode, restart=restart)
        torch.cuda.synchronize()
        xo, info = fgmres(lambda v: A @ v, bn, H.vcycle, tol=tol, tol_mode=mode, restart=restart)
        assert st["converged"] and info["converged"]
        assert abs(st["iterations"] - info["iterations"]) <= 1
        xg = to_np(x)
        assert np.linalg.norm(xg - xo) <= 1e-8 * np.linalg.norm(xo)
        r = np.linalg.norm(bn - A @ xg)
        if mode == TOL_ABS:
            assert r <= tol * (1 + 1e-6)
        if restart == 2:
            assert st["restarts"] >= 1 and st["restarts"] == info["restarts"]


def test_maxit_returns_not_converged_with_last_iterate(pair):
    import torch
    cfg, s, H = pair
    bn = uniform_load(H.fine.N, 94)
    x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
    st = s.solve(to_gpu(bn), x, tol=1e-14, restart=30, maxit=1)
    torch.cuda.synchronize()
    assert not st["converged"] and st["iterations"] == 1
    xg = to_np(x)
    assert np.all(np.isfinite(xg)) and np.linalg.norm(xg) > 0
    r = np.linalg.norm(bn - H.A[-1] @ xg) / np.linalg.norm(bn)
    assert abs(r - st["rel_residual"]) <= 1e-10 and r < 1.0


def test_nonzero_initial_guess_matches_oracle(pair):
    """x on entry is the initial guess X^(0) (r_0 = b - A X^(0)); device vs oracle FGMRES from the same X^(0)."""
    import torch
    from oracle.gmres import fgmres
    cfg, s, H = pair
    bn = uniform_load(H.fine.N, 95)
    x0 = random_vector(H.fine.N, 96, 1e-2)
    x = to_gpu(x0)
    st = s.solve(to_gpu(bn), x, tol=cfg["rtol"], restart=cfg["restart"])
    torch.cuda.synchronize()
    xo, info = fgmres(lambda v: H.A[-1] @ v, bn, H.vcycle, x0=x0, tol=cfg["rtol"], restart=cfg["restart"])
    assert st["converged"] and abs(st["iterations"] - info["iterations"]) <= 1
    assert np.linalg.norm(to_np(x) - xo) <= 1e-8 * np.linalg.norm(xo)


def test_zero_rhs_and_exact_initial_guess(pair):
    """Degenerate inputs: b = 0 returns at once (0 iterations, x = 0); an initial guess that already meets the
    tolerance returns at once with x unchanged (O11 step 1: beta <= target before any Arnoldi step)."""
    import torch
    cfg, s, H = pair
    N = H.fine.N
    b = torch.zeros(N, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    st = s.solve(b, x, tol=cfg["rtol"], restart=cfg["restart"])
    torch.cuda.synchronize()
    assert st["converged"] and st["iterations"] == 0 and torch.count_nonzero(x).item() == 0
    bn = to_gpu(uniform_load(N, 97))
    x = torch.zeros_like(bn)
    s.solve(bn, x, tol=1e-12, restart=cfg["restart"])
    x1 = x.clone()
    st = s.solve(bn, x, tol=1e-8, restart=cfg["restart"])
    torch.cuda.synchronize()
    assert st["converged"] and st["iterations"] == 0
    assert torch.equal(x, x1)


def test_single_level_is_a_direct_solve():
    """levels = 1: the preconditioner is the coarse direct solve A_0^{-1} (readings A16/A18), so FGMRES
    converges in one iteration (exact preconditioner -> 1 iteration) to the oracle's dense solve."""
    import torch
    from paper_2303_06742_b200 import Solver
    from stgmg_inputs import config
    from oracle.mg import Hierarchy
    from tests.gpu_common import oracle_params
    cfg = dict(config(0), levels=1)
    s = Solver(cfg)
    d = cfg["dim"]
    H = Hierarchy(d, cfg["cells"][:d], cfg["lo"][:d], cfg["hi"][:d], cfg["r"], cfg["k"], 1, oracle_params(cfg),
                  cfg["tau"], bc_u=list(cfg["bc_u"][:2 * d]), bc_p=list(cfg["bc_p"][:2 * d]))
    bn = uniform_load(H.fine.N, 98)
    x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
    st = s.solve(to_gpu(bn), x, tol=1e-10, restart=30)
    torch.cuda.synchronize()
    xd = np.linalg.solve(H.A[-1].toarray() if hasattr(H.A[-1], "toarray") else H.A[-1], bn)
    assert st["converged"] and st["iterations"] == 1
    assert np.linalg.norm(to_np(x) - xd) <= 1e-9 * np.linalg.norm(xd)
    s.close()


def test_level_seconds_filled(pair):
    """stgmg_stats.level_seconds (SPEC SolveStats per-level smoother timings): positive on every level
    that runs its own work (the folded sub-cycle, if any, is booked on the fold level), zero above the hierarchy, and
    their sum below the solve's own device time (the V-cycles are part of it)."""
    import torch
    cfg, s, H = pair
    b = to_gpu(uniform_load(H.fine.N, 95))
    x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
    st = s.solve(b, x, tol=cfg["rtol"], restart=cfg["restart"])
    st = s.solve(b, torch.zeros_like(x), tol=cfg["rtol"], restart=cfg["restart"])
    ls = st["level_seconds"]
    lo = s.fold_level()
    L = cfg["levels"]
    assert all(ls[l] > 0 for l in range(lo, L)), ls
    assert all(ls[l] == 0 for l in range(L, 16)) and all(ls[l] == 0 for l in range(0, lo)), ls
    assert sum(ls) < 1.5 * st["seconds"], (sum(ls), st["seconds"])


def test_binding_rejects_bad_buffers(pair):
    """The binding validates every pointer before the ABI call: wrong length, dtype, device, layout."""
    import torch
    cfg, s, H = pair
    N = H.fine.N
    good = torch.zeros(N, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        s.vcycle(torch.zeros(N - 1, dtype=torch.float64, device="cuda"), good)
    with pytest.raises(TypeError):
        s.vcycle(torch.zeros(N, dtype=torch.float32, device="cuda"), good)
    with pytest.raises(TypeError):
        s.vcycle(torch.zeros(N, dtype=torch.float64), good)
    with pytest.raises(TypeError):
        s.vcycle(torch.zeros(2 * N, dtype=torch.float64, device="cuda")[::2], good)
    with pytest.raises(ValueError):
        s.apply(good, torch.zeros(s.size(0), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        s.restrict(1, torch.zeros(s.size(1), dtype=torch.float64, device="cuda"),
                   torch.zeros(s.size(1), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        s.solve_host(np.zeros(N), np.zeros(N - 3))
    with pytest.raises(TypeError):
        s.solve_host(np.zeros(N), np.zeros(N, dtype=np.float32))
    with pytest.raises(TypeError):
        s.solve_host(np.zeros(N), good)
