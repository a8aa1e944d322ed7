"""GPU parity on the bench workload itself: BASELINE config 1 at full size (64 x 64 cells, 6 levels, 141,578 DoFs),
in the launch configuration bench.py times (default tile variants, dense K2 on the fine level, small-level CSR /
table path on levels 1-4), element by element against the full oracle (-m gpu).  Tolerances as test_gpu_parity.py;
the two-slab march uses the bench's load (uniform[-1,1) seed 1, reading A21) and zero initial state."""
import numpy as np
import pytest

from stgmg_inputs import config, uniform_load, random_vector
from tests.gpu_common import oracle_hierarchy, cfg_key, to_gpu, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bench_pair():
    import torch
    from paper_2303_06742_b200 import Solver
    cfg = config(1)
    s = Solver(cfg)
    H = oracle_hierarchy(cfg_key(cfg))
    yield cfg, s, H
    s.close()
    torch.cuda.synchronize()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_bench_operator_every_level(bench_pair):
    import torch
    cfg, s, H = bench_pair
    for l, lev in enumerate(H.levels):
        x = random_vector(lev.N, 400 + l)
        y = torch.zeros(lev.N, dtype=torch.float64, device="cuda")
        s.apply(to_gpu(x), y, level=l)
        torch.cuda.synchronize()
        assert rel(to_np(y), H.A[l] @ x) < 1e-13, l


def test_bench_sweep_every_level(bench_pair):
    import torch
    cfg, s, H = bench_pair
    for l in range(1, len(H.levels)):
        N = H.levels[l].N
        b, d0 = random_vector(N, 410 + l), random_vector(N, 420 + l, 1e-3)
        d = to_gpu(d0)
        s.smooth_sweep(to_gpu(b), d, level=l)
        torch.cuda.synchronize()
        assert rel(to_np(d), H.smoothers[l].sweep(b, d0)) < 1e-9, l


def test_bench_vcycle(bench_pair):
    import torch
    cfg, s, H = bench_pair
    b = uniform_load(H.fine.N, 1)
    x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), x)
    torch.cuda.synchronize()
    assert rel(to_np(x), H.vcycle(b)) < 1e-8


def test_bench_two_slab_march(bench_pair):
    """The bench step twice: F_n = L + J X_{n-1} (K8) then the FGMRES-GMG solve, against the oracle."""
    import torch
    from oracle.gmres import fgmres
    from oracle.loads import slab_rhs, end_state
    cfg, s, H = bench_pair
    lev, op = H.fine, H.ops[-1]
    S = op.assemble_spatial()
    L = uniform_load(lev.N, cfg["seed"])
    Lg = to_gpu(L)
    X = torch.zeros(lev.N, dtype=torch.float64, device="cuda")
    F = torch.zeros_like(X)
    Xprev = np.zeros(lev.N)   # the GPU's previous slab (each slab is compared on identical input data)
    for _ in range(2):
        s.slab_rhs(Lg, X, F)
        X.zero_()
        st = s.solve(F, X, tol=cfg["rtol"], restart=cfg["restart"])
        U, V, P = end_state(lev, Xprev)
        Fo = slab_rhs(lev, S, op.chi_m1, op.th, U, V, P, None, None) + L
        Xo, info = fgmres(lambda v: H.A[-1] @ v, Fo, H.vcycle, tol=cfg["rtol"], restart=cfg["restart"])
        torch.cuda.synchronize()
        assert st["converged"] and info["converged"]
        assert abs(st["iterations"] - info["iterations"]) <= 1
        assert rel(to_np(F), Fo) < 1e-12
        assert rel(to_np(X), Xo) <= 1e-8
        assert np.linalg.norm(H.A[-1] @ (to_np(X) - Xo)) / np.linalg.norm(Fo) <= 1e-10
        Xprev = to_np(X)
