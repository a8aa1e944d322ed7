"""Pins of the oracle's V-cycle composition (oracle/mg.py) against textbook multigrid identities (CPU, -m "not gpu").

P:L433-440: one V-cycle = J_max pre-smoothing sweeps of Alg. 1 from d = 0, residual, restriction by P^T, the
coarser V-cycle (direct solve on T_0), prolongation-add, J_max post-smoothing sweeps continuing from the corrected
iterate (reading A13).  Two pins that do not re-type mg.Hierarchy.vcycle:

* V1 — error propagation.  A V-cycle with zero initial guess is a linear map B_l; its error operator
  E_l = I - B_l A_l obeys the textbook recursion (Hackbusch, Multi-Grid Methods, Ch. 2/7)
      E_0 = 0 (exact coarse solve),
      E_l = S_l^{nu2} (I - P_l (I - E_{l-1}) A_{l-1}^{-1} P_l^T A_l) S_l^{nu1},
  with S_l = the iteration matrix of ONE Alg. 1 sweep, built column by column as S_l e_i = sweep(b = 0, d = e_i)
  (the sweep itself is pinned by P10/P11), P_l the interpolation (P9) and A_l the level matrices (P8).  The V-cycle
  is evaluated as a black box; the recursion is applied to the same random vectors.  A V-cycle that skips the
  post-smoothing, restarts it from 0 or restricts b instead of the residual violates it.
* V2 — two-grid projection.  With a frozen h_F the coarse matrix is the Galerkin product A_0 = P^T A_1 P (P8), so
  the iterate handed to the post-smoother satisfies P^T (b - A_1 d) = 0 exactly (up to rounding); post-smoothing
  starts from that iterate, not from 0.
"""
import numpy as np
import pytest

from oracle.mg import Hierarchy

P0 = dict(rho=1.0, alpha=0.9, c0=0.01, lam=1.0, mu=1.0, K=[0.01, 0, 0, 0.01])
P3D = dict(P0, K=[0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01])


def E_apply(H, l, x):
    """E_l x by the recursion: E_0 = 0, E_l = S^nu (I - P (I - E_{l-1}) A_{l-1}^{-1} P^T A_l) S^nu, where S is one
    Alg. 1 sweep with b = 0 (S e = sweep(0, e)) and A_{l-1}^{-1} is a dense direct solve."""
    sm, nu = H.smoothers[l], H.jmax
    z = np.zeros_like(x)
    for _ in range(nu):
        x = sm.sweep(z, x)
    y = H.P[l].T @ (H.A[l] @ x)
    c = np.linalg.solve(H.A[l - 1].toarray(), y)                # A_{l-1}^{-1} P^T A_l S^nu x
    if l - 1 >= 1:
        c = c - E_apply(H, l - 1, c)                            # (I - E_{l-1}) A_{l-1}^{-1} ...
    x = x - H.P[l] @ c
    for _ in range(nu):
        x = sm.sweep(z, x)
    return x


def E_vcycle(H, vcycle, x):
    """(I - B A) x with B = the V-cycle as a black box."""
    return x - vcycle(H.A[-1] @ x)


CASES = [
    ("2d_q2_dg1_4levels_mixedbc", dict(d=2, cells=[8, 8], r=2, k=1, levels=4, bc_u=[0, 1, 0, 0], bc_p=[1, 0, 0, 0])),
    ("2d_q3_dg2_3levels", dict(d=2, cells=[4, 4], r=3, k=2, levels=3, bc_u=None, bc_p=None)),
    ("3d_q2_dg0_2levels", dict(d=3, cells=[2, 2, 2], r=2, k=0, levels=2, bc_u=[0, 1, 1, 1, 1, 1],
                               bc_p=[1, 1, 1, 1, 1, 0])),
]


def hierarchy(c):
    d = c["d"]
    return Hierarchy(d, c["cells"], [0.0] * d, [1.0] * d, c["r"], c["k"], c["levels"], P0 if d == 2 else P3D, 0.01,
                     bc_u=c["bc_u"], bc_p=c["bc_p"])


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def hier(request):
    return hierarchy(request.param[1])


def test_V1_vcycle_error_propagation(hier):
    H = hier
    rng = np.random.default_rng(1)
    for _ in range(2):
        x = rng.standard_normal(H.fine.N)
        a, b = E_vcycle(H, H.vcycle, x), E_apply(H, len(H.levels) - 1, x)
        assert np.linalg.norm(a - b) < 1e-9 * np.linalg.norm(x), np.linalg.norm(a - b) / np.linalg.norm(x)
        assert np.linalg.norm(b) > 1e-4 * np.linalg.norm(x)     # non-trivial error operator


def _mutants(H):
    """Three plausible composition bugs: no post-smoothing; post-smoothing restarted from 0; restriction
    of b instead of the residual."""
    def no_post(b, l=None):
        l = len(H.levels) - 1 if l is None else l
        if l == 0:
            return H.coarse_inv @ b
        sm = H.smoothers[l]
        d = sm.smooth(b, None, H.jmax)
        d = d + H.P[l] @ no_post(H.P[l].T @ (b - H.A[l] @ d), l - 1)
        return d

    def post_from_zero(b, l=None):
        l = len(H.levels) - 1 if l is None else l
        if l == 0:
            return H.coarse_inv @ b
        sm = H.smoothers[l]
        d = sm.smooth(b, None, H.jmax)
        d = d + H.P[l] @ post_from_zero(H.P[l].T @ (b - H.A[l] @ d), l - 1)
        return d + sm.smooth(b, None, H.jmax)

    def restrict_b(b, l=None):
        l = len(H.levels) - 1 if l is None else l
        if l == 0:
            return H.coarse_inv @ b
        sm = H.smoothers[l]
        d = sm.smooth(b, None, H.jmax)
        d = d + H.P[l] @ restrict_b(H.P[l].T @ b, l - 1)
        return sm.smooth(b, d, H.jmax)

    return {"no_post": no_post, "post_from_zero": post_from_zero, "restrict_b": restrict_b}


def test_V1_pin_detects_composition_mutants(hier):
    """The pin has teeth: each mutant V-cycle violates the recursion by far more than rounding."""
    H = hier
    x = np.random.default_rng(2).standard_normal(H.fine.N)
    ref = E_apply(H, len(H.levels) - 1, x)
    for name, vc in _mutants(H).items():
        dev = np.linalg.norm(E_vcycle(H, vc, x) - ref) / np.linalg.norm(x)
        assert dev > 1e-4, (name, dev)


def test_V2_two_grid_projection_frozen_hF(monkeypatch):
    """Frozen h_F: P^T (b - A_1 d_corr) = 0 for the iterate d_corr that the post-smoother receives."""
    H = Hierarchy(2, [4, 4], [0, 0], [1, 1], 2, 1, 2, P0 | {"hF_fixed": 0.05}, 0.01)
    A1, P = H.A[1], H.P[1]
    G = (P.T @ A1 @ P).toarray()
    assert np.abs(G - H.A[0].toarray()).max() < 1e-11 * np.abs(G).max()     # the Galerkin identity holds (P8)
    sm = H.smoothers[1]
    seen = []
    orig = sm.smooth

    def spy(b, d=None, *a, **kw):
        seen.append(None if d is None else d.copy())
        return orig(b, d, *a, **kw)

    monkeypatch.setattr(sm, "smooth", spy)
    b = np.random.default_rng(3).standard_normal(H.fine.N)
    H.vcycle(b)
    assert len(seen) == 2 and seen[0] is None and seen[1] is not None    # pre from 0, post continues (A13)
    r = b - A1 @ seen[1]
    proj = P.T @ r
    assert np.abs(proj).max() < 1e-9 * np.abs(P.T @ b).max(), np.abs(proj).max()
    assert np.abs(r).max() > 1e-6 * np.abs(b).max()                       # the fine residual itself is not zero
