"""Pins of the oracle against what the paper and the mathematics fix.

CPU only (-m "not gpu").  Each test names the pin and the passage it follows.  None of these re-types the
oracle's own formula: they check printed paper values, closed forms, textbook special cases, invariants and
brute force on tiny inputs.
"""
import json
import math
import os

import numpy as np
import pytest
import scipy.sparse.linalg as spla
from numpy.polynomial import polynomial as Pn

from oracle.basis import radau_right, gauss_lobatto_nodes01, lagrange_values
from oracle.temporal import temporal_constants
from oracle.mesh import Level, FIELD_V, FIELD_U, FIELD_P
from oracle.assembly import SlabOperator
from oracle.transfer import prolongation
from oracle.vanka import Patches, VankaSmoother, equilibrated_inverse
from oracle.mg import Hierarchy
from oracle.gmres import fgmres
from oracle.loads import (manufactured_eq53, manufactured_eq51, manufactured_baseline, load_vectors, slab_rhs,
                          end_state, interpolate_initial)
from oracle.errors import march_errors
from stgmg_inputs import config, dof_count, uniform_load

GOLD = os.path.join(os.path.dirname(__file__), "golden")
P0 = dict(rho=1.0, alpha=0.9, c0=0.01, lam=1.0, mu=1.0, K=[0.01, 0, 0, 0.01])


def lame(E, nu):
    return E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))


# ---------------------------------------------------------------- P1 / P2: temporal constants -------
def test_P1_closed_form_k0_k1():
    """P1 (P:L122-128 Eq:GF): k=0 backward Euler, k=1 Radau IIA(2)."""
    t, w, c, T = temporal_constants(0)
    assert np.allclose(t, [1.0]) and np.allclose(w, [2.0]) and np.allclose(c, [1.0]) and np.allclose(T, [[1.0]])
    t, w, c, T = temporal_constants(1)
    assert np.allclose(t, [-1 / 3, 1], atol=1e-15)
    assert np.allclose(w, [1.5, 0.5], atol=1e-15)
    assert np.allclose(c, [1.5, -0.5], atol=1e-15)
    assert np.allclose(T, [[9 / 8, 3 / 8], [-9 / 8, 5 / 8]], atol=1e-14)


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_P1_radau_exactness(k):
    """Eq:GF: exact on P_{2k}, last node t = +1; not exact on P_{2k+1}."""
    t, w = radau_right(k)
    assert t[-1] == 1.0
    for deg in range(2 * k + 1):
        exact = (1 - (-1) ** (deg + 1)) / (deg + 1)
        assert abs(np.sum(w * t ** deg) - exact) < 1e-13
    deg = 2 * k + 1
    assert abs(np.sum(w * t ** deg) - (1 - (-1) ** (deg + 1)) / (deg + 1)) > 1e-6


def _radau_iia_butcher(k):
    """Textbook collocation Butcher matrix on [0,1]: c = (t+1)/2, A_ij = int_0^{c_i} l_j(s) ds."""
    t, _ = radau_right(k)
    c = 0.5 * (t + 1.0)
    A = np.zeros((k + 1, k + 1))
    for j in range(k + 1):
        poly = np.array([1.0])
        for m in range(k + 1):
            if m != j:
                poly = Pn.polymul(poly, np.array([-c[m], 1.0]) / (c[j] - c[m]))
        integ = Pn.polyint(poly)
        for i in range(k + 1):
            A[i, j] = Pn.polyval(c[i], integ)
    return A


@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_P2_radau_iia_identity(k):
    """P2: T = diag(w/2) A_RIIA^{-1}; row sums of T = chi(-1)."""
    t, w, c, T = temporal_constants(k)
    A = _radau_iia_butcher(k)
    assert np.allclose(T, np.diag(w / 2) @ np.linalg.inv(A), atol=1e-12)
    assert np.allclose(T.sum(axis=1), c, atol=1e-13)


def _pade(k, z):
    """Pade(k, k+1) approximant of e^z (textbook closed form; Radau IIA stability function)."""
    num = sum(math.factorial(2 * k + 1 - j) * math.factorial(k) /
              (math.factorial(2 * k + 1) * math.factorial(j) * math.factorial(k - j)) * z ** j for j in range(k + 1))
    den = sum(math.factorial(2 * k + 1 - j) * math.factorial(k + 1) /
              (math.factorial(2 * k + 1) * math.factorial(j) * math.factorial(k + 1 - j)) * (-z) ** j
              for j in range(k + 2))
    return num / den


@pytest.mark.parametrize("k", [0, 1, 2, 3])
@pytest.mark.parametrize("z", [-0.5, -3.0, -50.0, 2j])
def test_P2_pade_amplification(k, z):
    """dG(k) slab for y' = lambda y: (T - z diag(w)/2) Y = chi(-1) y0; end value = Pade(k,k+1)(z)."""
    t, w, c, T = temporal_constants(k)
    Y = np.linalg.solve(T.astype(complex) - z * np.diag(w) / 2, c.astype(complex))
    assert abs(Y[-1] - _pade(k, z)) < 1e-12 * max(1.0, abs(_pade(k, z)))


# ---------------------------------------------------------------- element / assembly invariants -----
def test_element_invariants_2d():
    """Mass sums to |Omega|; A_gamma, B_gamma symmetric; C(chi, 1) = 0 when G_D^u = dOmega
    (divergence theorem); rigid translations in the kernel of the volume part of A."""
    lev = Level(2, [3, 3], [0, 0], [1, 2], 2, 1)
    op = SlabOperator(lev, P0, 0.01)
    S = op.assemble_spatial()
    assert abs(S["Mq"].sum() - 2.0) < 1e-13
    assert abs(S["Mp"].sum() - 2.0) < 1e-13
    for name in ("A", "B", "Mrho", "Mc"):
        M = S[name].toarray()
        assert np.abs(M - M.T).max() < 1e-9 * np.abs(M).max()
    assert np.abs(S["C"].T @ np.ones(lev.np_)).max() < 1e-12
    interior = SlabOperator(lev, P0, 0.01).forms.matrices((), ())
    ones = np.ones(interior["A"].shape[0] // 2)
    assert np.abs(interior["A"] @ np.concatenate([ones, 0 * ones])).max() < 1e-12
    assert np.abs(interior["B"] @ np.ones(interior["B"].shape[0])).max() < 1e-12


@pytest.mark.parametrize("d,h", [(2, (0.5, 0.125)), (3, (0.5, 0.25, 0.0625))])
def test_penalty_length_is_cell_measure(d, h):
    """"For boundary faces we set h_F := |K|_d" (reading A6).  On constants the consistency terms of
    a_gamma / b_gamma vanish (sigma(const) = 0, grad const = 0) and the bases are partitions of unity, so the sum of
    all entries of one component block of the element A with ONE Dirichlet face F (normal to axis a) is
    gamma_a |F| / h_F = gamma_a / h_a, and the sum of all entries of B is gamma_b / h_a — on an anisotropic cell the
    edge reading h_F = h_a gives gamma_a |K| / h_a^2 instead."""
    from oracle.element import ElementForms
    K = np.eye(d).ravel().tolist()
    prm = P0 | {"K": K, "gamma_a": 5e4 * 2 * 3, "gamma_b": 0.5 * 2 * 1}      # P:L207-210 with r = 2
    ef = ElementForms(d, 2, h, prm)
    nb = 3 ** d
    for a in range(d):
        for s in (0, 1):
            M = ef.matrices((2 * a + s,), (2 * a + s,))
            for c in range(d):
                blk = M["A"][c * nb:(c + 1) * nb, c * nb:(c + 1) * nb]
                assert abs(blk.sum() - prm["gamma_a"] / h[a]) <= 1e-9 * prm["gamma_a"] / h[a]
            assert abs(M["B"].sum() - prm["gamma_b"] / h[a]) <= 1e-9 * prm["gamma_b"] / h[a]


def test_element_rotation_kernel_3d():
    """Infinitesimal rotations are strain-free: volume part of A annihilates (-y, x, 0) on a 3D cell."""
    lev = Level(3, [1, 1, 1], [0, 0, 0], [1, 1, 1], 2, 0)
    op = SlabOperator(lev, P0 | {"K": [0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01]}, 0.01)
    A = op.forms.matrices((), ())["A"]
    x = lev.node_coords(2, gauss_lobatto_nodes01(2))
    rot = np.concatenate([-x[:, 1], x[:, 0], 0 * x[:, 0]])
    assert np.abs(A @ rot).max() < 1e-12


def test_P15_dof_counts():
    """F8/P15: (k+1)(2R+S) without eliminated DoFs (Nitsche) for the BASELINE configs."""
    assert [dof_count(config(i)) for i in range(5)] == [698, 141578, 7885839, 3367374, 26568846]
    for i in range(5):
        c = config(i)
        lev = Level(c["dim"], c["cells"], c["lo"], c["hi"], c["r"], c["k"])
        assert lev.N == dof_count(c)


# ---------------------------------------------------------------- P4: Tab:3 --------------------------
@pytest.fixture(scope="module")
def tab3_runs():
    """The oracle's Tab:3 marches (Q5/Q4, k = 2, Eq. 5.3, 4x4 cells, interval length 1) at tau0 / 2^0..2^3."""
    lam, mu = lame(100.0, 0.35)
    params = dict(rho=1.0, alpha=0.9, c0=0.01, lam=lam, mu=mu, K=[1, 0, 0, 1])
    lev = Level(2, [4, 4], [0, 0], [1, 1], r=5, k=2)
    sol = manufactured_eq53(params)
    return [march_errors(lev, params, sol, 0.0, 1.0, 50 * 2 ** level) for level in range(4)]


@pytest.mark.parametrize("level", [0, 1, 2, 3])
def test_P4_table3_reproduction(level, tab3_runs):
    """P4: PAPER Tab:3 printed errors, Q5/Q4, k=2, Eq. 5.3, within 2 %."""
    gold = json.load(open(os.path.join(GOLD, "tab3.json")))
    res = tab3_runs[level]
    assert np.allclose(res["L2"], gold["L2"][str(level)], rtol=0.02, atol=0)
    assert np.allclose(res["linf_tn"], gold["linf_tn"][str(level)], rtol=0.02, atol=0)


def test_P4_table3_eoc(tab3_runs):
    """P4: the printed EOC columns of Tab:3 (order 2k+1 = 5 in the time nodes, k+1 = 3 in
    L2(L2) for grad u and v, the pre-asymptotic pressure rates 4.13 / 4.77 / 4.09) within +-0.1."""
    gold = json.load(open(os.path.join(GOLD, "tab3.json")))
    for key, gkey in (("L2", "eoc_L2"), ("linf_tn", "eoc_linf_tn")):
        e = np.array([r[key] for r in tab3_runs])
        eoc = np.log2(e[:-1] / e[1:])
        for lvl in (1, 2, 3):
            assert np.all(np.abs(eoc[lvl - 1] - np.array(gold[gkey][str(lvl)])) <= 0.1), (key, lvl, eoc[lvl - 1])


# ---------------------------------------------------------------- P5: Tab:App1 rates (k = 3) ---------
def test_P5_tab_app1_eoc_k3():
    """P5 (rates only; reading R1): Tab:App1 (Q4/Q3 Taylor-Hood, dG(3), Eq. 5.1 with
    omega_1 = omega_2 = pi, I = (1, 2], tau_0 = 0.1, 4x4 cells, E = 100, nu = 0.35, K = I) prints L2(L2) EOCs that
    approach 4 (4.00 / 4.09 / 4.03 on its finest level).  The oracle's errors fall by 2^4 per joint h/tau halving
    already between levels 0 and 1 (|EOC - 4| <= 0.25 for grad u, v and p): a wrong k = 3 time discretisation
    (temporal constants, RHS jump weights, Radau-node loads) or a wrong Q4/Q3 form drops the rate.  The absolute
    values stay 1.8-7x below the printed ones (R1), so they are not pinned."""
    lam, mu = lame(100.0, 0.35)
    params = dict(rho=1.0, alpha=0.9, c0=0.01, lam=lam, mu=mu, K=[1, 0, 0, 1])
    sol = manufactured_eq51(params, "ones")
    errs = []
    for lvl in range(2):
        n = 4 * 2 ** lvl
        errs.append(march_errors(Level(2, [n, n], [0, 0], [1, 1], r=4, k=3), params, sol, 1.0, 2.0,
                                 10 * 2 ** lvl)["L2"])
    eoc = np.log2(np.array(errs[0]) / np.array(errs[1]))
    assert np.all(np.abs(eoc - 4.0) <= 0.25), eoc


# ---------------------------------------------------------------- P6: EOC of the BASELINE family ----
def test_P6_eoc_baseline_family():
    """P6: Q2/Q1 dG(1) with the config-0 manufactured solution, joint h/tau halving -> grad u and p
    errors converge with order ~2 = min(r, k+1) (Eq:ApFES)."""
    errs = []
    for lvl in range(3):
        n = 4 * 2 ** lvl
        lev = Level(2, [n, n], [0, 0], [1, 1], 2, 1)
        res = march_errors(lev, P0, manufactured_baseline(2, P0), 0.0, 0.2, 2 * 2 ** lvl)
        errs.append(res["L2"])
    errs = np.array(errs)
    eoc = np.log2(errs[:-1] / errs[1:])
    assert np.all(eoc[-1][[0, 2]] > 1.7) and np.all(eoc[-1] < 4.0)


# ---------------------------------------------------------------- P7: energy ------------------------
def test_P7_energy_monotone():
    """P7 (Eq:ExUniDS_3 P:L300-306): zero loads -> E_n = A(u,u) + <rho v, v> + <c0 p, p> at t_n
    is non-increasing."""
    lev = Level(2, [4, 4], [0, 0], [1, 1], 2, 1)
    op = SlabOperator(lev, P0, 0.05)
    S = op.assemble_spatial()
    lu = spla.splu(op.assemble().tocsc())
    rng = np.random.default_rng(0)
    U, V, P = rng.standard_normal(lev.R) * 1e-3, rng.standard_normal(lev.R), rng.standard_normal(lev.S)

    def energy(U, V, P):
        return U @ (S["A"] @ U) + V @ (S["Mrho"] @ V) + P @ (S["Mc"] @ P)

    E_prev = energy(U, V, P)
    for _ in range(10):
        X = lu.solve(slab_rhs(lev, S, op.chi_m1, op.th, U, V, P, None, None))
        U, V, P = end_state(lev, X)
        E = energy(U, V, P)
        assert E <= E_prev * (1 + 1e-12)
        E_prev = E


# ---------------------------------------------------------------- P8 / P9: transfer -------------------
def test_P8_galerkin_identity_frozen_hF():
    """P8: nested conforming spaces + exact quadrature => P^T A_l P = A_{l-1} when h_F is frozen."""
    coarse = Level(2, [2, 2], [0, 0], [1, 1], 2, 1)
    fine = Level(2, [4, 4], [0, 0], [1, 1], 2, 1)
    hF = 0.25
    Ac = SlabOperator(coarse, P0 | {"hF_fixed": hF}, 0.01).assemble().toarray()
    Af = SlabOperator(fine, P0 | {"hF_fixed": hF}, 0.01).assemble()
    P = prolongation(coarse, fine)
    G = (P.T @ Af @ P).toarray()
    assert np.abs(G - Ac).max() < 1e-12 * np.abs(Ac).max()


def test_P8_galerkin_identity_frozen_hF_3d():
    """P8 in 3D (Q2/Q1, dG(1), mixed Dirichlet / Neumann faces, anisotropic box): with a frozen h_F the rediscretised
    coarse slab operator is exactly the Galerkin product P^T A_l P: a value pin of every 3D form (volume terms,
    Nitsche face terms of A_gamma, C and B_gamma) against the 3D interpolation."""
    bcu, bcp = [0, 1, 0, 0, 1, 0], [1, 0, 1, 0, 0, 1]
    P3 = P0 | {"K": [0.02, 0.005, 0, 0.005, 0.01, 0, 0, 0, 0.015], "hF_fixed": 0.1}
    coarse = Level(3, [2, 1, 1], [0, 0, 0], [2, 1, 0.5], 2, 1, bc_u=bcu, bc_p=bcp)
    fine = Level(3, [4, 2, 2], [0, 0, 0], [2, 1, 0.5], 2, 1, bc_u=bcu, bc_p=bcp)
    Ac = SlabOperator(coarse, P3, 0.01).assemble().toarray()
    Af = SlabOperator(fine, P3, 0.01).assemble()
    P = prolongation(coarse, fine)
    G = (P.T @ Af @ P).toarray()
    assert np.abs(G - Ac).max() < 1e-11 * np.abs(Ac).max(), np.abs(G - Ac).max() / np.abs(Ac).max()
    # and the identity is not vacuous: the level operators differ when h_F follows the level
    P3l = dict(P3)
    del P3l["hF_fixed"]
    Acl = SlabOperator(coarse, P3l, 0.01).assemble().toarray()
    Afl = SlabOperator(fine, P3l, 0.01).assemble()
    assert np.abs((P.T @ Afl @ P).toarray() - Acl).max() > 1e-6 * np.abs(Acl).max()


def test_P8_galerkin_identity_level_hF_boundary_only():
    """P8 with level h_F: the difference lives only in Nitsche penalty entries of boundary DoFs."""
    coarse = Level(2, [2, 2], [0, 0], [1, 1], 2, 1)
    fine = Level(2, [4, 4], [0, 0], [1, 1], 2, 1)
    Ac = SlabOperator(coarse, P0, 0.01).assemble().toarray()
    Af = SlabOperator(fine, P0, 0.01).assemble()
    P = prolongation(coarse, fine)
    Dm = (P.T @ Af @ P).toarray() - Ac
    xq = coarse.node_coords(2, gauss_lobatto_nodes01(2))
    on_bd = np.any((xq < 1e-12) | (xq > 1 - 1e-12), axis=1)
    interior_nodes = np.nonzero(~on_bd)[0]
    rows = np.concatenate([coarse.offset(m, f, c) + interior_nodes for m in range(2) for f in (0, 1) for c in range(2)])
    assert np.abs(Dm[rows]).max() < 1e-12 * np.abs(Ac).max()
    assert np.abs(Dm).max() > 1.0


def test_P9_prolongation_reproduces_polynomials():
    """P9: interpolation reproduces coarse Q_r / Q_{r-1} polynomials exactly at the fine nodes."""
    for r in (2, 3):
        coarse = Level(2, [2, 3], [0, 0], [1, 1], r, 0)
        fine = Level(2, [4, 6], [0, 0], [1, 1], r, 0)
        P = prolongation(coarse, fine)
        f = lambda x: x[:, 0] ** r * x[:, 1] ** (r - 1) + 0.5 * x[:, 1] ** r
        g = lambda x: x[:, 0] ** (r - 1) * x[:, 1] ** (r - 1) - x[:, 0]
        xc = coarse.node_coords(r, gauss_lobatto_nodes01(r))
        xf = fine.node_coords(r, gauss_lobatto_nodes01(r))
        pc = coarse.node_coords(r - 1, gauss_lobatto_nodes01(r - 1))
        pf = fine.node_coords(r - 1, gauss_lobatto_nodes01(r - 1))
        vc = np.concatenate([f(xc), g(xc), f(xc), g(xc), g(pc)])
        vf = np.concatenate([f(xf), g(xf), f(xf), g(xf), g(pf)])
        assert np.abs(P @ vc - vf).max() < 1e-12


# ---------------------------------------------------------------- P10-P12: Vanka ----------------------
@pytest.fixture(scope="module")
def cfg0():
    c = config(0)
    H = Hierarchy(2, c["cells"], c["lo"], c["hi"], c["r"], c["k"], c["levels"], P0, c["tau"])
    return H


def test_P10_vanka_fixed_point(cfg0):
    """P10 (Eq:VankaOP0): b = A d => a sweep returns d."""
    sm = cfg0.smoothers[1]
    d = np.random.default_rng(3).standard_normal(cfg0.fine.N)
    b = cfg0.A[1] @ d
    assert np.abs(sm.sweep(b, d) - d).max() < 1e-12 * np.abs(d).max()


def test_P11_multiplicities():
    """P11: interior counts p_mu (2D Q2: 9/6/4 vertex/edge/cell; Q1 vertex 9; 3D 27/18/12/8, Q1 27)."""
    lev = Level(2, [4, 4], [0, 0], [1, 1], 2, 0)
    p = Patches(lev).p
    q = lambda i, j: p[lev.offset(0, FIELD_U, 0) + i + j * lev.q_shape[0]]
    assert (q(4, 4), q(5, 4), q(5, 5), q(4, 5)) == (9, 6, 4, 6)
    assert p[lev.offset(0, FIELD_P) + 2 + 2 * lev.p_shape[0]] == 9
    assert q(0, 0) == 4 and q(1, 0) == 4 and q(2, 0) == 6      # boundary: fewer patches
    lev3 = Level(3, [4, 4, 4], [0, 0, 0], [1, 1, 1], 2, 0)
    p3 = Patches(lev3).p
    s = lev3.q_strides
    qq = lambda i, j, k: p3[lev3.offset(0, FIELD_V, 1) + i * s[0] + j * s[1] + k * s[2]]
    assert (qq(4, 4, 4), qq(5, 4, 4), qq(5, 5, 4), qq(5, 5, 5)) == (27, 18, 12, 8)
    ps = lev3.p_strides
    assert p3[lev3.offset(0, FIELD_P) + 2 * ps[0] + 2 * ps[1] + 2 * ps[2]] == 27


def test_P11_literal_alg1_equals_averaged_form(cfg0):
    """P11(iii), reading A17: literal (sum_P (d + w y_P))/p equals d + w sum y_P / p to rounding."""
    sm = cfg0.smoothers[1]
    rng = np.random.default_rng(4)
    b, d = rng.standard_normal(cfg0.fine.N), rng.standard_normal(cfg0.fine.N)
    s1, s2 = sm.sweep(b, d), sm.sweep_literal(b, d)
    assert np.abs(s1 - s2).max() < 1e-13 * np.abs(s1).max()


def test_P11_centre_patch_is_direct_solve():
    """P11(iv): on the 2x2 mesh the centre patch holds every DoF, so A_P^{-1} R_P b = A^{-1} b."""
    lev = Level(2, [2, 2], [0, 0], [1, 1], 2, 1)
    A = SlabOperator(lev, P0, 0.01).assemble()
    pa = Patches(lev)
    centre = pa.verts.index((1, 1))
    assert len(pa.dofs[centre]) == lev.N
    b = np.random.default_rng(5).standard_normal(lev.N)
    Ainv = equilibrated_inverse(pa.extract(A, centre))
    y = np.empty(lev.N)
    y[pa.dofs[centre]] = Ainv @ b[pa.dofs[centre]]
    x = spla.spsolve(A.tocsc(), b)
    assert np.abs(y - x).max() < 1e-9 * np.abs(x).max()


@pytest.mark.parametrize("dim,cells", [(2, (6, 5)), (3, (4, 4, 5))])
def test_P12_class_sharing_bitwise(dim, cells):
    """P12 (App. A.4): A_P extracted per patch is identical within a per-axis class, up to the summation
    order of the global assembly (scipy sums duplicate entries in its own order: differences <= 1e-15 rel)."""
    lo, hi = [0.0] * dim, [1.0] * dim
    lev = Level(dim, cells, lo, hi, 2, 1, bc_u=[0, 1, 0, 0, 1, 0][:2 * dim], bc_p=[1, 0, 0, 1, 0, 0][:2 * dim])
    P3 = P0 | {"K": [0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01]} if dim == 3 else P0
    A = SlabOperator(lev, P3, 0.01).assemble()
    pa = Patches(lev)
    nclass = 0
    for c in pa.classes:
        mem = pa.members[c]
        ref = pa.extract(A, mem[0])
        for i in mem[1:min(len(mem), 6)]:
            assert np.abs(pa.extract(A, i) - ref).max() <= 1e-15 * np.abs(ref).max()
        nclass += 1
    assert nclass == np.prod([min(n, 4) + 1 for n in cells])


def test_P12_shared_equals_unshared_smoother():
    """Class-shared inverses give the same sweep as one inverse per patch, on a 16x16 mesh where the
    interior class holds 169 patches (on config 0 every patch is its own class, which would make this vacuous)."""
    lev = Level(2, [16, 16], [0, 0], [1, 1], 2, 1)
    A = SlabOperator(lev, P0, 0.01).assemble()
    pa = Patches(lev)
    assert max(len(m) for m in pa.members.values()) == 13 * 13 and len(pa.classes) == 25
    sm1 = VankaSmoother(A, pa, 0.7, share_classes=True)
    sm2 = VankaSmoother(A, pa, 0.7, share_classes=False)
    rng = np.random.default_rng(6)
    b, d = rng.standard_normal(lev.N), rng.standard_normal(lev.N)
    s1, s2 = sm1.sweep(b, d), sm2.sweep(b, d)
    # per-patch inverses of bitwise-equal-up-to-assembly-order matrices (R2): agreement to rounding, not bitwise
    assert np.abs(s1 - s2).max() <= 1e-11 * np.abs(s2).max(), np.abs(s1 - s2).max()


# ---------------------------------------------------------------- P13: coercivity -------------------
@pytest.mark.parametrize("n", [2, 4, 8])
def test_P13_coercivity(n):
    """P13 (Eq:CoercA P:L1018, Eq:CoercB P:L1046): lambda_min(sym A_gamma), lambda_min(sym B_gamma) > 0."""
    lev = Level(2, [n, n], [0, 0], [1, 1], 2, 1)
    S = SlabOperator(lev, P0, 0.01).assemble_spatial()
    for name in ("A", "B"):
        M = S[name].toarray()
        assert np.linalg.eigvalsh(0.5 * (M + M.T)).min() > 0


# ---------------------------------------------------------------- P3 / P14: solver ------------------
def test_P3_fgmres_gmg_matches_direct_solve(cfg0):
    """P3 (Lemma 3.1): FGMRES-GMG with rtol 1e-13 reaches the dense direct solution of config 0."""
    A = cfg0.A[1]
    b = np.random.default_rng(7).standard_normal(cfg0.fine.N)
    xs = np.linalg.solve(A.toarray(), b)
    x, info = fgmres(lambda v: A @ v, b, cfg0.vcycle, tol=1e-13, restart=30)
    assert info["converged"]
    assert np.linalg.norm(x - xs) <= 1e-9 * np.linalg.norm(xs)


def test_P3_vcycle_single_level_is_direct():
    """a V-cycle with one level is the coarse direct solve."""
    H = Hierarchy(2, [2, 2], [0, 0], [1, 1], 2, 1, 1, P0, 0.01)
    b = np.random.default_rng(8).standard_normal(H.fine.N)
    x = np.linalg.solve(H.A[0].toarray(), b)
    assert np.abs(H.vcycle(b) - x).max() < 1e-10 * np.abs(x).max()


def test_P14_gmres_minimal_residual_bruteforce():
    """P14: after j steps the FGMRES iterate minimises ||b - A x|| over span{Z_j}; with a fixed linear
    preconditioner M that is M K_j(AM, b): compare with dense least squares."""
    rng = np.random.default_rng(9)
    n = 12
    A = rng.standard_normal((n, n)) + 6 * np.eye(n)
    M = np.eye(n) + 0.1 * rng.standard_normal((n, n))
    b = rng.standard_normal(n)
    for j in (1, 2, 3, 5):
        x, info = fgmres(lambda v: A @ v, b, lambda v: M @ v, tol=1e-300, restart=j, maxit=j)
        K = [b]
        for _ in range(j - 1):
            K.append(A @ (M @ K[-1]))
        Zb = M @ np.array(K).T
        y = np.linalg.lstsq(A @ Zb, b, rcond=None)[0]
        assert abs(np.linalg.norm(b - A @ x) - np.linalg.norm(b - A @ Zb @ y)) < 1e-10


def test_P14_exact_preconditioner_one_iteration():
    """FGMRES with M = A^{-1} converges in one iteration."""
    rng = np.random.default_rng(10)
    A = rng.standard_normal((20, 20)) + 8 * np.eye(20)
    Ai = np.linalg.inv(A)
    b = rng.standard_normal(20)
    x, info = fgmres(lambda v: A @ v, b, lambda v: Ai @ v, tol=1e-10)
    assert info["iterations"] == 1 and info["converged"]


def test_P16_grid_robustness_cfg0_cfg1():
    """P16 (plausibility): iteration counts of config 0 (2 levels) and a 16x16 / 4-level version
    of the same problem stay within +-50 %; parity of counts is otherwise unpinned."""
    its = []
    for cells, lv in (((4, 4), 2), ((16, 16), 4)):
        H = Hierarchy(2, cells, [0, 0], [1, 1], 2, 1, lv, P0, 0.01)
        b = uniform_load(H.fine.N, 1)
        _, info = fgmres(lambda v: H.A[-1] @ v, b, H.vcycle, tol=1e-8, restart=30)
        its.append(info["iterations"])
    assert max(its) <= 1.5 * min(its) + 1


# ---------------------------------------------------------------- sampled evaluations (full-size parity) ---
@pytest.mark.parametrize("dim,cells,r,k", [(2, (6, 5), 2, 1), (2, (5, 4), 3, 2), (3, (5, 4, 4), 2, 1)])
def test_sampled_helpers_match_global_definitions(dim, cells, r, k):
    """oracle/sampled.py (used at BASELINE sizes) reproduces the assembled-matrix definitions: rows of A x,
    A_P = A[Z,Z] and one Alg. 1 step at sampled DoFs."""
    from oracle.sampled import LiteOperator
    bc = [0, 1, 0, 0, 1, 0][:2 * dim]
    lev = Level(dim, cells, [0.0] * dim, [1.0] * dim, r, k, bc_u=bc, bc_p=bc[::-1])
    P3 = P0 | {"K": [0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01]} if dim == 3 else P0
    op = SlabOperator(lev, P3, 0.01)
    A = op.assemble()
    lite = LiteOperator(lev, P3, 0.01)
    rng = np.random.default_rng(11)
    x, b = rng.standard_normal(lev.N), rng.standard_normal(lev.N)
    rows = rng.choice(lev.N, 25, replace=False)
    assert np.abs(lite.rows(x, rows) - (A @ x)[rows]).max() < 1e-12 * np.abs(A @ x).max()
    pa = Patches(lev)
    for i in (0, len(pa.verts) // 2, len(pa.verts) - 1):
        Z, AP, _ = lite.patch_system(pa.verts[i])
        assert np.array_equal(Z, pa.dofs[i])
        ref = pa.extract(A, i)
        assert np.abs(AP - ref).max() <= 1e-13 * np.abs(ref).max()
    sm = VankaSmoother(A, pa, 0.7)
    d = 1e-3 * rng.standard_normal(lev.N)
    full = sm.sweep(b, d)
    sample = rng.choice(lev.N, 6, replace=False)
    got = lite.sampled_sweep(b, d, sample)
    assert np.abs(got - full[sample]).max() <= 1e-9 * np.abs(full).max()


# ---------------------------------------------------------------- N2(i): multiplicative coloured Vanka -------
@pytest.fixture(scope="module")
def mesh8():
    """8 x 6 cells, Q2/Q1, dG(1): large enough for several patches per colour (vertex colours v mod 4)."""
    lev = Level(2, [8, 6], [0, 0], [1, 0.75], 2, 1)
    A = SlabOperator(lev, P0, 0.01).assemble()
    return lev, A, VankaSmoother(A, Patches(lev), omega=0.7)


def test_N2_same_colour_patches_share_no_cell(mesh8):
    """Colour batching is exact only if A_l couples no two patches of one colour: A[Z(P), Z(Q)] = 0."""
    lev, A, sm = mesh8
    Ad = A.tocsr()
    for group in sm.colour_order():
        assert len(group) >= 1
        for a in range(len(group)):
            for b in range(a + 1, len(group)):
                zp, zq = sm.P.dofs[group[a]], sm.P.dofs[group[b]]
                assert len(np.intersect1d(zp, zq)) == 0
                assert abs(Ad[zp][:, zq]).sum() == 0.0


def test_N2_colour_batched_equals_sequential_overwrite(mesh8):
    """P:L527-529 ('overwriting successively ... within the patch loop'): the colour-batched sweep equals the
    literal one-patch-at-a-time overwrite loop in the same order (a different computation: one residual per patch)."""
    lev, A, sm = mesh8
    rng = np.random.default_rng(11)
    b, d = rng.standard_normal(lev.N), rng.standard_normal(lev.N)
    s1, s2 = sm.sweep_colored(b, d), sm.sweep_sequential(b, d)
    assert np.abs(s1 - s2).max() < 1e-12 * np.abs(s2).max()


def test_N2_fixed_point_and_exact_local_solves(mesh8):
    """Eq:VankaOP0: b = A d is a fixed point; with omega = 1 each patch update is an exact local solve, so right after
    a colour is processed the residual vanishes on every DoF of that colour's patches."""
    lev, A, sm = mesh8
    rng = np.random.default_rng(12)
    d = rng.standard_normal(lev.N)
    assert np.abs(sm.sweep_colored(A @ d, d) - d).max() < 1e-12 * np.abs(d).max()
    sm1 = VankaSmoother(A, sm.P, omega=1.0)
    b, x = rng.standard_normal(lev.N), np.zeros(lev.N)
    for group in sm1.colour_order():
        r = b - A @ x
        for i in group:
            z = sm1.P.dofs[i]
            x[z] = x[z] + sm1.inv[i] @ r[z]
        res = b - A @ x
        for i in group:
            assert np.abs(res[sm1.P.dofs[i]]).max() < 1e-9 * np.abs(b).max()


def test_N2_multiplicative_gmg_converges(cfg0):
    """The colour-ordered multiplicative smoother inside the V-cycle preconditions FGMRES to the direct solution."""
    c = config(0)
    Hm = Hierarchy(2, c["cells"], c["lo"], c["hi"], c["r"], c["k"], c["levels"], P0, c["tau"], colored=True)
    b = uniform_load(Hm.fine.N, 7)
    x, info = fgmres(lambda v: Hm.A[-1] @ v, b, Hm.vcycle, tol=1e-10, restart=30)
    xs = spla.spsolve(Hm.A[-1].tocsc(), b)
    assert info["iterations"] <= 30
    assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)


# ---------------------------------------------------------------- N4: Problem B.1 (DS) -----------------------
def test_N4_ds_equals_dsa_on_steady_states():
    """Problem B.1 couples d_t u (not v) into the pressure equation, via -sum_a T_ba C U_a on the left and, on the
    right (Eq:DPQ_3), <alpha div u^{n-1}, psi^+> - alpha <u_D.n, psi^+>_{G_D^u} with u_D = 0.  For a state
    steady in time (V = 0, U_a = U^{n-1} = U0, P_a = P^{n-1} = P0) whose trace satisfies the Dirichlet data
    (U0 = 0 on the boundary nodes), d_t u = v = 0 in both formulations, so F_n - A_n X must be the same for DS and
    DSA: the row sums of T equal chi(-1) (App. A.2), which makes the DS coupling cancel exactly; a wrong sign or slot
    breaks it."""
    lev = Level(2, [4, 4], [0, 0], [1, 1], 2, 1)
    rng = np.random.default_rng(21)
    xq = lev.node_coords(2, gauss_lobatto_nodes01(2))
    interior = np.all((xq > 1e-12) & (xq < 1 - 1e-12), axis=1).astype(float)
    U0 = rng.standard_normal(lev.R) * np.concatenate([interior, interior])
    P0_ = rng.standard_normal(lev.S)
    V0 = np.zeros(lev.R)
    X = np.zeros(lev.N)
    for m in range(lev.k + 1):
        o = m * lev.block
        X[o + lev.R: o + 2 * lev.R] = U0
        X[o + 2 * lev.R: o + lev.block] = P0_
    res = []
    for ds in (False, True):
        op = SlabOperator(lev, P0_params(), 0.01, ds)
        S = op.assemble_spatial()
        F = slab_rhs(lev, S, op.chi_m1, op.th, U0, V0, P0_, None, None, ds)
        res.append(F - op.assemble() @ X)
    assert np.abs(res[0] - res[1]).max() < 1e-12 * np.abs(res[0]).max()
    # and the DS operator really differs from DSA on a non-steady state
    opd, opa = SlabOperator(lev, P0_params(), 0.01, True), SlabOperator(lev, P0_params(), 0.01, False)
    Y = rng.standard_normal(lev.N)
    assert np.abs(opd.assemble() @ Y - opa.assemble() @ Y).max() > 1e-6


def test_N4_ds_rhs_is_volume_divergence_only():
    """Eq:DPQ_3 right-hand side with homogeneous Dirichlet data: the psi-row jump datum is
    chi_b(-1) <c0 p^{n-1} + alpha div u^{n-1}, psi>, WITHOUT the boundary trace alpha <u^{n-1}.n, psi>_{G_D^u} that
    -C(u^{n-1}, psi) would add.  u^{n-1} = (x^2, x y) (in Q2) has div u = 3x (in Q1) and a nonzero normal trace, so
    <alpha div u, psi_s> = 3 alpha (M_p X1)_s with X1 the Q1 interpolant of x: a closed form independent of C."""
    lev = Level(2, [4, 3], [0, 0], [1, 1], 2, 1)
    op = SlabOperator(lev, P0_params(), 0.01, True)
    S = op.assemble_spatial()
    xq = lev.node_coords(2, gauss_lobatto_nodes01(2))
    xp = lev.node_coords(1, gauss_lobatto_nodes01(1))
    U = np.concatenate([xq[:, 0] ** 2, xq[:, 0] * xq[:, 1]])
    F = slab_rhs(lev, S, op.chi_m1, op.th, U, np.zeros(lev.R), np.zeros(lev.S), None, None, ds=True)
    want = 3.0 * P0_params()["alpha"] * (S["Mp"] @ xp[:, 0])
    for b in range(lev.k + 1):
        o = b * lev.block + 2 * lev.R
        got = F[o: o + lev.S] / op.chi_m1[b]
        assert np.abs(got - want).max() < 1e-12 * np.abs(want).max(), np.abs(got - want).max()
    # the trace term this excludes is not small for this u (so the pin tells the two readings apart)
    trace = S["C"] @ U - S["Cvol"] @ U
    assert np.abs(trace).max() > 0.1 * np.abs(want).max()


def P0_params():
    return dict(P0)


def test_N4_ds_eoc_baseline_family():
    """P6 for Problem B.1: the DS discretisation converges with the same order ~2 ('identical convergence
    behaviour' of both formulations), and its errors stay within a factor 2 of the DSA errors."""
    errs, errs_a = [], []
    for lvl in range(3):
        n = 4 * 2 ** lvl
        lev = Level(2, [n, n], [0, 0], [1, 1], 2, 1)
        errs.append(march_errors(lev, P0, manufactured_baseline(2, P0), 0.0, 0.2, 2 * 2 ** lvl, ds=True)["L2"])
        errs_a.append(march_errors(lev, P0, manufactured_baseline(2, P0), 0.0, 0.2, 2 * 2 ** lvl)["L2"])
    errs, errs_a = np.array(errs), np.array(errs_a)
    eoc = np.log2(errs[:-1] / errs[1:])
    assert np.all(eoc[-1][[0, 2]] > 1.7) and np.all(eoc[-1] < 4.0)
    assert np.all(errs[-1] < 2 * errs_a[-1]) and np.all(errs_a[-1] < 2 * errs[-1])


# ---------------------------------------------------------------- N2(ii): element-wise Vanka -------------------
@pytest.mark.parametrize("dim,cells", [(2, (7, 6)), (3, (4, 3, 5))])
def test_N2ii_cell_class_sharing(dim, cells):
    """Element-wise patches Z(K) (one cell): A_K = A_l[Z(K), Z(K)] is the same matrix for all cells of a per-axis
    class {0}, {1..n-2}, {n-1} (mixed boundary conditions), up to the global assembly's summation order."""
    d = dim
    bcu = [0, 1, 0, 0, 1, 0][:2 * d]
    bcp = [1, 0, 0, 1, 0, 0][:2 * d]
    lev = Level(d, list(cells), [0] * d, [1] * d, 2, 1, bc_u=bcu, bc_p=bcp)
    par = dict(P0) if d == 2 else dict(P0, K=[0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01])
    A = SlabOperator(lev, par, 0.01).assemble()
    pa = Patches(lev, cells=True)
    assert len(pa.verts) == int(np.prod(cells)) and len(pa.classes) == 3 ** d
    for c in pa.classes:
        mem = pa.members[c]
        A0 = pa.extract(A, mem[0])
        for i in mem[1:]:
            assert np.abs(pa.extract(A, i) - A0).max() <= 1e-15 * np.abs(A0).max()


def test_N2ii_cell_multiplicities_and_fixed_point(cfg0):
    """p_mu = number of cells containing mu (2D interior Q2: vertex 4, edge 2, cell-interior 1); b = A d is a fixed
    point of the element-wise sweep."""
    lev = cfg0.fine
    A = cfg0.A[-1]
    sm = VankaSmoother(A, Patches(lev, cells=True))
    q = lambda i, j: sm.P.p[lev.offset(0, FIELD_U, 0) + i + j * lev.q_shape[0]]
    assert (q(4, 4), q(5, 4), q(5, 5)) == (4, 2, 1)
    d = np.random.default_rng(31).standard_normal(lev.N)
    assert np.abs(sm.sweep(A @ d, d) - d).max() < 1e-12 * np.abs(d).max()


# ---------------------------------------------------------------- N2(iii): overwrite without averaging ----------
def test_N2iii_overwrite_equals_literal_loop_and_fixed_point(cfg0):
    """The vectorised last-writer form equals the literal overwriting patch loop; b = A d stays a fixed point; and it
    differs from the averaged sweep (DoFs shared by patches take one patch's update, not the mean)."""
    sm = cfg0.smoothers[1]
    rng = np.random.default_rng(41)
    b, d = rng.standard_normal(cfg0.fine.N), rng.standard_normal(cfg0.fine.N)
    s1, s2 = sm.sweep_overwrite(b, d), sm.sweep_overwrite_literal(b, d)
    assert np.abs(s1 - s2).max() == 0.0
    assert np.abs(sm.sweep_overwrite(cfg0.A[1] @ d, d) - d).max() < 1e-12 * np.abs(d).max()
    assert np.abs(s1 - sm.sweep(b, d)).max() > 1e-3 * np.abs(s1).max()


# ---------------------------------------------------------------- N1: goal quantities (Eq:DefGQ) ---------------
def test_N1_goal_quantities_exact_for_fe_functions():
    """b_u = int_face u.n, b_p = int_face p on box faces are exact for interpolants of polynomials in the FE spaces:
    u = (1 + x + 2y, 3 - y), p = 2 + x y on [0,2] x [0,1] (closed-form face integrals)."""
    from oracle.loads import goal_quantities
    lev = Level(2, [4, 3], [0, 0], [2, 1], 2, 1)
    xq = lev.node_coords(2, gauss_lobatto_nodes01(2))
    xp = lev.node_coords(1, gauss_lobatto_nodes01(1))
    X = np.zeros(lev.N)
    o = lev.k * lev.block
    X[o + lev.R: o + lev.R + lev.nq] = 1 + xq[:, 0] + 2 * xq[:, 1]      # U_x
    X[o + lev.R + lev.nq: o + 2 * lev.R] = 3 - xq[:, 1]                 # U_y
    X[o + 2 * lev.R: o + lev.block] = 2 + xp[:, 0] * xp[:, 1]           # P
    want = {0: (-2.0, 2.0),            # x = 0: n = -e_x, int (1 + 2y) dy = 2 ; int 2 dy = 2
            1: (4.0, 3.0),             # x = 2: int (3 + 2y) dy = 4 ; int (2 + 2y) dy = 3
            2: (-6.0, 4.0),            # y = 0: n = -e_y, int 3 dx = 6 ; int 2 dx = 4
            3: (4.0, 6.0)}             # y = 1: int 2 dx = 4 ; int (2 + x) dx = 6
    for face, (bu, bp) in want.items():
        gu, gp = goal_quantities(lev, X, face)
        assert abs(gu - bu) < 1e-12 and abs(gp - bp) < 1e-12, (face, gu, gp)
