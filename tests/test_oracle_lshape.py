"""Pins of the L-shaped benchmark oracle (oracle/lshape.py) against what the paper prints and what
the mathematics fixes (CPU, -m "not gpu").  None of them re-types the oracle's formulas:

* L1  DoF counts of Table 4 for every printed row, the (k+1) 390 DoFs of the initial grid (caption) and
      the 98,304 cells of ref_5.  Rows beyond ref_3 by the closed count the oracle's levels match up to ref_3.
* L2  SIP consistency: for the globally linear q = 1 - y (in P_1^disc, continuous, zero on Gamma_p^D), integration by
      parts on every cell leaves only the Neumann boundary flux: B_gamma q = sum_{F Neumann} <K grad q . n, psi>_F,
      evaluated with the exact face moments of the monomials (Def:B second option).
* L3  A_gamma with directional and Dirichlet faces: for w = (0, y, 0) (w = 0 on y = 0, w.n = 0 on the directional
      faces, sigma(w) constant, sigma(w) n normal on them) A_gamma w = sum_{traction-free / traction faces} <sigma n,
      chi>, with Simpson's weights as the exact face integrals of the Q_2 basis (Def:A + Eq:BCd).
* L4  C(chi, 1) = -alpha sum_{Neumann faces of u} <chi . n, 1> (divergence theorem + the face terms on Dirichlet
      and directional faces, Def:C and reading R5).
* L5  Galerkin identity with frozen h_F: P^T A_l P = A_{l-1} (interior SIP faces inside a coarse cell see zero
      jumps of prolonged functions) — pins the P_{r-1}^disc transfer and every face term at once.
* L6  Prolongation reproduces quadratic u and linear p exactly; symmetry and coercivity of A_gamma and B_gamma
      (Eq:CoercA/B).
* L7  Traction load: partition of unity and first moment give -5e9 int g and -5e9 int x g in closed form.
* L8  FGMRES with the L-shape V-cycle reaches the sparse direct solution; the V-cycle obeys the error-propagation
      recursion (tests/test_oracle_pins_mg.py::E_apply).
* L9  Goal quantities of constant fields: b_u = b_p = |Gamma_m| = 1/4.
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import lshape as LS

# Table 4: (k, r, ref) -> DoF per slab
TABLE4 = {(0, 2, 4): 682950, (1, 2, 2): 25836, (1, 2, 3): 182220, (1, 2, 4): 1365900, (1, 2, 5): 10571532,
          (1, 2, 6): 83172876, (1, 3, 5): 34596492, (1, 3, 6): 273640716}


def closed_count(k, r, ref):
    """DoFs of Q_r^3 x Q_r^3 x P_{r-1}^disc on the 3-cube L-shape with 2^ref cells per cube edge."""
    N = 2 ** ref
    nq = ((2 * r * N + 1) ** 2 - (r * N) ** 2) * (r * N + 1)
    npc = {2: 4, 3: 10}[r]
    return (k + 1) * (6 * nq + npc * 3 * N ** 3)


def test_L1_dof_counts_table4():
    for ref in range(0, 4):
        for r in (2, 3):
            for k in (0, 1):
                lv = LS.LLevel(ref, r, k)
                assert lv.N == closed_count(k, r, ref)
                assert lv.n_cells == 3 * 8 ** ref
    assert LS.LLevel(0, 2, 1).N == 2 * 390                       # caption: (k+1) 390 for r = 2
    for (k, r, ref), n in TABLE4.items():
        assert closed_count(k, r, ref) == n, (k, r, ref)
    assert 3 * 8 ** 5 == 98304
    assert LS.LLevel(1, 2, 1).N == 2 * 2046                     # reading R7 (caption prints 2013)


@pytest.fixture(scope="module")
def lev1():
    lv = LS.LLevel(1, 2, 1)
    S = LS.LSpatial(lv, LS.lshape_params(2))
    return lv, S


def test_L2_sip_consistency_linear_pressure(lev1):
    lv, S = lev1
    h = lv.h[0]
    q = np.zeros(lv.np_)
    expect = np.zeros(lv.np_)
    for cid, c in enumerate(lv.cells):
        yc = (c[1] + 0.5) * h
        q[cid * 4:(cid + 1) * 4] = [1.0 - yc, 0.0, -0.5 * h, 0.0]   # 1 - y = (1 - y_c) - (h/2) xi_y
        # K grad q . n on Neumann faces with n = -+e_y; face moments of (1, xi_x, xi_y, xi_z): h^2 (1, 0, xi_y, 0)
        if c[1] == 0:                                                # y = 0, n = -e_y: flux +1, xi_y = -1
            expect[cid * 4:(cid + 1) * 4] += h * h * np.array([1.0, 0.0, -1.0, 0.0])
        if c[1] == lv.Ncube - 1 and c[0] >= lv.Ncube:                # y = 0.5, x > 0.5, n = +e_y: flux -1, xi_y = 1
            expect[cid * 4:(cid + 1) * 4] -= h * h * np.array([1.0, 0.0, 1.0, 0.0])
    got = S.B @ q
    assert np.allclose(got, expect, rtol=0, atol=1e-12 * np.abs(expect).max())


def _simpson_face(lv, cid, f):
    """(local node index, weight) of int_face phi_J for the Q_2 basis on face f of cell cid (exact)."""
    h = lv.h[0]
    w1 = np.array([1.0, 4.0, 1.0]) / 6.0
    a, s = f // 2, f % 2
    out = []
    for J, loc in enumerate(lv.q_loc):
        if loc[a] != 2 * s:
            continue
        wt = h * h
        for b in range(3):
            if b != a:
                wt *= w1[loc[b]]
        out.append((lv.cell_q[cid][J], wt))
    return out


def test_L3_directional_and_dirichlet_faces(lev1):
    lv, S = lev1
    p = S.p
    lam, mu = p["lam"], p["mu"]
    r = lv.r
    ys = np.zeros(lv.nq)
    for cid, c in enumerate(lv.cells):
        for J, loc in enumerate(lv.q_loc):
            ys[lv.cell_q[cid][J]] = (r * c[1] + loc[1]) * lv.h[1] / r
    w = np.zeros(3 * lv.nq)
    w[lv.nq:2 * lv.nq] = ys                                    # w = (0, y, 0)
    expect = np.zeros(3 * lv.nq)
    N = lv.Ncube
    for cid, c in enumerate(lv.cells):
        for f in range(6):
            if lv.neighbour(c, f) >= 0:
                continue
            kind = lv.u_bc(c, f)
            if kind not in (LS.U_NEUMANN, LS.U_TRACTION):
                continue
            a, s = f // 2, f % 2
            assert s == 1 and a in (0, 1)
            # sigma(w) = lam E + 2 mu e_y e_y^T: sigma e_x = lam e_x, sigma e_y = (lam + 2 mu) e_y
            comp, val = (0, lam) if a == 0 else (1, lam + 2 * mu)
            for node, wt in _simpson_face(lv, cid, f):
                expect[comp * lv.nq + node] += val * wt
    got = S.A @ w
    scale = np.abs(expect).max()
    assert np.abs(got - expect).max() <= 1e-9 * scale
    assert N == 2


def test_L4_pressure_coupling_row_sums(lev1):
    lv, S = lev1
    alpha = S.p["alpha"]
    one = np.zeros(lv.np_)
    one[0::4] = 1.0
    expect = np.zeros(3 * lv.nq)
    for cid, c in enumerate(lv.cells):
        for f in range(6):
            if lv.neighbour(c, f) >= 0 or lv.u_bc(c, f) not in (LS.U_NEUMANN, LS.U_TRACTION):
                continue
            a = f // 2
            for node, wt in _simpson_face(lv, cid, f):
                expect[a * lv.nq + node] -= alpha * wt           # outward n = +e_a on these faces
    got = S.C.T @ one
    assert np.abs(got - expect).max() <= 1e-12 * np.abs(expect).max()


def test_L5_galerkin_identity_frozen_hF():
    params = dict(LS.lshape_params(2), hF_fixed=0.37)
    H = LS.LHierarchy(0, 2, 2, 1, 0.01, params=params)
    G = (H.P[1].T @ H.A[1] @ H.P[1]).toarray()
    A0 = H.A[0].toarray()
    assert np.abs(G - A0).max() <= 1e-10 * np.abs(A0).max()
    # the level penalty (h_F = |K|_d, reading A6) breaks it only through the face penalty terms
    H2 = LS.LHierarchy(0, 2, 2, 1, 0.01)
    G2 = (H2.P[1].T @ H2.A[1] @ H2.P[1]).toarray()
    assert np.abs(G2 - H2.A[0].toarray()).max() > 1e-3 * np.abs(A0).max()


def test_L6_prolongation_polynomials_and_coercivity(lev1):
    lc, lf = LS.LLevel(0, 2, 0), LS.LLevel(1, 2, 0)
    P = LS.prolongation(lc, lf)

    def q_nodes_xyz(lv):
        xyz = np.zeros((lv.nq, 3))
        for cid, c in enumerate(lv.cells):
            for J, loc in enumerate(lv.q_loc):
                xyz[lv.cell_q[cid][J]] = (2 * c + loc) * lv.h / 2
        return xyz

    def field(lv):
        x = q_nodes_xyz(lv)
        u = x[:, 0] ** 2 - 3 * x[:, 1] * x[:, 2] + x[:, 2]
        v = np.zeros(lv.N)
        v[lv.R + lv.nq:lv.R + 2 * lv.nq] = u                    # U_1
        for cid, c in enumerate(lv.cells):                       # p = 2 + x - 4 z, as monomial coefficients
            ctr = (c + 0.5) * lv.h
            v[2 * lv.R + cid * 4: 2 * lv.R + cid * 4 + 4] = [2 + ctr[0] - 4 * ctr[2], 0.5 * lv.h[0], 0.0,
                                                             -2.0 * lv.h[2]]
        return v
    assert np.abs(P @ field(lc) - field(lf)).max() <= 1e-13
    lv, S = lev1
    for M in (S.A, S.B):
        D = M.toarray()
        assert np.abs(D - D.T).max() <= 1e-12 * np.abs(D).max()
        assert np.linalg.eigvalsh(D)[0] > 0


def test_L7_traction_moments():
    lv = LS.LLevel(1, 2, 1)
    f = LS.traction_vector(lv)
    assert np.all(f[:lv.nq] == 0) and np.all(f[2 * lv.nq:] == 0)
    fy = f[lv.nq:2 * lv.nq]
    assert abs(fy.sum() - (-5e9 * 0.875)) <= 1e-12 * 5e9
    xs = np.zeros(lv.nq)
    for cid, c in enumerate(lv.cells):
        for J, loc in enumerate(lv.q_loc):
            xs[lv.cell_q[cid][J]] = (2 * c[0] + loc[0]) * lv.h[0] / 2
    assert abs(xs @ fy - (-5e9 / 6.0)) <= 1e-12 * 5e9


@pytest.fixture(scope="module")
def hier():
    return LS.LHierarchy(0, 2, 2, 1, 0.01)


def test_L8_fgmres_vcycle_reaches_direct_solve(hier):
    from oracle.gmres import fgmres
    H = hier
    rng = np.random.default_rng(7)
    b = rng.uniform(-1, 1, H.fine.N)
    x, info = fgmres(lambda v: H.A[-1] @ v, b, H.vcycle, tol=1e-10, restart=30)
    xd = spla.spsolve(H.A[-1].tocsc(), b)
    assert info["converged"] and info["iterations"] < 30
    assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd)


def test_L8_vcycle_error_propagation(hier):
    from tests.test_oracle_pins_mg import E_apply, E_vcycle
    H = hier
    rng = np.random.default_rng(3)
    for _ in range(2):
        x = rng.standard_normal(H.fine.N)
        e1 = E_apply(H, 1, x)
        e2 = E_vcycle(H, H.vcycle, x)
        assert np.linalg.norm(e1 - e2) <= 1e-9 * np.linalg.norm(x)


def test_L9_goal_quantities_of_constants():
    lv = LS.LLevel(1, 2, 1)
    x = np.zeros(lv.N)
    o = lv.k * lv.block
    x[o + lv.R:o + lv.R + lv.nq] = 1.0          # u_x = 1 at t_n
    x[o + 2 * lv.R:o + lv.block:4] = 1.0         # p = 1
    bu, bp = LS.goal_quantities(lv, x)
    assert abs(bu - 0.25) <= 1e-14 and abs(bp - 0.25) <= 1e-14


def test_penalty_length_modes_enter_as_gamma_over_hF():
    """The experiment modes of DESIGN.md §7.6 change only the penalty lengths: B_gamma(mode) - B_gamma(|K|_d) =
    gamma_b (1 / h_P - 1 / h^3) M_pen with ONE penalty form M_pen for every mode (4: h_P = h, 6: h_P = h^2), and
    mode 5 leaves B_gamma unchanged; likewise A_gamma for the u lengths (5: h, 6: h^2) — Def:ab / Def:B."""
    lv = LS.LLevel(1, 2, 1)
    h = lv.h[0]
    S = {m: LS.LSpatial(lv, dict(LS.lshape_params(2), hF_mode=m)) for m in (0, 4, 5, 6)}
    dB4 = (S[4].B - S[0].B).toarray() / (1.0 / h - 1.0 / h ** 3)
    dB6 = (S[6].B - S[0].B).toarray() / (1.0 / h ** 2 - 1.0 / h ** 3)
    assert np.abs(dB4).max() > 0
    assert np.allclose(dB4, dB6, rtol=0, atol=1e-9 * np.abs(dB4).max())
    assert np.abs((S[5].B - S[0].B).toarray()).max() == 0.0
    dA5 = (S[5].A - S[0].A).toarray() / (1.0 / h - 1.0 / h ** 3)
    dA6 = (S[6].A - S[0].A).toarray() / (1.0 / h ** 2 - 1.0 / h ** 3)
    assert np.abs(dA5).max() > 0
    assert np.allclose(dA5, dA6, rtol=0, atol=1e-9 * np.abs(dA5).max())
    assert np.abs((S[4].A - S[0].A).toarray()).max() == 0.0


def test_L10_slab_energy_identity():
    """L10: the homogeneous slab problem (P:L233-256 with f = 0, no traction) dissipates the energy
    E(v, u, p) = (rho |v|^2 + a_gamma(u, u) + c0 |p|^2) / 2 exactly as the continuous system does, up to the dG(k)
    jump: testing the rows (phi, chi, psi) with (M_rho^-1 A_gamma u, v, p) — polynomials of degree k in time, so
    admissible rows of the algebraic system — and using that the k+1 point right Radau rule integrates d/dt E
    (degree 2k - 1) and b_gamma(p, p) (degree 2k) exactly gives

        E(x(t_n)) - E(x(t_{n-1}^-)) + E(x(t_{n-1}^+) - x(t_{n-1}^-)) + Q_n(b_gamma(p, p)) = 0.

    The coupling terms cancel only if C enters the chi row as +C^T p and the psi row as -C v: a sign
    slip in either, a wrong T, a wrong chi_hat(-1) or a wrong jump term in slab_rhs breaks the identity at O(1).
    Radau data typed from the textbook rule for k = 1: nodes (-1/3, 1), weights (3/2, 1/2), chi_hat(-1) = (3/2, -1/2).
    """
    tau = 0.05
    H = LS.LHierarchy(0, 1, 2, 1, tau)
    lev, S = H.fine, H.spatial[-1]
    R, blk = lev.R, lev.block
    th = 0.5 * tau * np.array([1.5, 0.5])
    cm1 = np.array([1.5, -0.5])
    lu = spla.splu(H.A[-1].tocsc())

    def split(xb):
        return xb[:R], xb[R:2 * R], xb[2 * R:]

    def energy(xb):
        V, U, P = split(xb)
        return 0.5 * (V @ (S.Mr @ V) + U @ (S.A @ U) + P @ (S.Mc @ P))

    rng = np.random.default_rng(11)
    x_prev = np.zeros(lev.N)
    x_prev[blk:] = rng.uniform(-1, 1, blk)
    # scale the three fields so that the three energies and the coupling are of comparable size
    V, U, P = split(x_prev[blk:])
    V *= 1.0 / np.sqrt(V @ (S.Mr @ V))
    U *= 1.0 / np.sqrt(U @ (S.A @ U))
    P *= 1.0 / np.sqrt(P @ (S.Mc @ P))
    coupling = 0.0
    for _ in range(3):
        F = LS.slab_rhs(H, np.zeros(lev.N), x_prev)
        x = lu.solve(F)
        xm = x_prev[blk:]
        xp = cm1[0] * x[:blk] + cm1[1] * x[blk:]
        diss = sum(th[b] * (split(x[b * blk:(b + 1) * blk])[2] @ (S.B @ split(x[b * blk:(b + 1) * blk])[2]))
                   for b in range(2))
        coupling = max(coupling, max(abs(split(x[b * blk:(b + 1) * blk])[0] @ (S.C.T @ split(x[b * blk:(b + 1) * blk])[2]))
                                     * th[b] for b in range(2)))
        E0, E1 = energy(xm), energy(x[blk:])
        defect = E1 - E0 + energy(xp - xm) + diss
        assert diss > 0 and E1 < E0
        assert abs(defect) <= 1e-9 * E0, (defect, E0)
        x_prev = x
    # the identity is a real constraint on the coupling sign: the terms that cancel are 10^5 tolerances large
    assert coupling >= 1e-4


def test_L11_slab_load_is_radau_quadrature_of_sin():
    """L11: L_n = Q_n(<sin(8 pi t) t_N, chi>) (P:L241-251 with the load of P:L757-783): summed over the Radau rows
    it is F times the (k+1)-point Radau value of int_{I_n} sin(8 pi t) dt, and weighted with (t_{n,b} - t_{n-1})
    the first moment; the rule is exact to degree 2k, so both approach the closed forms
    (cos(8 pi t0) - cos(8 pi t1)) / (8 pi) and int (t - t0) sin(8 pi t) dt at relative O(tau^(2k+1)) — halving tau
    gains 2^(2k+1) — and only the chi rows carry load.  Nodes typed from the textbook rule (k = 1: -1/3, 1)."""
    w8 = 8.0 * np.pi
    t0 = 0.013

    def moments(tau):
        t1 = t0 + tau
        m0 = (np.cos(w8 * t0) - np.cos(w8 * t1)) / w8
        # int (t - t0) sin(w t) dt = [-(t - t0) cos(w t) / w + sin(w t) / w^2]
        m1 = -(t1 - t0) * np.cos(w8 * t1) / w8 + (np.sin(w8 * t1) - np.sin(w8 * t0)) / w8 ** 2
        return m0, m1

    errs = []
    for tau in (0.01, 0.005):
        H = LS.LHierarchy(0, 1, 2, 1, tau)
        lev = H.fine
        fN = LS.traction_vector(lev, H.params)
        L = LS.slab_load(H, t0).reshape(2, lev.block)
        chi = L[:, lev.R:2 * lev.R]
        assert np.all(L[:, :lev.R] == 0) and np.all(L[:, 2 * lev.R:] == 0)      # phi and psi rows carry no load
        nodes = t0 + 0.5 * tau * (1.0 + np.array([-1.0 / 3.0, 1.0]))
        m0, m1 = moments(tau)
        s0 = chi.sum(axis=0)
        s1 = ((nodes - t0)[:, None] * chi).sum(axis=0)
        j = int(np.argmax(abs(fN)))
        assert np.allclose(s0 * fN[j], s0[j] * fN, rtol=0, atol=1e-12 * abs(s0[j] * fN[j]))   # parallel to F
        errs.append((abs(s0[j] / fN[j] - m0) / abs(m0), abs(s1[j] / fN[j] - m1) / abs(m1)))
    (e0a, e1a), (e0b, e1b) = errs
    assert e0a <= 2e-4 and e1a <= 2e-3, errs
    assert 5.0 <= e0a / e0b <= 12.0, errs                                        # O(tau^3) for k = 1
