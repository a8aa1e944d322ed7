"""The element-by-element oracle (oracle/ebe.py, used at BASELINE sizes) computes what the assembled-matrix oracle
(oracle/assembly.py, transfer.py, vanka.py, mg.py — pinned in test_oracle_pins*.py) computes: operator, transfers,
patch index sets and multiplicities, one Alg. 1 sweep, the V-cycle, FGMRES iterates and the slab right-hand sides,
on small meshes of every BASELINE family with mixed boundary conditions (CPU, -m "not gpu")."""
import numpy as np
import pytest

from oracle.ebe import EbeHierarchy, ebe_slab_rhs, fgmres_iterations
from oracle.gmres import fgmres
from oracle.mg import Hierarchy
from oracle.vanka import Patches
from stgmg_inputs import config

P2 = dict(rho=1.0, alpha=0.9, c0=0.01, lam=1.0, mu=1.0, K=[0.01, 0, 0, 0.01])
P2b = dict(rho=1.0, alpha=0.9, c0=1e-3, lam=10.0, mu=1.0, K=[1e-3, 0, 0, 1e-3])
P3 = dict(P2, K=[0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01])

CASES = [
    ("2d_q2_dg1", dict(d=2, cells=[8, 4], r=2, k=1, levels=3, p=P2, bc_u=[0, 1, 0, 0], bc_p=[1, 0, 0, 0])),
    ("2d_q3_dg2", dict(d=2, cells=[4, 4], r=3, k=2, levels=2, p=P2b, bc_u=None, bc_p=None)),
    ("3d_q2_dg1", dict(d=3, cells=[4, 2, 2], r=2, k=1, levels=2, p=P3, bc_u=[0, 1, 1, 1, 1, 1],
                       bc_p=[1, 1, 1, 1, 1, 0])),
]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def pair(request):
    c = request.param[1]
    d = c["d"]
    args = (d, c["cells"], [0.0] * d, [1.0] * d, c["r"], c["k"], c["levels"], c["p"], 0.01)
    H = Hierarchy(*args, bc_u=c["bc_u"], bc_p=c["bc_p"])
    E = EbeHierarchy(*args, bc_u=c["bc_u"], bc_p=c["bc_p"])
    return H, E


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_operator_every_level(pair):
    H, E = pair
    rng = np.random.default_rng(0)
    for l in range(len(H.levels)):
        x = rng.standard_normal(H.levels[l].N)
        assert rel(E.ops[l].apply(x), H.A[l] @ x) < 1e-14


def test_transfer(pair):
    H, E = pair
    rng = np.random.default_rng(1)
    for l in range(1, len(H.levels)):
        xc, xf = rng.standard_normal(H.levels[l - 1].N), rng.standard_normal(H.levels[l].N)
        assert rel(E.T[l].prolong(xc), H.P[l] @ xc) < 1e-14
        assert rel(E.T[l].restrict(xf), H.P[l].T @ xf) < 1e-14


def test_patch_sets_and_multiplicities(pair):
    H, E = pair
    for l in range(1, len(H.levels)):
        pa = Patches(H.levels[l])
        sm = E.smoother(l)
        Z = sm.patch_dofs()
        assert len(Z) == len(pa.verts)
        for v, z in zip(pa.verts, pa.dofs):
            assert np.array_equal(Z[tuple(v)], z)
        assert np.array_equal(sm.p, pa.p)
        assert len(sm.classes) == len(pa.classes)


def test_sweep_and_vcycle(pair):
    H, E = pair
    rng = np.random.default_rng(2)
    L = len(H.levels) - 1
    b, d = rng.standard_normal(H.fine.N), 1e-2 * rng.standard_normal(H.fine.N)
    assert rel(E.smoother(L).sweep(b, d), H.smoothers[L].sweep(b, d)) < 1e-12
    assert rel(E.smoother(L).sweep(b, None), H.smoothers[L].sweep(b, 0 * b)) < 1e-12
    assert rel(E.vcycle(b), H.vcycle(b)) < 1e-10


def test_fgmres(pair):
    H, E = pair
    b = np.random.default_rng(3).standard_normal(H.fine.N)
    x1, i1 = fgmres(lambda v: H.A[-1] @ v, b, H.vcycle, tol=1e-8, restart=30)
    x2, i2 = fgmres(E.fine_op.apply, b, E.vcycle, tol=1e-8, restart=30)
    assert i1["iterations"] == i2["iterations"] and i2["converged"]
    assert rel(x2, x1) < 1e-9
    x3, i3 = fgmres_iterations(E, b, 2)
    assert i3["iterations"] == 2


@pytest.mark.parametrize("ci", [1, 3, 4])
def test_slab_rhs_matches_assembled(ci):
    """ebe_slab_rhs (slab 1 and a later slab) = loads.slab_rhs with the assembled spatial matrices, on shrunken
    versions of configs 1 (random load), 3 (manufactured, interpolated initial data) and 4 (beam traction)."""
    from oracle.loads import slab_rhs, manufactured_baseline, load_vectors, traction_face_vector, interpolate_initial
    from stgmg_inputs import uniform_load
    cfg = config(ci)
    d = cfg["dim"]
    cfg["cells"] = (8, 4, 4) if d == 3 else (8, 8, 1)
    cfg["levels"] = 2
    E = EbeHierarchy.from_config(cfg)
    op = E.fine_op
    lev = E.fine
    from oracle.assembly import SlabOperator
    S = SlabOperator(lev, op.params, cfg["tau"]).assemble_spatial()
    n = 2
    t_nodes = n * cfg["tau"] + 0.5 * cfg["tau"] * (op.t_hat + 1.0)
    Xp = np.random.default_rng(4).standard_normal(lev.N)
    o = lev.k * lev.block
    V, U, P = Xp[o:o + lev.R], Xp[o + lev.R:o + 2 * lev.R], Xp[o + 2 * lev.R:o + lev.block]
    if cfg["load"] == "random":
        want = slab_rhs(lev, S, op.chi_m1, op.th, U, V, P, None, None) + uniform_load(lev.N, cfg["seed"])
    elif cfg["load"] == "manufactured":
        sol = manufactured_baseline(d, op.params)
        FG = [load_vectors(lev, sol, t) for t in t_nodes]
        want = slab_rhs(lev, S, op.chi_m1, op.th, U, V, P, [f for f, g in FG], [g for f, g in FG])
        U0, V0, P0 = interpolate_initial(lev, sol, 0.0)
        FG0 = [load_vectors(lev, sol, t) for t in 0.5 * cfg["tau"] * (op.t_hat + 1.0)]
        want0 = slab_rhs(lev, S, op.chi_m1, op.th, U0, V0, P0, [f for f, g in FG0], [g for f, g in FG0])
        assert rel(ebe_slab_rhs(E, cfg, 0), want0) < 1e-13
    else:
        Fl = [traction_face_vector(lev, 1, d - 1, np.sin(np.pi * t / 2)) for t in t_nodes]
        want = slab_rhs(lev, S, op.chi_m1, op.th, U, V, P, Fl, None)
    assert rel(ebe_slab_rhs(E, cfg, n, Xp), want) < 1e-13
