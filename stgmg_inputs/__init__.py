"""Workload definitions and seeded input generators shared by the product path, the tests and the oracle.

This module holds NONE of the method's arithmetic: only the BASELINE.json configuration data (mesh, orders,
physical parameters, solver settings) and seeded random draws.  Both ``paper_2303_06742_b200`` and
``oracle`` may import it; they never import each other.

Config data: /root/repo/BASELINE.json "configs" 0..4, with SURVEY.md §8(d) readings A20-A26 for the
unspecified parts (boundary faces of config 4, GMRES restart of config 4, t0 = 0).
Boundary codes: 0 = Dirichlet (Nitsche), 1 = Neumann.  Face order: x-, x+, y-, y+, z-, z+.
"""
import numpy as np

D, N = 0, 1

CONFIGS = {
    0: dict(name="cfg0_2d_q2q1_dg1_4x4", dim=2, cells=(4, 4, 1), lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0),
            levels=2, r=2, k=1, tau=0.01, slabs=1,
            params=dict(rho=1.0, alpha=0.9, c0=0.01, lam=1.0, mu=1.0, K=(0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01)),
            bc_u=(D,) * 6, bc_p=(D,) * 6, restart=30, rtol=1e-10, load="manufactured", seed=None),
    1: dict(name="cfg1_2d_q2q1_dg1_64x64", dim=2, cells=(64, 64, 1), lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0),
            levels=6, r=2, k=1, tau=0.01, slabs=10,
            params=dict(rho=1.0, alpha=0.9, c0=0.01, lam=1.0, mu=1.0, K=(0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01)),
            bc_u=(D,) * 6, bc_p=(D,) * 6, restart=30, rtol=1e-8, load="random", seed=1),
    2: dict(name="cfg2_2d_q3q2_dg2_256x256", dim=2, cells=(256, 256, 1), lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0),
            levels=8, r=3, k=2, tau=0.005, slabs=5,
            params=dict(rho=1.0, alpha=0.9, c0=1e-3, lam=10.0, mu=1.0, K=(1e-3, 0, 0, 0, 1e-3, 0, 0, 0, 1e-3)),
            bc_u=(D,) * 6, bc_p=(D,) * 6, restart=50, rtol=1e-8, load="random", seed=2),
    3: dict(name="cfg3_3d_q2q1_dg1_32cube", dim=3, cells=(32, 32, 32), lo=(0.0, 0.0, 0.0), hi=(1.0, 1.0, 1.0),
            levels=5, r=2, k=1, tau=0.01, slabs=5,
            params=dict(rho=1.0, alpha=0.9, c0=0.01, lam=1.0, mu=1.0, K=(0.01, 0, 0, 0, 0.01, 0, 0, 0, 0.01)),
            bc_u=(D,) * 6, bc_p=(D,) * 6, restart=30, rtol=1e-8, load="manufactured", seed=None),
    4: dict(name="cfg4_3d_beam_256x32x32", dim=3, cells=(256, 32, 32), lo=(0.0, 0.0, 0.0), hi=(8.0, 1.0, 1.0),
            levels=6, r=2, k=1, tau=0.01, slabs=20,
            params=dict(rho=1.0, alpha=0.9, c0=0.01, lam=1.0, mu=1.0, K=(1e-3, 0, 0, 0, 1e-3, 0, 0, 0, 1e-3)),
            bc_u=(D, N, N, N, N, N), bc_p=(N, N, N, N, N, D), restart=30, rtol=1e-8, load="beam", seed=None),
}


def config(i):
    return dict(CONFIGS[i])


def dof_count(cfg, level_from_fine=0):
    """N = (k+1)(2 d n_q + n_p) of a level (layout bookkeeping only, SURVEY §8 'Shared notation')."""
    d, r, k = cfg["dim"], cfg["r"], cfg["k"]
    n = [c // (2 ** level_from_fine) for c in cfg["cells"][:d]]
    nq = int(np.prod([r * c + 1 for c in n]))
    npp = int(np.prod([(r - 1) * c + 1 for c in n]))
    return (k + 1) * (2 * d * nq + npp)


def uniform_load(n, seed):
    """i.i.d. U[-1, 1) vector of length n from numpy's default_rng(seed) (reading A21)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def random_vector(n, seed, scale=1.0):
    """Generic seeded test vector (parity inputs)."""
    return scale * np.random.default_rng(seed).standard_normal(n)
