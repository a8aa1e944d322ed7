"""Space-time error norms and the slab-marching driver used by the Tab:3 / Tab:App1 pins (oracle; test only).

Norms (P:L552-556 Eq:DiscNorm, P:L673-677 Eq:MDN, reading A30):
  L2(L2):   sum over slabs of a Gauss rule in time (nt points) x (r+2)^d Gauss in space
  Linf(L2): max over the M = 100 Gauss–Legendre nodes of every slab
  linf(L2): max over the slab end points t_n
Errors are || grad(u - u_h) ||, || v - v_h ||, || p - p_h ||.
Each slab is solved by a sparse direct solve (reading A28: the printed errors need a much tighter solve than
the paper's 1e-8 GMRES tolerance).
"""
import numpy as np
import scipy.sparse.linalg as spla
from .basis import gauss_legendre, lagrange_values
from .mesh import FIELD_V, FIELD_P
from .loads import CellQuad, load_vectors, slab_rhs, end_state, interpolate_initial
from .assembly import SlabOperator


def _field_errors(lev, quad, sol, U, V, P, t):
    """Squared spatial L2 errors (grad u, v, p) at time t for nodal vectors U, V (length R), P (length S)."""
    d = lev.d
    nc, nq = quad.x.shape[0], quad.x.shape[1]
    D = quad.dofs
    nql, npl = quad.nql, quad.npl
    qn = D[:, :nql] - lev.offset(0, FIELD_V, 0)
    pn = D[:, 2 * d * nql: 2 * d * nql + npl] - lev.offset(0, FIELD_P)
    pts = quad.points()
    gu_ex = sol.grad_u(pts, t).reshape(nc, nq, d, d)
    v_ex = sol.v(pts, t).reshape(nc, nq, d)
    p_ex = sol.p(pts, t).reshape(nc, nq)
    e_gu = 0.0
    e_v = 0.0
    for c in range(d):
        Uc = U[c * lev.nq + qn]                                    # (nc, nql)
        Vc = V[c * lev.nq + qn]
        gh = np.einsum("cj,jqb->cqb", Uc, quad.gq)
        e_gu += np.einsum("cqb,q->", (gh - gu_ex[:, :, c, :]) ** 2, quad.w)
        vh = Vc @ quad.phq
        e_v += np.einsum("cq,q->", (vh - v_ex[:, :, c]) ** 2, quad.w)
    ph = P[pn] @ quad.php
    e_p = np.einsum("cq,q->", (ph - p_ex) ** 2, quad.w)
    return np.array([e_gu, e_v, e_p])


def march_errors(lev, params, sol, t0, T_end, n_slabs, nt=None, linf_M=0, ds=False):
    """March n_slabs slabs of length (T_end - t0)/n_slabs with direct solves; return the error norms.

    Returns dict with 'L2' (3,), 'linf_tn' (3,), and 'Linf' (3,) if linf_M > 0."""
    tau = (T_end - t0) / n_slabs
    op = SlabOperator(lev, params, tau, ds)
    A = op.assemble().tocsc()
    lu = spla.splu(A)
    spatial = op.assemble_spatial()
    quad = CellQuad(lev, lev.r + 2)
    k = lev.k
    nt = nt or (k + 4)
    tg, wg = gauss_legendre(nt)
    Lg = lagrange_values(op.t_hat, tg)                     # (k+1, nt)
    if linf_M:
        tm, _ = gauss_legendre(linf_M)
        Lm = lagrange_values(op.t_hat, tm)
    U, V, P = interpolate_initial(lev, sol, t0)
    L2 = np.zeros(3)
    linf_tn = np.zeros(3)
    Linf = np.zeros(3)
    for n in range(1, n_slabs + 1):
        ta = t0 + (n - 1) * tau
        t_nodes = ta + 0.5 * tau * (op.t_hat + 1.0)
        Fl, Gl = [], []
        for b in range(k + 1):
            F, G = load_vectors(lev, sol, t_nodes[b], quad)
            Fl.append(F)
            Gl.append(G)
        rhs = slab_rhs(lev, spatial, op.chi_m1, op.th, U, V, P, Fl, Gl, ds)
        X = lu.solve(rhs)
        blocks = [(X[m * lev.block + lev.R: m * lev.block + 2 * lev.R],
                   X[m * lev.block: m * lev.block + lev.R],
                   X[m * lev.block + 2 * lev.R: (m + 1) * lev.block]) for m in range(k + 1)]

        def at(Lcol):
            Ut = sum(Lcol[m] * blocks[m][0] for m in range(k + 1))
            Vt = sum(Lcol[m] * blocks[m][1] for m in range(k + 1))
            Pt = sum(Lcol[m] * blocks[m][2] for m in range(k + 1))
            return Ut, Vt, Pt

        for q in range(nt):
            tq = ta + 0.5 * tau * (tg[q] + 1.0)
            L2 += 0.5 * tau * wg[q] * _field_errors(lev, quad, sol, *at(Lg[:, q]), tq)
        U, V, P = end_state(lev, X)
        e_end = _field_errors(lev, quad, sol, U, V, P, ta + tau)
        linf_tn = np.maximum(linf_tn, np.sqrt(e_end))
        if linf_M:
            for q in range(linf_M):
                tq = ta + 0.5 * tau * (tm[q] + 1.0)
                Linf = np.maximum(Linf, np.sqrt(_field_errors(lev, quad, sol, *at(Lm[:, q]), tq)))
    out = {"L2": np.sqrt(L2), "linf_tn": linf_tn}
    if linf_M:
        out["Linf"] = Linf
    return out
