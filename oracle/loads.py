"""Load functionals, slab right-hand side, initial data and manufactured solutions (oracle; test only).

P:L215-228 (Def:LG): F_gamma(chi) = <f, chi> - <t_N, chi>_{G_N^u} + a_gamma(u_D, chi);
                     G_gamma(psi) = <g, psi> - alpha <v_D.n, psi>_{G_D^u} - <p_N, psi>_{G_N^p} + b_gamma(p_D, psi).
All Dirichlet data used here are homogeneous (readings A26, A31), so the a_gamma / b_gamma / v_D terms vanish.
The body load is the exact solution's residual (reading A8): f = rho d_tt u - div(C eps(u)) + alpha grad p,
g = c0 d_t p + alpha div(d_t u) - div(K grad p) (Eq:HPS_1-2), differentiated symbolically (sympy).
Slab RHS, at Radau node b:
  phi-row (V slot): chi_b(-1) M_rho U^{n-1}
  chi-row (U slot): chi_b(-1) M_rho V^{n-1} + theta_b F_gamma(t_{n,b})
  psi-row (P slot): chi_b(-1) M_c  P^{n-1} + theta_b G_gamma(t_{n,b})
Load quadrature: (r+2)^d Gauss points per cell (reading A10).
"""
import numpy as np
import sympy as sy
from .basis import gauss_legendre01, gauss_lobatto_nodes01
from .element import _tensor_eval, _tensor_weights
from .mesh import FIELD_V, FIELD_U, FIELD_P
from .assembly import all_cell_dofs


class Manufactured:
    """Exact solution (u, p) given as sympy expressions in x_0..x_{d-1}, t."""

    def __init__(self, d, u_exprs, p_expr, X, t, params):
        self.d = d
        lam, mu, alpha, rho, c0 = (params[k] for k in ("lam", "mu", "alpha", "rho", "c0"))
        K = np.asarray(params["K"], dtype=np.float64).reshape(d, d)
        u = sy.Matrix(u_exprs)
        p = p_expr
        grad_u = sy.Matrix(d, d, lambda i, j: sy.diff(u[i], X[j]))
        eps = (grad_u + grad_u.T) / 2
        sig = 2 * mu * eps + lam * eps.trace() * sy.eye(d)
        div_sig = [sum(sy.diff(sig[i, j], X[j]) for j in range(d)) for i in range(d)]
        f = [rho * sy.diff(u[i], t, 2) - div_sig[i] + alpha * sy.diff(p, X[i]) for i in range(d)]
        Kgp = [sum(float(K[i, j]) * sy.diff(p, X[j]) for j in range(d)) for i in range(d)]
        g = c0 * sy.diff(p, t) + alpha * sum(sy.diff(sy.diff(u[i], t), X[i]) for i in range(d)) \
            - sum(sy.diff(Kgp[i], X[i]) for i in range(d))
        args = list(X) + [t]
        lam_ = lambda e: sy.lambdify(args, e, "numpy")
        self._u = [lam_(e) for e in u]
        self._v = [lam_(sy.diff(e, t)) for e in u]
        self._p = lam_(p)
        self._gu = [[lam_(grad_u[i, j]) for j in range(d)] for i in range(d)]
        self._f = [lam_(e) for e in f]
        self._g = lam_(g)

    @staticmethod
    def _ev(fn, pts, t):
        val = fn(*[pts[:, a] for a in range(pts.shape[1])], t)
        return np.broadcast_to(np.asarray(val, dtype=np.float64), (pts.shape[0],)).copy()

    def u(self, pts, t):
        return np.stack([self._ev(f, pts, t) for f in self._u], axis=1)

    def v(self, pts, t):
        return np.stack([self._ev(f, pts, t) for f in self._v], axis=1)

    def p(self, pts, t):
        return self._ev(self._p, pts, t)

    def grad_u(self, pts, t):
        return np.stack([np.stack([self._ev(f, pts, t) for f in row], axis=1) for row in self._gu], axis=1)

    def f(self, pts, t):
        return np.stack([self._ev(fn, pts, t) for fn in self._f], axis=1)

    def g(self, pts, t):
        return self._ev(self._g, pts, t)


def sym_vars(d):
    X = sy.symbols("x0:%d" % d, real=True)
    t = sy.Symbol("t", real=True)
    return X, t


def manufactured_baseline(d, params):
    """BASELINE configs 0/1/3: u_i = S sin(2 pi t), p = S cos(2 pi t), S = prod sin(pi x_i)."""
    X, t = sym_vars(d)
    S = sy.Integer(1)
    for a in range(d):
        S = S * sy.sin(sy.pi * X[a])
    return Manufactured(d, [S * sy.sin(2 * sy.pi * t)] * d, S * sy.cos(2 * sy.pi * t), X, t, params)


def manufactured_eq51(params, vector_reading="ones", omega1=sy.pi, omega2=sy.pi):
    """Eq. 5.1: u = phi E_2 (reading A32), p = phi, phi = sin(w1 t^2) sin(w2 x) sin(w2 y)."""
    X, t = sym_vars(2)
    phi = sy.sin(omega1 * t ** 2) * sy.sin(omega2 * X[0]) * sy.sin(omega2 * X[1])
    u = [phi, phi] if vector_reading == "ones" else [sy.Integer(0), phi]
    return Manufactured(2, u, phi, X, t, params)


def manufactured_eq53(params):
    """Eq. 5.3: polynomial in space, w1 = 40 pi, w2 = 10 pi."""
    X, t = sym_vars(2)
    x, y = X
    w1, w2 = 40 * sy.pi, 10 * sy.pi
    a = -2 * (x - 1) ** 2 * x ** 2 * (y - 1) * y * (2 * y - 1)
    b = 2 * (x - 1) * x * (2 * x - 1) * (y - 1) ** 2 * y ** 2
    return Manufactured(2, [a * sy.sin(w1 * t), b * sy.sin(w1 * t)], a * sy.sin(w2 * t), X, t, params)


class CellQuad:
    """Reference basis values at an (nq1)^d Gauss rule and the physical points of every cell."""

    def __init__(self, lev, nq1):
        self.lev = lev
        d, r = lev.d, lev.r
        xg, wg = gauss_legendre01(nq1)
        pts = [xg] * d
        self.phq, self.gq = _tensor_eval(d, gauss_lobatto_nodes01(r), pts, lev.h)
        self.php, self.gp = _tensor_eval(d, gauss_lobatto_nodes01(r - 1), pts, lev.h)
        self.w = _tensor_weights([wg] * d, float(np.prod(lev.h)))
        self.dofs, cells = all_cell_dofs(lev)
        qi = np.array(np.unravel_index(np.arange(nq1 ** d), [nq1] * d, order="F")).T
        ref = xg[qi]                                        # (nq, d)
        self.x = lev.lo[None, None, :] + (cells[:, None, :] + ref[None, :, :]) * lev.h[None, None, :]
        self.nql = (r + 1) ** d
        self.npl = r ** d

    def points(self):
        return self.x.reshape(-1, self.lev.d)


def load_vectors(lev, sol, t, quad=None, rho_scale=False):
    """Spatial load vectors (F_gamma as length-R vector, G_gamma as length-S vector) at time t."""
    quad = quad or CellQuad(lev, lev.r + 2)
    d = lev.d
    nc, nq = quad.x.shape[0], quad.x.shape[1]
    pts = quad.points()
    f = sol.f(pts, t).reshape(nc, nq, d)
    g = sol.g(pts, t).reshape(nc, nq)
    F = np.zeros(lev.R)
    G = np.zeros(lev.S)
    D = quad.dofs
    nql, npl = quad.nql, quad.npl
    qn = D[:, :nql] - lev.offset(0, FIELD_V, 0)
    pn = D[:, 2 * d * nql: 2 * d * nql + npl] - lev.offset(0, FIELD_P)
    for c in range(d):
        np.add.at(F, c * lev.nq + qn, np.einsum("cq,jq,q->cj", f[:, :, c], quad.phq, quad.w))
    np.add.at(G, pn, np.einsum("cq,sq,q->cs", g, quad.php, quad.w))
    return F, G


def traction_face_vector(lev, face, comp, amplitude=1.0):
    """Vector of int_{face} amplitude * chi_comp over the boundary face (2a+s) of the box (length R)."""
    d, r = lev.d, lev.r
    a, s = face // 2, face % 2
    xg, wg = gauss_legendre01(r + 2)
    pts = [xg] * d
    pts[a] = np.array([float(s)])
    wts = [wg] * d
    wts[a] = np.array([1.0])
    phq, _ = _tensor_eval(d, gauss_lobatto_nodes01(r), pts, lev.h)
    w = _tensor_weights(wts, float(np.prod(lev.h)) / lev.h[a])
    loc = phq @ w
    D, cells = all_cell_dofs(lev)
    sel = cells[:, a] == (0 if s == 0 else lev.n[a] - 1)
    qn = D[sel][:, :(r + 1) ** d] - lev.offset(0, FIELD_V, 0)
    F = np.zeros(lev.R)
    np.add.at(F, comp * lev.nq + qn, amplitude * loc[None, :])
    return F


def goal_quantities(lev, X, face):
    """Goal quantities of Eq:DefGQ on a whole box face at t_n (last Radau block of X):
    b_u = int_face u . n do, b_p = int_face p do, with the (r+2)^{d-1} Gauss rule on the face cells."""
    d, r = lev.d, lev.r
    a, s = face // 2, face % 2
    U, V, P = end_state(lev, X)
    nrm = 1.0 if s == 1 else -1.0
    Fu = traction_face_vector(lev, face, a, 1.0)            # int_face chi_a for every Q_r basis function
    bu = nrm * (Fu @ U)
    # pressure: int_face xi_s over the Q_{r-1} basis
    xg, wg = gauss_legendre01(r + 2)
    pts = [xg] * d
    pts[a] = np.array([float(s)])
    wts = [wg] * d
    wts[a] = np.array([1.0])
    php, _ = _tensor_eval(d, gauss_lobatto_nodes01(r - 1), pts, lev.h)
    w = _tensor_weights(wts, float(np.prod(lev.h)) / lev.h[a])
    loc = php @ w
    D, cells = all_cell_dofs(lev)
    sel = cells[:, a] == (0 if s == 0 else lev.n[a] - 1)
    nql, npl = (r + 1) ** d, r ** d
    pn = D[sel][:, 2 * d * nql: 2 * d * nql + npl] - lev.offset(0, FIELD_P)
    Fp = np.zeros(lev.S)
    np.add.at(Fp, pn, loc[None, :])
    bp = Fp @ P
    return bu, bp


def slab_rhs(lev, spatial, chi_m1, th, U_prev, V_prev, P_prev, Floads, Gloads, ds=False, uD_trace=None):
    """Assemble F_n in ABI layout.  Floads[b], Gloads[b]: spatial loads at t_{n,b} (None = 0).
    ds=True (Problem B.1, Eq:DPQ_3): the right-hand side of the pressure equation carries
    <c0 p^{n-1} + alpha div u^{n-1}, psi^+(t_{n-1})> - alpha <u_D(t_{n-1}).n, psi^+(t_{n-1})>_{G_D^u}, i.e. at node b
    chi_b(-1) (M_c P^{n-1} - Cvol U^{n-1}) - chi_b(-1) uD_trace, with Cvol = -alpha <div chi, q> (the volume part of
    C) and uD_trace = alpha <u_D(t_{n-1}).n, xi_s>_{G_D^u} (None = 0: homogeneous Dirichlet data, readings A25/A26).
    The discrete trace u_h^{n-1}.n does NOT enter the right-hand side (it does enter the operator through
    -C(u^+(t_{n-1}), psi^+))."""
    Rv = np.zeros(lev.N)
    MU = spatial["Mrho"] @ U_prev
    MV = spatial["Mrho"] @ V_prev
    MP = spatial["Mc"] @ P_prev
    if ds:
        MP = MP - spatial["Cvol"] @ U_prev
        if uD_trace is not None:
            MP = MP - uD_trace
    for b in range(lev.k + 1):
        o = b * lev.block
        Rv[o: o + lev.R] = chi_m1[b] * MU
        Rv[o + lev.R: o + 2 * lev.R] = chi_m1[b] * MV
        Rv[o + 2 * lev.R: o + lev.block] = chi_m1[b] * MP
        if Floads is not None and Floads[b] is not None:
            Rv[o + lev.R: o + 2 * lev.R] += th[b] * Floads[b]
        if Gloads is not None and Gloads[b] is not None:
            Rv[o + 2 * lev.R: o + lev.block] += th[b] * Gloads[b]
    return Rv


def end_state(lev, X):
    """(U, V, P) at t_n = last Radau node (t_{n,k+1} = t_n)."""
    o = lev.k * lev.block
    return X[o + lev.R: o + 2 * lev.R].copy(), X[o: o + lev.R].copy(), X[o + 2 * lev.R: o + lev.block].copy()


def interpolate_initial(lev, sol, t0):
    """Nodal interpolation (reading A20) of u(t0), v(t0) = d_t u(t0), p(t0)."""
    xq = lev.node_coords(lev.r, gauss_lobatto_nodes01(lev.r))
    xp = lev.node_coords(lev.r - 1, gauss_lobatto_nodes01(lev.r - 1))
    U = sol.u(xq, t0).T.ravel()
    V = sol.v(xq, t0).T.ravel()
    P = sol.p(xp, t0)
    return U, V, P
