"""Element matrices of the spatial forms by tensor Gauss quadrature (oracle; test infrastructure only).

Forms (Def:ACB and Def:ab), Taylor–Hood option Q_h = Q_h^{l,cont}:
  A_gamma(w, chi) = <C eps(w), eps(chi)> - <C eps(w) n, chi>_{G_D^u} - <w, C eps(chi) n>_{G_D^u}
                    + gamma_a/h_F <w, chi>_{G_D^u}
  C(chi, q)       = -alpha <div chi, q> + alpha <chi . n, q>_{G_D^u}
  B_gamma(q, psi) = <K grad q, grad psi> - <K grad q . n, psi>_{G_D^p} - <q, K grad psi . n>_{G_D^p}
                    + gamma_b/h_F <q, psi>_{G_D^p}
with isotropic C: C eps = lambda tr(eps) E + 2 mu eps, h_F = |K|_d on boundary faces (P:L205,
reading A6), gamma_a = 5e4 r(r+1), gamma_b = r(r-1)/2 (reading A7).
Masses: M_rho = rho <psi_j, psi_i>, M_c = c0 <xi_s, xi_r>.

Plain evaluation: every basis function's value and gradient is formed at every quadrature point and the
integrands are summed point by point (no sum factorisation).  Quadrature (r+1)^d Gauss points in the cell,
(r+1)^{d-1} on faces (reading A10) — exact for all these polynomial integrands on axis-aligned cells.
Matrix convention: M[test, trial].
"""
import numpy as np
from .basis import gauss_legendre01, gauss_lobatto_nodes01, lagrange_values, lagrange_derivs


def default_gammas(r):
    return 5.0e4 * r * (r + 1), 0.5 * r * (r - 1)


def _tensor_eval(d, nodes01, pts_per_axis, h):
    """phi[j, q] and grad[j, q, b] of the tensor Lagrange basis at a tensor point set.

    pts_per_axis[a] = 1D reference points on [0,1] for axis a; local node / point multi-indices are
    lexicographic with axis 0 fastest."""
    n1 = len(nodes01)
    V = [lagrange_values(nodes01, p) for p in pts_per_axis]
    D = [lagrange_derivs(nodes01, p) for p in pts_per_axis]
    node_idx = np.array(np.unravel_index(np.arange(n1 ** d), [n1] * d, order="F")).T      # (nb, d)
    npts = [len(p) for p in pts_per_axis]
    q_idx = np.array(np.unravel_index(np.arange(int(np.prod(npts))), npts, order="F")).T  # (nq, d)
    nb, nq = node_idx.shape[0], q_idx.shape[0]
    phi = np.ones((nb, nq))
    grad = np.ones((nb, nq, d))
    for a in range(d):
        va = V[a][node_idx[:, a]][:, q_idx[:, a]]
        da = D[a][node_idx[:, a]][:, q_idx[:, a]] / h[a]
        phi *= va
        for b in range(d):
            grad[:, :, b] *= da if b == a else va
    return phi, grad


def _tensor_weights(wts_per_axis, scale):
    w = np.ones(1)
    for wa in wts_per_axis:          # axis 0 fastest
        w = np.kron(wa, w)
    return w * scale


class ElementForms:
    """Spatial element matrices for one cell size h and a given set of Dirichlet faces."""

    def __init__(self, d, r, h, params):
        self.d, self.r = d, r
        self.h = np.asarray(h, dtype=np.float64)
        self.p = params
        self.nodes_q = gauss_lobatto_nodes01(r)
        self.nodes_p = gauss_lobatto_nodes01(r - 1)
        self.xg, self.wg = gauss_legendre01(r + 1)
        self.vol = float(np.prod(self.h))

    # volume quadrature -------------------------------------------------------------------------
    def _volume(self):
        d = self.d
        pts = [self.xg] * d
        phq, gq = _tensor_eval(d, self.nodes_q, pts, self.h)
        php, gp = _tensor_eval(d, self.nodes_p, pts, self.h)
        w = _tensor_weights([self.wg] * d, self.vol)
        return phq, gq, php, gp, w

    def _face(self, face):
        d = self.d
        a, s = face // 2, face % 2
        pts = [self.xg] * d
        pts[a] = np.array([float(s)])
        wts = [self.wg] * d
        wts[a] = np.array([1.0])
        area = self.vol / self.h[a]
        phq, gq = _tensor_eval(d, self.nodes_q, pts, self.h)
        php, gp = _tensor_eval(d, self.nodes_p, pts, self.h)
        w = _tensor_weights(wts, area)
        n = np.zeros(d)
        n[a] = -1.0 if s == 0 else 1.0
        return phq, gq, php, gp, w, n

    def hF(self, face):
        if self.p.get("hF_fixed") is not None:
            return float(self.p["hF_fixed"])  # frozen h_F (Galerkin-identity pin P8 only)
        mode = self.p.get("hF_mode", 0)
        if mode == 0:
            return self.vol                 # |K|_d, P:L205 (reading A6)
        return float(self.h[face // 2])     # edge reading (flag)

    # vector basis helpers -------------------------------------------------------------------------
    def _vec_grad(self, gq):
        """G[I, q, i, j] = d_j (psi_I)_i for psi_I = phi_J e_c, I = c*nb + J (component-major)."""
        nb, nq, d = gq.shape
        G = np.zeros((d * nb, nq, d, d))
        for c in range(d):
            G[c * nb:(c + 1) * nb, :, c, :] = gq
        return G

    def _vec_val(self, phq):
        nb, nq = phq.shape
        d = self.d
        Vv = np.zeros((d * nb, nq, d))
        for c in range(d):
            Vv[c * nb:(c + 1) * nb, :, c] = phq
        return Vv

    def _stress(self, G):
        lam, mu = self.p["lam"], self.p["mu"]
        eps = 0.5 * (G + np.swapaxes(G, 2, 3))
        tr = np.trace(eps, axis1=2, axis2=3)
        sig = 2.0 * mu * eps
        for i in range(self.d):
            sig[:, :, i, i] += lam * tr
        return eps, sig

    # matrices -------------------------------------------------------------------------------------
    def matrices(self, dir_u_faces=(), dir_p_faces=()):
        """Return dict with Mq (scalar Q_r mass), Mrho (vector, rho), Mc (c0 Q_{r-1} mass), A, C, B."""
        p = self.p
        d = self.d
        phq, gq, php, gp, w = self._volume()
        Mq = np.einsum("iq,jq,q->ij", phq, phq, w)
        Mp = np.einsum("iq,jq,q->ij", php, php, w)
        G = self._vec_grad(gq)
        eps, sig = self._stress(G)
        A = np.einsum("Jqab,Iqab,q->IJ", sig, eps, w)
        div = np.trace(G, axis1=2, axis2=3)                    # (nv, nq)
        C = -p["alpha"] * np.einsum("Jq,sq,q->sJ", div, php, w)
        Cvol = C.copy()                                       # volume part -alpha <div chi, q> only
        K = np.asarray(p["K"], dtype=np.float64).reshape(d, d)
        Kg = np.einsum("ab,sqb->sqa", K, gp)
        B = np.einsum("sqa,rqa,q->rs", Kg, gp, w)
        ga, gb = p["gamma_a"], p["gamma_b"]
        for f in dir_u_faces:
            fphq, fgq, fphp, fgp, fw, n = self._face(f)
            Gf = self._vec_grad(fgq)
            Vf = self._vec_val(fphq)
            _, sigf = self._stress(Gf)
            sn = np.einsum("Iqab,b->Iqa", sigf, n)              # sigma(psi_I) n
            pen = ga / self.hF(f)
            A += (-np.einsum("Jqa,Iqa,q->IJ", sn, Vf, fw)       # -<sigma(w) n, chi>
                  - np.einsum("Jqa,Iqa,q->IJ", Vf, sn, fw)      # -<w, sigma(chi) n>
                  + pen * np.einsum("Jqa,Iqa,q->IJ", Vf, Vf, fw))
            vn = np.einsum("Jqa,a->Jq", Vf, n)
            C += p["alpha"] * np.einsum("Jq,sq,q->sJ", vn, fphp, fw)
        for f in dir_p_faces:
            fphq, fgq, fphp, fgp, fw, n = self._face(f)
            Kgn = np.einsum("ab,sqb,a->sq", K, fgp, n)          # K grad xi_s . n
            pen = gb / self.hF(f)
            B += (-np.einsum("sq,rq,q->rs", Kgn, fphp, fw)
                  - np.einsum("sq,rq,q->rs", fphp, Kgn, fw)
                  + pen * np.einsum("sq,rq,q->rs", fphp, fphp, fw))
        Mrho = p["rho"] * np.kron(np.eye(d), Mq)
        Mc = p["c0"] * Mp
        return {"Mq": Mq, "Mp": Mp, "Mrho": Mrho, "Mc": Mc, "A": A, "C": C, "B": B, "Cvol": Cvol}


def slab_element_matrix(mats, T, th, ds=False):
    """Element slab matrix in element DoF order (m, f in (V,U,P), c, node), P:L233-256 (Eq:DPQ_A0).

    Rows are the test slots (phi, chi, psi) at node b aligned with the columns (V, U, P) at node a
    (reading A5):
      [phi_b, V_a] = -theta_b d_ab M_rho   [phi_b, U_a] = T_ba M_rho
      [chi_b, V_a] = T_ba M_rho            [chi_b, U_a] = theta_b d_ab A   [chi_b, P_a] = theta_b d_ab C^T
      [psi_b, V_a] = -theta_b d_ab C       [psi_b, P_a] = T_ba M_c + theta_b d_ab B
    ds=True: Problem B.1 (DS): the pressure equation keeps d_t u instead of v,
    -Q_n(C(d_t u, psi)) - C(u^+(t_{n-1}), psi^+) = -sum_a T_ba C U_a, i.e. [psi_b, U_a] = -T_ba C, [psi_b, V_a] = 0.
    """
    Mr, Mc, A, C, B = mats["Mrho"], mats["Mc"], mats["A"], mats["C"], mats["B"]
    nv, ns = Mr.shape[0], Mc.shape[0]
    nb = 2 * nv + ns
    k1 = T.shape[0]
    E = np.zeros((k1 * nb, k1 * nb))
    sV, sU, sP = slice(0, nv), slice(nv, 2 * nv), slice(2 * nv, nb)
    for b in range(k1):
        for a in range(k1):
            blk = np.zeros((nb, nb))
            blk[sV, sU] = T[b, a] * Mr
            blk[sU, sV] = T[b, a] * Mr
            blk[sP, sP] = T[b, a] * Mc
            if ds:
                blk[sP, sU] = -T[b, a] * C
            if a == b:
                blk[sV, sV] = -th[b] * Mr
                blk[sU, sU] = th[b] * A
                blk[sU, sP] = th[b] * C.T
                if not ds:
                    blk[sP, sV] = -th[b] * C
                blk[sP, sP] += th[b] * B
            E[b * nb:(b + 1) * nb, a * nb:(a + 1) * nb] = blk
    return E
