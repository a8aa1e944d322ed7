"""3D L-shaped benchmark of Sec. 5.2 with the Q_r^d / P_{r-1}^disc pair (oracle, test
infrastructure only).

Passages followed:
  P:L130-148 (Def:VhQh)   Q_r^d for u, v (continuous), P_{r-1}^disc for p (discontinuous, "broken polynomial space").
  P:L177-212 (Def:ACB, Def:ab)  A_gamma, C as for Taylor-Hood; B_gamma = the SIP option (second case of Def:B):
      sum_K <K grad q, grad psi>_K - sum_F (<{K grad q}.n, [psi]>_F + <[q], {K grad psi}.n>_F)
      + sum_F gamma/h_F <[q], [psi]>_F,   {w} = (w+ + w-)/2, [w] = w+ - w-, h_F = (|K+|_d + |K-|_d)/2,
      boundary faces: {w} = [w] = w|_K, h_F = |K|_d; gamma = gamma_b = r(r-1)/2.
  P:L757-781 (Eq:BCd)  directional condition u.n = 0, (sigma(u) n).t_i = 0 on Gamma^d_u, implemented by
      a^d_gamma(w, chi) = -<w.n, C eps(chi) n.n> + gamma_a h^-1 <w.n, chi.n> and the consistency term
      -<C eps(u) n.n, n.chi> in place of -<C eps(u) n, chi> of Def:A.
  P:L782-790  traction t_N = (0, 5e9 (32xz - 18x - 16z + 10) sin(8 pi t), 0) on Gamma^N_u = (0,.5) x {1} x (0,.5);
      p = 0 on Gamma^D_p = [0,.5] x {1} x [0,.5], no flux elsewhere; rho = 1, alpha = 0.9, c0 = 0.01, K = E_3,
      E = 20000, nu = 0.3, T = 4 (exact Lame conversion, reading A33).
  P:L805-810 (Eq:DefGQ)  b_u = int_{Gamma_m} u.n, b_p = int_{Gamma_m} p, Gamma_m = {1} x (0,.5) x (0,.5).
  P:L838-856 (tab:3d_L_results)  DoF counts per slab; ref_n = n uniform refinements of the 3-cell initial grid.
  P:L894  ref_5 has 98,304 cells.

Readings (N3-R1 .. N3-R7):
  R1 geometry: Omega = ([0,1] x [0,.5] U [0,.5] x [.5,1]) x [0,.5], three cubes of side 0.5; ref_n has 2^n cells per
     cube edge (the DoF counts of Table 4 and the 98,304 cells of ref_5 follow).
  R2 boundary parts of u (the figure is not in PAPER.md): y = 0 Dirichlet (u = 0); x = 0 and z = 0, z = 0.5
     directional; y = 1 (x < .5) traction t_N; x = 1 (Gamma_m) and the re-entrant faces x = .5 (y > .5), y = .5
     (x > .5) traction free.
  R3 the boundary faces in the SIP sums of B_gamma are the Dirichlet faces of p (F_h^{D,p}); Def:LG's disc option
     names F_h^{D,p} and F_h^{N,p} separately and only the former carries data of a Dirichlet term.
  R4 h in a^d_gamma and in the SIP penalty = h_F (cell measure, reading A6), as in a_gamma.
  R5 the C face term alpha <chi.n, q> of Def:C also acts on the directional faces (consistency of
     -div(sigma - alpha p E) tested with chi, whose normal component is constrained there).
  R6 P_{r-1}^disc basis: monomials xi^a, |a| <= r-1, of the cell coordinates xi = 2 x_hat - 1 in [-1,1]^3, ordered by
     total degree, then x before y before z (the basis changes vectors, not the discrete functions).
  R7 Table 4's caption gives (k+1) 2013 DoFs for ref_1; the counting of every other printed row gives (k+1) 2046 there
     (6 * 325 Q2 nodes + 4 * 24 cells); the printed rows are pinned, the caption value is not.
"""
import itertools

import numpy as np
import scipy.sparse as sp

from .basis import gauss_legendre01, gauss_lobatto_nodes01
from .element import ElementForms, _tensor_eval, _tensor_weights, default_gammas
from .temporal import temporal_constants
from .transfer import interp_1d
from .vanka import VankaSmoother, equilibrated_inverse

U_DIRICHLET, U_DIRECTIONAL, U_NEUMANN, U_TRACTION = 0, 1, 2, 3
P_DIRICHLET, P_NEUMANN = 0, 1
TRACTION_AMP = 5.0e9


def lshape_params(r, E=20000.0, nu=0.3):
    """Sec. 5.2 parameters: exact Lame conversion (reading A33), gammas of P:L209-211."""
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    ga, gb = default_gammas(r)
    return dict(rho=1.0, alpha=0.9, c0=0.01, lam=lam, mu=mu, K=[1.0, 0, 0, 0, 1.0, 0, 0, 0, 1.0],
                gamma_a=ga, gamma_b=gb, hF_mode=0)


def p_exponents(deg, d=3):
    """Exponents of the P_deg monomial basis (reading R6): total degree first, then x before y before z."""
    ex = [a for a in itertools.product(range(deg + 1), repeat=d) if sum(a) <= deg]
    return sorted(ex, key=lambda a: (sum(a), tuple(reversed(a))))


def p_eval(exps, pts_axes, h):
    """Values phi[s, q] and gradients grad[s, q, b] of the monomials xi^a at the tensor point set pts_axes (reference
    coordinates x_hat in [0,1], axis 0 fastest), xi = 2 x_hat - 1, d/dx = (2/h) d/dxi."""
    d = len(pts_axes)
    npts = [len(p) for p in pts_axes]
    qi = np.array(np.unravel_index(np.arange(int(np.prod(npts))), npts, order="F")).T
    xi = np.stack([2.0 * np.asarray(pts_axes[a])[qi[:, a]] - 1.0 for a in range(d)], axis=1)   # (nq, d)
    phi = np.zeros((len(exps), xi.shape[0]))
    grad = np.zeros((len(exps), xi.shape[0], d))
    for s, a in enumerate(exps):
        phi[s] = np.prod([xi[:, b] ** a[b] for b in range(d)], axis=0)
        for b in range(d):
            if a[b] == 0:
                continue
            g = a[b] * xi[:, b] ** (a[b] - 1) * (2.0 / h[b])
            for c in range(d):
                if c != b:
                    g = g * xi[:, c] ** a[c]
            grad[s, :, b] = g
    return phi, grad


class LLevel:
    """Level ref_n of the L-shaped domain (reading R1): structured (2N, 2N, N) cell grid of [0,1] x [0,1] x [0,.5],
    N = 2^ref, cells (i, j, l) active unless i >= N and j >= N.  Active cells and Q_r nodes are numbered
    lexicographically (x fastest) over the structured grid.  Slab layout (Eq:DefXn): per Radau node
    m: V_0..V_2 (nq each), U_0..U_2, P (npc per active cell, cells in order)."""

    def __init__(self, ref, r, k):
        self.ref, self.r, self.k, self.d = int(ref), int(r), int(k), 3
        N = 2 ** self.ref
        self.Ncube = N
        self.h = np.full(3, 0.5 / N)
        self.n = (2 * N, 2 * N, N)
        act = np.ones(self.n, dtype=bool)
        act[N:, N:, :] = False
        self.active = act
        cl = np.array(np.unravel_index(np.arange(int(np.prod(self.n))), self.n, order="F")).T
        cl = cl[act[cl[:, 0], cl[:, 1], cl[:, 2]]]
        self.cells = cl                                           # (ncell, 3) lexicographic
        self.n_cells = len(cl)
        self.cell_id = -np.ones(self.n, dtype=np.int64)
        self.cell_id[cl[:, 0], cl[:, 1], cl[:, 2]] = np.arange(self.n_cells)
        self.q_shape = tuple(r * n + 1 for n in self.n)
        loc = np.array(np.unravel_index(np.arange((r + 1) ** 3), [r + 1] * 3, order="F")).T
        self.q_loc = loc
        qact = np.zeros(self.q_shape, dtype=bool)
        for c in cl:
            qact[r * c[0]:r * c[0] + r + 1, r * c[1]:r * c[1] + r + 1, r * c[2]:r * c[2] + r + 1] = True
        flat = qact.ravel(order="F")
        self.qmap = -np.ones(flat.size, dtype=np.int64)
        self.qmap[flat] = np.arange(int(flat.sum()))
        self.qmap = self.qmap.reshape(self.q_shape, order="F")
        self.nq = int(flat.sum())
        self.exps = p_exponents(r - 1)
        self.npc = len(self.exps)
        self.np_ = self.npc * self.n_cells
        self.R = 3 * self.nq
        self.S = self.np_
        self.block = 2 * self.R + self.S
        self.N = (self.k + 1) * self.block
        q = r * cl[:, None, :] + loc[None, :, :]
        self.cell_q = self.qmap[q[..., 0], q[..., 1], q[..., 2]]   # (ncell, (r+1)^3) compact Q nodes
        assert np.all(self.cell_q >= 0)

    def offset(self, m, f, c=0):
        base = m * self.block
        if f == 0:
            return base + c * self.nq
        if f == 1:
            return base + self.R + c * self.nq
        return base + 2 * self.R

    def cell_p(self, cid):
        return np.arange(cid * self.npc, (cid + 1) * self.npc)

    def u_bc(self, c, f):
        """Boundary part of u on face f = 2a + s of active cell c (reading R2); the caller checks that f is a
        boundary face."""
        a, s = f // 2, f % 2
        if a == 1 and s == 0:
            return U_DIRICHLET                      # y = 0
        if a == 0 and s == 0:
            return U_DIRECTIONAL                    # x = 0
        if a == 2:
            return U_DIRECTIONAL                    # z = 0, z = 0.5
        if a == 1 and s == 1 and c[1] == self.n[1] - 1:
            return U_TRACTION                       # y = 1, x < 0.5
        return U_NEUMANN                            # x = 1 (Gamma_m), re-entrant faces

    def p_bc(self, c, f):
        a, s = f // 2, f % 2
        return P_DIRICHLET if (a == 1 and s == 1 and c[1] == self.n[1] - 1) else P_NEUMANN

    def neighbour(self, c, f):
        a, s = f // 2, f % 2
        nb = np.array(c)
        nb[a] += 1 if s else -1
        if nb[a] < 0 or nb[a] >= self.n[a]:
            return -1
        return int(self.cell_id[nb[0], nb[1], nb[2]])


class LForms:
    """Element-local matrices on a cube of side h (all cells of a level are congruent).  Vector Q_r index
    I = c (r+1)^3 + J (component-major), P index s (monomial order, reading R6).  M[test, trial]."""

    def __init__(self, r, h, params):
        self.r, self.d = r, 3
        self.h = np.asarray(h, dtype=np.float64)
        self.p = params
        self.ef = ElementForms(3, r, self.h, params)      # tensor Q_r tables, vector helpers, stress
        self.exps = p_exponents(r - 1)
        self.vol = float(np.prod(self.h))
        # |K|_d, also the SIP average on a uniform mesh (R4); hF_fixed: frozen h_F (Galerkin-identity pin only)
        if params.get("hF_fixed") is not None:
            self.hF = float(params["hF_fixed"])
        else:   # |K|_d (reading A6), or the edge length with hF_mode = 1 (the flag of the structured path)
            self.hF = float(self.h[0]) if params.get("hF_mode", 0) == 1 else self.vol
        # penalty length of the directional faces: h_F (reading R4), or the literal h of a^d_gamma (hF_mode = 2)
        self.hD = float(self.h[0]) if params.get("hF_mode", 0) in (1, 2) else self.hF
        # penalty length of the SIP faces of B_gamma: h_F as the u faces, except for the experiment modes of DESIGN.md
        # §7.6 (4: h^3 for u, h for p; 5: h for u, h^3 for p; 6: the face measure h^2 for both)
        self.hP = self.hF
        mode, hh = params.get("hF_mode", 0), float(self.h[0])
        if params.get("hF_fixed") is None and mode in (4, 5, 6):
            self.hF = self.hD = {4: self.vol, 5: hh, 6: hh * hh}[mode]
            self.hP = {4: hh, 5: self.vol, 6: hh * hh}[mode]
        self.K = np.asarray(params["K"], dtype=np.float64).reshape(3, 3)

    def _pts(self, face=None):
        xg, wg = self.ef.xg, self.ef.wg
        pts, wts = [xg] * 3, [wg] * 3
        scale = self.vol
        n = None
        if face is not None:
            a, s = face // 2, face % 2
            pts = list(pts)
            wts = list(wts)
            pts[a] = np.array([float(s)])
            wts[a] = np.array([1.0])
            scale = self.vol / self.h[a]
            n = np.zeros(3)
            n[a] = 1.0 if s else -1.0
        phq, gq = _tensor_eval(3, self.ef.nodes_q, pts, self.h)
        php, gp = p_eval(self.exps, pts, self.h)
        return phq, gq, php, gp, _tensor_weights(wts, scale), n

    def volume(self):
        p = self.p
        phq, gq, php, gp, w, _ = self._pts()
        Mq = np.einsum("iq,jq,q->ij", phq, phq, w)
        G = self.ef._vec_grad(gq)
        eps, sig = self.ef._stress(G)
        A = np.einsum("Jqab,Iqab,q->IJ", sig, eps, w)
        div = np.trace(G, axis1=2, axis2=3)
        C = -p["alpha"] * np.einsum("Jq,sq,q->sJ", div, php, w)
        Kg = np.einsum("ab,sqb->sqa", self.K, gp)
        B = np.einsum("sqa,rqa,q->rs", Kg, gp, w)
        Mp = np.einsum("iq,jq,q->ij", php, php, w)
        return dict(Mq=Mq, Mrho=p["rho"] * np.kron(np.eye(3), Mq), Mc=p["c0"] * Mp, Mp=Mp, A=A, C=C, B=B)

    def face_u(self, f, kind):
        """(A_face, C_face) of a Dirichlet (Def:A, Def:agam) or directional (a^d_gamma, Eq:BCd) face f."""
        phq, gq, php, _, w, n = self._pts(f)
        Gf = self.ef._vec_grad(gq)
        Vf = self.ef._vec_val(phq)
        _, sig = self.ef._stress(Gf)
        sn = np.einsum("Iqab,b->Iqa", sig, n)               # sigma(psi_I) n
        pen = self.p["gamma_a"] / (self.hF if kind == U_DIRICHLET else self.hD)
        vn = np.einsum("Jqa,a->Jq", Vf, n)                    # psi_J . n
        if kind == U_DIRICHLET:
            A = (-np.einsum("Jqa,Iqa,q->IJ", sn, Vf, w) - np.einsum("Jqa,Iqa,q->IJ", Vf, sn, w)
                 + pen * np.einsum("Jqa,Iqa,q->IJ", Vf, Vf, w))
        else:
            snn = np.einsum("Jqa,a->Jq", sn, n)              # sigma(psi_J) n . n
            A = (-np.einsum("Jq,Iq,q->IJ", snn, vn, w) - np.einsum("Jq,Iq,q->IJ", vn, snn, w)
                 + pen * np.einsum("Jq,Iq,q->IJ", vn, vn, w))
        C = self.p["alpha"] * np.einsum("Jq,sq,q->sJ", vn, php, w)
        return A, C

    def face_p_dirichlet(self, f):
        """SIP boundary face (reading R3): -<K grad q.n, psi> - <q, K grad psi.n> + gamma/h_F <q, psi>."""
        _, _, php, gp, w, n = self._pts(f)
        Kgn = np.einsum("ab,sqb,a->sq", self.K, gp, n)
        pen = self.p["gamma_b"] / self.hP
        return (-np.einsum("sq,rq,q->rs", Kgn, php, w) - np.einsum("sq,rq,q->rs", php, Kgn, w)
                + pen * np.einsum("sq,rq,q->rs", php, php, w))

    def face_p_interior(self, a):
        """SIP interior face normal to axis a between K- (lower) and K+ = K- + e_a.  With n = e_a (outward of K-) and
        [w] = w- - w+ (the product of normal and jump is the same as with P:L201's convention).  Returns the 2x2
        blocks Bf[i][j] (test side i, trial side j; 0 = K-, 1 = K+)."""
        pm = self._pts(2 * a + 1)    # K-'s face x_a = 1
        pp = self._pts(2 * a)        # K+'s face x_a = 0 (same physical points, same order)
        w = pm[4]
        n = np.zeros(3)
        n[a] = 1.0
        ph = [pm[2], pp[2]]
        kgn = [np.einsum("ab,sqb,a->sq", self.K, pm[3], n), np.einsum("ab,sqb,a->sq", self.K, pp[3], n)]
        sg = [1.0, -1.0]
        pen = self.p["gamma_b"] / self.hP
        Bf = [[None, None], [None, None]]
        for i in range(2):
            for j in range(2):
                Bf[i][j] = (-0.5 * sg[i] * np.einsum("sq,rq,q->rs", kgn[j], ph[i], w)
                            - 0.5 * sg[j] * np.einsum("sq,rq,q->rs", ph[j], kgn[i], w)
                            + pen * sg[i] * sg[j] * np.einsum("sq,rq,q->rs", ph[j], ph[i], w))
        return Bf


class LSpatial:
    """Assembled spatial matrices of one level: Mrho, Mc (masses), A (A_gamma), C, B (SIP B_gamma) — plain COO
    summation over cells and faces (library primitive scipy.sparse)."""

    def __init__(self, lev, params):
        self.lev = lev
        self.p = params
        F = LForms(lev.r, lev.h, params)
        self.forms = F
        vol = F.volume()
        nq, npc, nc = lev.nq, lev.npc, lev.n_cells
        nbq = (lev.r + 1) ** 3
        vdofs = np.concatenate([c * nq + lev.cell_q for c in range(3)], axis=1)     # (nc, 3 nbq)
        pdofs = np.arange(nc * npc).reshape(nc, npc)
        trip = {k: ([], [], []) for k in ("Mr", "Mc", "A", "C", "B")}

        def add(key, rows, cols, M):
            trip[key][0].append(np.repeat(rows, len(cols)))
            trip[key][1].append(np.tile(cols, len(rows)))
            trip[key][2].append(M.ravel())

        face_u = {}
        face_pd = {}
        face_pi = {a: F.face_p_interior(a) for a in range(3)}
        for cid in range(nc):
            c = lev.cells[cid]
            vd, pd = vdofs[cid], pdofs[cid]
            add("Mr", vd, vd, vol["Mrho"])
            add("Mc", pd, pd, vol["Mc"])
            A = vol["A"].copy()
            C = vol["C"].copy()
            B = vol["B"].copy()
            for f in range(6):
                nb = lev.neighbour(c, f)
                if nb >= 0:
                    if f % 2 == 1:                         # interior face, assembled once from the lower cell
                        Bf = face_pi[f // 2]
                        sides = [pd, pdofs[nb]]
                        for i in range(2):
                            for j in range(2):
                                add("B", sides[i], sides[j], Bf[i][j])
                    continue
                ub = lev.u_bc(c, f)
                if ub in (U_DIRICHLET, U_DIRECTIONAL):
                    if (f, ub) not in face_u:
                        face_u[(f, ub)] = F.face_u(f, ub)
                    Af, Cf = face_u[(f, ub)]
                    A += Af
                    C += Cf
                if lev.p_bc(c, f) == P_DIRICHLET:
                    if f not in face_pd:
                        face_pd[f] = F.face_p_dirichlet(f)
                    B += face_pd[f]
            add("A", vd, vd, A)
            add("C", pd, vd, C)
            add("B", pd, pd, B)
        shp = dict(Mr=(3 * nq, 3 * nq), Mc=(nc * npc, nc * npc), A=(3 * nq, 3 * nq), C=(nc * npc, 3 * nq),
                   B=(nc * npc, nc * npc))
        for key, (ri, ci, vv) in trip.items():
            M = sp.coo_matrix((np.concatenate(vv), (np.concatenate(ri), np.concatenate(ci))), shape=shp[key]).tocsr()
            setattr(self, key, M)


def slab_matrix(S, T, th):
    """A_n = T (x) calM + diag(theta) (x) calK, rows (phi, chi, psi), columns (V, U, P) (reading A5;
    Problem 3.1)."""
    calM = sp.bmat([[None, S.Mr, None], [S.Mr, None, None], [None, None, S.Mc]], format="csr")
    calK = sp.bmat([[-S.Mr, None, None], [None, S.A, S.C.T], [-S.C, None, S.B]], format="csr")
    return (sp.kron(sp.csr_matrix(T), calM) + sp.kron(sp.diags(th), calK)).tocsr()


def prolongation(coarse, fine):
    """P: coarse -> fine: Q_r nodal interpolation (structured 1D tables, Kronecker, restricted to active
    nodes) and, for P_{r-1}^disc, the coarse cell polynomial restricted to each child, per (m, f, c)."""
    r = fine.r
    Ps = sp.identity(1, format="csr")
    for a in range(3):
        Ps = sp.kron(sp.csr_matrix(interp_1d(coarse.n[a], r)), Ps, format="csr")
    fa = np.nonzero(fine.qmap.ravel(order="F") >= 0)[0]
    ca = np.nonzero(coarse.qmap.ravel(order="F") >= 0)[0]
    Pfull = Ps[fa]
    assert abs(Pfull).sum() == abs(Pfull[:, ca]).sum(), "interpolation reaches an inactive coarse node"
    Pq = Pfull[:, ca].tocsr()
    # P_{r-1}^disc: coefficients of the coarse monomials restricted to child with position bits sb (exact fit at
    # a unisolvent point set of the child; library primitive lstsq)
    xg, _ = gauss_legendre01(r + 1)
    blocks = {}
    for sb in itertools.product((0, 1), repeat=3):
        pts_child = [xg] * 3
        pts_parent = [0.5 * (xg + sb[a]) for a in range(3)]
        Vc, _ = p_eval(fine.exps, pts_child, fine.h)
        Vp, _ = p_eval(coarse.exps, pts_parent, coarse.h)
        X, *_ = np.linalg.lstsq(Vc.T, Vp.T, rcond=None)     # Vc^T X = Vp^T: child coefficients of each coarse fn
        blocks[sb] = X
    rows, cols, vals = [], [], []
    for cid in range(fine.n_cells):
        c = fine.cells[cid]
        pc = coarse.cell_id[c[0] // 2, c[1] // 2, c[2] // 2]
        X = blocks[tuple(int(v % 2) for v in c)]
        for i in range(fine.npc):
            for j in range(coarse.npc):
                rows.append(cid * fine.npc + i)
                cols.append(pc * coarse.npc + j)
                vals.append(X[i, j])
    Pp = sp.coo_matrix((vals, (rows, cols)), shape=(fine.np_, coarse.np_)).tocsr()
    Pp.eliminate_zeros()
    blocks = []
    for _ in range(fine.k + 1):
        blocks += [Pq] * 6 + [Pp]
    return sp.block_diag(blocks, format="csr")


class LPatches:
    """Vertex patches (Eq:DefPlm) of the active vertices: cells = the active cells around the vertex;
    Z(P) = all DoFs of those cells (reading A11), ordered (m, f, c, node / P DoF ascending) (reading A12).  Every
    patch is its own class (no class sharing on the L-shape)."""

    def __init__(self, lev):
        self.lev = lev
        nv = tuple(n + 1 for n in lev.n)
        verts = np.array(np.unravel_index(np.arange(int(np.prod(nv))), nv, order="F")).T
        self.verts, self.dofs = [], []
        for v in verts:
            cids = []
            for off in itertools.product((-1, 0), repeat=3):
                c = v + np.array(off)
                if np.all(c >= 0) and np.all(c < np.array(lev.n)) and lev.active[c[0], c[1], c[2]]:
                    cids.append(int(lev.cell_id[c[0], c[1], c[2]]))
            if not cids:
                continue
            cids.sort()
            qn = np.unique(lev.cell_q[cids].ravel())
            pn = np.concatenate([lev.cell_p(c) for c in cids])
            idx = []
            for m in range(lev.k + 1):
                for c in range(3):
                    idx.append(lev.offset(m, 0, c) + qn)
                for c in range(3):
                    idx.append(lev.offset(m, 1, c) + qn)
                idx.append(lev.offset(m, 2) + pn)
            self.verts.append(tuple(int(x) for x in v))
            self.dofs.append(np.concatenate(idx))
        self.classes = list(range(len(self.dofs)))
        self.members = {i: [i] for i in self.classes}
        cnt = np.zeros(lev.N)
        for idx in self.dofs:
            np.add.at(cnt, idx, 1.0)
        self.p = cnt
        self.flat_idx = np.concatenate(self.dofs)

    def extract(self, A, i):
        z = self.dofs[i]
        return A[z][:, z].toarray()


class LHierarchy:
    """GMG hierarchy ref_c .. ref_c + nlevels - 1 (Table 4: the coarse level is ref_1), V-cycle as oracle.mg
    (readings A13-A16), per-patch inverses (share_classes=False)."""

    def __init__(self, ref_coarse, nlevels, r, k, tau, params=None, omega=0.7, jmax=4):
        self.params = params or lshape_params(r)
        self.levels = [LLevel(ref_coarse + l, r, k) for l in range(nlevels)]
        self.t_hat, self.w_hat, self.chi_m1, self.T = temporal_constants(k)
        self.tau = float(tau)
        self.th = 0.5 * self.tau * self.w_hat
        self.spatial = [LSpatial(lv, self.params) for lv in self.levels]
        self.A = [slab_matrix(S, self.T, self.th) for S in self.spatial]
        self.P = [None] + [prolongation(self.levels[l - 1], self.levels[l]) for l in range(1, nlevels)]
        self.jmax = jmax
        self.patches = [None] + [LPatches(self.levels[l]) for l in range(1, nlevels)]
        self.smoothers = [None] + [VankaSmoother(self.A[l], self.patches[l], omega, share_classes=False)
                                   for l in range(1, nlevels)]
        self.coarse_inv = equilibrated_inverse(self.A[0].toarray())

    @property
    def fine(self):
        return self.levels[-1]

    def vcycle(self, b, l=None):
        if l is None:
            l = len(self.levels) - 1
        if l == 0:
            return self.coarse_inv @ b
        sm = self.smoothers[l]
        d = sm.smooth(b, None, self.jmax)
        r = b - self.A[l] @ d
        dc = self.vcycle(self.P[l].T @ r, l - 1)
        d = d + self.P[l] @ dc
        return sm.smooth(b, d, self.jmax)


def traction_vector(lev, params=None):
    """Spatial load of the chi rows per unit sin(8 pi t): F_gamma = -<t_N, chi>_{Gamma^N_u} (Def:L P:L220, sign as
    reading A23), t_N = (0, 5e9 g(x, z), 0), g = 32xz - 18x - 16z + 10; (r+2)-point Gauss per face axis (reading
    A10).  Returns a vector of length 3 nq (U components, component-major)."""
    r = lev.r
    xg, wg = gauss_legendre01(r + 2)
    pts = [xg, np.array([1.0]), xg]
    wts = [wg, np.array([1.0]), wg]
    phq, _ = _tensor_eval(3, gauss_lobatto_nodes01(r), pts, lev.h)
    w = _tensor_weights(wts, lev.h[0] * lev.h[2])
    qi = np.array(np.unravel_index(np.arange(len(w)), [len(xg), 1, len(xg)], order="F")).T
    out = np.zeros(3 * lev.nq)
    for cid in range(lev.n_cells):
        c = lev.cells[cid]
        if c[1] != lev.n[1] - 1 or lev.u_bc(c, 3) != U_TRACTION:
            continue
        x = (c[0] + xg[qi[:, 0]]) * lev.h[0]
        z = (c[2] + xg[qi[:, 2]]) * lev.h[2]
        g = TRACTION_AMP * (32.0 * x * z - 18.0 * x - 16.0 * z + 10.0)
        np.add.at(out, lev.nq + lev.cell_q[cid], -(phq * (g * w)[None, :]).sum(axis=1))
    return out


def slab_load(H, t_prev, fN=None):
    """L_n of the slab (t_prev, t_prev + tau]: chi_b rows = theta_b sin(8 pi t_{n,b}) F."""
    lev = H.fine
    fN = traction_vector(lev, H.params) if fN is None else fN
    L = np.zeros(lev.N)
    for b in range(lev.k + 1):
        t = t_prev + 0.5 * H.tau * (1.0 + H.t_hat[b])
        o = lev.offset(b, 1, 0)
        L[o:o + 3 * lev.nq] += H.th[b] * np.sin(8.0 * np.pi * t) * fN
    return L


def slab_rhs(H, L, x_prev):
    """F_n = L_n + J X_{n-1}: chi_hat_b(-1) (M_rho U, M_rho V, M_c P) of the last Radau block of X_{n-1}
    (SURVEY a10)."""
    lev, S = H.fine, H.spatial[-1]
    k = lev.k
    o = k * lev.block
    V = x_prev[o:o + lev.R]
    U = x_prev[o + lev.R:o + 2 * lev.R]
    P = x_prev[o + 2 * lev.R:o + lev.block]
    F = L.copy()
    MU, MV, MP = S.Mr @ U, S.Mr @ V, S.Mc @ P
    for b in range(k + 1):
        ob = b * lev.block
        F[ob:ob + lev.R] += H.chi_m1[b] * MU
        F[ob + lev.R:ob + 2 * lev.R] += H.chi_m1[b] * MV
        F[ob + 2 * lev.R:ob + lev.block] += H.chi_m1[b] * MP
    return F


def goal_quantities(lev, x):
    """(b_u, b_p) of Eq:DefGQ for the last Radau block of x (the value at t_n): integrals over
    Gamma_m = {1} x (0,.5) x (0,.5) with (r+1)-point Gauss per face axis."""
    r = lev.r
    xg, wg = gauss_legendre01(r + 1)
    pts = [np.array([1.0]), xg, xg]
    wts = [np.array([1.0]), wg, wg]
    phq, _ = _tensor_eval(3, gauss_lobatto_nodes01(r), pts, lev.h)
    php, _ = p_eval(lev.exps, pts, lev.h)
    w = _tensor_weights(wts, lev.h[1] * lev.h[2])
    o = lev.k * lev.block
    bu = bp = 0.0
    for cid in range(lev.n_cells):
        c = lev.cells[cid]
        if c[0] != lev.n[0] - 1:
            continue
        ux = x[o + lev.R + lev.cell_q[cid]]
        pp = x[o + 2 * lev.R + lev.cell_p(cid)]
        bu += float((ux @ phq) @ w)
        bp += float((pp @ php) @ w)
    return bu, bp
