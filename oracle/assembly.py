"""Slab operator A_n of Problem 3.1: element slab matrices, global assembly, element-wise apply.

P:L233-256 (Eq:DPQ_A0, Problem 3.1 DSA) defines A_n; P:L384-431 (Eq:ALS_In, Eq:DefAn) its block form, read
per reading A5 (rows = test (phi, chi, psi) at node b, columns = trial (V, U, P) at node a).  Each level is
rediscretised with its own h_F (reading A14).  The global matrix is the sum of element slab matrices over
cells (standard FE assembly; the library primitive is scipy.sparse COO -> CSR summation).
(oracle; test infrastructure only)
"""
import numpy as np
import scipy.sparse as sp
from .element import ElementForms, slab_element_matrix, default_gammas
from .temporal import temporal_constants
from .mesh import FIELD_V, FIELD_U, FIELD_P


def full_params(params, r):
    p = dict(params)
    ga, gb = default_gammas(r)
    if p.get("gamma_a") is None or p.get("gamma_a", -1) < 0:
        p["gamma_a"] = ga
    if p.get("gamma_b") is None or p.get("gamma_b", -1) < 0:
        p["gamma_b"] = gb
    p.setdefault("hF_mode", 0)
    return p


def all_cell_dofs(lev):
    """(n_cells, n_e) global DoF indices of every cell (lexicographic cells), element order (m, f, c, node)."""
    d, r = lev.d, lev.r
    cells = np.array(np.unravel_index(np.arange(lev.n_cells), lev.n, order="F")).T   # (nc, d)

    def nodes(deg, strides):
        loc = np.array(np.unravel_index(np.arange((deg + 1) ** d), [deg + 1] * d, order="F")).T
        g = np.zeros((cells.shape[0], loc.shape[0]), dtype=np.int64)
        for a in range(d):
            g += (deg * cells[:, a][:, None] + loc[None, :, a]) * strides[a]
        return g

    qn = nodes(r, lev.q_strides)
    pn = nodes(r - 1, lev.p_strides)
    parts = []
    for m in range(lev.k + 1):
        for c in range(d):
            parts.append(lev.offset(m, FIELD_V, c) + qn)
        for c in range(d):
            parts.append(lev.offset(m, FIELD_U, c) + qn)
        parts.append(lev.offset(m, FIELD_P) + pn)
    return np.concatenate(parts, axis=1), cells


class SlabOperator:
    """A_n on one level: T (x) calM + diag(theta) (x) calK."""

    def __init__(self, lev, params, tau, ds=False):
        self.lev = lev
        self.ds = ds   # Problem B.1 (DS) instead of Problem 3.1 (DSA), SURVEY N4
        self.params = full_params(params, lev.r)
        self.tau = float(tau)
        self.t_hat, self.w_hat, self.chi_m1, self.T = temporal_constants(lev.k)
        self.th = 0.5 * self.tau * self.w_hat
        self.forms = ElementForms(lev.d, lev.r, lev.h, self.params)
        self._mats = {}
        self._slab = {}
        self.dofs, self.cells = all_cell_dofs(lev)
        types = [lev.cell_type(tuple(c)) for c in self.cells]
        self.type_keys = sorted(set(types))
        key_index = {key: i for i, key in enumerate(self.type_keys)}
        self.cell_type_id = np.array([key_index[t] for t in types])

    def mats(self, key):
        if key not in self._mats:
            self._mats[key] = self.forms.matrices(*key)
        return self._mats[key]

    def slab(self, key):
        if key not in self._slab:
            self._slab[key] = slab_element_matrix(self.mats(key), self.T, self.th, self.ds)
        return self._slab[key]

    def assemble(self):
        """Global sparse A_n (CSR)."""
        rows, cols, vals = [], [], []
        for ti, key in enumerate(self.type_keys):
            E = self.slab(key)
            D = self.dofs[self.cell_type_id == ti]
            rows.append(np.repeat(D, D.shape[1], axis=1).ravel())
            cols.append(np.tile(D, (1, D.shape[1])).ravel())
            vals.append(np.broadcast_to(E.ravel(), (D.shape[0], E.size)).ravel())
        N = self.lev.N
        A = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(N, N))
        return A.tocsr()

    def apply(self, x):
        """y = A_n x element by element (gather, dense element matvec, scatter-add)."""
        y = np.zeros(self.lev.N)
        for ti, key in enumerate(self.type_keys):
            E = self.slab(key)
            D = self.dofs[self.cell_type_id == ti]
            np.add.at(y, D, x[D] @ E.T)
        return y

    def apply_rows(self, x, rows):
        """(A_n x)[rows] computed element by element for the cells that touch each row (sampled parity)."""
        out = np.zeros(len(rows))
        for ti, key in enumerate(self.type_keys):
            E = self.slab(key)
            sel = np.nonzero(self.cell_type_id == ti)[0]
            D = self.dofs[sel]
            for i, rw in enumerate(rows):
                hit = np.nonzero(D == rw)
                for ci, li in zip(*hit):
                    out[i] += E[li] @ x[D[ci]]
        return out

    # spatial matrices (for closed-form pins) ---------------------------------------------------------
    def assemble_spatial(self):
        """Global Mq (scalar Q_r mass), Mp, Mrho, Mc, A, C, B and Cvol (volume part of C) of the level (CSR)."""
        lev = self.lev
        d = lev.d
        out = {}
        qn_all, pn_all = [], []
        D = self.dofs
        nq_loc = (lev.r + 1) ** d
        np_loc = lev.r ** d
        qn = D[:, :nq_loc] - lev.offset(0, FIELD_V, 0)
        pn = D[:, 2 * d * nq_loc: 2 * d * nq_loc + np_loc] - lev.offset(0, FIELD_P)
        vec = np.concatenate([qn + c * lev.nq for c in range(d)], axis=1)
        spec = {"Mq": (qn, qn, lev.nq, lev.nq), "Mp": (pn, pn, lev.np_, lev.np_),
                "Mrho": (vec, vec, lev.R, lev.R), "Mc": (pn, pn, lev.np_, lev.np_),
                "A": (vec, vec, lev.R, lev.R), "C": (pn, vec, lev.np_, lev.R), "B": (pn, pn, lev.np_, lev.np_),
                "Cvol": (pn, vec, lev.np_, lev.R)}
        for name, (Rm, Cm, nr, nc) in spec.items():
            rows, cols, vals = [], [], []
            for ti, key in enumerate(self.type_keys):
                M = self.mats(key)[name]
                sel = self.cell_type_id == ti
                Rs, Cs = Rm[sel], Cm[sel]
                rows.append(np.repeat(Rs, Cs.shape[1], axis=1).ravel())
                cols.append(np.tile(Cs, (1, Rs.shape[1])).ravel())
                vals.append(np.broadcast_to(M.ravel(), (Rs.shape[0], M.size)).ravel())
            out[name] = sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                      shape=(nr, nc)).tocsr()
        return out
