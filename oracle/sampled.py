"""Sampled oracle evaluations for full-size parity (oracle; test infrastructure only).

At BASELINE sizes (up to 26.5 M DoFs) the global matrices cannot be assembled on the CPU in seconds, so these
helpers evaluate the same definitions locally, cell by cell:
  * rows of y = A_l x (Problem 3.1) from the element slab matrices of the <= 2^d cells containing the
    node of each row;
  * A_P = A_l[Z(P), Z(P)] by summing the element slab matrices of every cell that touches Z(P)
    (SURVEY O8), restricted to Z(P);
  * one step of Algorithm 1 (reading A17) at sampled DoFs: d_mu + omega/p_mu * sum_{P containing mu}
    (A_P^{-1} R_P (b - A_l d))[mu_hat], with the same equilibrated inverse as vanka.py.
"""
import itertools

import numpy as np

from .assembly import full_params
from .element import ElementForms, slab_element_matrix
from .temporal import temporal_constants
from .mesh import FIELD_V, FIELD_U, FIELD_P
from .vanka import axis_class, equilibrated_inverse


class LiteOperator:
    """Element slab matrices per cell type, without any global array (for huge levels)."""

    def __init__(self, lev, params, tau):
        self.lev = lev
        self.params = full_params(params, lev.r)
        t_hat, w_hat, self.chi_m1, self.T = temporal_constants(lev.k)
        self.th = 0.5 * float(tau) * w_hat
        self.forms = ElementForms(lev.d, lev.r, lev.h, self.params)
        self._E = {}

    def E(self, cell):
        key = self.lev.cell_type(tuple(cell))
        if key not in self._E:
            self._E[key] = slab_element_matrix(self.forms.matrices(*key), self.T, self.th)
        return self._E[key]

    def decode(self, mu):
        lev = self.lev
        m, rem = divmod(int(mu), lev.block)
        if rem < 2 * lev.R:
            pres, node, deg, shape = False, rem % lev.nq, lev.r, lev.q_shape
        else:
            pres, node, deg, shape = True, rem - 2 * lev.R, lev.r - 1, lev.p_shape
        idx = np.unravel_index(node, shape, order="F")
        return m, pres, deg, [int(i) for i in idx]

    def cells_of(self, mu):
        lev = self.lev
        _, _, deg, idx = self.decode(mu)
        per_axis = []
        for a in range(lev.d):
            i = idx[a]
            if i % deg == 0:
                cs = [c for c in (i // deg - 1, i // deg) if 0 <= c < lev.n[a]]
            else:
                cs = [i // deg]
            per_axis.append(cs)
        return [tuple(reversed(t)) for t in itertools.product(*reversed(per_axis))]   # lexicographic, x fastest

    def rows(self, x, rows):
        """(A x)[rows], cell by cell."""
        out = np.zeros(len(rows))
        for i, mu in enumerate(rows):
            for cell in self.cells_of(mu):
                D = self.lev.cell_dofs(cell)
                li = int(np.nonzero(D == mu)[0][0])
                out[i] += self.E(cell)[li] @ x[D]
        return out

    # --- patches ------------------------------------------------------------------------------------------
    def patch_dofs(self, v):
        lev, r, d = self.lev, self.lev.r, self.lev.d
        lo_c = [max(v[a] - 1, 0) for a in range(d)]
        hi_c = [min(v[a], lev.n[a] - 1) for a in range(d)]

        def lex(deg, strides):
            boxes = [np.arange(deg * lo_c[a], deg * (hi_c[a] + 1) + 1) * strides[a] for a in range(d)]
            return sum(np.meshgrid(*boxes, indexing="ij")).ravel(order="F").astype(np.int64)

        qn, pn = lex(r, lev.q_strides), lex(r - 1, lev.p_strides)
        idx = []
        for m in range(lev.k + 1):
            for c in range(d):
                idx.append(lev.offset(m, FIELD_V, c) + qn)
            for c in range(d):
                idx.append(lev.offset(m, FIELD_U, c) + qn)
            idx.append(lev.offset(m, FIELD_P) + pn)
        return np.concatenate(idx)

    def neighbourhood(self, v):
        """Cells that touch Z(P): per axis v-2 .. v+1."""
        lev = self.lev
        ranges = [range(max(v[a] - 2, 0), min(v[a] + 1, lev.n[a] - 1) + 1) for a in range(lev.d)]
        return [tuple(reversed(t)) for t in itertools.product(*reversed(ranges))]

    def patch_system(self, v, x=None):
        """A_P (dense) and, if x is given, (A_l x)[Z(P)], both from the neighbourhood cells."""
        Z = self.patch_dofs(v)
        pos = {int(g): i for i, g in enumerate(Z)}
        AP = np.zeros((len(Z), len(Z)))
        Ax = np.zeros(len(Z)) if x is not None else None
        for cell in self.neighbourhood(v):
            D = self.lev.cell_dofs(cell)
            loc = np.array([pos.get(int(g), -1) for g in D])
            sel = np.nonzero(loc >= 0)[0]
            if len(sel) == 0:
                continue
            E = self.E(cell)
            AP[np.ix_(loc[sel], loc[sel])] += E[np.ix_(sel, sel)]
            if x is not None:
                Ax[loc[sel]] += E[sel] @ x[D]
        return Z, AP, Ax

    def patches_of(self, mu):
        lev = self.lev
        _, _, deg, idx = self.decode(mu)
        per_axis = []
        for a in range(lev.d):
            i, n = idx[a], lev.n[a]
            if i % deg == 0:
                vv = i // deg
                cand = [w for w in (vv - 1, vv, vv + 1) if 0 <= w <= n and
                        any(0 <= c < n for c in {w - 1, w} & {vv - 1, vv})]
            else:
                cand = [i // deg, i // deg + 1]
            per_axis.append(cand)
        return [tuple(reversed(t)) for t in itertools.product(*reversed(per_axis))]

    def sampled_sweep(self, b, d, sample, omega=0.7):
        """One Alg. 1 step (A17 form) evaluated at the sampled DoFs only."""
        inv_cache = {}
        out = np.zeros(len(sample))
        for i, mu in enumerate(sample):
            z = 0.0
            pats = self.patches_of(mu)
            for v in pats:
                Z, AP, Ad = self.patch_system(v, d)
                key = tuple(axis_class(v[a], self.lev.n[a]) for a in range(self.lev.d))
                if key not in inv_cache:
                    inv_cache[key] = equilibrated_inverse(AP)
                y = inv_cache[key] @ (b[Z] - Ad)
                z += y[int(np.nonzero(Z == mu)[0][0])]
            out[i] = d[mu] + omega * z / len(pats)
        return out
