"""Patch-wise Vanka smoother, Algorithm 1 (oracle; test infrastructure only).

P:L449-453 (Eq:DefPlm): one patch per grid vertex, the cells whose closure contains the vertex.
P:L454-466: Z_l(P) = all global DoFs of the patch cells, for all k+1 Radau nodes, fields and components
(reading A11: closure); local order (m, f, c, node lexicographic in the patch node box) (reading A12).
P:L469-485 (Def:VankaOP): S_P(d) = R_P d + omega A_P^{-1} R_P (b - A_l d), A_P = A_l[Z(P), Z(P)].
P:L486: omega = 0.7, explicit inverse (reading A18), here LU with partial pivoting from LAPACK (library
primitive numpy.linalg.inv) after power-of-2 symmetric equilibration s_i = 2^-round(log2 sqrt|a_ii|)
(readings A19): Ainv = S (S A S)^{-1} S.
P:L488-524 (alg:smoother): additive patch loop with counters p and accumulator z, averaging after the loop.
Main form (reading A17): d <- d + omega * (sum_P E_P A_P^{-1} R_P r) / p, patches accumulated in
lexicographic vertex order; the literal form d <- (sum_P E_P S_P(d)) / p is ``sweep_literal``.
Class sharing: A_P depends only on the per-axis class of the vertex index
({0}, {1}, {2..n-2}, {n-1}, {n} for n >= 4; every index its own class for n < 4).

Smoother variant (the north star's "cell-coloured multiplicative patch sweeps"): the patch
loop of Def:VankaOP with SUCCESSIVE OVERWRITING, which P:L527-529 (Remark after alg:smoother) names as the
alternative to averaging: d[Z(P)] <- S_P(d) for one patch after the other, each with the current d.  Patches are
ordered by vertex colour (v_a mod 4 per axis, colours lexicographic, x fastest; patches of one colour in
lexicographic vertex order).  Two patches of one colour share no cell (their vertices differ by >= 4 along some
axis), so A_l does not couple their DoFs and the colour's patches can be updated from ONE residual: that is
``sweep_colored`` (what the GPU computes); ``sweep_sequential`` is the literal one-patch-at-a-time loop, used as
its pin.
"""
import itertools
import numpy as np
from .mesh import FIELD_V, FIELD_U, FIELD_P


def axis_class(v, n):
    if n < 4:
        return v
    if v == 0:
        return 0
    if v == 1:
        return 1
    if v == n:
        return 4
    if v == n - 1:
        return 3
    return 2


def equilibrated_inverse(A):
    """Ainv = S (S A S)^{-1} S with power-of-two s_i (exact scaling), LU with partial pivoting (LAPACK)."""
    dg = np.abs(np.diag(A))
    if np.any(dg == 0.0):
        raise np.linalg.LinAlgError("zero diagonal")
    s = np.exp2(-np.round(0.5 * np.log2(dg)))
    As = A * s[:, None] * s[None, :]
    inv = np.linalg.inv(As)
    return inv * s[:, None] * s[None, :]


def axis_class_cell(c, n):
    """Per-axis class of a cell for element-wise Vanka (N2(ii)): {0}, {1..n-2}, {n-1} (n >= 3), every cell its own
    class for n < 3.  A_K = A_l[Z(K), Z(K)] also sums the neighbours' element matrices on K's boundary DoFs, but a
    Nitsche face term of a boundary neighbour couples only DoFs ON that face, which a cell one away does not own, so
    one class per side suffices (pinned bitwise up to assembly order in test_oracle_pins.py)."""
    if n < 3:
        return c
    return 0 if c == 0 else (2 if c == n - 1 else 1)


class Patches:
    """Vertex patches (Eq:DefPlm) of one level with their DoF index sets Z(P) in local order.
    cells=True: one patch per CELL instead (element-wise Vanka, the alternative P:L529-531 rejects);
    ``verts`` then holds cell + 1 per axis, so that the patch cell range below is the single cell."""

    def __init__(self, lev, cells=False):
        self.lev = lev
        d, r = lev.d, lev.r
        self.cells = cells
        if cells:
            self.verts = [tuple(c + 1 for c in reversed(t))
                          for t in itertools.product(*[range(n) for n in reversed(lev.n)])]
        else:
            self.verts = [tuple(reversed(t)) for t in itertools.product(*[range(n + 1) for n in reversed(lev.n)])]
        self.dofs = []
        self.keys = []
        for v in self.verts:
            lo_c = [max(v[a] - 1, 0) for a in range(d)]
            hi_c = [min(v[a], lev.n[a] - 1) for a in range(d)]       # inclusive cell range
            if cells:
                hi_c = list(lo_c)
            qbox = [np.arange(r * lo_c[a], r * (hi_c[a] + 1) + 1) for a in range(d)]
            pbox = [np.arange((r - 1) * lo_c[a], (r - 1) * (hi_c[a] + 1) + 1) for a in range(d)]
            qn = self._lex(qbox, lev.q_strides)
            pn = self._lex(pbox, lev.p_strides)
            idx = []
            for m in range(lev.k + 1):
                for c in range(d):
                    idx.append(lev.offset(m, FIELD_V, c) + qn)
                for c in range(d):
                    idx.append(lev.offset(m, FIELD_U, c) + qn)
                idx.append(lev.offset(m, FIELD_P) + pn)
            self.dofs.append(np.concatenate(idx))
            if cells:
                self.keys.append(tuple(axis_class_cell(v[a] - 1, lev.n[a]) for a in range(d)))
            else:
                self.keys.append(tuple(axis_class(v[a], lev.n[a]) for a in range(d)))
        self.classes = sorted(set(self.keys))
        self.members = {c: [i for i, kk in enumerate(self.keys) if kk == c] for c in self.classes}
        cnt = np.zeros(lev.N)
        for idx in self.dofs:
            np.add.at(cnt, idx, 1.0)
        self.p = cnt
        self.flat_idx = np.concatenate(self.dofs)

    @staticmethod
    def _lex(boxes, strides):
        grids = np.meshgrid(*[b * strides[a] for a, b in enumerate(boxes)], indexing="ij")
        return sum(grids).ravel(order="F").astype(np.int64)   # axis 0 fastest

    def extract(self, A, i):
        """A_P = A_l[Z(P), Z(P)], dense."""
        z = self.dofs[i]
        return A[z][:, z].toarray()


class VankaSmoother:
    """Algorithm 1 on one level with per-class (or per-patch) equilibrated inverses."""

    def __init__(self, A, patches, omega=0.7, share_classes=True):
        self.A = A
        self.P = patches
        self.omega = omega
        self.share = share_classes
        self.inv = {}
        if share_classes:
            for c in patches.classes:
                rep = patches.members[c][0]                     # lexicographically first patch of the class
                Ainv = equilibrated_inverse(patches.extract(A, rep))
                for i in patches.members[c]:
                    self.inv[i] = Ainv
        else:
            for i in range(len(patches.dofs)):
                self.inv[i] = equilibrated_inverse(patches.extract(A, i))
        if np.any(patches.p == 0):
            raise ValueError("a DoF lies in no patch (S:L357)")

    def patch_updates(self, r):
        """y_P = A_P^{-1} R_P r for every patch, in lexicographic patch order (concatenated)."""
        out = []
        for c in self.P.classes:
            mem = self.P.members[c]
            if self.share:
                Z = np.stack([self.P.dofs[i] for i in mem])
                Y = r[Z] @ self.inv[mem[0]].T
                for j, i in enumerate(mem):
                    out.append((i, Y[j]))
            else:
                for i in mem:
                    out.append((i, self.inv[i] @ r[self.P.dofs[i]]))
        out.sort(key=lambda t: t[0])
        return np.concatenate([y for _, y in out])

    def sweep(self, b, d):
        """One smoothing step (reading A17): d + omega * (sum_P E_P y_P) / p."""
        r = b - self.A @ d
        z = np.zeros_like(d)
        np.add.at(z, self.P.flat_idx, self.patch_updates(r))
        return d + self.omega * z / self.P.p

    def sweep_literal(self, b, d):
        """Literal Alg. 1 lines 3-9: z += E_P S_P(d), p++, d = z / p."""
        r = b - self.A @ d
        y = self.patch_updates(r)
        z = np.zeros_like(d)
        np.add.at(z, self.P.flat_idx, d[self.P.flat_idx] + self.omega * y)
        return z / self.P.p

    # ---------------------------------------------------------------- overwrite variant (N2(iii))
    def sweep_overwrite(self, b, d):
        """Alg. 1 without averaging (P:L527-529 names it as what averaging replaces): lines 7-9 become
        z[dof(P, mu_hat)] = S_P(d)[mu_hat] (overwrite, no counter) and d = z, so every DoF keeps the update of the LAST
        patch (lexicographic vertex order) that contains it.  Vectorised: the last writer of each DoF."""
        r = b - self.A @ d
        y = self.patch_updates(r)
        last = np.full(len(d), -1, dtype=np.int64)
        last[self.P.flat_idx] = np.arange(len(self.P.flat_idx))   # numpy keeps the last assignment per index
        z = d.copy()
        hit = last >= 0
        z[hit] = d[hit] + self.omega * y[last[hit]]
        return z

    def sweep_overwrite_literal(self, b, d):
        """The same, written as the literal patch loop (pin of ``sweep_overwrite``)."""
        r = b - self.A @ d
        z = d.copy()
        for i in range(len(self.P.dofs)):
            Z = self.P.dofs[i]
            yP = self.inv[i] @ r[Z]
            for j, mu in enumerate(Z):
                z[mu] = d[mu] + self.omega * yP[j]
        return z

    # ---------------------------------------------------------------- multiplicative variant (N2(i))
    NCOL = 4   # colours per axis: same-colour patches share no cell

    def colour_order(self):
        """Patch indices grouped by vertex colour (v mod 4 per axis, lexicographic, x fastest)."""
        d = self.P.lev.d
        key = [sum((v[a] % self.NCOL) * self.NCOL ** a for a in range(d)) for v in self.P.verts]
        groups = {}
        for i, c in enumerate(key):            # self.P.verts is in lexicographic vertex order
            groups.setdefault(c, []).append(i)
        return [groups[c] for c in sorted(groups)]

    def sweep_colored(self, b, d):
        """One multiplicative sweep: for each colour, r = b - A d, then d[Z(P)] += omega A_P^{-1} R_P r for the
        colour's patches (Eq:VankaOP0 with overwriting)."""
        d = d.copy()
        for group in self.colour_order():
            r = b - self.A @ d
            for i in group:
                z = self.P.dofs[i]
                d[z] = d[z] + self.omega * (self.inv[i] @ r[z])
        return d

    def sweep_sequential(self, b, d):
        """Literal successive overwriting d[Z(P)] <- S_P(d), one patch at a time with its own residual."""
        d = d.copy()
        for group in self.colour_order():
            for i in group:
                z = self.P.dofs[i]
                d[z] = d[z] + self.omega * (self.inv[i] @ (b - self.A @ d)[z])
        return d

    def smooth(self, b, d=None, steps=4, colored=False, overwrite=False):
        """Alg. 1: d initialised with 0 (pre-smoothing) or continued (post-smoothing, reading A13)."""
        d = np.zeros_like(b) if d is None else d.copy()
        for _ in range(steps):
            if colored:
                d = self.sweep_colored(b, d)
            elif overwrite:
                d = self.sweep_overwrite(b, d)
            else:
                d = self.sweep(b, d)
        return d
