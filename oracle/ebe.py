"""Element-by-element oracle for BASELINE sizes (oracle; test infrastructure only).

SURVEY §8(c) O5: "the §8(a) formula, applied element-by-element with a dense element slab matrix per cell type ...
Memory stays low and the algorithm is independent of K1's sum factorisation."  This module computes exactly what
assembly.py / transfer.py / vanka.py / mg.py compute, without any global sparse matrix, so that the full V-cycle and
FGMRES of configs 2-4 (up to 26.6 M DoFs) run on the host:

  * EbeOperator  y = A_n x (Problem 3.1, Eq:DPQ_A0; block form per reading A5): per cell type the
    element slab matrix of element.slab_element_matrix, applied to the gathered cell vectors x[D_K] (library
    matmul), contributions summed into y (np.bincount = the sequential loop y[D_K[j]] += (E x_K)[j]).
  * EbeTransfer  prolongation by nodal interpolation = the Kronecker product of the 1D interpolation
    matrices of transfer.interp_1d, applied axis by axis (the definition of the Kronecker product); restriction =
    the transpose, applied the same way.
  * EbeSmoother  Algorithm 1 (reading A17): patches = vertex patches (Eq:DefPlm), Z(P) in local order
    (m, f, c, node lexicographic, readings A11/A12), A_P = A_l[Z(P), Z(P)] summed from the element slab matrices of
    the cells that touch Z(P) (sampled.LiteOperator.patch_system), one equilibrated inverse per per-axis
    class (reading R2; vanka.equilibrated_inverse), y_P = Ainv R_P r for all patches of a class as
    one matmul, z accumulated, d <- d + omega z / p.
  * EbeHierarchy V-cycle with the same composition as mg.Hierarchy.vcycle (pre from 0, residual,
    restriction, coarser cycle, prolongation-add, post continuing, reading A13); direct coarse solve with the
    equilibrated inverse of the assembled (small) A_0.
  * fgmres from gmres.py unchanged.

Pinned against the assembled-matrix oracle (whose own pins are in tests/test_oracle_pins*.py) on small meshes of
every family: tests/test_oracle_ebe.py (operator, transfer, patch sets and multiplicities, sweep, V-cycle, FGMRES).
"""
import itertools

import numpy as np

from .assembly import SlabOperator, all_cell_dofs, full_params
from .basis import gauss_lobatto_nodes01
from .element import ElementForms, slab_element_matrix
from .gmres import fgmres
from .mesh import BC_DIRICHLET, FIELD_P, FIELD_U, FIELD_V, hierarchy
from .sampled import LiteOperator
from .temporal import temporal_constants
from .transfer import interp_1d
from .vanka import axis_class, equilibrated_inverse

CHUNK = 1 << 15          # cells / patches per gathered block (memory bound only; no effect on the arithmetic order)
FLUSH = 1 << 26          # accumulate at most this many (index, value) pairs before summing them into z


class _Accumulator:
    """z[idx[j]] += val[j] in the order the pairs are added (np.bincount sums sequentially)."""

    def __init__(self, n):
        self.n = n
        self.z = np.zeros(n)
        self.idx, self.val, self.size = [], [], 0

    def add(self, idx, val):
        self.idx.append(idx.ravel())
        self.val.append(val.ravel())
        self.size += idx.size
        if self.size >= FLUSH:
            self.flush()

    def flush(self):
        if self.idx:
            self.z += np.bincount(np.concatenate(self.idx), np.concatenate(self.val), minlength=self.n)
        self.idx, self.val, self.size = [], [], 0

    def result(self):
        self.flush()
        return self.z


class EbeOperator:
    """A_n of one level, element by element (no global matrix)."""

    def __init__(self, lev, params, tau, ds=False):
        self.lev = lev
        self.ds = ds
        self.params = full_params(params, lev.r)
        self.tau = float(tau)
        self.t_hat, self.w_hat, self.chi_m1, self.T = temporal_constants(lev.k)
        self.th = 0.5 * self.tau * self.w_hat
        self.forms = ElementForms(lev.d, lev.r, lev.h, self.params)
        self.dofs, self.cells = all_cell_dofs(lev)
        d = lev.d
        code = np.zeros(lev.n_cells, dtype=np.int64)
        for f in range(2 * d):
            a, s = f // 2, f % 2
            on = self.cells[:, a] == (0 if s == 0 else lev.n[a] - 1)
            if lev.bc_u[f] == BC_DIRICHLET:
                code |= on.astype(np.int64) << f
            if lev.bc_p[f] == BC_DIRICHLET:
                code |= on.astype(np.int64) << (6 + f)
        self.groups = []     # (key, cell indices) per cell type, types in ascending code order
        for c in np.unique(code):
            du = tuple(f for f in range(2 * d) if (c >> f) & 1)
            dp = tuple(f for f in range(2 * d) if (c >> (6 + f)) & 1)
            self.groups.append(((du, dp), np.nonzero(code == c)[0]))
        self._mats, self._E = {}, {}

    def mats(self, key):
        if key not in self._mats:
            self._mats[key] = self.forms.matrices(*key)
        return self._mats[key]

    def E(self, key):
        if key not in self._E:
            self._E[key] = slab_element_matrix(self.mats(key), self.T, self.th, self.ds)
        return self._E[key]

    def apply(self, x, xcells=None):
        """y = A_n x: y[D_K] += E_type(K) x[D_K] over all cells K (xcells = (c0, c1): only the cells with x-index in
        [c0, c1), i.e. the rows of those cells' DoFs get partial sums; used for bounded timing samples)."""
        acc = _Accumulator(self.lev.N)
        for key, cells in self.groups:
            E = self.E(key)
            if xcells is not None:
                cx = self.cells[cells, 0]
                cells = cells[(cx >= xcells[0]) & (cx < xcells[1])]
            for i in range(0, len(cells), CHUNK):
                D = self.dofs[cells[i:i + CHUNK]]
                acc.add(D, x[D] @ E.T)
        return acc.result()

    def residual(self, b, x):
        return b - self.apply(x)

    def spatial_apply(self, name, v):
        """One spatial matrix of the level (``Mrho``, ``Mc``, ``A``, ``C``, ``Cvol``, ...) applied element by element to
        a node vector: Mrho / A act on length-R vectors, Mc / B on length-S ones, C / Cvol map R -> S."""
        lev = self.lev
        d, nql, npl = lev.d, (lev.r + 1) ** lev.d, lev.r ** lev.d
        qn = self.dofs[:, :nql] - lev.offset(0, FIELD_V, 0)
        pn = self.dofs[:, 2 * d * nql: 2 * d * nql + npl] - lev.offset(0, FIELD_P)
        vec = np.concatenate([qn + c * lev.nq for c in range(d)], axis=1)
        rows, cols, nout = {"Mrho": (vec, vec, lev.R), "A": (vec, vec, lev.R), "Mc": (pn, pn, lev.S),
                            "B": (pn, pn, lev.S), "C": (pn, vec, lev.S), "Cvol": (pn, vec, lev.S)}[name]
        acc = _Accumulator(nout)
        for key, cells in self.groups:
            M = self.mats(key)[name]
            for i in range(0, len(cells), CHUNK):
                sel = cells[i:i + CHUNK]
                acc.add(rows[sel], v[cols[sel]] @ M.T)
        return acc.result()


class EbeTransfer:
    """P: level l-1 -> l by nodal interpolation, per (Radau node, field, component) block (reading A15)."""

    def __init__(self, coarse, fine):
        self.coarse, self.fine = coarse, fine
        d, r = fine.d, fine.r
        self.Pq = [interp_1d(coarse.n[a], r) for a in range(d)]
        self.Pp = [interp_1d(coarse.n[a], r - 1) for a in range(d)]

    @staticmethod
    def _kron_apply(v, shape_in, mats, transpose):
        """(M_{d-1} (x) ... (x) M_0) v for a lexicographic (axis 0 fastest) node vector v."""
        d = len(shape_in)
        X = v.reshape(tuple(reversed(shape_in)))          # C order: the last array axis is axis 0
        for a in range(d):
            M = mats[a].T if transpose else mats[a]
            ax = d - 1 - a
            X = np.moveaxis(np.tensordot(M, X, axes=([1], [ax])), 0, ax)
        return np.ascontiguousarray(X).ravel()

    def _blocks(self, lev):
        for m in range(lev.k + 1):
            for f, nc in ((FIELD_V, lev.d), (FIELD_U, lev.d), (FIELD_P, 1)):
                for c in range(nc):
                    o = lev.offset(m, f, c)
                    yield f, o, (lev.np_ if f == FIELD_P else lev.nq)

    def prolong(self, xc):
        c, f = self.coarse, self.fine
        out = np.empty(f.N)
        for (fld, oc, nc), (_, of, nf) in zip(self._blocks(c), self._blocks(f)):
            shape, mats = (c.p_shape, self.Pp) if fld == FIELD_P else (c.q_shape, self.Pq)
            out[of:of + nf] = self._kron_apply(xc[oc:oc + nc], shape, mats, False)
        return out

    def restrict(self, xf):
        c, f = self.coarse, self.fine
        out = np.empty(c.N)
        for (fld, oc, nc), (_, of, nf) in zip(self._blocks(c), self._blocks(f)):
            shape, mats = (f.p_shape, self.Pp) if fld == FIELD_P else (f.q_shape, self.Pq)
            out[oc:oc + nc] = self._kron_apply(xf[of:of + nf], shape, mats, True)
        return out


class EbeSmoother:
    """Algorithm 1 on one level with one equilibrated inverse per patch class, patch index sets built per class."""

    def __init__(self, op, omega=0.7):
        self.op, self.lev, self.omega = op, op.lev, omega
        lev, d, r = op.lev, op.lev.d, op.lev.r
        self.lite = LiteOperator(lev, op.params, op.tau)
        self.lite._E = {key: op.E(key) for key, _ in op.groups}    # the same element slab matrices
        if op.ds:
            raise NotImplementedError("EbeSmoother: DS formulation not wired (assembled oracle only)")
        per_axis = []
        for a in range(d):
            cls = {}
            for v in range(lev.n[a] + 1):
                cls.setdefault(axis_class(v, lev.n[a]), []).append(v)
            per_axis.append(cls)
        self.classes = []     # (key, member vertex array (nm, d) lexicographic, Z_rep, isP mask, inverse)
        for key in itertools.product(*[sorted(per_axis[a]) for a in reversed(range(d))]):
            key = tuple(reversed(key))                              # x fastest over the class keys
            axes = [np.array(per_axis[a][key[a]]) for a in range(d)]
            grids = np.meshgrid(*axes, indexing="ij")
            verts = np.stack([g.ravel(order="F") for g in grids], axis=1)   # lexicographic, x fastest
            rep = tuple(int(t) for t in verts[0])
            Zrep, AP, _ = self.lite.patch_system(rep)
            isP = np.zeros(len(Zrep), dtype=bool)
            for m in range(lev.k + 1):
                o = lev.offset(m, FIELD_P)
                isP |= (Zrep >= o) & (Zrep < o + lev.np_)
            self.classes.append((key, verts, Zrep, isP, equilibrated_inverse(AP)))
        acc = _Accumulator(lev.N)
        for Z in self._index_blocks():
            acc.add(Z, np.ones(Z.shape))
        self.p = acc.result()
        if np.any(self.p == 0):
            raise ValueError("a DoF lies in no patch (S:L357)")

    def _anchors(self, verts):
        lev, r = self.lev, self.lev.r
        lo = np.maximum(verts - 1, 0)
        qa = sum(r * lo[:, a] * int(lev.q_strides[a]) for a in range(lev.d))
        pa = sum((r - 1) * lo[:, a] * int(lev.p_strides[a]) for a in range(lev.d))
        return qa, pa

    def _class_blocks(self, ci):
        """Z(P) of the members of class ci in lexicographic blocks: Z = Z_rep + shift of the patch box."""
        key, verts, Zrep, isP, _ = self.classes[ci]
        qa, pa = self._anchors(verts)
        for i in range(0, len(verts), CHUNK):
            dq = qa[i:i + CHUNK] - qa[0]
            dp = pa[i:i + CHUNK] - pa[0]
            yield Zrep[None, :] + np.where(isP[None, :], dp[:, None], dq[:, None])

    def _index_blocks(self):
        for ci in range(len(self.classes)):
            yield from self._class_blocks(ci)

    def partial_sweep(self, b, d, x0, x1):
        """The work of one sweep restricted to the patches whose vertex x-index lies in [x0, x1): the residual on the
        cells that touch their Z(P) (x-index x0-2 .. x1), their local solves and their contributions to z.  A bounded
        timing sample of ``sweep`` (bench.py); returns the partial z."""
        r = b if d is None else b - self.op.apply(d, (x0 - 2, x1 + 1))
        acc = _Accumulator(self.lev.N)
        for ci, (_key, verts, _Z, _isP, inv) in enumerate(self.classes):
            sel = (verts[:, 0] >= x0) & (verts[:, 0] < x1)
            if not sel.any():
                continue
            for j, Z in enumerate(self._class_blocks(ci)):
                lo, hi = j * CHUNK, min((j + 1) * CHUNK, len(verts))
                m = sel[lo:hi]
                if m.any():
                    acc.add(Z[m], r[Z[m]] @ inv.T)
        return acc.result()

    def patch_dofs(self):
        """{vertex tuple: Z(P)} (tests)."""
        out = {}
        for ci, (key, verts, *_rest) in enumerate(self.classes):
            rows = np.concatenate(list(self._class_blocks(ci)))
            for v, Z in zip(verts, rows):
                out[tuple(int(t) for t in v)] = Z
        return out

    def sweep(self, b, d):
        """One smoothing step (reading A17): d + omega * (sum_P E_P A_P^{-1} R_P r) / p, r = b - A d."""
        r = b if d is None else b - self.op.apply(d)
        acc = _Accumulator(self.lev.N)
        for ci, (_key, _verts, _Z, _isP, inv) in enumerate(self.classes):
            for Z in self._class_blocks(ci):
                acc.add(Z, r[Z] @ inv.T)
        z = acc.result()
        base = np.zeros_like(b) if d is None else d
        return base + self.omega * z / self.p

    def smooth(self, b, d=None, steps=4):
        """Alg. 1 from d = 0 (pre-smoothing) or continuing from d (post-smoothing, reading A13)."""
        for _ in range(steps):
            d = self.sweep(b, d)
        return d

    def k2_flops(self):
        return sum(2.0 * len(Z) ** 2 * len(v) for _k, v, Z, _p, _i in self.classes)


class EbeHierarchy:
    """Levels, element-by-element operators, transfers, lazily built smoothers, V-cycle."""

    def __init__(self, d, cells, lo, hi, r, k, nlevels, params, tau, bc_u=None, bc_p=None, omega=0.7, jmax=4):
        self.levels = hierarchy(d, cells, lo, hi, r, k, nlevels, bc_u, bc_p)
        self.ops = [EbeOperator(lv, params, tau) for lv in self.levels]
        self.T = [None] + [EbeTransfer(self.levels[l - 1], self.levels[l]) for l in range(1, nlevels)]
        self.params, self.tau, self.omega, self.jmax = params, tau, omega, jmax
        self._sm = {}
        self._coarse_inv = None

    @classmethod
    def from_config(cls, cfg, levels=None):
        d = cfg["dim"]
        p = dict(cfg["params"])
        p["K"] = np.array(p["K"], dtype=float).reshape(3, 3)[:d, :d].ravel().tolist()
        return cls(d, cfg["cells"][:d], cfg["lo"][:d], cfg["hi"][:d], cfg["r"], cfg["k"], levels or cfg["levels"],
                   p, cfg["tau"], bc_u=list(cfg["bc_u"][:2 * d]), bc_p=list(cfg["bc_p"][:2 * d]))

    @property
    def fine(self):
        return self.levels[-1]

    @property
    def fine_op(self):
        return self.ops[-1]

    def smoother(self, l):
        if l not in self._sm:
            self._sm[l] = EbeSmoother(self.ops[l], self.omega)
        return self._sm[l]

    def coarse_inv(self):
        if self._coarse_inv is None:
            A0 = SlabOperator(self.levels[0], self.params, self.tau).assemble().toarray()
            self._coarse_inv = equilibrated_inverse(A0)
        return self._coarse_inv

    def vcycle(self, b, l=None):
        if l is None:
            l = len(self.levels) - 1
        if l == 0:
            return self.coarse_inv() @ b
        sm = self.smoother(l)
        d = sm.smooth(b, None, self.jmax)
        r = b - self.ops[l].apply(d)
        dc = self.vcycle(self.T[l].restrict(r), l - 1)
        d = d + self.T[l].prolong(dc)
        return sm.smooth(b, d, self.jmax)


def ebe_slab_rhs(H, cfg, n, X_prev=None):
    """F_{n+1} = L_{n+1} + J X_n of slab n (0-based, t_n = n tau) for a BASELINE config (loads.py).
    X_prev None: the config's initial state X_0 (zero, or the interpolated manufactured data, reading A20)."""
    from stgmg_inputs import uniform_load
    from .loads import manufactured_baseline, load_vectors, traction_face_vector, interpolate_initial
    op, lev = H.fine_op, H.fine
    d = lev.d
    tn = n * cfg["tau"]
    t_nodes = tn + 0.5 * cfg["tau"] * (op.t_hat + 1.0)
    F = np.zeros(lev.N)
    if X_prev is not None:
        o = lev.k * lev.block
        V, U, P = X_prev[o:o + lev.R], X_prev[o + lev.R:o + 2 * lev.R], X_prev[o + 2 * lev.R:o + lev.block]
    elif cfg["load"] == "manufactured":
        sol = manufactured_baseline(d, op.params)
        U, V, P = interpolate_initial(lev, sol, 0.0)
    else:
        U = V = P = None
    if U is not None:
        MU, MV, MP = op.spatial_apply("Mrho", U), op.spatial_apply("Mrho", V), op.spatial_apply("Mc", P)
        for b in range(lev.k + 1):
            o = b * lev.block
            F[o:o + lev.R] += op.chi_m1[b] * MU
            F[o + lev.R:o + 2 * lev.R] += op.chi_m1[b] * MV
            F[o + 2 * lev.R:o + lev.block] += op.chi_m1[b] * MP
    if cfg["load"] == "random":
        F += uniform_load(lev.N, cfg["seed"] or 1)
    elif cfg["load"] == "manufactured":
        sol = manufactured_baseline(d, op.params)
        for b, t in enumerate(t_nodes):
            Fl, Gl = load_vectors(lev, sol, t)
            o = b * lev.block
            F[o + lev.R:o + 2 * lev.R] += op.th[b] * Fl
            F[o + 2 * lev.R:o + lev.block] += op.th[b] * Gl
    else:   # beam: + sin(pi t / 2) int_{x = hi} chi_{d-1} (reading A23)
        face = traction_face_vector(lev, 1, d - 1, 1.0)
        for b, t in enumerate(t_nodes):
            o = b * lev.block
            F[o + lev.R:o + 2 * lev.R] += op.th[b] * np.sin(np.pi * t / 2.0) * face
    return F


def fgmres_iterations(H, b, iterations, restart=30):
    """`iterations` Arnoldi steps of FGMRES(restart) preconditioned by the V-cycle (x0 = 0, tol 0: no early stop)."""
    A = H.fine_op.apply
    return fgmres(A, b, H.vcycle, tol=0.0, restart=restart, maxit=iterations)


def level_k2_flops(lev, params, tau):
    """2 sum_P C_P^2 of one sweep on a level, from the patch shapes alone (no inverses)."""
    lite = LiteOperator(lev, params, tau)
    total = 0.0
    counts = {}
    for v in itertools.product(*[range(n + 1) for n in lev.n]):
        key = tuple(axis_class(v[a], lev.n[a]) for a in range(lev.d))
        counts[key] = (counts.get(key, (v, 0))[0], counts.get(key, (v, 0))[1] + 1)
    for key, (rep, cnt) in counts.items():
        total += 2.0 * len(lite.patch_dofs(rep)) ** 2 * cnt
    return total


def vcycle_k2_flops(H):
    """K2 flops of one V-cycle: 2 J_max sweeps per smoothed level, 2 sum_P C_P^2 each."""
    return sum(2 * H.jmax * level_k2_flops(H.levels[l], H.params, H.tau) for l in range(1, len(H.levels)))
