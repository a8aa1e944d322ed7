"""Structured multigrid levels and the slab DoF layout (oracle; test infrastructure only).

P:L130: nested quad/hex hierarchy, h_l = gamma h_{l-1}; here gamma = 1/2 on an axis-aligned box.
P:L379-382 (Eq:DefXn): X_n = (V_1, U_1, P_1, ..., V_{k+1}, U_{k+1}, P_{k+1}).
Within V and U the d components are stored one after another; nodes are lexicographic, x fastest
(reading O1 / A12).  Q_r nodes per axis: r*n+1; Q_{r-1} nodes per axis: (r-1)*n+1 (Taylor–Hood,
continuous pressure, P:L138 Def:Qh).  Dirichlet data are imposed by Nitsche, so no DoF is
eliminated.
"""
import itertools
import numpy as np

FIELD_V, FIELD_U, FIELD_P = 0, 1, 2
BC_DIRICHLET, BC_NEUMANN = 0, 1


def lex_strides(shape):
    s = [1]
    for n in shape[:-1]:
        s.append(s[-1] * n)
    return np.array(s, dtype=np.int64)


class Level:
    """One level T_l of the hierarchy: a box [lo, hi] split into cells[a] equal cells per axis."""

    def __init__(self, d, cells, lo, hi, r, k, bc_u=None, bc_p=None):
        self.d = int(d)
        self.n = tuple(int(c) for c in cells[:d])
        self.lo = np.array(lo[:d], dtype=np.float64)
        self.hi = np.array(hi[:d], dtype=np.float64)
        self.h = (self.hi - self.lo) / np.array(self.n, dtype=np.float64)
        self.r, self.k = int(r), int(k)
        self.bc_u = list(bc_u) if bc_u is not None else [BC_DIRICHLET] * (2 * d)
        self.bc_p = list(bc_p) if bc_p is not None else [BC_DIRICHLET] * (2 * d)
        self.q_shape = tuple(self.r * n + 1 for n in self.n)
        self.p_shape = tuple((self.r - 1) * n + 1 for n in self.n)
        self.nq = int(np.prod(self.q_shape))
        self.np_ = int(np.prod(self.p_shape))
        self.R = self.d * self.nq
        self.S = self.np_
        self.block = 2 * self.R + self.S
        self.N = (self.k + 1) * self.block
        self.q_strides = lex_strides(self.q_shape)
        self.p_strides = lex_strides(self.p_shape)
        self.n_cells = int(np.prod(self.n))

    def coarsen(self):
        return Level(self.d, [n // 2 for n in self.n], self.lo, self.hi, self.r, self.k, self.bc_u, self.bc_p)

    # --- DoF layout (Eq:DefXn) ---------------------------------------------------------------
    def offset(self, m, f, c=0):
        base = m * self.block
        if f == FIELD_V:
            return base + c * self.nq
        if f == FIELD_U:
            return base + self.R + c * self.nq
        return base + 2 * self.R

    def cells(self):
        """All cells, lexicographic (x fastest)."""
        return [tuple(reversed(t)) for t in itertools.product(*[range(n) for n in reversed(self.n)])]

    def cell_local_nodes(self, deg):
        """Local node multi-indices of Q_deg on a cell, lexicographic x fastest."""
        return [tuple(reversed(t)) for t in itertools.product(*[range(deg + 1)] * self.d)]

    def cell_q_nodes(self, cell):
        loc = self.cell_local_nodes(self.r)
        return np.array([sum((self.r * cell[a] + j[a]) * self.q_strides[a] for a in range(self.d)) for j in loc],
                        dtype=np.int64)

    def cell_p_nodes(self, cell):
        deg = self.r - 1
        loc = self.cell_local_nodes(deg)
        return np.array([sum((deg * cell[a] + j[a]) * self.p_strides[a] for a in range(self.d)) for j in loc],
                        dtype=np.int64)

    def cell_dofs(self, cell):
        """Global DoFs of a cell in element order (m, f, c, local node)."""
        qn = self.cell_q_nodes(cell)
        pn = self.cell_p_nodes(cell)
        out = []
        for m in range(self.k + 1):
            for c in range(self.d):
                out.append(self.offset(m, FIELD_V, c) + qn)
            for c in range(self.d):
                out.append(self.offset(m, FIELD_U, c) + qn)
            out.append(self.offset(m, FIELD_P) + pn)
        return np.concatenate(out)

    def cell_boundary_faces(self, cell):
        """Faces (2a + s) of the cell that lie on the boundary of the box."""
        fs = []
        for a in range(self.d):
            if cell[a] == 0:
                fs.append(2 * a)
            if cell[a] == self.n[a] - 1:
                fs.append(2 * a + 1)
        return tuple(fs)

    def cell_type(self, cell):
        """Element matrices depend only on which faces are Dirichlet faces for u and for p."""
        bf = self.cell_boundary_faces(cell)
        du = tuple(f for f in bf if self.bc_u[f] == BC_DIRICHLET)
        dp = tuple(f for f in bf if self.bc_p[f] == BC_DIRICHLET)
        return du, dp

    # --- node coordinates -----------------------------------------------------------------------
    def node_coords(self, deg, nodes01):
        """Coordinates of all global Q_deg nodes (lexicographic), for 1D node set ``nodes01`` on [0,1]."""
        axes = []
        for a in range(self.d):
            n = self.n[a]
            xs = np.empty(deg * n + 1)
            for c in range(n):
                xs[deg * c: deg * c + deg + 1] = self.lo[a] + (c + nodes01) * self.h[a]
            axes.append(xs)
        grids = np.meshgrid(*axes, indexing="ij")
        # lexicographic x fastest = Fortran order of the ij grid
        return np.stack([g.ravel(order="F") for g in grids], axis=1)


def hierarchy(d, cells, lo, hi, r, k, nlevels, bc_u=None, bc_p=None):
    """Levels 0 (coarse) .. nlevels-1 (fine); BASELINE's 'levels' counts the coarse level (reading O1)."""
    fine = Level(d, cells, lo, hi, r, k, bc_u, bc_p)
    for a in range(d):
        if fine.n[a] % (2 ** (nlevels - 1)) != 0:
            raise ValueError("cells must be divisible by 2^(levels-1)")
    levs = [fine]
    for _ in range(nlevels - 1):
        levs.append(levs[-1].coarsen())
    return levs[::-1]
