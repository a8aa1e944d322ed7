"""Geometric multigrid V-cycle (oracle; test infrastructure only).

P:L433-440: one V-cycle per preconditioner application; prolongation by interpolation, restriction by its
transpose; J_max = 4 pre- and post-smoothing steps on every level l = 1..L; direct solve on T_0.
Level operators are rediscretised (reading A14).  Coarse solve = equilibrated explicit inverse (reading A16).
Pre-smoothing starts from 0, post-smoothing continues from the corrected iterate (reading A13); no
coarse-correction damping.
"""
import numpy as np
from .mesh import hierarchy
from .assembly import SlabOperator
from .transfer import prolongation
from .vanka import Patches, VankaSmoother, equilibrated_inverse


class Hierarchy:
    def __init__(self, d, cells, lo, hi, r, k, nlevels, params, tau, bc_u=None, bc_p=None,
                 omega=0.7, jmax=4, share_classes=True, colored=False, ds=False, cell_patches=False,
                 overwrite=False):
        self.levels = hierarchy(d, cells, lo, hi, r, k, nlevels, bc_u, bc_p)
        self.ops = [SlabOperator(lv, params, tau, ds) for lv in self.levels]
        self.A = [op.assemble() for op in self.ops]
        self.P = [None] + [prolongation(self.levels[l - 1], self.levels[l]) for l in range(1, nlevels)]
        self.jmax = jmax
        self.colored = colored   # N2(i): multiplicative colour-ordered smoother instead of Alg. 1
        self.overwrite = overwrite   # N2(iii): Alg. 1 without averaging
        self.smoothers = [None] + [VankaSmoother(self.A[l], Patches(self.levels[l], cell_patches), omega, share_classes)
                                   for l in range(1, nlevels)]
        self.coarse_inv = equilibrated_inverse(self.A[0].toarray())

    @property
    def fine(self):
        return self.levels[-1]

    def vcycle(self, b, l=None):
        """d = V-cycle(b) on level l (default: finest)."""
        if l is None:
            l = len(self.levels) - 1
        if l == 0:
            return self.coarse_inv @ b
        sm = self.smoothers[l]
        d = sm.smooth(b, None, self.jmax, self.colored, self.overwrite)
        r = b - self.A[l] @ d
        dc = self.vcycle(self.P[l].T @ r, l - 1)
        d = d + self.P[l] @ dc
        return sm.smooth(b, d, self.jmax, self.colored, self.overwrite)
