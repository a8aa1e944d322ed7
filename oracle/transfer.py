"""Grid transfer (oracle; test infrastructure only).

P:L436: "prolongation to grids by interpolation and application of the transpose operator for restriction".
Prolongation P_l: level l-1 -> l is nodal interpolation of the coarse Q_r (velocity, displacement components)
and Q_{r-1} (pressure) functions at the fine nodes, per Radau node and field (no temporal coarsening, reading
A15).  Restriction = P_l^T.  Built as the Kronecker product of 1D interpolation matrices (the coarse
Lagrange basis evaluated at the fine nodes), then block-diagonal over (m, f, c).
"""
import numpy as np
import scipy.sparse as sp
from .basis import gauss_lobatto_nodes01, lagrange_values


def interp_1d(n_coarse, deg):
    """(deg*2n+1) x (deg*n+1) matrix: coarse Q_deg function on n cells evaluated at the fine nodes (2n cells)."""
    nodes = gauss_lobatto_nodes01(deg)
    nf, nc = deg * 2 * n_coarse + 1, deg * n_coarse + 1
    P = np.zeros((nf, nc))
    for cf in range(2 * n_coarse):
        cc = cf // 2
        xf = 0.5 * ((cf % 2) + nodes)          # fine nodes of fine cell cf in coarse-cell coordinates
        V = lagrange_values(nodes, xf)         # V[j, i] = l_j(xf_i)
        for i in range(deg + 1):
            for j in range(deg + 1):
                P[deg * cf + i, deg * cc + j] = V[j, i]
    return P


def prolongation(coarse, fine):
    """Sparse P: R^{N_coarse} -> R^{N_fine}."""
    d, r = fine.d, fine.r

    def kron_axes(deg):
        M = sp.identity(1, format="csr")
        for a in range(d):                      # axis 0 fastest -> outermost Kronecker factor is the last axis
            Pa = sp.csr_matrix(interp_1d(coarse.n[a], deg))
            M = sp.kron(Pa, M, format="csr")
        return M

    Pq = kron_axes(r)
    Pp = kron_axes(r - 1)
    blocks = []
    for m in range(fine.k + 1):
        blocks += [Pq] * (2 * d) + [Pp]
    return sp.block_diag(blocks, format="csr")
