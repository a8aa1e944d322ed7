"""1D quadrature rules and Lagrange bases (oracle; test infrastructure only).

P:L122-128 (Eq:GF): right-sided (k+1)-point Gauss–Radau rule on [-1,1], exact on P_{2k}, last node = +1.
P:L148 (Def:VhQh): Q_r / Q_{r-1} Lagrange elements.  Node layout is unstated; reading A9 = Gauss–Lobatto
nodes (equispaced for r = 2).
Spatial quadrature: (r+1)-point Gauss–Legendre per axis (reading A10), exact for every operator integrand on
affine axis-aligned cells.
"""
import numpy as np
from numpy.polynomial import legendre as L


def gauss_legendre(n):
    """n-point Gauss–Legendre rule on [-1, 1] (library primitive numpy.leggauss)."""
    x, w = L.leggauss(n)
    return np.asarray(x, dtype=np.float64), np.asarray(w, dtype=np.float64)


def gauss_legendre01(n):
    """n-point Gauss–Legendre rule mapped to [0, 1]."""
    x, w = gauss_legendre(n)
    return 0.5 * (x + 1.0), 0.5 * w


def gauss_lobatto_nodes(r):
    """r+1 Gauss–Lobatto–Legendre nodes on [-1, 1]: the endpoints and the roots of P_r' (reading A9)."""
    if r < 1:
        raise ValueError("r >= 1")
    if r == 1:
        return np.array([-1.0, 1.0])
    c = np.zeros(r + 1)
    c[r] = 1.0
    inner = np.sort(np.real(L.legroots(L.legder(c))))
    return np.concatenate([[-1.0], inner, [1.0]])


def gauss_lobatto_nodes01(r):
    return 0.5 * (gauss_lobatto_nodes(r) + 1.0)


def radau_right(k):
    """Right (k+1)-point Gauss–Radau rule on [-1,1] (Eq:GF).

    Nodes: roots of P_{k+1} - P_k (these include t = +1).  Weights: solution of the moment equations
    sum_j w_j t_j^i = int_{-1}^{1} t^i dt, i = 0..k (a (k+1)x(k+1) Vandermonde solve)."""
    if k == 0:
        return np.array([1.0]), np.array([2.0])
    c = np.zeros(k + 2)
    c[k + 1] = 1.0
    c[k] -= 1.0
    t = np.sort(np.real(L.legroots(c)))
    t[-1] = 1.0  # the root at +1 is exact; remove its rounding
    V = np.vander(t, k + 1, increasing=True).T  # V[i, j] = t_j^i
    mom = np.array([(1.0 - (-1.0) ** (i + 1)) / (i + 1) for i in range(k + 1)])
    w = np.linalg.solve(V, mom)
    return t, w


def lagrange_values(nodes, x):
    """V[i, q] = l_i(x_q) for the Lagrange basis on ``nodes`` (plain product formula)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    V = np.ones((n, len(x)))
    for i in range(n):
        for j in range(n):
            if j != i:
                V[i] *= (x - nodes[j]) / (nodes[i] - nodes[j])
    return V


def lagrange_derivs(nodes, x):
    """D[i, q] = l_i'(x_q) by the product rule: l_i' = sum_m 1/(x_i-x_m) prod_{j != i,m} (x-x_j)/(x_i-x_j)."""
    nodes = np.asarray(nodes, dtype=np.float64)
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    n = len(nodes)
    D = np.zeros((n, len(x)))
    for i in range(n):
        for m in range(n):
            if m == i:
                continue
            term = np.full(len(x), 1.0 / (nodes[i] - nodes[m]))
            for j in range(n):
                if j != i and j != m:
                    term = term * (x - nodes[j]) / (nodes[i] - nodes[j])
            D[i] += term
    return D
