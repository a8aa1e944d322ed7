"""dG(k) temporal constants of the slab system (oracle; test infrastructure only).

P:L356-362 (Eq:TimeExp): Lagrange basis chi_{n,m} at the k+1 right Gauss–Radau nodes of I_n.
P:L233-256 (Eq:DPQ_A0): the slab problem uses Q_n (Eq:GF) and the jump terms at t_{n-1}^+.
With chi_a(t) = chi_hat_a(t_hat), d/dt = (2/tau) d/dt_hat:
  Q_n(<chi_a, chi_b>)                               = theta_b delta_ab,   theta_b = (tau/2) omega_hat_b
  Q_n(<chi_a', chi_b>) + chi_a(t_{n-1}^+) chi_b(..) = T_ba = omega_hat_b chi_hat_a'(t_hat_b) + chi_hat_a(-1) chi_hat_b(-1)
T is indexed [b, a] (test node b = row, trial node a = column).
"""
import numpy as np
from .basis import radau_right, lagrange_values, lagrange_derivs


def radau(k):
    return radau_right(k)


def temporal_constants(k):
    """Return (t_hat, omega_hat, chi_m1, T) for dG(k): chi_m1[b] = chi_hat_b(-1), T[b, a] as above."""
    t, w = radau_right(k)
    Vm1 = lagrange_values(t, [-1.0])[:, 0]          # chi_hat_a(-1)
    D = lagrange_derivs(t, t)                          # D[a, q] = chi_hat_a'(t_q)
    T = np.zeros((k + 1, k + 1))
    for b in range(k + 1):
        for a in range(k + 1):
            T[b, a] = w[b] * D[a, b] + Vm1[a] * Vm1[b]
    return t, w, Vm1, T


def theta(k, tau):
    """theta_b = (tau/2) omega_hat_b (Eq:GF)."""
    _, w = radau_right(k)
    return 0.5 * tau * w
