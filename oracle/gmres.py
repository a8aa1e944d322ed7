"""Flexible GMRES(m), right preconditioned (oracle; test infrastructure only).

P:L354: flexible GMRES [S03] preconditioned by one V-cycle per iteration.  Readings: A2 (right,
flexible; stores Z), A3 (stop when the Givens estimate |g_{j+1}| <= target, confirmed by the true residual),
A4 (restart m, restart from the true residual), A35 (happy breakdown h_{j+1,j} <= 1e-14 beta_cycle; maxit
counts Arnoldi steps).  Modified Gram–Schmidt.
"""
import numpy as np

TOL_REL, TOL_ABS = 0, 1


def fgmres(apply_A, b, precond, x0=None, tol=1e-8, tol_mode=TOL_REL, restart=30, maxit=1000):
    """Return (x, info) with info = dict(iterations, converged, rel_residual, abs_residual, history)."""
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else x0.astype(np.float64).copy()
    bnorm = float(np.sqrt(b @ b))
    target = tol * bnorm if tol_mode == TOL_REL else tol
    its = 0
    history = []
    restarts = 0
    r = b - apply_A(x)
    beta = float(np.sqrt(r @ r))
    history.append(beta)
    if beta <= target:
        return x, dict(iterations=0, converged=True, abs_residual=beta,
                       rel_residual=beta / bnorm if bnorm > 0 else 0.0, history=history, restarts=0)
    while its < maxit:
        m = restart
        Vb = np.zeros((m + 1, n))
        Zb = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        Vb[0] = r / beta
        j_done = 0
        for j in range(m):
            Zb[j] = precond(Vb[j])
            w = apply_A(Zb[j])
            for i in range(j + 1):                          # modified Gram–Schmidt
                H[i, j] = w @ Vb[i]
                w = w - H[i, j] * Vb[i]
            hn = float(np.sqrt(w @ w))
            H[j + 1, j] = hn
            for i in range(j):                              # previous Givens rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            rho = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j] = H[j, j] / rho
            sn[j] = H[j + 1, j] / rho
            H[j, j] = rho
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            its += 1
            j_done = j + 1
            history.append(abs(g[j + 1]))
            if abs(g[j + 1]) <= target or hn <= 1e-14 * beta or its >= maxit:
                break
            Vb[j + 1] = w / hn
        y = np.zeros(j_done)
        for i in range(j_done - 1, -1, -1):                 # back substitution
            y[i] = (g[i] - H[i, i + 1:j_done] @ y[i + 1:j_done]) / H[i, i]
        x = x + Zb[:j_done].T @ y
        r = b - apply_A(x)
        beta = float(np.sqrt(r @ r))
        if beta <= target:
            return x, dict(iterations=its, converged=True, abs_residual=beta, rel_residual=beta / bnorm,
                           history=history, restarts=restarts)
        if its >= maxit:
            break
        restarts += 1
    return x, dict(iterations=its, converged=False, abs_residual=beta, rel_residual=beta / bnorm,
                   history=history, restarts=restarts)
