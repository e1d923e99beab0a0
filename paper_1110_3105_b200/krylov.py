"""Full GMRES (reference solver.py:321-408): the Krylov
driver around the GPU operators (``apply`` of a compressed matrix, ``solve``
of a factorization as the preconditioner, or any callable / dense matrix).

Same recurrence and stopping rule as the reference, so iteration counts
agree: modified Gram-Schmidt with one DGKS re-orthogonalisation pass when
the projection removed nearly everything, Givens rotations, relative
residual |g_{j+1}| / beta of the (left-)preconditioned system, no restart,
``NotConverged`` carrying the best iterate.  The small Hessenberg algebra
runs on the host; the operator applications are wherever the callables run.
"""

import numpy as np

from .errors import InvalidInput, NotConverged


def _operator(op):
    if callable(op):
        return op
    M = np.asarray(op)
    return lambda v: M @ v


def gmres(apply_fn, b, tol=1e-9, max_iter=None, precond=None):
    """Returns (x, iterations); raises NotConverged(x, residual, max_iter)."""
    if not tol > 0:
        raise InvalidInput("tol must be positive")
    A = _operator(apply_fn)
    M = _operator(precond) if precond is not None else None
    b = np.asarray(b)
    n = b.shape[0]
    kmax = n if max_iter is None else min(int(max_iter), n)
    r0 = np.asarray(M(b) if M is not None else b)
    dt = np.result_type(r0.dtype, np.float64)
    beta = np.linalg.norm(r0)
    if beta == 0:
        return np.zeros(n, dtype=dt), 0
    V = np.empty((kmax + 1, n), dtype=dt)
    V[0] = r0 / beta
    H = np.zeros((kmax + 1, kmax), dtype=dt)
    cs = np.zeros(kmax + 1, dtype=dt)
    sn = np.zeros(kmax + 1, dtype=dt)
    g = np.zeros(kmax + 1, dtype=dt)
    g[0] = beta

    def solution(j):
        y = np.zeros(j, dtype=dt)
        for i in range(j - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:j] @ y[i + 1:j]) / H[i, i]
        return V[:j].T @ y

    res, j = 1.0, 0
    for j in range(kmax):
        w = A(V[j])
        if M is not None:
            w = M(w)
        w = np.array(w, dtype=dt)
        w0 = np.linalg.norm(w)
        for i in range(j + 1):                      # modified Gram-Schmidt
            h = np.vdot(V[i], w)
            H[i, j] = h
            w -= h * V[i]
        c = V[:j + 1].conj() @ w                    # one DGKS correction pass
        if np.linalg.norm(c) > 1e-10 * max(w0, 1e-300):
            w -= V[:j + 1].T @ c
            H[:j + 1, j] += c
        H[j + 1, j] = np.linalg.norm(w)
        if H[j + 1, j] > 0:
            V[j + 1] = w / H[j + 1, j]
        for i in range(j):                          # previous rotations
            t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
            H[i + 1, j] = -np.conj(sn[i]) * H[i, j] + cs[i] * H[i + 1, j]
            H[i, j] = t
        d = np.sqrt(np.abs(H[j, j]) ** 2 + np.abs(H[j + 1, j]) ** 2)
        if d == 0:
            res = 0.0
            j += 1
            break
        cs[j] = np.abs(H[j, j]) / d
        ph = H[j, j] / np.abs(H[j, j]) if H[j, j] != 0 else 1.0
        sn[j] = ph * np.conj(H[j + 1, j]) / d
        H[j, j] = ph * d
        H[j + 1, j] = 0.0
        g[j + 1] = -np.conj(sn[j]) * g[j]
        g[j] = cs[j] * g[j]
        res = abs(g[j + 1]) / beta
        if res <= tol:
            return solution(j + 1), j + 1
    raise NotConverged(solution(j + 1), float(res), int(kmax))
