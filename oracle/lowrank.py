"""Oracle interpolative decompositions.  TEST INFRASTRUCTURE ONLY.

Restates:
  * pivoted_qr             lowrank.py:48-119  (Householder CPQR, squared-norm
                           downdating, renormalisation every 32 steps, stale
                           recompute below 1e-8 of the reference norm,
                           first-max pivot, stop at pn <= eps*p0 after
                           min_rank steps, stop at pn == 0)
  * _proj_from_qr          lowrank.py:122-133 (P[:, skel] = I, R11^-1 R12)
  * id_fixed_precision     lowrank.py:136-161 (min_rank padding)
  * _spectral_norm_estimate, id_randomized  lowrank.py:169-231
"""

import numpy as np
from scipy.linalg import solve_triangular

RENORM_EVERY = 32          # lowrank.py:19


def _colnorm2(W):
    return np.real(np.einsum("ij,ij->j", W.conj(), W))


def cpqr(A, eps, min_rank=0):
    """Returns (piv, R, rank, ratio) like lowrank.py:48-119."""
    W = np.array(A, order="F", copy=True)
    m, n = W.shape
    cplx = np.iscomplexobj(W)
    piv = np.arange(n)
    nrm = _colnorm2(W)
    ref = nrm.copy()            # by position; not swapped (lowrank.py:64)
    rank, p0, trailing = 0, 0.0, 0.0
    for s in range(min(m, n)):
        if s and s % RENORM_EVERY == 0:
            nrm[s:] = _colnorm2(W[s:, s:])
            ref[s:] = nrm[s:]
        bad = np.nonzero(nrm[s:] < 1e-8 * ref[s:])[0]
        if bad.size:
            cols = s + bad
            nrm[cols] = _colnorm2(W[s:, cols])
            ref[cols] = nrm[cols]
        j = s + int(np.argmax(nrm[s:]))
        pn = np.sqrt(max(nrm[j], 0.0))
        if s == 0:
            p0 = pn
            if p0 == 0.0:
                return piv, W[:0, :], 0, 0.0
        if s >= min_rank and pn <= eps * p0:
            trailing = pn
            break
        if pn == 0.0:
            break
        if j != s:
            W[:, [s, j]] = W[:, [j, s]]
            nrm[[s, j]] = nrm[[j, s]]
            piv[[s, j]] = piv[[j, s]]
        x = W[s:, s]
        x0 = x[0]
        alpha = -(x0 / abs(x0) if x0 != 0 else 1.0) * np.linalg.norm(x)
        v = x.copy()
        v[0] -= alpha
        vv = np.real(np.vdot(v, v))
        if vv > 0:
            W[s:, s + 1:] -= np.outer(v, (v.conj() @ W[s:, s + 1:]) * (2.0 / vv))
        W[s, s] = alpha
        W[s + 1:, s] = 0
        r = W[s, s + 1:]
        nrm[s + 1:] -= (r * r.conj()).real if cplx else r * r
        np.clip(nrm[s + 1:], 0.0, None, out=nrm[s + 1:])
        nrm[s] = 0.0
        rank = s + 1
    return piv, W[:rank, :], rank, (trailing / p0 if p0 > 0 else 0.0)


def interp_matrix(piv, R, rank, n, dtype):
    """lowrank.py:122-133 (without the warning; returns (P, max|P|))."""
    P = np.zeros((rank, n), dtype=dtype)
    if rank:
        P[np.arange(rank), piv[:rank]] = 1.0
        if rank < n:
            P[:, piv[rank:]] = solve_triangular(R[:, :rank], R[:, rank:])
    return P, float(np.abs(P).max(initial=0.0))


def id_fixed(A, eps, min_rank=0):
    """Column ID (lowrank.py:136-161).  Returns (skel, proj, rank, ratio)."""
    A = np.asarray(A)
    if A.dtype.kind not in "fc":
        A = A.astype(np.float64)
    n = A.shape[1]
    piv, R, rank, ratio = cpqr(A, eps, min_rank)
    P, _ = interp_matrix(piv, R, rank, n, A.dtype)
    if rank < min_rank:
        extra = min(min_rank, n) - rank
        padded = piv[rank:rank + extra]
        P[:, padded] = 0.0
        pad = np.zeros((extra, n), dtype=A.dtype)
        pad[np.arange(extra), padded] = 1.0
        P = np.vstack([P, pad])
        rank += extra
    return piv[:rank].copy(), P, rank, ratio


def _norm_estimate(A, rng, iters=8):
    """lowrank.py:169-183."""
    cplx = np.iscomplexobj(A)
    v = rng.standard_normal(A.shape[1])
    if cplx:
        v = v + 1j * rng.standard_normal(A.shape[1])
    v /= np.linalg.norm(v)
    s = 0.0
    for _ in range(iters):
        v = A.conj().T @ (A @ v)
        nv = np.linalg.norm(v)
        s = nv ** 0.5
        if nv == 0:
            return 0.0
        v /= nv
    return float(s)


def id_randomized(A, eps, oversampling=10, seed=0):
    """lowrank.py:186-231: Gaussian sketch with doubling, 5-probe check,
    deterministic fallback.  Returns (skel, proj, rank, err)."""
    A = np.asarray(A)
    m, n = A.shape
    rng = np.random.default_rng(seed)
    cplx = np.iscomplexobj(A)
    normA = _norm_estimate(A, rng)
    if normA == 0.0:
        return np.empty(0, dtype=np.int64), np.zeros((0, n), dtype=A.dtype), 0, 0.0
    ell = 2 * oversampling
    while True:
        if ell >= m:
            return id_fixed(A, eps)
        Om = rng.standard_normal((ell, m))
        if cplx:
            Om = Om + 1j * rng.standard_normal((ell, m))
        piv, R, rank, _ = cpqr(Om @ A, eps)
        if rank <= ell - oversampling:
            break
        ell *= 2
    P, _ = interp_matrix(piv, R, rank, n, A.dtype)
    skel = piv[:rank].copy()
    worst = 0.0
    for _ in range(5):
        v = rng.standard_normal(n)
        if cplx:
            v = v + 1j * rng.standard_normal(n)
        err = np.linalg.norm(A @ v - A[:, skel] @ (P @ v))
        worst = max(worst, err / (normA * np.linalg.norm(v)))
    if worst > 3 * eps:
        return id_fixed(A, eps)
    return skel, P, rank, worst
