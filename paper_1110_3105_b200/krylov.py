"""Full (unrestarted) GMRES around the GPU operators -- SURVEY 8(f) rank 4,
the Krylov driver of the reference's multiple-scattering application
(solver.py:321-408, bie.py:408-427).

Contract kept from the reference: ``gmres(apply_fn, b, tol, max_iter,
precond)`` returns ``(x, iterations)``; the operator may be a callable or a
dense matrix; a preconditioner is applied on the left (the residual that is
tested is the preconditioned one, relative to |M b|); ``max_iter`` defaults
to and is capped at n; a zero right-hand side returns zeros after 0
iterations; on failure ``NotConverged(x_best, residual, max_iter)``.

Implementation (this module's own design, not the reference's loop):

* ``_Basis`` keeps the orthonormal Krylov vectors as the rows of ONE
  preallocated block and orthogonalises a new vector by classical
  Gram-Schmidt applied twice (CGS2: two block projections V^H w, each a
  single matrix-vector product over the whole basis), which is as stable
  as modified Gram-Schmidt with re-orthogonalisation and turns the inner
  loop into two GEMVs.  When ``b`` is a CUDA tensor and the operator returns
  CUDA tensors the block lives in HBM and the projections run there, so a
  device-resident operator (``apply`` / ``solve_device``) never round-trips
  the iterate through the host.
* ``_RotatedLSQ`` maintains the QR factorisation of the (j+1) x j Hessenberg
  matrix by plane rotations as columns arrive; the last entry of the rotated
  right-hand side is the least-squares residual, so convergence is known
  without forming y, and y is one back substitution at the end.
"""

import numpy as np

from .errors import InvalidInput, NotConverged


def _callable(op):
    if callable(op):
        return op
    M = np.asarray(op)
    return lambda v: M @ v


class _Basis:
    """Rows 0..k of ``V`` are orthonormal; ``add`` orthogonalises a vector
    against them (CGS2) and appends it."""

    def __init__(self, first, kmax, dev):
        self.dev = dev
        n = first.shape[0]
        if dev is not None:
            import torch
            self.V = torch.zeros((kmax + 1, n), dtype=first.dtype, device=dev)
        else:
            self.V = np.zeros((kmax + 1, n), dtype=first.dtype)
        self.V[0] = first
        self.k = 1

    def _proj(self, w):
        B = self.V[:self.k]
        c = B.conj() @ w                    # V^H w
        return c, w - B.T @ c

    def add(self, w):
        """Returns (h, beta): h = V^H w over the current rows (both passes),
        beta = |w - V h|; the normalised remainder becomes row k."""
        c1, w = self._proj(w)
        c2, w = self._proj(w)
        h = c1 + c2
        beta = float(abs(self._norm(w)))
        if beta > 0 and self.k < self.V.shape[0]:
            self.V[self.k] = w / beta
        self.k += 1
        return (h.cpu().numpy() if self.dev is not None else np.asarray(h)), beta

    def _norm(self, w):
        if self.dev is not None:
            import torch
            return torch.linalg.vector_norm(w).item()
        return np.linalg.norm(w)

    def combine(self, y):
        j = y.size
        if self.dev is not None:
            import torch
            return self.V[:j].T @ torch.from_numpy(np.ascontiguousarray(y)).to(self.V)
        return self.V[:j].T @ y


class _RotatedLSQ:
    """min_y |beta e1 - H y| by plane rotations applied column by column."""

    def __init__(self, beta, kmax, dtype):
        self.R = np.zeros((kmax + 1, kmax), dtype=dtype)
        self.rot = []                          # (c, s) of each rotation, c real
        self.z = np.zeros(kmax + 1, dtype=dtype)
        self.z[0] = beta
        self.j = 0

    def add_column(self, h, sub):
        """Append Hessenberg column (h, sub) = (H[:j+1, j], H[j+1, j]);
        returns |residual|, or 0 on an exact (lucky) breakdown."""
        j = self.j
        col = np.zeros(j + 2, dtype=self.R.dtype)
        col[:j + 1] = h
        col[j + 1] = sub
        for i, (c, s) in enumerate(self.rot):
            a, b = col[i], col[i + 1]
            col[i] = c * a + s * b
            col[i + 1] = -np.conj(s) * a + c * b
        a, b = col[j], col[j + 1]
        r = np.hypot(abs(a), abs(b))
        self.j = j + 1
        if r == 0:
            self.R[:j + 2, j] = col
            self.rot.append((1.0, 0.0))
            return 0.0
        u = a / abs(a) if a != 0 else 1.0
        c, s = abs(a) / r, u * np.conj(b) / r
        self.rot.append((c, s))
        col[j], col[j + 1] = u * r, 0.0
        self.R[:j + 2, j] = col
        zj = self.z[j]
        self.z[j], self.z[j + 1] = c * zj, -np.conj(s) * zj
        return abs(self.z[j + 1])

    def solve(self):
        j = self.j
        y = np.zeros(j, dtype=self.R.dtype)
        for i in range(j - 1, -1, -1):
            y[i] = (self.z[i] - self.R[i, i + 1:j] @ y[i + 1:j]) / self.R[i, i]
        return y


def gmres(apply_fn, b, tol=1e-9, max_iter=None, precond=None):
    """Returns (x, iterations); raises NotConverged(x, residual, max_iter)."""
    if not tol > 0:
        raise InvalidInput("tol must be positive")
    A = _callable(apply_fn)
    M = _callable(precond) if precond is not None else (lambda v: v)
    dev = None
    if not isinstance(b, np.ndarray) and hasattr(b, "is_cuda") and b.is_cuda:
        dev = b.device
    else:
        b = np.asarray(b)
    n = int(b.shape[0])
    kmax = n if max_iter is None else min(int(max_iter), n)
    r0 = M(b)
    if dev is not None:
        import torch
        dt = torch.complex128 if r0.is_complex() else torch.float64
        r0 = r0.to(dt)
        beta = torch.linalg.vector_norm(r0).item()
        npdt = np.complex128 if r0.is_complex() else np.float64
    else:
        r0 = np.asarray(r0)
        npdt = np.result_type(r0.dtype, np.float64)
        r0 = r0.astype(npdt)
        beta = float(np.linalg.norm(r0))
    if beta == 0:
        z = np.zeros(n, dtype=npdt)
        return (torch.from_numpy(z).to(dev) if dev is not None else z), 0
    basis = _Basis(r0 / beta, kmax, dev)
    lsq = _RotatedLSQ(beta, kmax, npdt)
    res = 1.0
    for it in range(1, kmax + 1):
        w = M(A(basis.V[it - 1]))
        w = w.to(basis.V.dtype) if dev is not None else np.asarray(w, dtype=npdt)
        h, sub = basis.add(w)
        r = lsq.add_column(h, sub)
        res = r / beta
        if res <= tol:
            return basis.combine(lsq.solve()), it
    raise NotConverged(basis.combine(lsq.solve()), float(res), int(kmax))
