"""Oracle matrix sources (the matrix-source protocol of skel.py:289-290).
TEST INFRASTRUCTURE ONLY (see oracle/__init__).

  * BieSource     -- bie.py:135-176 + bie.py:233-262 (tree-ordered 2D
                     double-layer Nystrom system, single-layer proxies, row
                     proxies scaled by the mean weight)
  * KernelSource  -- skel.py:100-124, plus an optional ``diag`` added where
                     row == col (BASELINE config 4: "diagonal set to 1",
                     SURVEY App. B ``DiagOneSource``)
  * CfieSource    -- BASELINE config 3 composed from reference pieces
                     (SURVEY F2 / App. B): (D_k - i*kappa*S_k) * KR10 + 1/2 I
"""

import numpy as np

from .entries import eval_block, kr10_factor


class BieSource:
    """Laplace (or Helmholtz) double-layer interior-Dirichlet system in tree
    order.  identity_coef defaults to the reference's -1/2 (bie.py:145)."""

    def __init__(self, curve, perm, equation="laplace", k=0.0,
                 identity_coef=-0.5, quad=None):
        self.equation = equation
        self.k = float(k)
        self.wavenumber = self.k
        self.dim = 2
        self.perm = np.asarray(perm, dtype=np.int64)
        self.n = self.perm.size
        self.ic = float(identity_coef)
        self.quad = quad or ("plain_trapezoid" if equation == "laplace" else "kapur_rokhlin_10")
        self.xy = curve["xy"][self.perm]
        self.nrm = curve["normals"][self.perm]
        self.w = curve["weights"][self.perm]
        self.kap = curve["curvature"][self.perm]
        self.dtype = np.float64 if equation == "laplace" else np.complex128
        self.wscale = float(np.mean(self.w))        # bie.py:251

    def block(self, rows, cols):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        si = "curvature_limit" if self.equation == "laplace" else "zero"
        G = eval_block(self.equation, 2, "double", self.k, self.xy[rows],
                       self.xy[cols], self.nrm[cols], self.w[cols],
                       self.kap[cols], si)
        oi, oj = self.perm[rows], self.perm[cols]
        if self.quad == "kapur_rokhlin_10":
            G = G * kr10_factor(oi, oj, self.n)
        same = oi[:, None] == oj[None, :]
        if same.any():
            G = G + np.where(same, self.ic, 0.0)
        return G

    def proxy_row_block(self, rows, pxy):
        return self.wscale * eval_block(self.equation, 2, "single", self.k,
                                        self.xy[rows], pxy)

    def proxy_col_block(self, cols, pxy):
        return eval_block(self.equation, 2, "single", self.k, pxy,
                          self.xy[cols], src_weights=self.w[cols])


class KernelSource:
    """Plain kernel matrix in tree order (skel.py:100-124); ``diag`` is added
    on coincident tree positions when non-zero."""

    def __init__(self, equation, dim, layer, coords, perm, k=0.0, normals=None,
                 weights=None, diag=0.0):
        self.equation = equation
        self.dim = dim
        self.layer = layer
        self.k = float(k)
        self.wavenumber = self.k
        self.perm = np.asarray(perm, dtype=np.int64)
        self.n = self.perm.size
        self.x = np.asarray(coords, dtype=np.float64)[self.perm]
        self.nrm = None if normals is None else np.asarray(normals)[self.perm]
        self.w = None if weights is None else np.asarray(weights, dtype=np.float64)[self.perm]
        self.diag = float(diag)
        self.dtype = np.float64 if equation == "laplace" else np.complex128

    def block(self, rows, cols):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        G = eval_block(self.equation, self.dim, self.layer, self.k, self.x[rows],
                       self.x[cols],
                       None if self.nrm is None else self.nrm[cols],
                       None if self.w is None else self.w[cols])
        if self.diag != 0.0:
            same = rows[:, None] == cols[None, :]
            if same.any():
                G = G + np.where(same, self.diag, 0.0)
        return G

    def proxy_row_block(self, rows, pxy):
        return eval_block(self.equation, self.dim, "single", self.k, self.x[rows], pxy)

    def proxy_col_block(self, cols, pxy):
        return eval_block(self.equation, self.dim, "single", self.k, pxy, self.x[cols],
                          src_weights=None if self.w is None else self.w[cols])


class CfieSource(BieSource):
    """Combined field I/2 + D_k - i kappa S_k with KR10 on both terms and a
    zero self-interaction."""

    def __init__(self, curve, perm, k):
        super().__init__(curve, perm, equation="helmholtz", k=k,
                         identity_coef=0.5, quad="kapur_rokhlin_10")

    def block(self, rows, cols):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        dl = eval_block("helmholtz", 2, "double", self.k, self.xy[rows], self.xy[cols],
                        self.nrm[cols], self.w[cols])
        sl = eval_block("helmholtz", 2, "single", self.k, self.xy[rows], self.xy[cols],
                        src_weights=self.w[cols])
        oi, oj = self.perm[rows], self.perm[cols]
        G = (dl - 1j * self.k * sl) * kr10_factor(oi, oj, self.n)
        same = oi[:, None] == oj[None, :]
        if same.any():
            G = G + np.where(same, self.ic, 0.0)
        return G
