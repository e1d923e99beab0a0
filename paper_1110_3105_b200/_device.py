"""Device-resident geometry and the SkelSource descriptor (the GPU form of
the matrix-source protocol, skel.py:289-290)."""

import numpy as np

from . import _native


class DeviceGeometry:
    """Tree-ordered SoA geometry on the current CUDA device.

    ``coincide_tol`` = 1e-14 * max(extent, max|coord|, 1) over the whole point
    set: the reference's per-block threshold (kernels.py:111-118) can only be
    larger (proxy blocks include the proxy ring), and the two differ only for
    pairs closer than ~1e-13 -- which the BASELINE geometries never have
    (spacing >= 1e-5)."""

    def __init__(self, coords, perm, normals=None, weights=None, curvatures=None):
        torch = _native.require_cuda()
        coords = np.asarray(coords, dtype=np.float64)
        perm = np.asarray(perm, dtype=np.int64)
        self.n, self.dim = coords.shape
        dev = torch.device("cuda")
        ct = coords[perm]
        put = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
        self.x = put(ct[:, 0])
        self.y = put(ct[:, 1])
        self.z = put(ct[:, 2]) if self.dim == 3 else None
        if normals is not None:
            nt = np.asarray(normals, dtype=np.float64)[perm]
            self.nx, self.ny = put(nt[:, 0]), put(nt[:, 1])
            self.nz = put(nt[:, 2]) if self.dim == 3 else None
        else:
            self.nx = self.ny = self.nz = None
        self.w = None if weights is None else put(np.asarray(weights, dtype=np.float64)[perm])
        self.curv = None if curvatures is None else put(np.asarray(curvatures, dtype=np.float64)[perm])
        self.orig = put(perm)
        self.perm = perm
        span = max(float(np.ptp(coords, axis=0).max()), float(np.abs(coords).max()), 1.0)
        self.coincide_tol = 1e-14 * span
        self.host_weights = None if weights is None else np.asarray(weights, dtype=np.float64)[perm]

    def source(self, kind, equation, layer=1, k=0.0, identity_coef=0.0, diag=0.0, wscale=1.0,
               curvature_limit=False, kr10=False, weighted=True):
        p = _native.ptr
        s = _native.SkelSource()
        s.x, s.y, s.z = p(self.x), p(self.y), p(self.z)
        s.nx, s.ny, s.nz = p(self.nx), p(self.ny), p(self.nz)
        s.w = p(self.w) if weighted else None
        s.curv = p(self.curv)
        s.orig = p(self.orig)
        s.n = self.n
        s.dim = self.dim
        s.kind = kind
        s.equation = equation
        s.layer = layer
        s.curvature_limit = int(bool(curvature_limit))
        s.kr10 = int(bool(kr10))
        s.k = float(k)
        s.identity_coef = float(identity_coef)
        s.diag = float(diag)
        s.wscale = float(wscale)
        s.coincide_tol = self.coincide_tol
        return s
