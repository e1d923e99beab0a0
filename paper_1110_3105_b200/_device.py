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

    def __init__(self, coords, perm, normals=None, weights=None, curvatures=None, resident=None):
        """Upload (or reuse, via ``resident``: a ResidentPoints in original
        order) the point data and gather it into tree order on the device."""
        torch = _native.require_cuda()
        perm = np.asarray(perm, dtype=np.int64)
        if resident is None:
            resident = ResidentPoints(coords, normals, weights, curvatures)
        self.n, self.dim = resident.n, resident.dim
        self.perm = perm
        self.orig = torch.from_numpy(np.ascontiguousarray(perm)).to("cuda", non_blocking=False)
        L = _native.lib()
        st = _native.stream_ptr()

        def gather(src):
            if src is None:
                return None
            dst = torch.empty_like(src)
            _native.check(L.skel_permute_rows(_native.ptr(self.orig), self.n, _native.ptr(src),
                                              _native.ptr(dst), 1, 0, 0, st), "gather")
            return dst

        r = resident
        self.x, self.y, self.z = gather(r.x), gather(r.y), gather(r.z)
        self.nx, self.ny, self.nz = gather(r.nx), gather(r.ny), gather(r.nz)
        self.w, self.curv = gather(r.w), gather(r.curv)
        self.coincide_tol = r.coincide_tol


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


class ResidentPoints:
    """A point set's SoA arrays in ORIGINAL order on the device (uploaded
    once; tree orderings are gathered from it on the device)."""

    def __init__(self, coords, normals=None, weights=None, curvatures=None):
        _native.require_cuda()
        from ._staging import Packer
        coords = np.asarray(coords, dtype=np.float64)
        self.n, self.dim = coords.shape
        # one pinned staging block, one async copy for all SoA arrays
        pk = Packer()
        names = ["x", "y", "z"][:self.dim]
        cols = [np.ascontiguousarray(coords[:, j]) for j in range(self.dim)]
        for j, nm in enumerate(names):
            pk.add(nm, cols[j])
        if normals is not None:
            nt = np.asarray(normals, dtype=np.float64)
            for j, nm in enumerate(["nx", "ny", "nz"][:self.dim]):
                pk.add(nm, nt[:, j])
        if weights is not None:
            pk.add("w", np.asarray(weights, dtype=np.float64).reshape(-1))
        if curvatures is not None:
            pk.add("curv", np.asarray(curvatures, dtype=np.float64).reshape(-1))
        t = pk.upload()
        self._buf = t["_buffer"]
        for nm in ("x", "y", "z", "nx", "ny", "nz", "w", "curv"):
            setattr(self, nm, t.get(nm))
        # ptp / |.|max from per-column extrema (contiguous reductions; a
        # strided axis-0 reduce of an (N, d) array is ~20x slower)
        lo = [float(v.min()) for v in cols]
        hi = [float(v.max()) for v in cols]
        span = max(max(h - l for l, h in zip(lo, hi)), max(max(abs(l), abs(h)) for l, h in zip(lo, hi)),
                   1.0)
        self.coincide_tol = 1e-14 * span
