"""Kernel specifications and dense kernel blocks (drop-in for
skelkit/kernels.py).  Blocks are evaluated on the GPU by the same entry
routines the compression kernels use (csrc/entries.cuh)."""

from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import DeviceGeometry
from .errors import InvalidInput

COINCIDENT_RTOL = 1e-14   # kernels.py:24


@dataclass(frozen=True)
class KernelSpec:
    """Green's function selector (kernels.py:27-62 contract).

    2D Laplace -log r/(2 pi); 3D Laplace 1/(4 pi r); 2D Helmholtz (i/4) H0(kr);
    3D Helmholtz exp(ikr)/(4 pi r); ``layer="double"`` is the source-normal
    derivative."""

    equation: str
    dim: int
    layer: str = "single"
    wavenumber: float = 0.0
    self_interaction: str = "zero"

    def __post_init__(self):
        if self.equation not in ("laplace", "helmholtz"):
            raise InvalidInput(f"unknown equation {self.equation!r}")
        if self.dim not in (2, 3):
            raise InvalidInput("dim must be 2 or 3")
        if self.layer not in ("single", "double"):
            raise InvalidInput(f"unknown layer {self.layer!r}")
        if self.self_interaction not in ("zero", "curvature_limit"):
            raise InvalidInput(f"unknown self_interaction {self.self_interaction!r}")
        if self.equation == "helmholtz" and not self.wavenumber > 0:
            raise InvalidInput("helmholtz requires wavenumber > 0")
        if self.equation == "laplace" and self.wavenumber != 0:
            raise InvalidInput("laplace requires wavenumber == 0")

    @property
    def scalar_field(self):
        return "real" if self.equation == "laplace" else "complex"

    @property
    def dtype(self):
        return np.float64 if self.equation == "laplace" else np.complex128

    def single_layer(self):
        if self.layer == "single":
            return self
        return KernelSpec(self.equation, self.dim, "single", self.wavenumber, self.self_interaction)

    @property
    def eq_code(self):
        return _native.EQ_LAPLACE if self.equation == "laplace" else _native.EQ_HELMHOLTZ

    @property
    def layer_code(self):
        return _native.LAYER_DOUBLE if self.layer == "double" else _native.LAYER_SINGLE


def eval_block(spec: KernelSpec, targets, sources, source_curvature=None) -> np.ndarray:
    """Dense m x n block G(x_i, y_j) (or dG/dnu_y), columns scaled by source
    weights, coincident pairs by ``spec.self_interaction`` (kernels.py:82-161).
    Evaluated on the GPU."""
    torch = _native.require_cuda()
    if targets.dim != spec.dim or sources.dim != spec.dim:
        raise InvalidInput(f"dimension mismatch: spec is {spec.dim}D, targets {targets.dim}D, "
                           f"sources {sources.dim}D")
    if spec.layer == "double" and sources.normals is None:
        raise InvalidInput("double layer needs source normals")
    curv = source_curvature if source_curvature is not None else sources.curvatures
    climit = spec.self_interaction == "curvature_limit"
    m, n = targets.n, sources.n
    if climit and (spec.equation != "laplace" or spec.dim != 2 or spec.layer != "double"
                   or curv is None):
        # the reference only consults the self-interaction rule when the
        # block HAS a coincident pair (kernels.py:146-157): e.g. proxy blocks
        # of a curvature-limit spec's single layer are fine.  This host check
        # runs only for that unusual combination (an error path).
        span = max(float(np.ptp(targets.coords, axis=0).max()),
                   float(np.ptp(sources.coords, axis=0).max()),
                   float(np.abs(targets.coords).max()), float(np.abs(sources.coords).max()), 1.0)
        tol = COINCIDENT_RTOL * span
        hit = False
        for lo in range(0, m, 256):
            dd = targets.coords[lo:lo + 256, None, :] - sources.coords[None, :, :]
            if (np.sqrt(np.sum(dd * dd, axis=2)) < tol).any():
                hit = True
                break
        if hit:
            if spec.equation != "laplace" or spec.dim != 2 or spec.layer != "double":
                raise InvalidInput("curvature_limit only defined for the 2D Laplace double layer")
            raise InvalidInput("curvature_limit needs source curvatures")
        climit = False                   # no coincident pair: the rule never fires
    d = spec.dim
    coords = np.vstack([targets.coords, sources.coords])
    nrm = None
    if spec.layer == "double":
        nrm = np.vstack([np.zeros((m, d)), sources.normals])
    w = None
    if sources.weights is not None:
        w = np.concatenate([np.ones(m), sources.weights])
    kap = None
    if climit:
        kap = np.concatenate([np.zeros(m), np.broadcast_to(np.asarray(curv, dtype=np.float64), (n,))])
    geo = DeviceGeometry(coords, np.arange(m + n), nrm, w, kap)
    span = max(float(np.ptp(targets.coords, axis=0).max()), float(np.ptp(sources.coords, axis=0).max()),
               float(np.abs(targets.coords).max()), float(np.abs(sources.coords).max()), 1.0)
    geo.coincide_tol = COINCIDENT_RTOL * span
    src = geo.source(_native.SRC_KERNEL, spec.eq_code, spec.layer_code, spec.wavenumber,
                     curvature_limit=climit, weighted=w is not None)
    field = 1 if spec.equation == "helmholtz" else 0
    dev = torch.device("cuda")
    rows = torch.arange(m, dtype=torch.int32, device=dev)
    cols = torch.arange(m, m + n, dtype=torch.int32, device=dev)
    out = torch.empty((m, n), dtype=_native.torch_dtype(field), device=dev)
    _native.check(_native.lib().skel_eval_block(src, _native.ptr(rows), m, _native.ptr(cols), n,
                                                _native.ptr(out), field, _native.stream_ptr()),
                  "skel_eval_block")
    return out.cpu().numpy()


def bessel_h0(z):
    """H0^(1)(z) = J0(z) + i Y0(z) on the GPU (kernels.py:65-75); z > 0."""
    torch = _native.require_cuda()
    za = np.asarray(z, dtype=np.float64)
    if not np.all(za > 0):
        raise InvalidInput("bessel_h0 requires z > 0 (Y0 is singular at 0)")
    flat = np.ascontiguousarray(za.reshape(-1))
    dz = torch.from_numpy(flat).to("cuda")
    out = torch.empty(2 * flat.size, dtype=torch.float64, device="cuda")
    _native.check(_native.lib().skel_bessel_h0(_native.ptr(dz), flat.size, _native.ptr(out),
                                               _native.stream_ptr()), "skel_bessel_h0")
    h = out.cpu().numpy().view(np.complex128).reshape(za.shape)
    return complex(h) if h.ndim == 0 else h
