"""Second-kind boundary integral systems on closed 2D curves (drop-in for
the factor/solve-facing part of skelkit/bie.py).

Matrix entries are never materialised on the host: ``BieSystem`` and the
combined-field system expose a device descriptor (csrc/entries.cuh) that the
compression, S-assembly and dense-matvec kernels evaluate on the fly.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from ._device import DeviceGeometry, ResidentPoints
from .errors import InvalidInput
from .geom import PointSet, build_tree
from .kernels import KernelSpec, eval_block
from .skel import ProxyConfig, _DeviceSourceMixin, compress_source
from .solver import factor, solve

QUAD_RULES = ("plain_trapezoid", "kapur_rokhlin_10")


@dataclass
class Curve2D:
    """Closed curve sampled at n equispaced parameters: positions, outward
    unit normals, signed curvature, arclength weights |x'| 2 pi / n."""

    t: np.ndarray
    xy: np.ndarray
    normals: np.ndarray
    curvature: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        if np.any(self.weights <= 0):
            raise InvalidInput("curve weights must be positive")

    @property
    def n(self):
        return self.xy.shape[0]

    def point_set(self):
        return PointSet(self.xy, self.normals, self.weights, self.curvature)

    def node_spacing(self):
        return float(self.weights.max())

    def diameter(self):
        return float(np.linalg.norm(self.xy.max(axis=0) - self.xy.min(axis=0)))


def ellipse(a, b, n) -> Curve2D:
    """Counter-clockwise ellipse x = (a cos t, b sin t) (bie.py:81-91)."""
    if a <= 0 or b <= 0 or n < 4:
        raise InvalidInput("need positive semi-axes and n >= 4")
    t = 2 * np.pi * np.arange(n) / n
    c, s = np.cos(t), np.sin(t)
    speed = np.sqrt((a * s) ** 2 + (b * c) ** 2)
    return Curve2D(t, np.column_stack([a * c, b * s]),
                   np.column_stack([b * c, a * s]) / speed[:, None],
                   a * b / speed ** 3, speed * (2 * np.pi / n))


def circle(radius, n) -> Curve2D:
    return ellipse(radius, radius, n)


def winding_number(curve: Curve2D, point) -> int:
    d = curve.xy - np.asarray(point)
    ang = np.arctan2(d[:, 1], d[:, 0])
    dang = np.diff(np.concatenate([ang, ang[:1]]))
    dang = (dang + np.pi) % (2 * np.pi) - np.pi
    return int(np.round(dang.sum() / (2 * np.pi)))


def contains(curve: Curve2D, point) -> bool:
    return winding_number(curve, point) != 0


class BieSystem(_DeviceSourceMixin):
    """Nystrom system: K(x_i, x_j) w_j off the diagonal (times the KR10
    corrections when active) and identity_coef (+ the smooth Laplace limit)
    on it (bie.py:135-176).  ``block`` takes ORIGINAL indices."""

    def __init__(self, spec: KernelSpec, curve: Curve2D, quad: str, identity_coef: float = -0.5):
        self.spec = spec
        self.curve = curve
        self.quad = quad
        self.identity_coef = float(identity_coef)
        self.points = curve.point_set()
        self._geo = None
        self._res = None

    @property
    def n(self):
        return self.curve.n

    @property
    def dtype(self):
        return self.spec.dtype

    @property
    def wavenumber(self):
        return self.spec.wavenumber

    def resident(self):
        """Curve nodes resident on the device in original order (uploaded
        once per system; every tree ordering is gathered from it on the GPU)."""
        if self._res is None:
            self._res = ResidentPoints(self.curve.xy, self.curve.normals, self.curve.weights,
                                       self.curve.curvature)
        return self._res

    def geometry(self, perm=None):
        if perm is None:
            if self._geo is None:
                self._geo = DeviceGeometry(None, np.arange(self.n), resident=self.resident())
            return self._geo
        return DeviceGeometry(None, perm, resident=self.resident())

    def descriptor(self, geo, wscale=1.0):
        return geo.source(_native.SRC_BIE, self.spec.eq_code, _native.LAYER_DOUBLE,
                          self.spec.wavenumber, identity_coef=self.identity_coef, wscale=wscale,
                          curvature_limit=self.spec.self_interaction == "curvature_limit",
                          kr10=self.quad == "kapur_rokhlin_10")

    def _desc(self):
        return self.descriptor(self.geometry())

    def matrix(self):
        idx = np.arange(self.n)
        return self.block(idx, idx)


class CombinedFieldSystem(BieSystem):
    """BASELINE config 3: (D_k - i k S_k) x KR10 + 1/2 I on a closed curve
    (composed from the reference's entry rules)."""

    def __init__(self, curve: Curve2D, k: float):
        super().__init__(KernelSpec("helmholtz", 2, "double", k), curve, "kapur_rokhlin_10", 0.5)

    def descriptor(self, geo, wscale=1.0):
        return geo.source(_native.SRC_CFIE, _native.EQ_HELMHOLTZ, _native.LAYER_DOUBLE,
                          self.spec.wavenumber, identity_coef=self.identity_coef, wscale=wscale,
                          kr10=True)


def combined_field_system(curve: Curve2D, k: float) -> CombinedFieldSystem:
    if not k > 0:
        raise InvalidInput("wavenumber must be positive")
    return CombinedFieldSystem(curve, k)


def discretize_dirichlet(curve: Curve2D, spec: KernelSpec, quad: str | None = None) -> BieSystem:
    """Interior Dirichlet Nystrom system (bie.py:179-201): Laplace pairs with
    the plain trapezoid rule and the curvature-limit diagonal, Helmholtz with
    KR10."""
    if spec.dim != 2 or spec.layer != "double":
        spec = KernelSpec(spec.equation, 2, "double", spec.wavenumber,
                          "curvature_limit" if spec.equation == "laplace" else "zero")
    if quad is None:
        quad = "plain_trapezoid" if spec.equation == "laplace" else "kapur_rokhlin_10"
    if quad not in QUAD_RULES:
        raise InvalidInput(f"unknown quadrature {quad!r}")
    if spec.equation == "helmholtz" and quad == "plain_trapezoid":
        raise InvalidInput("helmholtz double layer is weakly singular; "
                           "plain trapezoid cannot meet the accuracy contract")
    if spec.equation == "laplace" and quad != "plain_trapezoid":
        raise InvalidInput("laplace double layer is smooth; use plain_trapezoid")
    if spec.equation == "laplace" and spec.self_interaction != "curvature_limit":
        spec = KernelSpec(spec.equation, 2, "double", 0.0, "curvature_limit")
    return BieSystem(spec, curve, quad)


class BieSource(_DeviceSourceMixin):
    """A BieSystem in tree order (bie.py:233-262): row proxies scaled by the
    mean quadrature weight, column proxies weighted."""

    def __init__(self, system: BieSystem, perm):
        self.system = system
        self.perm = np.asarray(perm)
        self.n = system.n
        self.dtype = system.dtype
        self.wavenumber = system.spec.wavenumber
        self.geo = system.geometry(self.perm)
        self.wscale = float(np.mean(system.curve.weights[self.perm]))

    def _desc(self):
        return self.system.descriptor(self.geo, self.wscale)


_BieSource = BieSource


def point_source_data(curve: Curve2D, source, spec: KernelSpec) -> np.ndarray:
    """f_i = G(x_i, source) for an exterior point source (bie.py:204-213)."""
    source = np.asarray(source, dtype=np.float64)
    if contains(curve, source):
        raise InvalidInput("point source must lie strictly outside the domain")
    sspec = KernelSpec(spec.equation, 2, "single", spec.wavenumber)
    return eval_block(sspec, PointSet(curve.xy), PointSet(source.reshape(1, 2)))[:, 0]


def compress_system(system: BieSystem, eps, max_leaf_size=None, proxy: ProxyConfig | None = None,
                    mode="proxy", seed=0, shard=None):
    """Tree over the curve nodes + GPU skeletonization (bie.py:265-272).
    ``shard`` (extension): see compress_source."""
    tree = build_tree(system.points, max_leaf_size)
    cm = compress_source(BieSource(system, tree.perm), tree, eps, proxy=proxy, mode=mode,
                         seed=seed, shard=shard)
    return tree, cm


def solve_dirichlet(system: BieSystem, rhs, eps, max_leaf_size=None, shard=None):
    """compress, factor, solve (bie.py:275-279).  Returns (density, cm, fi)."""
    _, cm = compress_system(system, eps, max_leaf_size, shard=shard)
    fi = factor(cm)
    return solve(fi, rhs), cm, fi


def dense_matvec(source, x):
    """y = A x with exact entries evaluated on the fly on the GPU (the
    residual oracle of SURVEY 8(a10), no N x N storage).  ``source`` is a
    tree-ordered device source (BieSource / KernelSource); x, y in ORIGINAL
    order."""
    torch = _native.require_cuda()
    desc, field = source.device_source()
    xa = np.asarray(x)
    single = xa.ndim == 1
    dt = np.complex128 if (field or np.iscomplexobj(xa)) else np.float64
    if field == 0 and np.iscomplexobj(xa):
        return dense_matvec(source, xa.real) + 1j * dense_matvec(source, xa.imag)
    X = np.ascontiguousarray(xa.reshape(source.n, -1), dtype=dt)
    perm = np.asarray(source.geo.perm)
    xt = torch.from_numpy(np.ascontiguousarray(X[perm])).to("cuda")
    yt = torch.empty_like(xt)
    _native.check(_native.lib().skel_dense_matvec(desc, _native.ptr(xt), _native.ptr(yt), xt.shape[1],
                                                  field, _native.stream_ptr()), "skel_dense_matvec")
    y = np.empty_like(X)
    y[perm] = yt.cpu().numpy()
    return y[:, 0] if single else y
