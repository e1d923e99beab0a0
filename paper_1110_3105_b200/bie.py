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
# Kapur-Rokhlin 10th-order endpoint corrections gamma_1..gamma_10 (bie.py:31-42);
# the kernels hold the same table as c_kr10 (csrc/entries.cuh)
KR10_GAMMA = np.array([
    7.832432020568779e+00, -4.565161670374749e+01, 1.452168846354677e+02,
    -2.901348302886379e+02, 3.870862162579900e+02, -3.523821383570681e+02,
    2.172421547519342e+02, -8.707796087382991e+01, 2.053584266072635e+01,
    -2.166984103403823e+00])


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


def perm_mean(w, perm):
    """np.mean(w[perm]) bit for bit (numpy's pairwise order), without the
    gathered copy: native, threaded over the top of the summation tree."""
    import ctypes
    w = np.ascontiguousarray(w, dtype=np.float64)
    perm = np.ascontiguousarray(perm, dtype=np.int64)
    out = ctypes.c_double()
    _native.check(_native.lib().skel_perm_mean(w.ctypes.data_as(ctypes.c_void_p),
                                                perm.ctypes.data_as(ctypes.c_void_p), perm.size,
                                                ctypes.byref(out)), "skel_perm_mean")
    return float(out.value)


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
        self.wscale = perm_mean(system.curve.weights, self.perm)

    def _desc(self):
        return self.system.descriptor(self.geo, self.wscale)

    # the reference's proxy protocol (bie.py:251-262), device-evaluated; the
    # fast sweep builds these blocks inside the ID kernel instead
    @property
    def points(self):
        return self.system.curve.point_set().subset(self.perm)

    def proxy_row_block(self, rows, pxy):
        return self.wscale * eval_block(self.system.spec.single_layer(), self.points.subset(rows), pxy)

    def proxy_col_block(self, cols, pxy):
        src = self.points.subset(cols)
        return eval_block(self.system.spec.single_layer(), pxy, PointSet(src.coords, None, src.weights))


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
    up = _upload_beside(system)
    try:
        tree = build_tree(system.points, max_leaf_size)
    except BaseException:
        up(False)                           # the tree's error wins
        raise
    up()
    cm = compress_source(BieSource(system, tree.perm), tree, eps, proxy=proxy, mode=mode,
                         seed=seed, shard=shard)
    return tree, cm


def _upload_beside(system):
    """Start the one-time upload of the system's geometry (host copies into
    the pinned staging block + one async H2D copy) on a helper thread, so it
    runs beside the native tree build instead of after it; returns the join
    function (re-raises what the upload raised).  Both sides are a handful of
    long GIL-free calls, unlike the per-level launch work."""
    if getattr(system, "_res", 0) is not None or not hasattr(system, "resident"):
        return lambda reraise=True: None
    import threading
    torch = _native.require_cuda()
    dev = torch.cuda.current_device()
    err = []

    def work():
        try:
            torch.cuda.set_device(dev)      # the CUDA current device is per host thread
            system.resident()
        except BaseException as e:          # noqa: BLE001 -- re-raised by join()
            err.append(e)

    th = threading.Thread(target=work, name="skel-geometry-upload")
    th.start()

    def join(reraise=True):
        th.join()
        if err and reraise:
            raise err[0]
    return join


def solve_dirichlet(system: BieSystem, rhs, eps, max_leaf_size=None, shard=None):
    """compress, factor, solve (bie.py:275-279).  Returns (density, cm, fi)."""
    pre = _prefetch_rhs(system, rhs)
    _, cm = compress_system(system, eps, max_leaf_size, shard=shard)
    fi = factor(cm)
    if pre is not None and pre[0].dtype == _native.torch_dtype(int(fi.dtype == np.complex128)):
        from .solver import solve_device
        torch = _native.require_cuda()
        torch.cuda.current_stream().wait_event(pre[1])
        x = _native.to_host(solve_device(fi, pre[0], _private=True))
        return (x[:, 0] if np.ndim(rhs) == 1 else x), cm, fi
    return solve(fi, rhs), cm, fi


def _prefetch_rhs(system, rhs):
    """A page-locked host RHS is copied to the device on a side stream while
    the system is compressed and factored (the solve needs it only at the
    very end); returns (device tensor, copy event) or None for anything else
    (pageable memory, other dtypes or layouts: ``solve`` handles those)."""
    if not isinstance(rhs, np.ndarray) or rhs.dtype not in (np.float64, np.complex128):
        return None
    if rhs.ndim not in (1, 2) or rhs.shape[0] != system.points.coords.shape[0] or not rhs.flags.c_contiguous:
        return None
    torch = _native.require_cuda()
    h = torch.from_numpy(rhs.reshape(rhs.shape[0], -1))
    if not h.is_pinned():
        return None
    from ._staging import side_streams
    s = side_streams(1, "rhs")[0]
    with torch.cuda.stream(s):
        d = torch.empty(h.shape, dtype=h.dtype, device="cuda")
        d.copy_(h, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
    d.record_stream(torch.cuda.current_stream())
    return d, ev


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


# ---------------------------------------------------------------------------
# more curves, post-processing and CSV output (bie.py:98-114, 216-230, 282-300)

def trefoil(n, center=(0.0, 0.0), scale=1.0) -> Curve2D:
    """Three-lobed curve r(theta) = (2 + cos 3 theta) / 6 (bie.py:98-114)."""
    if n < 8:
        raise InvalidInput("need n >= 8")
    t = 2 * np.pi * np.arange(n) / n
    r = (2 + np.cos(3 * t)) / 6
    dr = -np.sin(3 * t) / 2
    ddr = -1.5 * np.cos(3 * t)
    c, s = np.cos(t), np.sin(t)
    xy = np.asarray(center) + scale * r[:, None] * np.column_stack([c, s])
    tx = scale * (dr * c - r * s)
    ty = scale * (dr * s + r * c)
    speed = np.hypot(tx, ty)
    kap = (r * r + 2 * dr * dr - r * ddr) / (r * r + dr * dr) ** 1.5 / scale
    return Curve2D(t, xy, np.column_stack([ty, -tx]) / speed[:, None], kap,
                   speed * (2 * np.pi / n))


def eval_interior(curve: Curve2D, density, spec: KernelSpec, targets) -> np.ndarray:
    """Double-layer potential of ``density`` at interior targets (trapezoid
    rule, bie.py:216-230); the kernel block is evaluated on the GPU."""
    import warnings

    from .errors import AccuracyWarning
    targets = np.atleast_2d(np.asarray(targets, dtype=np.float64))
    for p in targets:
        if not contains(curve, p):
            raise InvalidInput(f"target {p} is not interior")
    d = np.min(np.linalg.norm(curve.xy[None, :, :] - targets[:, None, :], axis=2), axis=1)
    if np.any(d < 2 * curve.node_spacing()):
        warnings.warn("target within 2 node spacings of the boundary; quadrature accuracy "
                      "degrades near the curve", AccuracyWarning, stacklevel=2)
    blk = eval_block(KernelSpec(spec.equation, 2, "double", spec.wavenumber), PointSet(targets),
                     curve.point_set())
    return blk @ np.asarray(density)


def write_density_csv(path, curve: Curve2D, density):
    """t, x, y, re(sigma), im(sigma) per node (bie.py:282-289)."""
    density = np.asarray(density)
    with open(path, "w") as f:
        f.write("t,x,y,sigma_re,sigma_im\n")
        f.writelines(f"{curve.t[i]:.17g},{curve.xy[i, 0]:.17g},{curve.xy[i, 1]:.17g},"
                     f"{np.real(density[i]):.17g},{np.imag(density[i]):.17g}\n" for i in range(curve.n))


def write_field_csv(path, points, values):
    """x, y, re(u), im(u) per sample (bie.py:292-299)."""
    points = np.atleast_2d(np.asarray(points))
    values = np.asarray(values)
    with open(path, "w") as f:
        f.write("x,y,u_re,u_im\n")
        f.writelines(f"{p[0]:.17g},{p[1]:.17g},{np.real(v):.17g},{np.imag(v):.17g}\n"
                     for p, v in zip(points, values))


# ---------------------------------------------------------------------------
# multiple scattering by sound-hard obstacles (bie.py:305-459): single-layer
# representation, Neumann-trace system, block-diagonal skeletonized
# preconditioner, GMRES (krylov.gmres)

def _curves_resident(curves):
    xy = np.concatenate([c.xy for c in curves])
    nrm = np.concatenate([c.normals for c in curves])
    w = np.concatenate([c.weights for c in curves])
    kap = np.concatenate([c.curvature for c in curves])
    return ResidentPoints(xy, nrm, w, kap)


class ScattererSource(_DeviceSourceMixin):
    """Self-block of one scatterer in tree order (bie.py:326-349): Neumann
    trace of the Helmholtz single layer with KR10 and the -1/2 jump; row
    proxies are the Neumann trace of the proxy field, column proxies the
    weighted single layer (entries: csrc/entries.cuh, SKEL_SRC_NTRACE)."""

    def __init__(self, scat, perm):
        self.scat = scat
        self.perm = np.asarray(perm)
        self.n = scat.npts
        self.dtype = np.complex128
        self.wavenumber = scat.k
        self.geo = DeviceGeometry(None, self.perm, resident=scat.resident())

    def _desc(self):
        return self.geo.source(_native.SRC_NTRACE, _native.EQ_HELMHOLTZ, _native.LAYER_SINGLE,
                               self.scat.k, identity_coef=-0.5, kr10=True)


class Scatterer:
    def __init__(self, curve: Curve2D, k):
        self.curve = curve
        self.k = float(k)
        self.points = curve.point_set()
        self.npts = curve.n
        self._res = None

    def resident(self):
        if self._res is None:
            self._res = _curves_resident([self.curve])
        return self._res

    def self_block(self, rows, cols):
        """Dense self-interaction block on ORIGINAL indices (bie.py:359-367)."""
        src = ScattererSource(self, np.arange(self.npts))
        return src.block(np.asarray(rows), np.asarray(cols))


class _SystemSource(_DeviceSourceMixin):
    """All scatterers as one source (original order): KR10 only inside a
    scatterer (point groups), -1/2 on the diagonal, plain Neumann trace
    between scatterers (bie.py:386-398)."""

    def __init__(self, system):
        torch = _native.require_cuda()
        self.system = system
        off = system.offsets()
        self.n = int(off[-1])
        self.dtype = np.complex128
        self.wavenumber = system.k
        self.perm = np.arange(self.n)
        res = _curves_resident([s.curve for s in system.scatterers])
        self.geo = DeviceGeometry(None, self.perm, resident=res)
        grp = np.repeat(np.arange(len(system.scatterers)), np.diff(off)).astype(np.int32)
        self._grp = torch.from_numpy(grp).to("cuda")
        self._gstart = torch.from_numpy(off[:-1].astype(np.int64)).to("cuda")
        self._gsize = torch.from_numpy(np.diff(off).astype(np.int64)).to("cuda")

    def _desc(self):
        s = self.geo.source(_native.SRC_NTRACE, _native.EQ_HELMHOLTZ, _native.LAYER_SINGLE,
                            self.system.k, identity_coef=-0.5, kr10=True)
        s.grp = _native.ptr(self._grp)
        s.grp_start = _native.ptr(self._gstart)
        s.grp_size = _native.ptr(self._gsize)
        return s


@dataclass
class ScatteringSystem:
    """A_ii = -I/2 + K_ii (KR10), A_ij = K_ij: K the target-normal derivative
    of the Helmholtz single layer; incoming plane wave exp(i k x2)."""

    scatterers: list
    k: float

    def __post_init__(self):
        self._src = None

    @property
    def n(self):
        return sum(s.npts for s in self.scatterers)

    def offsets(self):
        return np.concatenate([[0], np.cumsum([s.npts for s in self.scatterers])]).astype(np.int64)

    def source(self):
        if self._src is None:
            self._src = _SystemSource(self)
        return self._src

    def matrix(self):
        """Dense system matrix (evaluated on the GPU)."""
        idx = np.arange(self.n)
        return self.source().block(idx, idx)

    def apply(self, x):
        """y = A x with exact entries evaluated on the fly (no N x N storage)."""
        return dense_matvec(self.source(), x)

    def rhs_plane_wave(self):
        """-d/dnu of u_inc = exp(i k x2) on every boundary (bie.py:400-406)."""
        return np.concatenate([-1j * self.k * s.curve.normals[:, 1] * np.exp(1j * self.k * s.curve.xy[:, 1])
                               for s in self.scatterers])

    def precond_blocks(self, eps=1e-6, max_leaf_size=None):
        """Skeletonized factorization of every isolated self-system (GPU)."""
        facs = []
        for s in self.scatterers:
            tree = build_tree(s.points, max_leaf_size)
            cm = compress_source(ScattererSource(s, tree.perm), tree, eps)
            facs.append(factor(cm))
        return facs

    def precond_apply(self, facs):
        off = self.offsets()

        def apply_pinv(x):
            x = np.asarray(x, dtype=np.complex128)
            out = np.empty_like(x)
            for i, fi in enumerate(facs):
                out[off[i]:off[i + 1]] = solve(fi, x[off[i]:off[i + 1]])
            return out

        return apply_pinv

    def scattered_field(self, densities, targets):
        """Single-layer field of the densities at exterior points (bie.py:429-438)."""
        targets = np.atleast_2d(np.asarray(targets, dtype=np.float64))
        off = self.offsets()
        spec = KernelSpec("helmholtz", 2, "single", self.k)
        out = np.zeros(targets.shape[0], dtype=np.complex128)
        for i, s in enumerate(self.scatterers):
            out += eval_block(spec, PointSet(targets), s.points) @ np.asarray(densities)[off[i]:off[i + 1]]
        return out


def scattering_system(scatterers, k) -> ScatteringSystem:
    """Validate the geometry (pairwise disjoint, bie.py:441-459) and build the system."""
    if k <= 0:
        raise InvalidInput("wavenumber must be positive")
    curves = list(scatterers)
    for i in range(len(curves)):
        for j in range(i + 1, len(curves)):
            a, b = curves[i], curves[j]
            la, ha = a.xy.min(0), a.xy.max(0)
            lb, hb = b.xy.min(0), b.xy.max(0)
            if (np.all(la <= hb) and np.all(lb <= ha)
                    and (contains(a, b.xy.mean(0)) or contains(b, a.xy.mean(0))
                         or contains(a, b.xy[0]) or contains(b, a.xy[0]))):
                raise InvalidInput(f"scatterers {i} and {j} overlap")
    return ScatteringSystem([Scatterer(c, k) for c in curves], k)
