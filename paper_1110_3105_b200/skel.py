"""Multilevel recursive skeletonization on the GPU (drop-in for
skelkit/skel.py).

``compress_source`` keeps the reference's level sweep (skel.py:286-411) as a
host loop over covers, but every box of a cover is processed by ONE launch of
``skel_id_level`` (csrc/id_level.cu): a 2-CTA cluster per box assembles
D = A(rd, cd) and the proxy-compressed targets t_row.T / t_col straight into
shared memory, runs both CPQR IDs, equalises the ranks through DSMEM and
writes sorted skeletons plus L / R.  The host only does O(p) integer
bookkeeping per level (offsets, buckets) and reads back the ranks.

The resulting ``CompressedMatrix`` stays on the device; its per-node numpy
view (``levels[l].nodes``) is materialised lazily for callers that inspect
it.
"""

import warnings
from dataclasses import dataclass, replace

import numpy as np

from . import _native, _profile
from ._device import DeviceGeometry
from .errors import InvalidInput, RefusedTooLarge
from .geom import OrthTree, PointSet
from .kernels import KernelSpec
from ._plan import plan_id_level
from ._staging import Packer, eager_stream, fork, join, on_stream

DEFAULT_N_PROXY = {2: 64, 3: 512}        # skel.py:29
_RANDOMIZED_CUTOFF = 4096                # skel.py:33
GLOBAL_MODE_LIMIT = 20000                # skel.py:35
# target-size classes (bytes of the m x n target) -> one launch each
# (boundaries chosen so a bucket's shared memory fits 8/6/5/4/3/2/1 CTAs per SM)
_W_CLASSES = (18 << 10, 27 << 10, 35 << 10, 46 << 10, 64 << 10, 100 << 10, 214 << 10)
# register-tile classes of the target height (see dispatch_id_level)
_M_CLASSES = (64, 128, 192, 256, 384, 512, 768)


@dataclass
class ProxyConfig:
    """Proxy surface: n_proxy points on the circle/sphere of radius
    3*sqrt(d)*halfwidth*radius_factor (skel.py:53-76)."""

    n_proxy: int | None = None
    radius_factor: float = 1.0
    shape: str = "auto"

    def resolve(self, dim):
        n = self.n_proxy if self.n_proxy is not None else DEFAULT_N_PROXY[dim]
        floor = 8 if dim == 2 else 32
        if n < floor:
            raise InvalidInput(f"n_proxy must be >= {floor} in {dim}D")
        shape = self.shape
        if shape == "auto":
            shape = "circle" if dim == 2 else "sphere"
        if (shape == "circle") != (dim == 2):
            raise InvalidInput(f"proxy shape {shape!r} incompatible with {dim}D")
        return replace(self, n_proxy=n, shape=shape)


def proxy_radius(halfwidth, config: ProxyConfig, dim):
    return config.radius_factor * 3.0 * halfwidth * np.sqrt(dim)


def unit_proxy(n, dim):
    """Unit proxy surface: equispaced circle from angle 0 / Fibonacci sphere
    (skel.py:87-96)."""
    if dim == 2:
        th = 2 * np.pi * np.arange(n) / n
        return np.column_stack([np.cos(th), np.sin(th)])
    i = np.arange(n) + 0.5
    z = 1.0 - 2.0 * i / n
    rho = np.sqrt(np.clip(1.0 - z * z, 0.0, None))
    th = np.pi * (3.0 - np.sqrt(5.0)) * i
    return np.column_stack([rho * np.cos(th), rho * np.sin(th), z])


def proxy_points(box, config: ProxyConfig, dim) -> PointSet:
    cfg = config.resolve(dim)
    r = proxy_radius(box.halfwidth, cfg, dim)
    return PointSet(np.asarray(box.center, dtype=np.float64) + r * unit_proxy(cfg.n_proxy, dim))


# ---------------------------------------------------------------------------
# matrix sources with a device descriptor

class _DeviceSourceMixin:
    """block(rows, cols) in tree positions, evaluated on the GPU."""

    def _desc(self):
        raise NotImplementedError

    def device_source(self):
        return self._desc(), self.field

    @property
    def field(self):
        return 1 if np.dtype(self.dtype) == np.complex128 else 0

    def block(self, rows, cols):
        torch = _native.require_cuda()
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        m, n = rows.size, cols.size
        if m == 0 or n == 0:
            return np.zeros((m, n), dtype=self.dtype)
        dev = torch.device("cuda")
        r = torch.from_numpy(rows.astype(np.int32)).to(dev)
        c = torch.from_numpy(cols.astype(np.int32)).to(dev)
        out = torch.empty((m, n), dtype=_native.torch_dtype(self.field), device=dev)
        _native.check(_native.lib().skel_eval_block(self._desc(), _native.ptr(r), m, _native.ptr(c),
                                                    n, _native.ptr(out), self.field,
                                                    _native.stream_ptr()), "skel_eval_block")
        return out.cpu().numpy()


class KernelSource(_DeviceSourceMixin):
    """Plain kernel matrix in tree order (skel.py:100-124); proxies use the
    single layer of the same equation.  ``diag`` (an extension used by
    BASELINE config 4) is added where row == col."""

    def __init__(self, spec: KernelSpec, points: PointSet, perm, diag=0.0):
        self.spec = spec
        self.points = points.subset(perm)
        self.proxy_spec = spec.single_layer()
        self.n = points.n
        self.dtype = spec.dtype
        self.wavenumber = spec.wavenumber
        self.diag = float(diag)
        self.geo = DeviceGeometry(points.coords, perm,
                                  points.normals if spec.layer == "double" else None,
                                  points.weights, None)

    # the reference's proxy protocol (skel.py:116-124), device-evaluated; the
    # fast sweep never calls these (it builds the proxies inside the ID kernel)
    def proxy_row_block(self, rows, proxy: PointSet):
        from .kernels import eval_block
        return eval_block(self.proxy_spec, self.points.subset(rows), proxy)

    def proxy_col_block(self, cols, proxy: PointSet):
        from .kernels import eval_block
        src = self.points.subset(cols)
        return eval_block(self.proxy_spec, proxy, PointSet(src.coords, None, src.weights))

    def _desc(self):
        return self.geo.source(_native.SRC_KERNEL, self.spec.eq_code, self.spec.layer_code,
                               self.spec.wavenumber, diag=self.diag,
                               weighted=self.points.weights is not None)


# ---------------------------------------------------------------------------
# compressed representation

@dataclass
class CompressedNode:
    row_skel: np.ndarray
    col_skel: np.ndarray
    D: np.ndarray
    L: np.ndarray
    R: np.ndarray
    children: np.ndarray | None

    @property
    def k_r(self):
        return self.row_skel.size

    @property
    def k_c(self):
        return self.col_skel.size


def _off(counts):
    return np.concatenate([[0], np.cumsum(np.asarray(counts, dtype=np.int64))]).astype(np.int64)


class DevLevel:
    """Device slabs of one compressed level (capacity layouts addressed by
    per-box element offsets).  ``t`` holds the device index arrays (one
    packed upload per level)."""

    def __init__(self, li, nr, nc, kr, kc, d_off, l_off, r_off, D, L, R, rskel, cskel, child_off,
                 dtype, t=None, mine=None):
        from ._staging import Packer
        self.li = li
        self.mine = mine          # sharded level: boolean mask of this rank's boxes
        self.p = nr.size
        self.nr, self.nc = nr.astype(np.int64), nc.astype(np.int64)
        self.kr, self.kc = kr.astype(np.int64), kc.astype(np.int64)
        self.d_off, self.l_off, self.r_off = d_off, l_off, r_off
        self.D, self.L, self.R = D, L, R
        self.rskel, self.cskel = rskel, cskel          # compacted, int32, device
        self.child_off = child_off
        self.dtype = dtype
        if t is None:
            pk = Packer()
            pk.add("d_off", d_off).add("l_off", l_off).add("r_off", r_off)
            pk.add("nr", self.nr.astype(np.int32)).add("kr", self.kr.astype(np.int32))
            pk.add("kc", self.kc.astype(np.int32))
            pk.add("rdof_off", _off(self.nr)).add("cdof_off", _off(self.nc))
            pk.add("kr_off", _off(self.kr)).add("kc_off", _off(self.kc))
            if child_off is not None:
                pk.add("child_off", child_off)
            t = pk.upload()
        self.t = t
        self.t_d_off, self.t_l_off, self.t_r_off = t["d_off"], t["l_off"], t["r_off"]
        self.t_nr, self.t_kr, self.t_kc = t["nr"], t["kr"], t["kc"]
        self.t_rdof_off, self.t_cdof_off = t["rdof_off"], t["cdof_off"]
        self.t_kr_off, self.t_kc_off = t["kr_off"], t["kc_off"]
        self.t_child_off = t.get("child_off")
        self.t_own = t.get("own")
        self.n_own = None if mine is None else int(mine.sum())


class CompressedLevel:
    """Per-level view with the reference's offset tables (skel.py:145-163)."""

    def __init__(self, nodes=None, dev: DevLevel | None = None):
        self._nodes = nodes
        self.dev = dev
        self.dev_from_compress = dev is not None
        if nodes is not None:
            self.row_dof_counts = np.array([nd.D.shape[0] for nd in nodes], dtype=np.int64)
            self.col_dof_counts = np.array([nd.D.shape[1] for nd in nodes], dtype=np.int64)
            self.kr_counts = np.array([nd.k_r for nd in nodes], dtype=np.int64)
            self.kc_counts = np.array([nd.k_c for nd in nodes], dtype=np.int64)
        else:
            self.row_dof_counts, self.col_dof_counts = dev.nr, dev.nc
            self.kr_counts, self.kc_counts = dev.kr, dev.kc
        self.row_dof_off = _off(self.row_dof_counts)
        self.col_dof_off = _off(self.col_dof_counts)
        self.kr_off = _off(self.kr_counts)
        self.kc_off = _off(self.kc_counts)

    @property
    def nodes(self):
        if self._nodes is None:
            d = self.dev
            if getattr(d, "mine", None) is not None:
                raise InvalidInput("per-node blocks of a sharded level live on their owning ranks")
            D = d.D.cpu().numpy()
            L = d.L.cpu().numpy()
            R = d.R.cpu().numpy()
            rs = d.rskel.cpu().numpy().astype(np.int64)
            cs = d.cskel.cpu().numpy().astype(np.int64)
            out = []
            for a in range(d.p):
                nr, nc, kr, kc = (int(d.nr[a]), int(d.nc[a]), int(d.kr[a]), int(d.kc[a]))
                out.append(CompressedNode(
                    row_skel=rs[self.kr_off[a]:self.kr_off[a + 1]].copy(),
                    col_skel=cs[self.kc_off[a]:self.kc_off[a + 1]].copy(),
                    D=D[d.d_off[a]:d.d_off[a] + nr * nc].reshape(nr, nc).copy(),
                    L=L[d.l_off[a]:d.l_off[a] + nr * kr].reshape(nr, kr).copy(),
                    R=R[d.r_off[a]:d.r_off[a] + kc * nc].reshape(kc, nc).copy(),
                    children=None if d.child_off is None else
                    np.arange(d.child_off[a], d.child_off[a + 1], dtype=np.int64)))
            self._nodes = out
        return self._nodes

    def skeleton_arrays(self):
        """(row_skel, col_skel) of every box, concatenated in box order (host
        int64) -- the skeleton lists without copying D / L / R to the host."""
        if self._nodes is not None or self.dev is None:
            nd = self.nodes
            cat = lambda xs: (np.concatenate(xs).astype(np.int64) if xs  # noqa: E731
                              else np.zeros(0, dtype=np.int64))
            return cat([x.row_skel for x in nd]), cat([x.col_skel for x in nd])
        d = self.dev
        rs = d.rskel.cpu().numpy()[:int(self.kr_off[-1])].astype(np.int64)
        cs = d.cskel.cpu().numpy()[:int(self.kc_off[-1])].astype(np.int64)
        return rs, cs

    @property
    def K_r(self):
        return int(self.kr_off[-1])

    @property
    def K_c(self):
        return int(self.kc_off[-1])


class CompressedMatrix:
    """Telescoping compressed form A ~ D1 + L1 [ ... S ... ] R1 (skel.py:166-203).
    ``S`` is materialised on the host on first access; the device copy is
    ``S_dev``."""

    def __init__(self, levels, S, n, eps, perm, scalar_field, tree=None, S_dev=None):
        self.levels = levels
        self._S = S
        self.S_dev = S_dev
        self.n = n
        self.eps = eps
        self.perm = perm
        self.scalar_field = scalar_field
        self.tree = tree
        self._eager = None
        self.shard = None          # shard.ShardPlan when compressed across ranks

    @property
    def S(self):
        if self._S is None:
            self._S = self.S_dev.cpu().numpy()
        return self._S

    @S.setter
    def S(self, v):
        self._S = v
        self.S_dev = None

    @property
    def nlevels(self):
        return len(self.levels)

    @property
    def dtype(self):
        return np.complex128 if self.scalar_field == "complex" else np.float64

    @property
    def field(self):
        return 1 if self.scalar_field == "complex" else 0

    def skeleton_counts(self):
        return [(lv.K_r, lv.K_c) for lv in self.levels]

    def storage_bytes(self):
        it = np.dtype(self.dtype).itemsize
        tot = int(np.prod(self.S_shape())) * it + self.perm.nbytes
        for lv in self.levels:
            nr, nc, kr, kc = lv.row_dof_counts, lv.col_dof_counts, lv.kr_counts, lv.kc_counts
            tot += int((nr * nc + nr * kr + kc * nc).sum()) * it + int((kr + kc).sum()) * 8
        return tot

    def S_shape(self):
        if self._S is not None:
            return self._S.shape
        return tuple(self.S_dev.shape)

    def apply(self, x):
        return apply(self, x)

    def matvec_dense(self):
        return apply(self, np.eye(self.n, dtype=self.dtype))

    # -- device view ----------------------------------------------------------
    def device_levels(self):
        """DevLevel per level; host-built levels are packed and uploaded once."""
        out = []
        for li, lv in enumerate(self.levels):
            if lv.dev is None:
                lv.dev = _pack_level(li, lv, self.dtype)
            out.append(lv.dev)
        return out

    def device_S(self):
        if self.S_dev is None:
            torch = _native.require_cuda()
            self.S_dev = torch.from_numpy(np.ascontiguousarray(self._S, dtype=self.dtype)).to("cuda")
        return self.S_dev


def _pack_level(li, lv, dtype):
    torch = _native.require_cuda()
    dev = torch.device("cuda")
    nodes = lv.nodes
    nr, nc = lv.row_dof_counts, lv.col_dof_counts
    kr, kc = lv.kr_counts, lv.kc_counts
    d_off, l_off, r_off = _off(nr * nc), _off(nr * kr), _off(kc * nc)
    cat = lambda arrs: (np.concatenate([np.asarray(a, dtype=dtype).ravel() for a in arrs])  # noqa: E731
                        if arrs else np.zeros(0, dtype=dtype))
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    D = up(cat([nd.D for nd in nodes]))
    L = up(cat([nd.L for nd in nodes]))
    R = up(cat([nd.R for nd in nodes]))
    rs = up(np.concatenate([nd.row_skel for nd in nodes]).astype(np.int32) if nodes else np.zeros(0, np.int32))
    cs = up(np.concatenate([nd.col_skel for nd in nodes]).astype(np.int32) if nodes else np.zeros(0, np.int32))
    child_off = None
    if li > 0:
        counts = [0 if nd.children is None else len(nd.children) for nd in nodes]
        child_off = _off(counts)
        firsts = [int(nd.children[0]) for nd in nodes if nd.children is not None and len(nd.children)]
        # children must be contiguous runs in order (as compress produces)
        flat = np.concatenate([np.asarray(nd.children, dtype=np.int64) for nd in nodes
                               if nd.children is not None and len(nd.children)]) if firsts else np.zeros(0, np.int64)
        if flat.size and not np.array_equal(flat, np.arange(flat.size)):
            raise InvalidInput("children of each level must be consecutive positions of the previous level")
    return DevLevel(li, nr, nc, kr, kc, d_off, l_off, r_off, D, L, R, rs, cs, child_off, dtype)


# ---------------------------------------------------------------------------
# compression sweep

def compress(spec: KernelSpec, points: PointSet, tree: OrthTree, eps, proxy=None, mode="proxy",
             equalize_ranks=True, seed=0, allow_large=False) -> CompressedMatrix:
    """Recursively skeletonize the kernel matrix of ``spec`` (skel.py:267-283)."""
    source = KernelSource(spec, points, tree.perm)
    return compress_source(source, tree, eps, proxy=proxy, mode=mode,
                           equalize_ranks=equalize_ranks, seed=seed, allow_large=allow_large)


def id_level_flops(m0, m1, nr, nc, kr, kc, c_entry=10.0):
    """Algorithmic flops of one box of skel_id_level: two CPQR
    IDs, 4mnk - 2k^2(m+n) + k^2(n-k) each, plus entry assembly at c_entry
    flops per entry (targets and D)."""
    def one(m, n, k):
        m, n, k = (np.asarray(v, dtype=np.float64) for v in (m, n, k))
        return 4 * m * n * k - 2 * k * k * (m + n) + k * k * (n - k)
    asm = c_entry * (np.asarray(m0) * nr + np.asarray(m1) * nc + np.asarray(nr) * nc)
    return one(m0, nr, kr) + one(m1, nc, kc) + asm


def _level_geometry(tree, li, cfg, dim, k_wave):
    """Rank-independent per-level inputs (neighbour lists, proxy circles /
    spheres, children ranges), uploaded in one async copy; computed for
    level l+1 while level l's ID kernels run."""
    from types import SimpleNamespace
    ids = tree.levels[li]
    p = ids.size
    noff, nidx = tree.cover_neighbors(li)
    rad = cfg.radius_factor * 3.0 * tree.hw[ids] * np.sqrt(dim)
    neff = np.full(p, cfg.n_proxy, dtype=np.int64)
    if k_wave > 0:
        neff += np.ceil(4.0 * k_wave * rad).astype(np.int64)
    uniq = np.unique(neff)
    tables = [unit_proxy(int(u), dim) for u in uniq]
    tstart = _off([t.shape[0] for t in tables])[:-1]
    pxy_begin = tstart[np.searchsorted(uniq, neff)].astype(np.int32)
    unit = np.concatenate(tables, axis=0)
    child_off = tree.cover_children(li) if li > 0 else None
    pk = Packer()
    pk.add("nbr_off", noff).add("nbr", nidx.astype(np.int32))
    pk.add("box_c", np.ascontiguousarray(tree.center[ids]).ravel()).add("box_r", rad)
    pk.add("pxy_begin", pxy_begin).add("pxy_count", neff.astype(np.int32)).add("pxy_unit", unit.ravel())
    if child_off is not None:
        pk.add("child_off", child_off)
    return SimpleNamespace(ids=ids, p=p, noff=noff, nidx=nidx, rad=rad, neff=neff,
                           n_unit=unit.shape[0], child_off=child_off, t=pk.upload())


def _frozen(a):
    """Read-only view: the tree, the compressed matrix and the factorization
    share ONE permutation array instead of 8 N-byte copies per step (the
    reference copies; nobody writes to it afterwards)."""
    v = a.view()
    v.flags.writeable = False
    return v


def _segment_sum(vals, off):
    cs = np.concatenate([[0], np.cumsum(vals)])
    return cs[off[1:]] - cs[off[:-1]]


def compress_source(source, tree: OrthTree, eps, proxy: ProxyConfig | None = None,
                    mode: str = "proxy", equalize_ranks: bool = True, seed: int = 0,
                    allow_large: bool = False, eager_factor: bool = True,
                    shard=None) -> CompressedMatrix:
    """GPU compression sweep over a matrix source with a device descriptor
    (skel.py:286-411).

    ``shard`` (extension): a ``shard.ShardPlan`` (or "auto" = one rank per
    process of the current torch.distributed job) splits the boxes of the
    levels at and below the plan's split level across ranks; every rank
    ends with the skeletons of all boxes and the blocks of its own (see
    shard.py).  Results are bit-identical to the unsharded sweep.

    ``eager_factor`` (extension, default on): each level's telescoping
    factorization is launched on a side stream as soon as the level is
    compressed, overlapping the next level's compression; ``factor(cm)``
    then only finalises (same kernels and results as a separate factor)."""
    if not 0 < eps < 1:
        raise InvalidInput("eps must lie in (0, 1)")
    if mode not in ("proxy", "global"):
        raise InvalidInput(f"unknown mode {mode!r}")
    n = tree.n_points
    if mode == "global" and n > GLOBAL_MODE_LIMIT and not allow_large:
        raise RefusedTooLarge(f"global-mode compression of N={n} is quadratic; "
                              "pass allow_large=True to force it")
    cfg = (proxy or ProxyConfig()).resolve(tree.dim)
    if mode == "global" or not hasattr(source, "device_source"):
        # the reference's plugin protocol / quadratic global mode: explicit
        # targets from the source, batched GPU IDs (hostsweep.py)
        if shard is not None:
            raise InvalidInput("sharded compression needs a source with a device descriptor "
                               "and mode='proxy'")
        for attr in ("block", "dtype") + (("proxy_row_block", "proxy_col_block")
                                          if mode == "proxy" else ()):
            if not hasattr(source, attr):
                raise InvalidInput(f"matrix source lacks {attr!r} (skel.py:286-290 protocol)")
        _native.require_cuda()
        from .hostsweep import compress_explicit
        return compress_explicit(source, tree, eps, cfg, mode, equalize_ranks, seed)
    torch = _native.require_cuda()
    dev = torch.device("cuda")
    desc, field = source.device_source()
    dtype = np.complex128 if field else np.float64
    sfield = "complex" if field else "real"
    tdt = _native.torch_dtype(field)
    covers = tree.levels
    top = next(i for i, c in enumerate(covers) if len(c) == 1)
    if isinstance(shard, str):
        if shard != "auto":
            raise InvalidInput(f"unknown shard option {shard!r}")
        from .shard import default_plan
        shard = default_plan(tree)
    top_run = min(top, _DEBUG_MAX_LEVELS[0]) if _DEBUG_MAX_LEVELS[0] else top
    L = _native.lib()
    st = _native.stream_ptr()
    p_ = _native.ptr
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731

    if top == 0:
        allidx = torch.arange(n, dtype=torch.int32, device=dev)
        S = torch.empty((n, n), dtype=tdt, device=dev)
        _native.check(L.skel_eval_block(desc, p_(allidx), n, p_(allidx), n, p_(S), field, st),
                      "skel_eval_block")
        return CompressedMatrix([], None, n, eps, tree.perm.copy(), sfield, tree, S_dev=S)

    k_wave = float(getattr(source, "wavenumber", 0.0))
    dim = tree.dim
    levels = []
    prev = None
    optin = _smem_optin()
    elem = 16 if field else 8
    allpos = torch.arange(n, dtype=torch.int32, device=dev)
    run = None
    if eager_factor:
        from .solver import FactorRun
        run = FactorRun(field, 0.0, stream=eager_stream(), shard=shard)
    nvtx = _NVTX
    geo_next = _level_geometry(tree, 0, cfg, dim, k_wave)
    pending = None          # (level, DevLevel, event): factor launch deferred into the next level
    for li in range(top_run):
        _ht = _HostTimer(li) if _HOST_TIMING else None
        lev_ctx = _profile.timed("level", level=li)
        lev_ctx.__enter__()
        if nvtx:
            torch.cuda.nvtx.range_push(f"level{li}")
        geo = geo_next
        ids, p = geo.ids, geo.p
        mine = shard.mine(li) if shard is not None else None
        own = np.ones(p, dtype=np.int64) if mine is None else mine.astype(np.int64)
        noff, nidx = geo.noff, geo.nidx
        if li == 0:
            nr = (tree.hi[ids] - tree.lo[ids]).astype(np.int64)
            nc = nr.copy()
            rdofs = cdofs = allpos
            child_off = None
        else:
            child_off = geo.child_off
            nr = _segment_sum(prev.kr, child_off)
            nc = _segment_sum(prev.kc, child_off)
            rdofs, cdofs = prev.rskel, prev.cskel
        neff = geo.neff
        # offsets, target heights, size classes, big boxes, launch buckets:
        # one native pass (csrc/plan.cpp)
        pl = plan_id_level(nr, nc, noff, nidx, neff, None if mine is None else own, elem, optin,
                           _W_CLASSES, _M_CLASSES, _BIG_N, 4096, _SMALL_LEVEL)
        rdof_off, cdof_off = pl.rdof_off, pl.cdof_off
        m0, m1 = pl.m0, pl.m1
        d_off, l_off, r_off = pl.d_off, pl.l_off, pl.r_off
        need_m, need_n = pl.need_m, pl.need_n
        big = pl.big
        buckets = pl.buckets
        merged = pl.merged if pl.merged_first else None
        _ht and _ht.mark("prep")
        pk = Packer()
        pk.add("rdof_off", rdof_off).add("cdof_off", cdof_off)
        pk.add("d_off", d_off).add("l_off", l_off).add("r_off", r_off)
        pk.add("nr", nr.astype(np.int32))
        for bi, sel in enumerate(buckets):
            pk.add(f"order{bi}", sel)
        own_idx = None
        if mine is not None:
            own_idx = np.nonzero(mine)[0].astype(np.int32)
            pk.add("own", own_idx)
        t = pk.upload()
        _ht and _ht.mark("pack.upload")
        tg = geo.t
        Dt = torch.empty(max(int(d_off[-1]), 1), dtype=tdt, device=dev)
        Lt = torch.empty(max(int(l_off[-1]), 1), dtype=tdt, device=dev)
        Rt = torch.empty(max(int(r_off[-1]), 1), dtype=tdt, device=dev)
        rskel = torch.empty(max(int(rdof_off[-1]), 1), dtype=torch.int32, device=dev)
        cskel = torch.empty(max(int(cdof_off[-1]), 1), dtype=torch.int32, device=dev)
        kk = torch.zeros(3 * p, dtype=torch.int32, device=dev)     # kr | kc | flags
        _ht and _ht.mark("pack.alloc")
        lvd = _native.SkelLevel()
        lvd.nbox, lvd.level, lvd.equalize, lvd.n_unit = p, li, int(bool(equalize_ranks)), geo.n_unit
        lvd.eps = float(eps)
        lvd.debug_skip = _DEBUG_SKIP[0]
        lvd.rdof_off, lvd.rdofs = p_(t["rdof_off"]), p_(rdofs)
        lvd.cdof_off, lvd.cdofs = p_(t["cdof_off"]), p_(cdofs)
        if li > 0:
            lvd.child_off = p_(tg["child_off"])
            lvd.prev_kr, lvd.prev_kc = p_(prev.t_kr), p_(prev.t_kc)
        lvd.nbr_off, lvd.nbr = p_(tg["nbr_off"]), p_(tg["nbr"])
        lvd.box_c, lvd.box_r = p_(tg["box_c"]), p_(tg["box_r"])
        lvd.pxy_begin, lvd.pxy_count, lvd.pxy_unit = (p_(tg["pxy_begin"]), p_(tg["pxy_count"]),
                                                      p_(tg["pxy_unit"]))
        lvd.d_off, lvd.l_off, lvd.r_off = p_(t["d_off"]), p_(t["l_off"]), p_(t["r_off"])
        lvd.D, lvd.L, lvd.R = p_(Dt), p_(Lt), p_(Rt)
        lvd.rskel, lvd.cskel = p_(rskel), p_(cskel)
        lvd.kr, lvd.kc, lvd.flags = p_(kk[:p]), p_(kk[p:2 * p]), p_(kk[2 * p:])
        scratch_keep = []
        recs = []
        _ht and _ht.mark("pack+upload+alloc")
        streams = fork(len(buckets) + 1)
        # D blocks on their own stream, concurrent with the ID buckets
        d_order = p_(t["own"]) if own_idx is not None else None
        d_nrun = 0 if own_idx is None else own_idx.size
        d_maxn = int(max(nr.max(initial=0), nc.max(initial=0), 1))
        on_stream(streams[-1], lambda sp: _native.check(
            L.skel_assemble_D(desc, lvd, d_order, d_nrun, d_maxn, field, sp), "skel_assemble_D"),
            "assemble_D", level=li)
        for bi, sel in enumerate(buckets):
            max_m, max_n = int(need_m[sel].max()), int(need_n[sel].max())
            max_w = int((need_m[sel] * need_n[sel]).max())
            if merged is not None and bi == 0:
                max_m, max_n, max_w = merged
            fixed = _level_smem_fixed(max_n, field)
            if fixed + max_w * elem > optin:
                sb = 2 * sel.size * max_w * elem
                scr = torch.empty(sb // 8 + 1, dtype=torch.float64, device=dev)
                scratch_keep.append(scr)
                lvd.scratch, lvd.scratch_bytes = p_(scr), sb
            else:
                lvd.scratch, lvd.scratch_bytes = None, 0
            order_p = p_(t[f"order{bi}"])
            rec = on_stream(streams[bi], lambda sp: _native.check(
                L.skel_id_level(desc, lvd, order_p, sel.size, max_m, max_n, max_w, field, sp),
                f"skel_id_level (level {li})"),
                "id_level", level=li, sel=sel, max_m=max_m, max_n=max_n, max_w=max_w)
            if rec is not None:
                recs.append(rec)
        big_boxes = np.nonzero(big)[0]
        if big_boxes.size:
            from . import _bigbox
            with _profile.timed("id_big", level=li):
                _bigbox.run_boxes(desc, lvd, big_boxes, li, noff, nidx, nr, nc, neff, eps,
                                  bool(equalize_ranks), seed, field)
        # host work overlapped with this level's ID kernels: the next level's
        # geometry and the deferred factor launch of the previous level
        # (all remaining levels' geometry while the finest level's kernels run:
        # that is the longest GPU stretch, and at the coarse levels -- a few
        # hundred microseconds of kernel time each -- the host is the chain)
        if li == 0:
            geo_ahead = {l: _level_geometry(tree, l, cfg, dim, k_wave) for l in range(1, top_run)}
        if li + 1 < top_run:
            geo_next = geo_ahead.pop(li + 1)
        if pending is not None:
            run.stream.wait_event(pending[2])
            run.add_level(pending[0], pending[1])
            pending = None
        _ht and _ht.mark("launch")
        join(streams)
        if mine is not None:
            shard.gather_boxes(kk, li, 3)   # kr | kc | flags of the owned boxes, everywhere
        _ht and _ht.mark("big+join")
        kk_h = kk.cpu().numpy()
        _ht and _ht.mark("kk-wait")
        kr = kk_h[:p].astype(np.int64)
        kc = kk_h[p:2 * p].astype(np.int64)
        fl = kk_h[2 * p:]
        for rec in recs:
            b = rec.meta["sel"]
            rec.flops = float(id_level_flops(m0[b], m1[b], nr[b], nc[b], kr[b], kc[b]).sum())
        if np.any(fl & 8):
            raise RuntimeError(f"level {li}: a box exceeds the kernel's neighbour/child limits")
        bad = np.nonzero(fl & 3)[0]
        if bad.size:
            # lowrank.py:128-132 warns once per ID call; aggregated per level here
            warnings.warn(f"interpolation matrix entries reach > 2 on {bad.size} block(s) at "
                          f"level {li} (first node {bad[0]}); pivoting quality degraded",
                          stacklevel=2)
        _ht and _ht.mark("post.flags")
        # the sorted skeletons, compacted, are the next level's dof lists
        kro, kco = _off(kr), _off(kc)
        pk2 = Packer()
        pk2.add("kr_off", kro).add("kc_off", kco)
        t2 = pk2.upload()
        t2.update({k: t[k] for k in ("rdof_off", "cdof_off", "nr", "d_off", "l_off", "r_off")})
        t2["kr"], t2["kc"] = kk[:p], kk[p:2 * p]      # the device ranks (full after the all-reduce)
        if own_idx is not None:
            t2["own"] = t["own"]
        if li > 0:
            t2["child_off"] = tg["child_off"]
        t2["_buffer0"] = t["_buffer"]
        t2["_buffer_geo"] = tg["_buffer"]
        t2["_kk"] = kk
        _ht and _ht.mark("post.upload")
        if mine is None:
            rsk = torch.empty(max(int(kro[-1]), 1), dtype=torch.int32, device=dev)
            csk = torch.empty(max(int(kco[-1]), 1), dtype=torch.int32, device=dev)
            klen_r, klen_c = t2["kr"], t2["kc"]
        else:
            # each rank compacts its own boxes' skeletons; all-gathering the
            # owned ranges of both lists gives every rank the full lists
            sk = torch.empty(max(int(kro[-1]) + int(kco[-1]), 1), dtype=torch.int32, device=dev)
            rsk, csk = sk[:int(kro[-1])], sk[int(kro[-1]):]
            pk3 = Packer()
            pk3.add("kr", (kr * own).astype(np.int32)).add("kc", (kc * own).astype(np.int32))
            t3 = pk3.upload()
            klen_r, klen_c = t3["kr"], t3["kc"]
            t2["_buffer3"] = t3["_buffer"]
        _native.check(L.skel_compact_i32(p, p_(t["rdof_off"]), p_(klen_r), p_(t2["kr_off"]),
                                         p_(rskel), p_(rsk), st), "skel_compact_i32")
        _native.check(L.skel_compact_i32(p, p_(t["cdof_off"]), p_(klen_c), p_(t2["kc_off"]),
                                         p_(cskel), p_(csk), st), "skel_compact_i32")
        if mine is not None:
            shard.gather_rows(rsk, kro, li)
            shard.gather_rows(csk, kco, li)
        rsk, csk = rsk[:int(kro[-1])], csk[:int(kco[-1])]
        _ht and _ht.mark("post.compact")
        # L is stored nr x kr inside an nr x nr slot, R kc x nc inside nc x nc
        dl = DevLevel(li, nr, nc, kr, kc, d_off, l_off, r_off, Dt, Lt, Rt, rsk, csk, child_off,
                      dtype, t=t2, mine=mine)
        levels.append(CompressedLevel(dev=dl))
        prev = dl
        _ht and _ht.mark("post")
        if run is not None:
            ev = torch.cuda.Event()
            ev.record()
            pending = (li, dl, ev)
        _ht and _ht.mark("factor-launch")
        _ht and _ht.done()
        lev_ctx.__exit__(None, None, None)
        if nvtx:
            torch.cuda.nvtx.range_pop()

    if pending is not None:
        run.stream.wait_event(pending[2])
        run.add_level(pending[0], pending[1])
    if top_run < top:      # developer benchmarking only: partial sweep
        return levels
    last = prev
    Kr, Kc = int(last.kr.sum()), int(last.kc.sum())
    S = torch.zeros((max(Kr, 0), max(Kc, 0)), dtype=tdt, device=dev)
    if Kr and Kc:
        rbox = up(np.repeat(np.arange(last.p), last.kr).astype(np.int32))
        cbox = up(np.repeat(np.arange(last.p), last.kc).astype(np.int32))
        _native.check(L.skel_assemble_S(desc, p_(last.rskel), p_(rbox), Kr, p_(last.cskel),
                                        p_(cbox), Kc, p_(S), field, st), "skel_assemble_S")
    cm = CompressedMatrix(levels, None, n, eps, _frozen(tree.perm), sfield, tree, S_dev=S)
    cm._eager = run
    cm.shard = shard
    return cm


_OPTIN = None
_HOST_TIMING = bool(__import__("os").environ.get("SKEL_HOST_TIMING"))   # developer: host phases per level


class _HostTimer:
    def __init__(self, li):
        import time
        self.li, self.t, self.parts = li, time.perf_counter(), []

    def mark(self, name):
        import time
        now = time.perf_counter()
        self.parts.append((name, now - self.t))
        self.t = now

    def done(self):
        print(f"  L{self.li:2d} host: " + "  ".join(f"{k} {1e3 * v:.2f}" for k, v in self.parts), flush=True)


_DEBUG_MAX_LEVELS = [0]      # developer benchmarking: stop the sweep after this many levels
_DEBUG_SKIP = [0]            # developer benchmarking: 1 = assembly only, 2 = + column norms
_NVTX = bool(__import__("os").environ.get("SKEL_NVTX"))   # per-level NVTX ranges (profiling)


class _nullctx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def _smem_optin():
    global _OPTIN
    if _OPTIN is None:
        import ctypes
        a, b, c, d = (ctypes.c_int32() for _ in range(4))
        _native.check(_native.lib().skel_device_query(ctypes.byref(a), ctypes.byref(b),
                                                      ctypes.byref(c), ctypes.byref(d)),
                      "skel_device_query")
        _OPTIN = b.value
    return _OPTIN


_BIG_N = 512                 # boxes wider than this take the whole-GPU path
_SMALL_LEVEL = 400           # levels with at most this many boxes: one ID launch


def _level_smem_fixed(max_n, field):
    """Host mirror of level_smem_fixed<T> in csrc/id_level.cu (upper bound)."""
    al = lambda v: (v + 15) // 16 * 16  # noqa: E731
    sh = al(96 + 8 * 32 + 4 * 32)
    hdr = al(4 * (257 + 256 + 9 + 9 + 2) + 8 * 32 + 8)
    return sh + hdr + al(80 * max_n) + al(24 * max_n) + al(8 * max_n) + al(48 * max_n)


# ---------------------------------------------------------------------------
# compressed apply (skel.py:206-249)

def _as_device_rhs(x, n, dtype):
    torch = _native.require_cuda()
    if hasattr(x, "is_cuda"):
        X = x.reshape(n, -1).to(_native.torch_dtype(int(np.dtype(dtype) == np.complex128)))
        return X.contiguous(), True
    X = np.ascontiguousarray(np.asarray(x).reshape(n, -1), dtype=dtype)
    return torch.from_numpy(X).to("cuda"), False


def apply(cm: CompressedMatrix, x) -> np.ndarray:
    """y = A x through the compressed form: R up-sweep, S, D + L down-sweep."""
    torch = _native.require_cuda()
    xa = x if hasattr(x, "is_cuda") else np.asarray(x)
    if xa.shape[0] != cm.n:
        raise InvalidInput(f"length mismatch: matrix is {cm.n}, vector {xa.shape[0]}")
    single = xa.ndim == 1
    xdt = np.complex128 if (hasattr(xa, "is_complex") and xa.is_complex()) else getattr(xa, "dtype", np.float64)
    dtype = np.result_type(cm.dtype, xdt if not hasattr(xa, "is_cuda") else
                           (np.complex128 if xa.is_complex() else np.float64))
    if dtype == np.complex128 and cm.dtype == np.float64:
        re = apply(cm, xa.real)
        im = apply(cm, xa.imag)
        return re + 1j * im
    field = int(dtype == np.complex128)
    X, on_dev = _as_device_rhs(xa, cm.n, dtype)
    Rn = X.shape[1]
    L = _native.lib()
    st = _native.stream_ptr()
    p_ = _native.ptr
    perm = torch.from_numpy(cm.perm).to("cuda")
    xt = torch.empty_like(X)
    _native.check(L.skel_permute_rows(p_(perm), cm.n, p_(X), p_(xt), Rn, 0, field, st), "permute")
    if cm.nlevels == 0:
        yt = _dense_apply(cm.device_S(), xt, field)
    else:
        dls = cm.device_levels()
        us = [xt]
        u = xt
        shard = getattr(cm, "shard", None)
        for dl in dls:
            sh = dl.mine is not None
            nxt = torch.empty((int(dl.kc.sum()), Rn), dtype=X.dtype, device="cuda")
            _native.check(L.skel_sweep_up_ex(dl.n_own if sh else dl.p, p_(dl.t_nr), p_(dl.t_kc),
                                             p_(dl.t_cdof_off), p_(dl.t_kc_off), p_(dl.t_r_off),
                                             p_(dl.R), p_(u), p_(nxt), Rn, field,
                                             int(max(dl.nc.max(), 1)), int(dl.kc.max(initial=0)),
                                             p_(dl.t_own) if sh else None, st),
                          "sweep_up")
            if sh and dl.li == shard.split:
                shard.gather_rows(nxt, _off(dl.kc), dl.li)
            us.append(nxt)
            u = nxt
        v = _dense_apply(cm.device_S(), u, field)
        for li in range(cm.nlevels - 1, -1, -1):
            dl = dls[li]
            sh = dl.mine is not None
            w = torch.empty((int(dl.nr.sum()), Rn), dtype=X.dtype, device="cuda")
            _native.check(L.skel_sweep_down_ex(dl.n_own if sh else dl.p, p_(dl.t_nr), p_(dl.t_kr),
                                               p_(dl.t_rdof_off), p_(dl.t_kr_off), p_(dl.t_d_off),
                                               p_(dl.D), p_(dl.t_l_off), p_(dl.L), p_(us[li]), p_(v),
                                               p_(w), Rn, field, int(max(dl.nr.max(), 1)),
                                               int(dl.kr.max(initial=0)),
                                               p_(dl.t_own) if sh else None, st),
                          "sweep_down")
            if sh and li == 0:
                shard.gather_rows(w, _off(dl.nr), 0)
            v = w
        yt = v
    out = torch.empty_like(yt)
    _native.check(L.skel_permute_rows(p_(perm), cm.n, p_(yt), p_(out), Rn, 1, field, st), "permute")
    if on_dev:
        return out[:, 0] if single else out
    res = _native.to_host(out)
    return res[:, 0] if single else res


def _dense_apply(M, x, field):
    torch = _native.require_cuda()
    K, Kc = M.shape
    Rn = x.shape[1]
    y = torch.empty((K, Rn), dtype=x.dtype, device="cuda")
    if K and Kc:
        _native.check(_native.lib().skel_dense_apply(_native.ptr(M), K, Kc, _native.ptr(x),
                                                     _native.ptr(y), Rn, field,
                                                     _native.stream_ptr()), "dense_apply")
    elif K:
        y.zero_()
    return y


# The reference keeps the SKLC container next to the data model
# (skel.py:428-511); here it lives in container.py and is re-exported lazily
# (container.py imports this module).
_CONTAINER_NAMES = ("serialize_compressed", "deserialize_compressed", "save_compressed",
                    "load_compressed")


def __getattr__(name):
    if name in _CONTAINER_NAMES:
        from . import container
        return getattr(container, name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
