"""Point sets and the adaptive orthtree (drop-in for skelkit/geom.py).

The tree, its covers and the same-cover neighbour lists are built by native
C++ in libskel_sm100.so (``skel_tree_*``): the reference's recursion
(geom.py:118-184) and its O(p^2) ``level_neighbors`` (geom.py:205-219) are
replaced by an explicit-stack build and an O(p) grid-hash search that keeps
the reference's box-touch predicate, so every list is identical.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import InvalidInput

DEFAULT_MAX_LEAF = {2: 64, 3: 128}


@dataclass
class PointSet:
    """N points in 2D or 3D with optional unit normals, quadrature weights and
    curvatures (validation as geom.py:35-61)."""

    coords: np.ndarray
    normals: np.ndarray | None = None
    weights: np.ndarray | None = None
    curvatures: np.ndarray | None = None

    def __post_init__(self):
        c = np.ascontiguousarray(self.coords, dtype=np.float64)
        if c.ndim != 2 or c.shape[1] not in (2, 3):
            raise InvalidInput(f"coords must be (N, d) with d in {{2,3}}, got {c.shape}")
        if c.shape[0] < 1:
            raise InvalidInput("need at least one point")
        nrm = None
        if self.normals is not None:
            nrm = np.ascontiguousarray(self.normals, dtype=np.float64)
        # finiteness, then (shape and) unit normals, in the reference's order;
        # the two numeric checks are one threaded native pass
        rc = _native.lib().skel_check_points(
            c.ctypes.data_as(ctypes.c_void_p),
            nrm.ctypes.data_as(ctypes.c_void_p) if nrm is not None and nrm.shape == c.shape else None,
            c.shape[0], c.shape[1])
        if rc == -3:
            raise InvalidInput("non-finite coordinate")
        _native.check(rc if rc != -4 else 0, "skel_check_points")
        self.coords = c
        if nrm is not None:
            if nrm.shape != c.shape:
                raise InvalidInput("normals must match coords shape")
            if rc == -4:
                raise InvalidInput("normals must be unit vectors (|n| = 1 within 1e-12)")
            self.normals = nrm
        for name in ("weights", "curvatures"):
            v = getattr(self, name)
            if v is None:
                continue
            v = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
            if v.shape[0] != c.shape[0]:
                raise InvalidInput(f"{name} must have one entry per point")
            setattr(self, name, v)

    @property
    def n(self):
        return self.coords.shape[0]

    @property
    def dim(self):
        return self.coords.shape[1]

    def subset(self, idx):
        pick = lambda a: None if a is None else a[idx]  # noqa: E731
        return PointSet(self.coords[idx], pick(self.normals), pick(self.weights),
                        pick(self.curvatures))


@dataclass
class TreeNode:
    center: np.ndarray
    halfwidth: float
    lo: int
    hi: int
    depth: int
    parent: int | None = None
    children: list = field(default_factory=list)

    @property
    def size(self):
        return self.hi - self.lo


class _TreeHandle:
    """Owns one native tree (csrc/tree.cpp); freed when the OrthTree AND every
    array that borrows native memory (the permutation) are gone."""

    def __init__(self, handle):
        self.ptr = ctypes.c_void_p(handle)

    def __del__(self):
        try:
            if self.ptr:
                _native.lib().skel_tree_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


class OrthTree:
    """Adaptive 2^d tree.  ``levels[0]`` is the finest cover, ``levels[-1]``
    the root alone; ``perm`` maps tree positions to original indices.  Node
    arrays (``center``, ``hw``, ``lo``, ``hi``, ``node_depth``, ``parent``,
    ``nchild``) are kept flat; ``nodes`` materialises TreeNode objects."""

    def __init__(self, handle, dim, n):
        L = _native.lib()
        self._owner = _TreeHandle(handle)
        self._handle = self._owner.ptr
        self.dim = dim
        nn = ctypes.c_int64()
        nc = ctypes.c_int32()
        _native.check(L.skel_tree_sizes(self._handle, ctypes.byref(nn), ctypes.byref(nc)),
                      "skel_tree_sizes")
        nn, nc = nn.value, nc.value
        self.center = np.empty((nn, dim))
        self.hw = np.empty(nn)
        self.lo = np.empty(nn, dtype=np.int64)
        self.hi = np.empty(nn, dtype=np.int64)
        self.node_depth = np.empty(nn, dtype=np.int64)
        self.parent = np.empty(nn, dtype=np.int64)
        self.nchild = np.empty(nn, dtype=np.int64)
        a = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        _native.check(L.skel_tree_nodes(self._handle, a(self.center), a(self.hw), a(self.lo),
                                        a(self.hi), a(self.node_depth), a(self.parent),
                                        a(self.nchild), None), "skel_tree_nodes")
        # the permutation is the native array itself (no 8 n-byte copy per
        # build): a read-only view whose base keeps the tree handle alive, so
        # it stays valid for cm.perm / fi.perm after this object is gone
        pp = ctypes.c_void_p()
        _native.check(L.skel_tree_perm_ptr(self._handle, ctypes.byref(pp)), "skel_tree_perm_ptr")
        if n > 0 and pp.value:
            buf = (ctypes.c_int64 * n).from_address(pp.value)
            buf._owner = self._owner
            self.perm = np.ctypeslib.as_array(buf)
            self.perm.flags.writeable = False
        else:
            self.perm = np.empty(n, dtype=np.int64)
        self.levels = []
        for li in range(nc):
            cnt = ctypes.c_int64()
            _native.check(L.skel_tree_cover(self._handle, li, ctypes.byref(cnt), None),
                          "skel_tree_cover")
            ids = np.empty(cnt.value, dtype=np.int64)
            _native.check(L.skel_tree_cover(self._handle, li, ctypes.byref(cnt), a(ids)),
                          "skel_tree_cover")
            self.levels.append(ids)
        self._nodes = None
        self._nbr_cache = {}

    @property
    def nodes(self):
        if self._nodes is None:
            out = [TreeNode(self.center[i].copy(), float(self.hw[i]), int(self.lo[i]),
                            int(self.hi[i]), int(self.node_depth[i]),
                            None if self.parent[i] < 0 else int(self.parent[i]))
                   for i in range(self.hw.size)]
            for i in range(self.hw.size):
                if self.parent[i] >= 0:
                    out[self.parent[i]].children.append(i)
            self._nodes = out
        return self._nodes

    @property
    def depth(self):
        return len(self.levels)

    @property
    def root(self):
        return self.nodes[int(self.levels[-1][0])]

    @property
    def n_points(self):
        return int(self.hi[0] - self.lo[0])

    def leaves(self):
        return [int(i) for i in np.nonzero(self.nchild == 0)[0]]

    def cover_neighbors(self, li):
        """CSR (offsets, positions) of cover ``li``'s adjacency (cached)."""
        if li not in self._nbr_cache:
            L = _native.lib()
            p = self.levels[li].size
            off = np.empty(p + 1, dtype=np.int64)
            cnt = ctypes.c_int64()
            a = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
            _native.check(L.skel_tree_neighbors(self._handle, li, a(off), ctypes.byref(cnt), None),
                          "skel_tree_neighbors")
            idx = np.empty(cnt.value, dtype=np.int64)
            _native.check(L.skel_tree_neighbors(self._handle, li, a(off), ctypes.byref(cnt), a(idx)),
                          "skel_tree_neighbors")
            self._nbr_cache[li] = (off, idx)
        return self._nbr_cache[li]

    def cover_children(self, li):
        """CSR offsets of cover ``li``'s nodes into cover ``li-1`` (children
        are contiguous runs; skel.py:252-264)."""
        starts = self.lo[self.levels[li - 1]]
        ends = self.hi[self.levels[li]]
        return np.concatenate([[0], np.searchsorted(starts, ends, side="left")]).astype(np.int64)


def build_tree(points: PointSet, max_leaf_size: int | None = None) -> OrthTree:
    """Adaptive orthtree with contiguous per-node ranges (geom.py:118-184),
    built natively."""
    d = points.dim
    if max_leaf_size is None:
        max_leaf_size = DEFAULT_MAX_LEAF[d]
    if max_leaf_size < 1:
        raise InvalidInput("max_leaf_size must be >= 1")
    coords = np.ascontiguousarray(points.coords, dtype=np.float64)
    h = ctypes.c_void_p()
    rc = _native.lib().skel_tree_build(coords.ctypes.data_as(ctypes.c_void_p), points.n, d,
                                       int(max_leaf_size), ctypes.byref(h))
    if rc == -3:        # checked in the native bounding-box pass (geom.py:133)
        raise InvalidInput("non-finite coordinate")
    _native.check(rc, "skel_tree_build")
    return OrthTree(h.value, d, points.n)


def _touch(tree, a, others, tol):
    gap = np.abs(tree.center[others] - tree.center[a]) - (tree.hw[others] + tree.hw[a])[:, None]
    return np.all(gap <= tol, axis=1)


def neighbors(tree: OrthTree, node_id: int) -> list:
    """Same-depth nodes touching ``node_id`` (geom.py:192-202), ascending id."""
    if not isinstance(node_id, (int, np.integer)) or not 0 <= node_id < tree.hw.size:
        raise InvalidInput(f"invalid node id {node_id!r}")
    tol = 1e-9 * tree.hw[0]
    cand = np.nonzero(tree.node_depth == tree.node_depth[node_id])[0]
    cand = cand[cand != node_id]
    return [int(i) for i in cand[_touch(tree, node_id, cand, tol)]]


def level_neighbors(tree: OrthTree, level: int) -> list:
    """Adjacency lists of cover ``level`` (geom.py:205-219), native O(p)."""
    off, idx = tree.cover_neighbors(level)
    return [idx[off[a]:off[a + 1]].tolist() for a in range(off.size - 1)]


# ---------------------------------------------------------------------------
# point-set files (geom.py:225-277): the text and "SKPT" binary layouts

ROOT_PAD = 1e-12          # relative root-box padding (geom.py:133-147), applied in csrc/tree.cpp
_SKPT = b"SKPT"
_SKPT_HEAD = "<IBB"       # N, dim, flags (bit 0: normals, bit 1: weights)


def _columns(dim, has_normals, has_weights):
    return dim * (2 if has_normals else 1) + (1 if has_weights else 0)


def read_points_text(path, dim, has_normals=False, has_weights=False) -> PointSet:
    """One point per row, whitespace separated: coordinates, then (optionally)
    the normal, then (optionally) the weight (geom.py:225-241)."""
    table = np.loadtxt(path, dtype=np.float64, ndmin=2)
    ncol = _columns(dim, has_normals, has_weights)
    if table.shape[1] != ncol:
        raise InvalidInput(f"expected {ncol} columns, found {table.shape[1]}")
    parts = np.split(table, [dim, 2 * dim] if has_normals else [dim], axis=1)
    coords = parts[0]
    normals = parts[1] if has_normals else None
    weights = parts[-1][:, 0] if has_weights else None
    return PointSet(coords, normals, weights)


def write_points_text(ps: PointSet, path):
    """Inverse of read_points_text, 17 significant digits (round-trip exact)."""
    blocks = [a for a in (ps.coords, ps.normals) if a is not None]
    if ps.weights is not None:
        blocks.append(np.asarray(ps.weights).reshape(-1, 1))
    np.savetxt(path, np.concatenate(blocks, axis=1), fmt="%.17g")


def write_points_binary(ps: PointSet, path):
    """"SKPT", u32 N, u8 dim, u8 flags, then little-endian float64 coordinates
    (row-major), normals, weights (geom.py:250-263)."""
    import struct
    flags = int(ps.normals is not None) | (int(ps.weights is not None) << 1)
    with open(path, "wb") as fh:
        fh.write(_SKPT + struct.pack(_SKPT_HEAD, ps.n, ps.dim, flags))
        for a in (ps.coords, ps.normals, ps.weights):
            if a is not None:
                fh.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def read_points_binary(path) -> PointSet:
    import struct
    with open(path, "rb") as fh:
        blob = fh.read()
    hs = struct.calcsize(_SKPT_HEAD)
    if blob[:4] != _SKPT or len(blob) < 4 + hs:
        raise InvalidInput(f"{path}: not a skelkit binary point file")
    n, dim, flags = struct.unpack_from(_SKPT_HEAD, blob, 4)
    shapes = [(n, dim)] + ([(n, dim)] if flags & 1 else []) + ([(n,)] if flags & 2 else [])
    pos, arrays = 4 + hs, []
    for shp in shapes:
        cnt = int(np.prod(shp))
        if pos + 8 * cnt > len(blob):
            raise InvalidInput(f"{path}: truncated point file")
        arrays.append(np.frombuffer(blob, dtype="<f8", count=cnt, offset=pos).reshape(shp).copy())
        pos += 8 * cnt
    coords = arrays.pop(0)
    normals = arrays.pop(0) if flags & 1 else None
    weights = arrays.pop(0) if flags & 2 else None
    return PointSet(coords, normals, weights)
