"""Oracle geometry: curves, point clouds, the adaptive orthtree, covers and
same-cover neighbour lists.  TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Restates:
  * ellipse nodes                 bie.py:81-91
  * Fibonacci sphere              bench.py:108-113
  * adaptive orthtree + covers    geom.py:118-184
  * box-touch predicate           geom.py:187-189
  * level_neighbors               geom.py:205-219 (O(p^2) there; here an O(p)
                                  grid-hash candidate search followed by the
                                  identical predicate, so the lists are equal)
  * cover children                skel.py:252-264
  * proxy surface unit points     skel.py:79-97
"""

from dataclasses import dataclass

import numpy as np

ROOT_PAD = 1e-12          # geom.py:20
MAX_DEPTH = 60            # geom.py:23
DEFAULT_MAX_LEAF = {2: 64, 3: 128}   # geom.py:17


def ellipse(a, b, n):
    """Counter-clockwise ellipse sampled at t_i = 2 pi i / n (bie.py:81-91).

    Returns a dict with xy (n,2), normals (n,2), curvature (n,), weights (n,).
    """
    t = (2.0 * np.pi) * np.arange(n) / n
    ct, st = np.cos(t), np.sin(t)
    xy = np.stack([a * ct, b * st], axis=1)
    speed = np.sqrt((a * st) ** 2 + (b * ct) ** 2)
    nrm = np.stack([b * ct, a * st], axis=1) / speed[:, None]
    return {"t": t, "xy": xy, "normals": nrm,
            "curvature": a * b / speed ** 3,
            "weights": speed * (2.0 * np.pi / n)}


def fib_sphere(n):
    """Fibonacci points on the unit sphere (bench.py:108-113)."""
    s = np.arange(n) + 0.5
    z = 1.0 - 2.0 * s / n
    rho = np.sqrt(np.clip(1.0 - z * z, 0.0, None))
    ang = np.pi * (3.0 - np.sqrt(5.0)) * s
    return np.stack([rho * np.cos(ang), rho * np.sin(ang), z], axis=1)


@dataclass
class Tree:
    """Flat orthtree.  Node arrays are indexed by DFS preorder id, exactly the
    node numbering of geom.py:146-172.  ``covers[0]`` is the finest cover."""
    center: np.ndarray      # (nnodes, d)
    hw: np.ndarray          # (nnodes,)
    lo: np.ndarray
    hi: np.ndarray
    depth: np.ndarray
    parent: np.ndarray
    nchild: np.ndarray
    perm: np.ndarray        # tree position -> original index
    covers: list            # list of int arrays of node ids, finest first
    dim: int

    @property
    def root_hw(self):
        return float(self.hw[0])

    @property
    def n(self):
        return int(self.hi[0])


def build_tree(coords, max_leaf=None):
    """Adaptive 2^d tree with centre splits, upper-child ties, pruning of
    empty children and a DFS permutation (geom.py:118-184)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    n, d = coords.shape
    if max_leaf is None:
        max_leaf = DEFAULT_MAX_LEAF[d]
    lo_c = coords.min(axis=0)
    hi_c = coords.max(axis=0)
    c0 = 0.5 * (lo_c + hi_c)
    hw0 = 0.5 * float((hi_c - lo_c).max())
    scale = max(hw0, float(np.abs(c0).max()), 1.0)
    hw0 = hw0 * (1.0 + ROOT_PAD) + ROOT_PAD * scale

    centers, hws, los, his, depths, parents, nch = [], [], [], [], [], [], []
    perm = np.empty(n, dtype=np.int64)
    cursor = 0
    # explicit stack of (point ids, centre, halfwidth, depth, parent);
    # children pushed in reverse code order -> same preorder as recursion
    stack = [(np.arange(n, dtype=np.int64), c0, hw0, 0, -1)]
    while stack:
        idx, cen, hw, dep, par = stack.pop()
        me = len(centers)
        centers.append(cen.copy())
        hws.append(hw)
        los.append(cursor)
        his.append(cursor + idx.size)
        depths.append(dep)
        parents.append(par)
        nch.append(0)
        if par >= 0:
            nch[par] += 1
        if idx.size <= max_leaf or dep >= MAX_DEPTH:
            perm[cursor:cursor + idx.size] = idx
            cursor += idx.size
            continue
        pts = coords[idx]
        code = np.zeros(idx.size, dtype=np.int64)
        for ax in range(d):
            code |= (pts[:, ax] >= cen[ax]).astype(np.int64) << ax
        kids = []
        for c in range(1 << d):
            sel = idx[code == c]
            if sel.size == 0:
                continue
            off = np.array([(0.5 if (c >> ax) & 1 else -0.5) * hw for ax in range(d)])
            kids.append((sel, cen + off, 0.5 * hw, dep + 1, me))
        stack.extend(reversed(kids))

    depth = np.array(depths, dtype=np.int64)
    nchild = np.array(nch, dtype=np.int64)
    lo = np.array(los, dtype=np.int64)
    maxd = int(depth.max())
    covers = []
    for f in range(maxd, -1, -1):
        sel = np.nonzero((depth == f) | ((nchild == 0) & (depth < f)))[0]
        covers.append(sel[np.argsort(lo[sel], kind="stable")])
    return Tree(center=np.array(centers), hw=np.array(hws, dtype=np.float64),
                lo=lo, hi=np.array(his, dtype=np.int64), depth=depth,
                parent=np.array(parents, dtype=np.int64), nchild=nchild,
                perm=perm, covers=covers, dim=d)


def _touch(ca, ha, cb, hb, tol):
    """Vectorised geom.py:187-189: every axis gap |ca-cb| - (ha+hb) <= tol."""
    gap = np.abs(ca - cb) - (ha + hb)[:, None]
    return np.all(gap <= tol, axis=1)


def level_neighbors(tree: Tree, li: int):
    """Adjacency of cover ``li`` as CSR (offsets, positions), each list sorted
    ascending by cover position -- the lists of geom.py:205-219."""
    ids = tree.covers[li]
    p = ids.size
    if p < 2:
        return np.zeros(p + 1, dtype=np.int64), np.zeros(0, dtype=np.int64)
    tol = 1e-9 * tree.root_hw
    cen = tree.center[ids]
    hw = tree.hw[ids]
    d = tree.dim
    cell = 2.0 * float(hw.min())
    origin = tree.center[0] - tree.hw[0] - 2.0 * cell
    lo_cell = np.floor((cen - hw[:, None] - tol - origin) / cell).astype(np.int64)
    hi_cell = np.floor((cen + hw[:, None] + tol - origin) / cell).astype(np.int64)
    span = hi_cell - lo_cell + 1
    ncells = np.prod(span, axis=1)
    owner = np.repeat(np.arange(p), ncells)
    # enumerate every cell of every box's (tol-expanded) extent
    local = np.arange(owner.size) - np.repeat(np.cumsum(ncells) - ncells, ncells)
    gdim = int(hi_cell.max()) + 2
    key = np.zeros(owner.size, dtype=np.int64)
    rem = local.copy()
    for ax in range(d):
        s = span[owner, ax]
        key = key * gdim + (lo_cell[owner, ax] + rem % s)
        rem //= s
    order = np.lexsort((owner, key))
    key, owner = key[order], owner[order]
    pa, pb = [], []
    for sh in range(1, owner.size):
        same = key[sh:] == key[:-sh]
        if not same.any():
            break
        pa.append(owner[:-sh][same])
        pb.append(owner[sh:][same])
    if pa:
        a = np.concatenate(pa)
        b = np.concatenate(pb)
        pair = np.unique(np.minimum(a, b) * p + np.maximum(a, b))
        a, b = pair // p, pair % p
        ok = _touch(cen[a], hw[a], cen[b], hw[b], tol)
        a, b = a[ok], b[ok]
    else:
        a = b = np.zeros(0, dtype=np.int64)
    src = np.concatenate([a, b])
    dst = np.concatenate([b, a])
    o = np.lexsort((dst, src))
    src, dst = src[o], dst[o]
    off = np.zeros(p + 1, dtype=np.int64)
    np.add.at(off, src + 1, 1)
    return np.cumsum(off), dst


def cover_children(tree: Tree, li: int):
    """CSR offsets of each node of cover ``li`` into cover ``li-1``
    (skel.py:252-264): members of the previous cover whose range starts
    before the node's end, consumed in order."""
    prev = tree.covers[li - 1]
    cur = tree.covers[li]
    starts = tree.lo[prev]
    ends = tree.hi[cur]
    off = np.searchsorted(starts, ends, side="left")
    return np.concatenate([[0], off]).astype(np.int64)


def proxy_unit_points(n, dim):
    """Unit proxy surface (skel.py:79-97) before scaling by r and shifting to
    the box centre: equispaced circle from angle 0, or Fibonacci sphere."""
    if dim == 2:
        th = 2 * np.pi * np.arange(n) / n
        return np.stack([np.cos(th), np.sin(th)], axis=1)
    s = np.arange(n) + 0.5
    z = 1.0 - 2.0 * s / n
    rho = np.sqrt(np.clip(1.0 - z * z, 0.0, None))
    th = np.pi * (3.0 - np.sqrt(5.0)) * s
    return np.stack([rho * np.cos(th), rho * np.sin(th), z], axis=1)


def proxy_radius(hw, dim, radius_factor=1.0):
    """skel.py:75-76."""
    return radius_factor * 3.0 * hw * np.sqrt(dim)
