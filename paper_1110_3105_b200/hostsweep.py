"""Compression sweep over EXPLICIT ID targets: the reference's plugin
protocol and ``mode="global"``.

The fast path (``skel.compress_source`` -> ``skel_id_level``) needs a matrix
source with a device descriptor, because it assembles the targets inside the
ID kernel.  The reference accepts ANY object exposing ``block(rows, cols)``,
``proxy_row_block(rows, proxy)``, ``proxy_col_block(cols, proxy)``, ``n``,
``dtype`` and ``wavenumber`` (skel.py:286-290; implemented there by
``KernelSource`` skel.py:100-124, ``_BieSource`` bie.py:233-262 and
``_ScattererSource`` bie.py:326-349), and a quadratic ``mode="global"`` that
compresses each box against its whole off-diagonal block row / column
(skel.py:369-373).  Both go through this module:

* the targets are materialised by the source itself -- its own callbacks for
  a protocol source (Python by contract), the device entry kernel
  (``skel_eval_block``) for sources that have a descriptor -- exactly as
  ``build_node`` composes them (skel.py:341-368): ``t_row = [A(rd, nbr_cols)
  | proxy_row_block(rd, pxy)]``, ``t_col = [A(nbr_rows, cd); proxy_col_block(cd,
  pxy)]``, the proxy count grown by ceil(4 kappa r) for oscillatory kernels;
* every box's two IDs run in ONE batched launch of ``skel_id_batched`` (the
  same CTA CPQR as the fast path, csrc/cpqr.cuh); sides above the randomized
  cut (m > max(4096, 4n + 256), skel.py:414-422) take the GPU randomized ID
  with the reference's seed rule;
* equalisation re-runs the smaller side with ``min_rank = k``
  (skel.py:377-382), again batched;
* skeletons are sorted, ``L = proj.T[:, order]``, ``R = proj[order, :]``
  (skel.py:384-391), and the top ``S`` is assembled block by block from the
  source (skel.py:396-408).

The result is an ordinary (host-built) ``CompressedMatrix``; ``factor`` /
``solve`` / ``apply`` upload it and run the same device kernels as for the
fast path.
"""

from dataclasses import replace

import numpy as np

from . import lowrank
from ._bigbox import randomized, sub_seed
from .errors import InvalidInput


def _blk(source, dtype, rows, cols):
    # nodes can be isolated (no neighbours) or fully compressed away
    if len(rows) == 0 or len(cols) == 0:
        return np.zeros((len(rows), len(cols)), dtype=dtype)
    return np.asarray(source.block(np.asarray(rows, dtype=np.int64),
                                   np.asarray(cols, dtype=np.int64)), dtype=dtype)


def _targets(source, tree, li, a, rd, cd, row, col, nbrs, mode, cfg, k_wave, dtype):
    """(t_row, t_col) of box ``a`` of cover ``li`` (skel.py:349-368)."""
    from .skel import proxy_points, proxy_radius
    if mode == "proxy":
        nb = nbrs[a]
        nbr_cols = np.concatenate([col[b] for b in nb]) if len(nb) else np.empty(0, np.int64)
        nbr_rows = np.concatenate([row[b] for b in nb]) if len(nb) else np.empty(0, np.int64)
        nid = int(tree.levels[li][a])
        hw = float(tree.hw[nid])
        n_eff = cfg.n_proxy
        if k_wave > 0:
            n_eff += int(np.ceil(4.0 * k_wave * proxy_radius(hw, cfg, tree.dim)))
        box = type("Box", (), {"center": tree.center[nid], "halfwidth": hw})
        pxy = proxy_points(box, replace(cfg, n_proxy=n_eff), tree.dim)
        if rd.size:
            t_row = np.hstack([_blk(source, dtype, rd, nbr_cols),
                               np.asarray(source.proxy_row_block(rd, pxy), dtype=dtype)])
        else:
            t_row = np.zeros((0, n_eff), dtype=dtype)
        if cd.size:
            t_col = np.vstack([_blk(source, dtype, nbr_rows, cd),
                               np.asarray(source.proxy_col_block(cd, pxy), dtype=dtype)])
        else:
            t_col = np.zeros((n_eff, 0), dtype=dtype)
    else:
        others = [b for b in range(len(row)) if b != a]
        other_c = np.concatenate([col[b] for b in others]) if others else np.empty(0, np.int64)
        other_r = np.concatenate([row[b] for b in others]) if others else np.empty(0, np.int64)
        t_row = _blk(source, dtype, rd, other_c)
        t_col = _blk(source, dtype, other_r, cd)
    return t_row, t_col


def _ids(mats, eps, seed, tags, min_ranks=None):
    """Column IDs of explicit targets: the deterministic ones in one batched
    launch, the randomized ones (skel.py:419-421) one by one."""
    out = [None] * len(mats)
    det = []
    for q, A in enumerate(mats):
        m, n = A.shape
        if min_ranks is None and randomized(m, n):
            li, a, side = tags[q]
            out[q] = lowrank.id_randomized(A, eps, seed=sub_seed(seed, li, a, side))
        else:
            det.append(q)
    if det:
        mr = None if min_ranks is None else [min_ranks[q] for q in det]
        res = lowrank.id_fixed_precision_batched([mats[q] for q in det], eps, mr)
        for q, r in zip(det, res):
            out[q] = r
    return out


def compress_explicit(source, tree, eps, cfg, mode, equalize_ranks, seed):
    """The level sweep of skel.py:286-411 over explicit targets; returns a
    host-built ``CompressedMatrix`` (see the module docstring)."""
    from .skel import CompressedLevel, CompressedMatrix, CompressedNode
    dtype = np.dtype(source.dtype)
    if dtype not in (np.dtype(np.float64), np.dtype(np.complex128)):
        raise InvalidInput(f"unsupported source dtype {dtype}")
    field = "complex" if dtype == np.complex128 else "real"
    n = tree.n_points
    covers = tree.levels
    top = next(i for i, c in enumerate(covers) if len(c) == 1)
    if top == 0:
        allidx = np.arange(n)
        S = np.ascontiguousarray(_blk(source, dtype, allidx, allidx))
        return CompressedMatrix([], S, n, eps, tree.perm.copy(), field, tree)
    k_wave = float(getattr(source, "wavenumber", 0.0) or 0.0)
    levels = []
    prev_row = prev_col = None
    for li in range(top):
        ids = covers[li]
        p = ids.size
        noff, nidx = tree.cover_neighbors(li)
        nbrs = [nidx[noff[a]:noff[a + 1]] for a in range(p)]
        if li == 0:
            row = [np.arange(tree.lo[i], tree.hi[i], dtype=np.int64) for i in ids]
            col = [r.copy() for r in row]
            children = [None] * p
        else:
            coff = tree.cover_children(li)
            children = [np.arange(coff[a], coff[a + 1], dtype=np.int64) for a in range(p)]
            row = [np.concatenate([prev_row[c] for c in ch]) if ch.size else np.empty(0, np.int64)
                   for ch in children]
            col = [np.concatenate([prev_col[c] for c in ch]) if ch.size else np.empty(0, np.int64)
                   for ch in children]
        Ds, mats, tags = [], [], []
        for a in range(p):
            rd, cd = row[a], col[a]
            D = np.ascontiguousarray(_blk(source, dtype, rd, cd))
            if li > 0:
                ro = np.concatenate([[0], np.cumsum([prev_row[c].size for c in children[a]])])
                co = np.concatenate([[0], np.cumsum([prev_col[c].size for c in children[a]])])
                for ci in range(children[a].size):
                    D[ro[ci]:ro[ci + 1], co[ci]:co[ci + 1]] = 0
            Ds.append(D)
            t_row, t_col = _targets(source, tree, li, a, rd, cd, row, col, nbrs, mode, cfg,
                                    k_wave, dtype)
            mats += [np.ascontiguousarray(t_row.T), t_col]      # row ID = column ID of t_row.T
            tags += [(li, a, 0), (li, a, 1)]
        res = _ids(mats, eps, seed, tags)
        if equalize_ranks:
            redo = []
            for a in range(p):
                kr, kc = res[2 * a].rank, res[2 * a + 1].rank
                if kr != kc:
                    redo.append((2 * a if kr < kc else 2 * a + 1, max(kr, kc)))
            if redo:
                again = _ids([mats[q] for q, _ in redo], eps, seed, [tags[q] for q, _ in redo],
                             [k for _, k in redo])
                for (q, _), r in zip(redo, again):
                    res[q] = r
        nodes = []
        for a in range(p):
            idr, idc = res[2 * a], res[2 * a + 1]
            ro, co = np.argsort(idr.skel), np.argsort(idc.skel)
            nodes.append(CompressedNode(
                row_skel=row[a][idr.skel[ro]], col_skel=col[a][idc.skel[co]], D=Ds[a],
                L=np.ascontiguousarray(np.asarray(idr.proj).T[:, ro], dtype=dtype),
                R=np.ascontiguousarray(np.asarray(idc.proj)[co, :], dtype=dtype),
                children=children[a]))
        levels.append(CompressedLevel(nodes))
        prev_row = [nd.row_skel for nd in nodes]
        prev_col = [nd.col_skel for nd in nodes]
    # dense top skeleton matrix, diagonal blocks zero (skel.py:396-408)
    lv = levels[-1]
    nodes = lv.nodes
    kro = np.concatenate([[0], np.cumsum([nd.k_r for nd in nodes])])
    kco = np.concatenate([[0], np.cumsum([nd.k_c for nd in nodes])])
    S = np.zeros((int(kro[-1]), int(kco[-1])), dtype=dtype)
    for a, nda in enumerate(nodes):
        for b, ndb in enumerate(nodes):
            if a == b or nda.k_r == 0 or ndb.k_c == 0:
                continue
            S[kro[a]:kro[a + 1], kco[b]:kco[b + 1]] = _blk(source, dtype, nda.row_skel, ndb.col_skel)
    return CompressedMatrix(levels, S, n, eps, tree.perm.copy(), field, tree)
