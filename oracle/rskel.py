"""Oracle recursive skeletonization: compression sweep, telescoping factor,
multi-RHS solve, compressed apply and a chunked dense matvec.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Restates:
  * compress_source + build_node + S   skel.py:286-411
  * _run_id selector                   skel.py:414-422
  * factor (+ _lu, _rcond1)            solver.py:179-276
  * solve                              solver.py:279-318
  * apply                              skel.py:206-249
  * dense residual matvec              bie.py:174-176 (without materialising A)
"""

from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import lu_factor, lu_solve

from .geometry import (Tree, cover_children, level_neighbors, proxy_radius,
                       proxy_unit_points)
from .lowrank import id_fixed, id_randomized

DEFAULT_N_PROXY = {2: 64, 3: 512}      # skel.py:29
RANDOMIZED_CUTOFF = 4096               # skel.py:33
RCOND_WARN = 1e-14                     # solver.py:30


class OracleSingular(Exception):
    def __init__(self, level, node, what):
        self.level, self.node, self.what = level, node, what
        super().__init__(f"singular {what} block at level {level}, node {node}")


class OracleNonSquare(Exception):
    pass


@dataclass
class OracleLevel:
    row_skel: list
    col_skel: list
    D: list
    L: list
    R: list
    child_off: np.ndarray | None      # CSR into previous level (None at li=0)
    box_ids: np.ndarray               # tree node ids of this cover

    @property
    def kr(self):
        return np.array([s.size for s in self.row_skel], dtype=np.int64)

    @property
    def kc(self):
        return np.array([s.size for s in self.col_skel], dtype=np.int64)

    @property
    def nr(self):
        return np.array([d.shape[0] for d in self.D], dtype=np.int64)

    @property
    def nc(self):
        return np.array([d.shape[1] for d in self.D], dtype=np.int64)


@dataclass
class OracleCompressed:
    levels: list
    S: np.ndarray
    n: int
    eps: float
    perm: np.ndarray
    dtype: type
    ids_randomized: int = 0


@dataclass
class OracleFactored:
    Dd: list          # per level list of arrays
    Ld: list
    Rd: list
    Lam: list
    S_lu: tuple | None
    n: int
    perm: np.ndarray
    dtype: type
    warnings: list = field(default_factory=list)


def _offsets(counts):
    return np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)


def run_id(A, eps, seed, tag):
    """skel.py:414-422 -- deterministic unless the target is very tall."""
    m, nn = A.shape
    if m > max(RANDOMIZED_CUTOFF, 4 * nn + 256):
        sub = (seed * 1000003 + hash(tag)) % (2 ** 31)
        return id_randomized(A, eps, seed=sub), True
    return id_fixed(A, eps), False


def _blk(src, r, c):
    if r.size == 0 or c.size == 0:
        return np.zeros((r.size, c.size), dtype=src.dtype)
    return src.block(r, c)


def compress_box(src, tree, li, a, nid, rd, cd, zero, ncols, nrows, eps, npx, radius_factor,
                 mode, equalize, seed):
    """build_node (skel.py:341-391) for box ``a`` of cover ``li`` (tree node
    ``nid``): D with the children's diagonal blocks (``zero`` = their (kr, kc))
    cleared, the proxy (or global) targets, both IDs, equalisation and the
    sorted skeletons.  Returns (row_skel, col_skel, D, L, R, n_randomized)."""
    dtype = src.dtype
    dim = tree.dim
    kw = float(getattr(src, "wavenumber", 0.0))
    D = np.ascontiguousarray(_blk(src, rd, cd), dtype=dtype)
    if zero:
        r0 = c0 = 0
        for kr_c, kc_c in zero:
            D[r0:r0 + kr_c, c0:c0 + kc_c] = 0
            r0 += kr_c
            c0 += kc_c
    if mode == "proxy":
        r = proxy_radius(tree.hw[nid], dim, radius_factor)
        neff = npx
        if kw > 0:
            neff += int(np.ceil(4.0 * kw * r))
        pxy = tree.center[nid] + r * proxy_unit_points(neff, dim)
        t_row = (np.hstack([_blk(src, rd, ncols), src.proxy_row_block(rd, pxy)])
                 if rd.size else np.zeros((0, neff), dtype=dtype))
        t_col = (np.vstack([_blk(src, nrows, cd), src.proxy_col_block(cd, pxy)])
                 if cd.size else np.zeros((neff, 0), dtype=dtype))
    else:
        t_row = _blk(src, rd, ncols)
        t_col = _blk(src, nrows, cd)
    (sr, Pr, kr, _), rz1 = run_id(t_row.T, eps, seed, (li, a, 0))
    (sc, Pc, kc, _), rz2 = run_id(t_col, eps, seed, (li, a, 1))
    if equalize and kr != kc:
        k = max(kr, kc)
        if kr < k:
            sr, Pr, kr, _ = id_fixed(t_row.T, eps, min_rank=k)
        else:
            sc, Pc, kc, _ = id_fixed(t_col, eps, min_rank=k)
    ro = np.argsort(sr)
    co = np.argsort(sc)
    return (rd[sr[ro]], cd[sc[co]], D, np.ascontiguousarray(Pr.T[:, ro], dtype=dtype),
            np.ascontiguousarray(Pc[co, :], dtype=dtype), int(rz1) + int(rz2))


def compress(src, tree: Tree, eps, n_proxy=None, radius_factor=1.0,
             mode="proxy", equalize=True, seed=0):
    """Level sweep of skel.py:286-411 over an oracle source."""
    dim = tree.dim
    dtype = src.dtype
    npx = n_proxy if n_proxy is not None else DEFAULT_N_PROXY[dim]
    n = tree.n
    covers = tree.covers
    top = next(i for i, c in enumerate(covers) if c.size == 1)
    if top == 0:
        allidx = np.arange(n)
        return OracleCompressed([], np.ascontiguousarray(src.block(allidx, allidx), dtype=dtype),
                                n, eps, tree.perm.copy(), dtype)

    levels = []
    prev = None
    n_rand = 0
    for li in range(top):
        ids = covers[li]
        p = ids.size
        noff, nidx = level_neighbors(tree, li)
        if li == 0:
            rows = [np.arange(tree.lo[i], tree.hi[i]) for i in ids]
            cols = [r.copy() for r in rows]
            coff = None
        else:
            coff = cover_children(tree, li)
            rows, cols = [], []
            for a in range(p):
                ch = range(coff[a], coff[a + 1])
                rows.append(np.concatenate([prev.row_skel[c] for c in ch]) if len(ch)
                            else np.empty(0, dtype=np.int64))
                cols.append(np.concatenate([prev.col_skel[c] for c in ch]) if len(ch)
                            else np.empty(0, dtype=np.int64))
        lv = OracleLevel([], [], [], [], [], coff, ids)
        for a in range(p):
            rd, cd = rows[a], cols[a]
            zero = None
            if li > 0:
                zero = [(prev.row_skel[c].size, prev.col_skel[c].size)
                        for c in range(coff[a], coff[a + 1])]
            nb = nidx[noff[a]:noff[a + 1]]
            if mode == "proxy":
                ncols = np.concatenate([cols[b] for b in nb]) if nb.size else np.empty(0, dtype=np.int64)
                nrows = np.concatenate([rows[b] for b in nb]) if nb.size else np.empty(0, dtype=np.int64)
            else:
                ncols = np.concatenate([cols[b] for b in range(p) if b != a])
                nrows = np.concatenate([rows[b] for b in range(p) if b != a])
            sr, sc, D, L, R, nr_ = compress_box(src, tree, li, a, ids[a], rd, cd, zero, ncols,
                                                nrows, eps, npx, radius_factor, mode, equalize,
                                                seed)
            n_rand += nr_
            lv.row_skel.append(sr)
            lv.col_skel.append(sc)
            lv.D.append(D)
            lv.L.append(L)
            lv.R.append(R)
        levels.append(lv)
        prev = lv

    last = levels[-1]
    kro, kco = _offsets(last.kr), _offsets(last.kc)
    S = np.zeros((kro[-1], kco[-1]), dtype=dtype)
    for a in range(len(last.D)):
        for b in range(len(last.D)):
            if a == b or last.row_skel[a].size == 0 or last.col_skel[b].size == 0:
                continue
            S[kro[a]:kro[a + 1], kco[b]:kco[b + 1]] = src.block(last.row_skel[a], last.col_skel[b])
    return OracleCompressed(levels, S, n, eps, tree.perm.copy(), dtype, n_rand)


def _rcond1(A, Ai):
    """solver.py:179-184."""
    if A.size == 0:
        return 1.0
    na = np.abs(A).sum(axis=0).max()
    nb = np.abs(Ai).sum(axis=0).max()
    return 1.0 / (na * nb) if na * nb > 0 else 0.0


def _lu(B, level, node, what, regularize, dtype):
    """solver.py:199-213."""
    if B.shape[0] != B.shape[1]:
        raise OracleNonSquare(f"non-square {what} block at level {level}, node {node}")
    if B.size == 0:
        return None
    if regularize:
        B = B + regularize * np.eye(B.shape[0], dtype=dtype)
    lu, piv = lu_factor(B, check_finite=False)
    if np.any(np.diag(lu) == 0):
        raise OracleSingular(level, node, what)
    return lu, piv


def factor_box(D, L, R, k, lams, li, a, regularize, dtype):
    """factor_node (solver.py:224-262) for box ``a`` of level ``li``: D_eff =
    D with the children's Lambda (``lams``) on the diagonal blocks, LU, D^-1,
    X, RD^-1, Lambda, Rd, Ld, Dd.  Returns (Dd, Ld, Rd, Lam, warnings)."""
    warns = []
    De = np.array(D, dtype=dtype)
    if lams:
        r0 = 0
        for lc in lams:
            De[r0:r0 + lc.shape[0], r0:r0 + lc.shape[1]] = lc
            r0 += lc.shape[0]
    nn = De.shape[0]
    luD = _lu(De, li + 1, a, "D", regularize, dtype)
    if luD is None:
        z = np.zeros((0, 0), dtype=dtype)
        return z, z, z, z, warns
    Dinv = lu_solve(luD, np.eye(nn, dtype=dtype), check_finite=False)
    rc = _rcond1(De, Dinv)
    if rc < RCOND_WARN:
        warns.append((li + 1, a, "D", rc))
    if k == 0:
        return (Dinv, np.zeros((nn, 0), dtype=dtype), np.zeros((0, nn), dtype=dtype),
                np.zeros((0, 0), dtype=dtype), warns)
    X = lu_solve(luD, L, check_finite=False)
    RD = lu_solve(luD, R.T, trans=1, check_finite=False).T
    M = R @ X
    luM = _lu(M, li + 1, a, "Lambda", regularize, dtype)
    Lam = lu_solve(luM, np.eye(k, dtype=dtype), check_finite=False)
    rc = _rcond1(M, Lam)
    if rc < RCOND_WARN:
        warns.append((li + 1, a, "Lambda", rc))
    Rd = Lam @ RD
    return Dinv - X @ Rd, X @ Lam, Rd, Lam, warns


def factor(oc: OracleCompressed, regularize=0.0):
    """Telescoping inverse (solver.py:187-276)."""
    dtype = oc.dtype
    warns = []
    if not oc.levels:
        return OracleFactored([], [], [], [], _lu(np.array(oc.S, dtype=dtype), "top", 0, "S",
                                                  regularize, dtype),
                              oc.n, oc.perm.copy(), dtype, warns)
    Dd_all, Ld_all, Rd_all, Lam_all = [], [], [], []
    lam_prev = None
    for li, lv in enumerate(oc.levels):
        Dd_l, Ld_l, Rd_l, Lam_l = [], [], [], []
        for a in range(len(lv.D)):
            lams = None
            if li > 0:
                lams = [lam_prev[c] for c in range(lv.child_off[a], lv.child_off[a + 1])]
            Dd, Ld, Rd, Lam, w = factor_box(lv.D[a], lv.L[a], lv.R[a], lv.row_skel[a].size,
                                            lams, li, a, regularize, dtype)
            warns.extend(w)
            Dd_l.append(Dd); Ld_l.append(Ld); Rd_l.append(Rd); Lam_l.append(Lam)
        Dd_all.append(Dd_l); Ld_all.append(Ld_l); Rd_all.append(Rd_l); Lam_all.append(Lam_l)
        lam_prev = Lam_l
    last = oc.levels[-1]
    Sh = np.array(oc.S, dtype=dtype)
    kro, kco = _offsets(last.kr), _offsets(last.kc)
    for a, lam in enumerate(lam_prev):
        Sh[kro[a]:kro[a + 1], kco[a]:kco[a + 1]] = lam
    S_lu = _lu(Sh, "top", 0, "S", regularize, dtype)
    return OracleFactored(Dd_all, Ld_all, Rd_all, Lam_all, S_lu, oc.n, oc.perm.copy(),
                          dtype, warns)


def solve(of: OracleFactored, B):
    """Multi-RHS telescoping solve (solver.py:279-318)."""
    B = np.asarray(B)
    single = B.ndim == 1
    dtype = np.result_type(of.dtype, B.dtype)
    bt = B.reshape(of.n, -1).astype(dtype, copy=False)[of.perm]
    if not of.Dd:
        xt = lu_solve(of.S_lu, bt, check_finite=False)
    else:
        ups = [bt]
        u = bt
        for li in range(len(of.Dd)):
            nr = _offsets([d.shape[0] for d in of.Dd[li]])
            kr = _offsets([r.shape[0] for r in of.Rd[li]])
            nxt = np.empty((kr[-1], bt.shape[1]), dtype=dtype)
            for a, Rd in enumerate(of.Rd[li]):
                if Rd.shape[0]:
                    nxt[kr[a]:kr[a + 1]] = Rd @ u[nr[a]:nr[a + 1]]
            ups.append(nxt)
            u = nxt
        v = lu_solve(of.S_lu, u, check_finite=False) if u.shape[0] else u
        for li in range(len(of.Dd) - 1, -1, -1):
            nr = _offsets([d.shape[0] for d in of.Dd[li]])
            nc = _offsets([d.shape[1] for d in of.Dd[li]])
            kc = _offsets([l.shape[1] for l in of.Ld[li]])
            w = np.empty((nc[-1], bt.shape[1]), dtype=dtype)
            for a, Dd in enumerate(of.Dd[li]):
                seg = Dd @ ups[li][nr[a]:nr[a + 1]]
                if of.Ld[li][a].shape[1]:
                    seg = seg + of.Ld[li][a] @ v[kc[a]:kc[a + 1]]
                w[nc[a]:nc[a + 1]] = seg
            v = w
        xt = v
    out = np.empty_like(bt)
    out[of.perm] = xt
    return out[:, 0] if single else out


def apply(oc: OracleCompressed, X):
    """Compressed matvec (skel.py:206-249)."""
    X = np.asarray(X)
    single = X.ndim == 1
    dtype = np.result_type(oc.dtype, X.dtype)
    xt = X.reshape(oc.n, -1).astype(dtype, copy=False)[oc.perm]
    if not oc.levels:
        yt = oc.S @ xt
    else:
        ups = [xt]
        u = xt
        for lv in oc.levels:
            nc = _offsets(lv.nc)
            kc = _offsets(lv.kc)
            nxt = np.zeros((kc[-1], xt.shape[1]), dtype=dtype)
            for a, R in enumerate(lv.R):
                if R.shape[0]:
                    nxt[kc[a]:kc[a + 1]] = R @ u[nc[a]:nc[a + 1]]
            ups.append(nxt)
            u = nxt
        v = oc.S @ u
        for li in range(len(oc.levels) - 1, -1, -1):
            lv = oc.levels[li]
            nr, nc, kr = _offsets(lv.nr), _offsets(lv.nc), _offsets(lv.kr)
            w = np.empty((nr[-1], xt.shape[1]), dtype=dtype)
            for a, D in enumerate(lv.D):
                seg = D @ ups[li][nc[a]:nc[a + 1]]
                if lv.L[a].shape[1]:
                    seg = seg + lv.L[a] @ v[kr[a]:kr[a + 1]]
                w[nr[a]:nr[a + 1]] = seg
            v = w
        yt = v
    out = np.empty_like(xt)
    out[oc.perm] = yt
    return out[:, 0] if single else out


def dense_matvec(src, X, chunk=1024):
    """y = A x with exact entries, row chunks of the tree-ordered matrix
    (the dense oracle of bie.py:174-176 without storing N x N)."""
    X = np.asarray(X)
    single = X.ndim == 1
    xt = X.reshape(src.n, -1)[src.perm]
    allc = np.arange(src.n)
    yt = np.empty((src.n, xt.shape[1]), dtype=np.result_type(src.dtype, X.dtype))
    for r0 in range(0, src.n, chunk):
        rows = np.arange(r0, min(src.n, r0 + chunk))
        yt[rows] = src.block(rows, allc) @ xt
    out = np.empty_like(yt)
    out[src.perm] = yt
    return out[:, 0] if single else out
