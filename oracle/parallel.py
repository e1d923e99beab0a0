"""Process-parallel driver of the oracle's compress + factor sweep.
TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__): this is how
``bench.py --impl reference`` (and the ``cpu_baseline`` leg) time the
reference algorithm on the GPU box's host cores at the FULL BASELINE size.

It is the reference's own parallel structure -- ``_map_nodes`` farms the
boxes of one level out to a pool (skel.py:38-50, 393; solver.py:264) -- with
processes instead of threads (the reference's threads serialise on the GIL,
SURVEY §8(d): SKELKIT_THREADS=8 is 2x slower).  Per level the parent builds
every box's dof / neighbour index lists (skel.py:316-352) and ships chunks of
boxes to the workers; a worker runs build_node (``rskel.compress_box``) and
then that box's factor_node (``rskel.factor_box``, solver.py:224-262, fed
with its children's Lambda), and returns the skeletons plus the factor
blocks the solve needs.  The per-box arithmetic is exactly the sequential
oracle's, so results are identical to ``rskel.compress`` + ``rskel.factor``
(checked in tests/test_host_cpu.py).  The compressed D/L/R blocks are
computed but stay in the workers (the solve does not read them).
"""

import multiprocessing as mp
import os

import numpy as np

from . import rskel
from .geometry import cover_children, level_neighbors

_G = {}


def _init(src, tree, eps, npx):
    # one BLAS thread per worker process: the pool is the parallelism (an
    # inherited multi-threaded OpenBLAS oversubscribes the cores)
    try:
        from threadpoolctl import threadpool_limits
        _G["limits"] = threadpool_limits(1)
    except Exception:
        pass
    _G.update(src=src, tree=tree, eps=eps, npx=npx)


def _work(job):
    li, items = job
    src, tree, eps, npx = _G["src"], _G["tree"], _G["eps"], _G["npx"]
    out = []
    for a, nid, rd, cd, zero, ncols, nrows, lams in items:
        sr, sc, D, L, R, _ = rskel.compress_box(src, tree, li, a, nid, rd, cd, zero, ncols,
                                                nrows, eps, npx, 1.0, "proxy", True, 0)
        Dd, Ld, Rd, Lam, w = rskel.factor_box(D, L, R, sr.size, lams, li, a, 0.0, src.dtype)
        out.append((a, sr, sc, Dd, Ld, Rd, Lam, w))
    return out


def workers_default():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


class ParallelRun:
    """Persistent worker pool bound to one (source, tree, eps)."""

    def __init__(self, src, tree, eps, workers=None):
        self.src, self.tree, self.eps = src, tree, eps
        self.workers = workers or workers_default()
        self.npx = rskel.DEFAULT_N_PROXY[tree.dim]
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(self.workers, initializer=_init,
                             initargs=(src, tree, eps, self.npx))

    def close(self):
        self.pool.close()
        self.pool.join()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def compress_factor(self):
        """Levels 0..top-1 then the top S / Shat LU.  Returns an
        ``OracleFactored`` (Dd/Ld/Rd/Lam per level + LU of Shat)."""
        src, tree = self.src, self.tree
        dtype = src.dtype
        covers = tree.covers
        top = next(i for i, c in enumerate(covers) if c.size == 1)
        Dd_all, Ld_all, Rd_all, Lam_all, warns = [], [], [], [], []
        prev_rs = prev_cs = prev_lam = None
        rows = cols = None
        for li in range(top):
            ids = covers[li]
            p = ids.size
            noff, nidx = level_neighbors(tree, li)
            coff = None
            if li == 0:
                rows = [np.arange(tree.lo[i], tree.hi[i]) for i in ids]
                cols = [r.copy() for r in rows]
            else:
                coff = cover_children(tree, li)
                rows, cols = [], []
                for a in range(p):
                    ch = range(coff[a], coff[a + 1])
                    rows.append(np.concatenate([prev_rs[c] for c in ch]) if len(ch)
                                else np.empty(0, dtype=np.int64))
                    cols.append(np.concatenate([prev_cs[c] for c in ch]) if len(ch)
                                else np.empty(0, dtype=np.int64))
            items = []
            empty = np.empty(0, dtype=np.int64)
            for a in range(p):
                nb = nidx[noff[a]:noff[a + 1]]
                ncols = np.concatenate([cols[b] for b in nb]) if nb.size else empty
                nrows = np.concatenate([rows[b] for b in nb]) if nb.size else empty
                zero = lams = None
                if li > 0:
                    ch = range(coff[a], coff[a + 1])
                    zero = [(prev_rs[c].size, prev_cs[c].size) for c in ch]
                    lams = [prev_lam[c] for c in ch]
                items.append((a, int(ids[a]), rows[a], cols[a], zero, ncols, nrows, lams))
            nchunk = max(1, min(p, 4 * self.workers))
            bounds = np.linspace(0, p, nchunk + 1).astype(int)
            jobs = [(li, items[bounds[c]:bounds[c + 1]]) for c in range(nchunk)
                    if bounds[c + 1] > bounds[c]]
            res = [None] * p
            for part in self.pool.imap(_work, jobs):
                for r in part:
                    res[r[0]] = r
            prev_rs = [r[1] for r in res]
            prev_cs = [r[2] for r in res]
            prev_lam = [r[6] for r in res]
            Dd_all.append([r[3] for r in res])
            Ld_all.append([r[4] for r in res])
            Rd_all.append([r[5] for r in res])
            Lam_all.append(prev_lam)
            for r in res:
                warns.extend(r[7])
        # top: S over the last level's skeletons (skel.py:399-408), Shat LU
        # (solver.py:269-274)
        kr = np.array([s.size for s in prev_rs])
        kc = np.array([s.size for s in prev_cs])
        kro, kco = rskel._offsets(kr), rskel._offsets(kc)
        Sh = np.zeros((kro[-1], kco[-1]), dtype=dtype)
        for a in range(len(prev_rs)):
            for b in range(len(prev_cs)):
                if a != b and prev_rs[a].size and prev_cs[b].size:
                    Sh[kro[a]:kro[a + 1], kco[b]:kco[b + 1]] = src.block(prev_rs[a], prev_cs[b])
        for a, lam in enumerate(prev_lam):
            Sh[kro[a]:kro[a + 1], kco[a]:kco[a + 1]] = lam
        S_lu = rskel._lu(Sh, "top", 0, "S", 0.0, dtype)
        fac = rskel.OracleFactored(Dd_all, Ld_all, Rd_all, Lam_all, S_lu, tree.n,
                                   tree.perm.copy(), dtype, warns)
        fac.kr_levels = [np.array([r.shape[0] for r in lv]) for lv in Rd_all]
        return fac
