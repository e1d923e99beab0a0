"""Full-size golden fixtures from the LIVE reference (skelkit 0.1.0) at the
BASELINE sizes: config 2 (+5) at N=2^20 / 1e-12, config 3 (CFIE) at N=2^18 /
1e-9, config 4 (3D sphere) at N=40000 / 1e-6.

Run in the build container only (the reference is not on GPU boxes):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_full.py c2
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_full.py c3
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_full.py c4

(about 10 min, 45 min and 45 min of one core each).  The only change to the
reference is the one SURVEY F4 validated: ``skelkit.skel.level_neighbors``
(O(p^2) Python, geom.py:205-219) is replaced by an O(p) grid-hash candidate
search followed by the reference's own ``_boxes_touch`` predicate, which
returns identical lists (checked here on every level against the reference
function wherever the cover has <= 3000 boxes).

The fixtures stay small: per level the per-box ranks (int16), dof counts and
an order-independent 64-bit hash of each box's row / column skeleton set (so
the count of boxes whose skeleton sets differ is exact without shipping the
sets), the top S shape, one solution column, and for config 5 a Gaussian
sketch of 64 solution columns.
"""

import os
import sys
import time
import types
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import skelkit  # noqa: E402
from skelkit import bie, geom  # noqa: E402
import skelkit.skel as rskel  # noqa: E402
from skelkit.kernels import KernelSpec  # noqa: E402
from skelkit.skel import compress_source  # noqa: E402

from make_golden import CfieSource, DiagOneSource, perimeter, sphere_points  # noqa: E402
from oracle.geometry import level_neighbors as _grid_neighbors  # noqa: E402
from skelhash import skel_set_hash  # noqa: E402

_REF_LEVEL_NEIGHBORS = geom.level_neighbors


def fast_level_neighbors(tree, level):
    """O(p) replacement for geom.level_neighbors with identical output."""
    t = types.SimpleNamespace(
        covers=[np.asarray(c, dtype=np.int64) for c in tree.levels],
        center=np.array([nd.center for nd in tree.nodes]),
        hw=np.array([nd.halfwidth for nd in tree.nodes]),
        root_hw=tree.root.halfwidth, dim=tree.dim)
    off, idx = _grid_neighbors(t, level)
    out = [idx[off[a]:off[a + 1]].tolist() for a in range(len(off) - 1)]
    if len(tree.levels[level]) <= 3000:
        assert out == _REF_LEVEL_NEIGHBORS(tree, level), level
    return out


rskel.level_neighbors = fast_level_neighbors


def pack_ranks(cm, tree):
    out = {"nlevels": np.array(cm.nlevels), "S_shape": np.array(cm.S.shape)}
    for li, lv in enumerate(cm.levels):
        out[f"L{li}_kr"] = lv.kr_counts.astype(np.int16)
        out[f"L{li}_kc"] = lv.kc_counts.astype(np.int16)
        out[f"L{li}_nr"] = lv.row_dof_counts.astype(np.int16)
        out[f"L{li}_nc"] = lv.col_dof_counts.astype(np.int16)
        rs = np.concatenate([nd.row_skel for nd in lv.nodes]) if lv.nodes else np.zeros(0, np.int64)
        cs = np.concatenate([nd.col_skel for nd in lv.nodes]) if lv.nodes else np.zeros(0, np.int64)
        out[f"L{li}_row_hash"] = skel_set_hash(rs, lv.kr_counts)
        out[f"L{li}_col_hash"] = skel_set_hash(cs, lv.kc_counts)
    # perm fingerprint: the GPU tree is checked against the oracle elsewhere
    out["perm_hash"] = skel_set_hash(tree.perm * 1048583 + np.arange(tree.perm.size),
                                     np.array([tree.perm.size]))
    return out


def _timed(label, fn):
    t0 = time.perf_counter()
    r = fn()
    print(f"  {label}: {time.perf_counter() - t0:.1f} s", flush=True)
    return r


def config2():
    n, eps = 1 << 20, 1e-12
    curve = bie.ellipse(2.0, 1.0, n)
    system = bie.discretize_dirichlet(curve, KernelSpec("laplace", 2))
    tree, cm = _timed("compress", lambda: bie.compress_system(system, eps, 64))
    fi = _timed("factor", lambda: skelkit.factor(cm))
    out = pack_ranks(cm, tree)
    out["factor_warnings"] = np.array(len(fi.warnings))
    # config 2: column 0 of the seeded 16-RHS draw
    B = np.random.default_rng(0).standard_normal((n, 16))
    X = _timed("solve16", lambda: skelkit.solve(fi, B))
    out["X0"] = X[:, 0].copy()
    out["X_colnorm"] = np.linalg.norm(X, axis=0)
    del B, X
    # config 5: first 64 columns of the seeded 1024-RHS draw, sketched
    B5 = np.random.default_rng(0).standard_normal((n, 1024))[:, :64].copy()
    X5 = _timed("solve64", lambda: skelkit.solve(fi, B5))
    Om = np.random.default_rng(1).standard_normal((n, 8))
    out["c5_sketch"] = Om.T @ X5
    out["c5_colnorm"] = np.linalg.norm(X5, axis=0)
    out.update({"eps": np.array(eps), "n": np.array(n)})
    return out


def config3():
    n, eps = 1 << 18, 1e-9
    k = 2 * np.pi * 8 / perimeter()
    curve = bie.ellipse(2.0, 1.0, n)
    tree = geom.build_tree(curve.point_set(), 64)
    src = CfieSource(curve, tree.perm, k)
    cm = _timed("compress", lambda: compress_source(src, tree, eps))
    fi = _timed("factor", lambda: skelkit.factor(cm))
    rng = np.random.default_rng(0)
    B = rng.standard_normal((n, 4)) + 1j * rng.standard_normal((n, 4))
    X = _timed("solve", lambda: skelkit.solve(fi, B))
    out = pack_ranks(cm, tree)
    out.update({"X0": X[:, 0].copy(), "X_colnorm": np.linalg.norm(X, axis=0),
                "eps": np.array(eps), "n": np.array(n), "k": np.array(k),
                "factor_warnings": np.array(len(fi.warnings))})
    return out


def config4():
    n, eps = 40000, 1e-6
    pts = skelkit.PointSet(sphere_points(n), None, np.full(n, 4 * np.pi / n))
    tree = geom.build_tree(pts, 64)
    src = DiagOneSource(KernelSpec("laplace", 3), pts, tree.perm)
    cm = _timed("compress", lambda: compress_source(src, tree, eps))
    fi = _timed("factor", lambda: skelkit.factor(cm))
    B = np.random.default_rng(0).standard_normal((n, 1))
    X = _timed("solve", lambda: skelkit.solve(fi, B))
    out = pack_ranks(cm, tree)
    out.update({"X": X, "eps": np.array(eps), "n": np.array(n),
                "factor_warnings": np.array(len(fi.warnings))})
    return out


JOBS = {"c2": ("full_c2_ellipse_1048576_1e-12", config2),
        "c3": ("full_c3_cfie_262144_1e-9", config3),
        "c4": ("full_c4_sphere_40000_1e-6", config4)}


def main():
    warnings.simplefilter("ignore")
    for key in sys.argv[1:] or list(JOBS):
        name, fn = JOBS[key]
        print(name, flush=True)
        t0 = time.perf_counter()
        data = fn()
        data["ref_seconds"] = np.array(time.perf_counter() - t0)
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **data)
        print(f"{name}: {os.path.getsize(path) / 1e6:.2f} MB, {time.perf_counter() - t0:.0f} s",
              flush=True)


if __name__ == "__main__":
    main()
