"""Developer probe: compression-only time at config 2 (N=2^20, eps=1e-12),
the k_id_level union time (CUDA events), and the rank / skeleton-set deltas
against the live-reference fixture tests/golden/full_c2_ellipse_1048576_1e-12.npz.

    python tools/idprof.py [reps]
"""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, time, warnings  # noqa: E401
import numpy as np
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile, skel

warnings.simplefilter("ignore")
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n, eps = 1 << 20, 1e-12
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)
ts = []
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cm = skel.compress_source(src, tree, eps, eager_factor=False)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
print(f"compress only: {1e3 * min(ts[1:] or ts):.2f} ms (min of {max(reps - 1, 1)})", flush=True)
_profile.enabled = True
_profile.reset()
cm = skel.compress_source(src, tree, eps, eager_factor=False)
torch.cuda.synchronize()
launches, tot, _, _ = _profile.summary("id_level")
print(f"id_level: {launches} launches, sum {tot:.2f} ms, union {_profile.union_ms('id_level'):.2f} ms")
per = {}
for rr in _profile.records:
    if rr.kind == "id_level":
        per.setdefault(rr.meta["level"], []).append(rr.ms())
print("per level (ms, sum of bucket launches):",
      " ".join(f"L{k}:{sum(v):.2f}" for k, v in sorted(per.items())))
_profile.enabled = False
gp = _os.path.join(_os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))), "tests", "golden",
                   "full_c2_ellipse_1048576_1e-12.npz")
if _os.path.exists(gp):
    g = np.load(gp)
    hist = {}
    for li in range(int(g["nlevels"])):
        for side, key in ((0, "kr"), (1, "kc")):
            mine = cm.levels[li].kr_counts if side == 0 else cm.levels[li].kc_counts
            d = mine.astype(np.int64) - g[f"L{li}_{key}"].astype(np.int64)
            for v, c in zip(*np.unique(d, return_counts=True)):
                hist[int(v)] = hist.get(int(v), 0) + int(c)
    print("rank delta histogram vs reference:", dict(sorted(hist.items())))
