"""Developer probe: phase breakdown of the level-0 k_id_level launches at config 2
(debug_skip 3 = launch only, 1 = + K1 assembly, 2 = + initial norms, 4 = + CPQR, 5 = + equalisation run,
6 = + interpolation solve, 0 = whole kernel),
per bucket, from CUDA-event records.

    python tools/idphase.py
"""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import warnings
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import skel, _profile
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)
skel._DEBUG_MAX_LEVELS[0] = 1
res = {}
ORDER = (3, 1, 2, 4, 5, 6, 0)
for skip in ORDER:
    skel._DEBUG_SKIP[0] = skip
    for r in range(2):
        skel.compress_source(src, tree, 1e-12, eager_factor=False)
    torch.cuda.synchronize()
    _profile.enabled = True; _profile.reset()
    skel.compress_source(src, tree, 1e-12, eager_factor=False); torch.cuda.synchronize()
    _profile.enabled = False
    res[skip] = [(r.meta.get("max_m"), r.meta.get("max_n"), r.meta["sel"].size if "sel" in r.meta else 0, r.ms())
                 for r in _profile.records if r.kind == "id_level"]
print("bucket (max_m, max_n, boxes): launch-only / +assembly / +norms / +cpqr / +equalise / +interp / all  [ms]")
for i, b in enumerate(res[0]):
    print(b[:3], " ".join(f"{res[s][i][3]:8.3f}" for s in ORDER))
print("sum", " ".join(f"{sum(x[3] for x in res[s]):8.3f}" for s in ORDER))
