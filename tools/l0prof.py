import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import cProfile, pstats, sys, time, warnings, os
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
for skip in (3, 0):
    skel._DEBUG_SKIP[0] = skip
    for r in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        skel.compress_source(src, tree, 1e-12, eager_factor=False)
        torch.cuda.synchronize(); t1 = time.perf_counter()
    print("skip", skip, "L0 ms", 1e3 * (t1 - t0))
skel._DEBUG_SKIP[0] = 3
pr = cProfile.Profile(); pr.enable()
skel.compress_source(src, tree, 1e-12, eager_factor=False); torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(12)
_profile.enabled = True; _profile.reset()
skel._DEBUG_SKIP[0] = 0
skel.compress_source(src, tree, 1e-12, eager_factor=False); torch.cuda.synchronize()
for r in _profile.records:
    print(r.kind, r.meta.get("level"), f"{r.ms():.3f} ms", r.meta.get("max_m"), r.meta.get("max_n"),
          r.meta["sel"].size if "sel" in r.meta else "")
