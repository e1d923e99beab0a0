"""Host-side profile (cProfile) of one factor step at a given N."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import cProfile, pstats, sys, time, warnings
import torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
def step():
    tree = sk.build_tree(system.points, 64)
    src = sk.bie.BieSource(system, tree.perm)
    cm = sk.compress_source(src, tree, 1e-12)
    fi = sk.factor(cm)
    torch.cuda.synchronize()
for _ in range(2): step()
t = time.perf_counter(); step(); print("step", time.perf_counter() - t)
pr = cProfile.Profile(); pr.enable(); step(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(40)
