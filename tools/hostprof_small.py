"""Developer probe: host cost per level when the levels are small (N=2^14:
every level <= ~500 boxes) -- cProfile of compress_source + factor, sorted by
cumulative time, after warm-up."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import cProfile, pstats, sys, time, warnings  # noqa: E401
import torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 14
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)


def step():
    cm = sk.compress_source(src, tree, 1e-12)
    sk.factor(cm)
    torch.cuda.synchronize()
    return cm


for _ in range(3):
    cm = step()
t = time.perf_counter()
for _ in range(5):
    step()
print(f"N={n} levels={cm.nlevels}: {1e3 * (time.perf_counter() - t) / 5:.2f} ms per compress+factor")
pr = cProfile.Profile()
pr.enable()
step()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(45)
