"""Developer probe: host time before the first ID launch at 2^20 (tree,
neighbours, BieSource, level-0 geometry)."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import time, warnings
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import skel
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = sk.build_tree(system.points, 64)
    t1 = time.perf_counter()
    tree.cover_neighbors(0)
    t2 = time.perf_counter()
    src = sk.bie.BieSource(system, tree.perm)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"tree {1e3*(t1-t0):.2f}  nbrs {1e3*(t2-t1):.2f}  BieSource {1e3*(t3-t2):.2f} ms", flush=True)
