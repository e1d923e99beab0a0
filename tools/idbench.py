"""Developer micro-benchmark: level-0 compression only, per variant."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import os, sys, time, warnings
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import skel
warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 20
nlev = int(sys.argv[2]) if len(sys.argv) > 2 else 1
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)
skel._DEBUG_MAX_LEVELS[0] = nlev
for skip in (3, 1, 2, 0):
    skel._DEBUG_SKIP[0] = skip
    ts = []
    for r in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        skel.compress_source(src, tree, 1e-12, eager_factor=False)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"mode={os.environ.get('SKEL_ID_MODE','1')} skip={skip} levels={nlev}: "
          f"{1e3*min(ts[1:]):.2f} ms (min of 3)", flush=True)
