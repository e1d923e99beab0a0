"""Host profile of FactorRun.add_level and compress_source internals at 2^20."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import cProfile, pstats, warnings, torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import solver
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)
for _ in range(2):
    cm = sk.compress_source(src, tree, 1e-12); sk.factor(cm); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
cm = sk.compress_source(src, tree, 1e-12); sk.factor(cm); torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumtime").print_callees("add_level")
st.sort_stats("tottime").print_stats(30)
