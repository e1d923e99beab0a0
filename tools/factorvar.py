"""Developer probe: spread of repeated factor steps (tree + compress + factor)
at 2^20, with and without the cyclic garbage collector (arg 'nogc')."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import gc, sys, time, warnings
import torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
if len(sys.argv) > 1 and sys.argv[1] == "nogc":
    gc.disable()
ts = []
for it in range(15):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tree = sk.build_tree(system.points, 64)
    cm = sk.compress_source(sk.bie.BieSource(system, tree.perm), tree, 1e-12)
    fi = sk.factor(cm)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
    del fi, cm, tree
print(" ".join(f"{t*1e3:.1f}" for t in ts[3:]))
