"""Does the eager (overlapped) factorization slow the compression down?
compress with / without the eager factor, and the separate factor time."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import time, warnings, torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)


def t(f):
    torch.cuda.synchronize(); a = time.perf_counter(); r = f(); torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - a)


for eager in (True, False) * 5:
    cm, tc = t(lambda: sk.compress_source(src, tree, 1e-12, eager_factor=eager))
    fi, tf = t(lambda: sk.factor(cm))
    print(f"eager={eager}: compress {tc:.1f} ms  factor {tf:.1f} ms  total {tc + tf:.1f} ms", flush=True)
