"""Developer probe: per-bucket k_factor_level times (CUDA events) of a separate
(non-eager) factor at config 2.

    python tools/facprof.py
"""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import time, warnings, torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)
cm = sk.compress_source(src, tree, 1e-12, eager_factor=False)
for r in range(2):
    fi = sk.factor(cm)
torch.cuda.synchronize()
_profile.enabled = True; _profile.reset()
t0 = time.perf_counter(); fi = sk.factor(cm); torch.cuda.synchronize(); t1 = time.perf_counter()
_profile.enabled = False
print(f"factor {1e3 * (t1 - t0):.2f} ms")
tot = 0.0
for r in _profile.records:
    if r.kind == "factor_level":
        tot += r.ms()
        if r.meta.get("level", 99) < 3:
            print("  L%d  %.3f ms" % (r.meta["level"], r.ms()), {k: v for k, v in r.meta.items() if k not in ("level", "sel")})
print(f"factor_level launches sum {tot:.2f} ms, union {_profile.union_ms('factor_level'):.2f} ms")
