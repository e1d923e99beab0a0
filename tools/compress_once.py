import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, warnings, torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
for r in range(2):
    tree, cm = sk.bie.compress_system(system, 1e-12, 64)
    fi = sk.factor(cm)
torch.cuda.synchronize()
print("ok")
