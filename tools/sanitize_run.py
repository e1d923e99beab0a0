"""Developer probe for compute-sanitizer (memcheck / racecheck / synccheck):
the config-1 pipeline (N=4096, eps=1e-9: 2-CTA cluster ID kernel with DSMEM
equalisation, factor, DMMA solve sweeps, dense matvec) and, with argv[1] ==
"big", the same pipeline with every box routed through the whole-GPU big-box
path (grid-synchronised CPQR / factor kernels of big.cu).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py [big]
"""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, warnings  # noqa: E401
import numpy as np
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import skel

warnings.simplefilter("ignore")
big = len(sys.argv) > 1 and sys.argv[1] == "big"
n = int(sys.argv[2]) if len(sys.argv) > 2 else (2048 if big else 4096)
if big:
    skel._BIG_N = 0
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree, cm = sk.bie.compress_system(system, 1e-9, 64)
fi = sk.factor(cm)
B = np.random.default_rng(0).standard_normal((n, 4))
X = sk.solve(fi, B)
B64 = np.random.default_rng(1).standard_normal((n, 64))
X64 = sk.solve(fi, B64)
torch.cuda.synchronize()
src = sk.bie.BieSource(system, tree.perm)
res = np.linalg.norm(sk.bie.dense_matvec(src, X) - B) / np.linalg.norm(B)
print(f"sanitize_run ok: big={big} N={n} levels={cm.nlevels} S={cm.S_shape()} residual={res:.2e}")
