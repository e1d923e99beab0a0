import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, time, torch, numpy as np, warnings
sys.path.insert(0, "/root/repo")
warnings.simplefilter("ignore")
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile
n = 2**20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
B = torch.from_numpy(np.random.default_rng(0).standard_normal((n, 16))).cuda()
flush = torch.empty(512 * 2**20 // 8, dtype=torch.float64, device="cuda")
def fs():
    tree = sk.build_tree(system.points, 64)
    cm = sk.compress_source(sk.bie.BieSource(system, tree.perm), tree, 1e-12)
    return sk.factor(cm)
for _ in range(3):
    fi = fs(); sk.solve_device(fi, B)
for _ in range(3):
    fi = fs()
_profile.reset(); _profile.enabled = True; fs(); torch.cuda.synchronize(); _profile.enabled = False
sk.solve_device(fi, B); sk.solve_device(fi, B); torch.cuda.synchronize()
for flushit in (False, True, False):
    ts = []
    for _ in range(5):
        if flushit: flush.fill_(1.0)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); X = sk.solve_device(fi, B); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print("flush", flushit, ["%.2f" % t for t in ts], flush=True)
