"""Does an eager solve between graph replays slow the replays down?"""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, torch, numpy as np, warnings
warnings.simplefilter("ignore")
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree, cm = sk.bie.compress_system(system, 1e-12, 64)
fi = sk.factor(cm)
B = torch.from_numpy(np.random.default_rng(0).standard_normal((n, 16))).cuda()
sk.solve_device(fi, B); sk.solve_device(fi, B); torch.cuda.synchronize()

def t(label, reps=5):
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); sk.solve_device(fi, B); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(label, ["%.2f" % x for x in ts], flush=True)

t("replay")
sk.solve_device(fi, B, graph=False); torch.cuda.synchronize()
t("after eager")
_profile.enabled = True; sk.solve_device(fi, B); torch.cuda.synchronize(); _profile.enabled = False
t("after profiled eager")
B2 = torch.from_numpy(np.random.default_rng(1).standard_normal((n, 16))).cuda()
sk.solve_device(fi, B2); torch.cuda.synchronize()
t("after new B")
