import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SKEL_HOST_TIMING"] = "1"
import io, contextlib, warnings, torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
keep = []
for r in range(5):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        tree, cm = sk.bie.compress_system(system, 1e-12, 64)
        fi = sk.factor(cm)
        torch.cuda.synchronize()
    keep = [cm, fi]
print("\n".join(buf.getvalue().splitlines()[:3]))
