"""Developer probe: per-replay times of the 16-RHS graph solve at 2^20 (L2
flushed between replays, CUDA events), to look at run-to-run spread."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import warnings
import torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree, cm = sk.bie.compress_system(system, 1e-12, 64)
fi = sk.factor(cm)
B = torch.randn(n, 16, dtype=torch.float64, device="cuda")
flush = torch.empty(512 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
sk.solve_device(fi, B); sk.solve_device(fi, B)
ts = []
for _ in range(30):
    flush.fill_(1.0)
    torch.cuda.synchronize()
    e1 = torch.cuda.Event(enable_timing=True); e2 = torch.cuda.Event(enable_timing=True)
    e1.record(); sk.solve_device(fi, B); e2.record(); torch.cuda.synchronize()
    ts.append(e1.elapsed_time(e2))
print(" ".join(f"{t:.2f}" for t in ts))
