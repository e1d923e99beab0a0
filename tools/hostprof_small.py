"""Developer probe: host-side cost of the level loop where the GPU work is negligible
(N = 2^14: every level is a 'coarse' level) -- cProfile of 20 compress + factor runs."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import cProfile, pstats, time, warnings
import torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = 2 ** 14
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))


def step():
    tree, cm = sk.bie.compress_system(system, 1e-12, 64)
    fi = sk.factor(cm)
    torch.cuda.synchronize()
    return fi


for _ in range(5):
    step()
t0 = time.perf_counter()
for _ in range(20):
    step()
print(f"{1e3 * (time.perf_counter() - t0) / 20:.2f} ms per compress+factor at N={n}")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(32)
