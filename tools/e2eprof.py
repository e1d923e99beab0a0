"""Host-side breakdown of the bench's e2e call (bie.solve_dirichlet with host
geometry and a pinned host RHS)."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import cProfile, pstats, sys, time, warnings
import numpy as np
import torch
import paper_1110_3105_b200 as sk
warnings.simplefilter("ignore")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
B = torch.from_numpy(np.random.default_rng(0).standard_normal((n, 16))).pin_memory().numpy()


def step():
    t0 = time.perf_counter()
    sys_e = sk.bie.discretize_dirichlet(sk.bie.Curve2D(curve.t, curve.xy, curve.normals,
                                                       curve.curvature, curve.weights),
                                        sk.KernelSpec("laplace", 2))
    t1 = time.perf_counter()
    tree, cm = sk.bie.compress_system(sys_e, 1e-12, 64)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    fi = sk.factor(cm)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    x = sk.solve(fi, B)
    t4 = time.perf_counter()
    print(f"discretize {1e3*(t1-t0):.1f}  compress {1e3*(t2-t1):.1f}  factor {1e3*(t3-t2):.1f}  "
          f"solve {1e3*(t4-t3):.1f}  total {1e3*(t4-t0):.1f} ms", flush=True)
    return x


for _ in range(3):
    step()
pr = cProfile.Profile(); pr.enable(); step(); pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
