"""Developer probe: factor once at N, then time solve_device for given R values."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, time, warnings
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile
warnings.simplefilter("ignore")
n = int(sys.argv[1]); Rs = [int(x) for x in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree, cm = sk.bie.compress_system(system, 1e-12, 64)
fi = sk.factor(cm)
for R in Rs:
    B = torch.randn(n, R, dtype=torch.float64, device="cuda")
    for _ in range(3): sk.solve_device(fi, B)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): sk.solve_device(fi, B)
    torch.cuda.synchronize(); t = (time.perf_counter() - t0) / reps
    _profile.enabled = True; _profile.reset(); sk.solve_device(fi, B); torch.cuda.synchronize(); _profile.enabled = False
    cnt, ms, fl, by = _profile.summary("sweep")
    print(f"R={R}: {t*1e3:.3f} ms  {n*R/t:.3e} N*RHS/s  sweeps {cnt} launches {ms:.3f} ms  "
          f"{fl/ms/1e9:.2f} TF/s  {by/ms/1e6:.1f} GB/s", flush=True)
    # per level / direction
    rs = [r for r in _profile.records if r.kind == "sweep"]
    nl = len(fi.levels)
    for i, r in enumerate(rs):
        li = i if i < nl else 2 * nl - 1 - i
        d = fi.levels[li].dev
        print(f"   {r.meta['dir']:4s} L{li:2d} boxes {d.p:6d} {r.ms()*1e3:8.1f} us  {r.nbytes/1e6:8.2f} MB  "
              f"{r.nbytes/max(r.ms(),1e-9)/1e6:8.1f} GB/s  buckets {len(d.solve_buckets)}", flush=True)
