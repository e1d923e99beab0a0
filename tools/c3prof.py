"""Developer probe: config 3 (CFIE, complex128, N = 2^18, eps = 1e-9) -- where the time goes
(per-kind kernel unions from CUDA-event records, host span)."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import time, warnings
import numpy as np
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile
import oracle
warnings.simplefilter("ignore")
n = 2 ** 18
k = 2 * np.pi * 8 / oracle.ellipse_perimeter(2.0, 1.0)
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.combined_field_system(curve, k)
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    tree, cm = sk.bie.compress_system(system, 1e-9, 64)
    fi = sk.factor(cm)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"compress+factor {1e3 * (t1 - t0):.1f} ms")
_profile.enabled = True; _profile.reset()
tree, cm = sk.bie.compress_system(system, 1e-9, 64); fi = sk.factor(cm); torch.cuda.synchronize()
_profile.enabled = False
for kind in ("id_level", "factor_level", "assemble_D"):
    c, ms, _, _ = _profile.summary(kind)
    print(f"{kind}: {c} launches, sum {ms:.1f} ms, union {_profile.union_ms(kind):.1f} ms")
per = {}
for r in _profile.records:
    if r.kind in ("id_level", "factor_level"):
        per.setdefault((r.kind, r.meta.get("level")), []).append(r.ms())
print(" ".join(f"{k[0][:2]}L{k[1]}:{sum(v):.1f}" for k, v in sorted(per.items())))
