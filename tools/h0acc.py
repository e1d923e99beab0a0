"""Developer probe: relative accuracy |H0_gpu - H0_mp| / |H0_mp| of bessel_h0 against mpmath
(30 digits) over (0, 700], by range."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import numpy as np
import mpmath as mp
import paper_1110_3105_b200 as sk
mp.mp.dps = 30
rng = np.random.default_rng(0)
edges = [1e-3, 0.5, 2, 5, 8, 12, 16, 20, 25, 30, 50, 100, 300, 700]
for lo, hi in zip(edges[:-1], edges[1:]):
    zs = np.sort(rng.uniform(lo, hi, 300))
    got = sk.bessel_h0(zs)
    worst, wz = 0.0, 0.0
    for z, g in zip(zs, got):
        ref = complex(mp.besselj(0, mp.mpf(float(z))) + 1j * mp.bessely(0, mp.mpf(float(z))))
        e = abs(g - ref) / abs(ref)
        if e > worst:
            worst, wz = e, z
    print(f"[{lo:g}, {hi:g}]: worst rel err {worst:.2e} at z={wz:.6f}", flush=True)
