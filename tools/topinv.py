"""Developer probe: time and checksum of the top-level dense inverse (skel_dense_inverse)
at the config-2 top size K = 160 (and 208, complex: config 3)."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import hashlib
import numpy as np
import torch
from paper_1110_3105_b200 import solver
rng = np.random.default_rng(0)
for K, field in ((160, 0), (208, 1), (130, 0), (250, 0)):
    A = rng.standard_normal((K, K)) + 4 * np.eye(K)
    if field:
        A = A + 1j * rng.standard_normal((K, K))
    A0 = torch.from_numpy(A).to("cuda")
    ts = []
    for it in range(6):
        S = A0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st, rc = solver._invert_top(S, 0.0, field)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    inv = S.cpu().numpy()
    err = np.abs(inv @ A - np.eye(K)).max()
    print(f"K={K} field={field}: {min(ts):.3f} ms  status {st}  |inv A - I| {err:.2e}  sha {hashlib.sha1(inv.tobytes()).hexdigest()[:12]}")
