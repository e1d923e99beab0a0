"""Developer check: the reference-side ctypes binding shown in INTEGRATION.md
(pivoted_qr_b200 over skel_pivoted_qr_batched) run verbatim against the built library and
compared with the package's own lowrank.pivoted_qr."""
import os as _os, sys as _sys  # noqa: E401
_ROOT = _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__)))
_sys.path.insert(0, _ROOT)
import ctypes, re  # noqa: E401
import numpy as np

_lib = ctypes.CDLL(_os.path.join(_ROOT, "paper_1110_3105_b200", "libskel_sm100.so"))
text = open(_os.path.join(_ROOT, "INTEGRATION.md")).read()
src = re.search(r"```python\n(def pivoted_qr_b200.*?)```", text, re.S).group(1)
exec(src)
rng = np.random.default_rng(2)
A = (np.linalg.qr(rng.standard_normal((80, 30)))[0] * 0.4 ** np.arange(30)) @ rng.standard_normal((30, 50))
piv, R, r, ratio = pivoted_qr_b200(A, 1e-9)            # noqa: F821
from paper_1110_3105_b200.lowrank import pivoted_qr
piv2, R2, r2, ratio2 = pivoted_qr(A, 1e-9)
assert r == r2 and np.array_equal(piv, piv2) and np.array_equal(R, R2) and ratio == ratio2
print(f"binding ok: rank {r}, ratio {ratio:.3e}, |A P - Q R| check via Gram: "
      f"{np.abs(R[:, :r].T @ R[:, :r] - A[:, piv[:r]].T @ A[:, piv[:r]]).max():.2e}")
