"""GPU busy fraction of one compress+factor at 2^20: union of the recorded
kernel intervals (id_level, assemble_D, factor_level, id_big, factor_big)
against the wall span of the sweep."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import time, warnings, torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile
warnings.simplefilter("ignore")
n = 2 ** 20
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)
for _ in range(2):
    sk.factor(sk.compress_source(src, tree, 1e-12)); torch.cuda.synchronize()
_profile.reset(); _profile.enabled = True
e0 = torch.cuda.Event(enable_timing=True); e0.record()
cm = sk.compress_source(src, tree, 1e-12); fi = sk.factor(cm)
e1 = torch.cuda.Event(enable_timing=True); e1.record(); torch.cuda.synchronize()
_profile.enabled = False
span = e0.elapsed_time(e1)
iv = sorted((e0.elapsed_time(r.start), e0.elapsed_time(r.end), r.kind) for r in _profile.records
            if r.kind != "level")
busy, cs, ce = 0.0, None, None
per = {}
gaps = []
for a, b, k in iv:
    per[k] = per.get(k, 0.0) + (b - a)
    if cs is None or a > ce:
        if cs is not None:
            busy += ce - cs
            gaps.append((ce, a - ce))
        else:
            gaps.append((0.0, a))
        cs, ce = a, b
    else:
        ce = max(ce, b)
busy += ce - cs
print(f"span {span:.1f} ms  GPU busy (union of kernels) {busy:.1f} ms  ({100 * busy / span:.0f}%)")
print("  per kind (sum of launch durations, overlapping):", {k: round(v, 1) for k, v in per.items()})
gaps.append((ce, span - ce))
lev = sorted((e0.elapsed_time(r.start), r.meta.get("level")) for r in _profile.records if r.kind == "id_level")
first = {}
for tt, l in lev:
    first.setdefault(l, tt)
print("  first id_level launch per level (ms):", {l: round(t, 2) for l, t in sorted(first.items())})
print("  idle gaps >= 0.15 ms (start ms, length ms):", [(round(a, 2), round(g, 2)) for a, g in gaps if g >= 0.15])
print("  idle total %.1f ms in %d gaps" % (sum(g for _, g in gaps), len(gaps)))
