"""Full-size probes of BASELINE configs 3 (CFIE 2^18) and 4 (3D sphere 40000):
wall time of each phase, ranks, residual against the exact on-the-fly matvec."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, time, warnings
import numpy as np
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile
import oracle
warnings.simplefilter("ignore")


def timed(f):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t


def report(name, tree, src, cm, fi, B, tc, tf):
    X, ts = timed(lambda: sk.solve(fi, B))
    res = np.linalg.norm(sk.bie.dense_matvec(src, X) - B) / np.linalg.norm(B)
    ks = [(int(lv.dev.kr.max()), int(lv.dev.nr.max())) for lv in cm.levels]
    print(f"{name}: levels {cm.nlevels} S {cm.S_shape()} compress {tc:.3f}s factor {tf:.3f}s "
          f"solve {ts*1e3:.1f}ms residual {res:.2e}", flush=True)
    print("   (max k, max n) per level:", ks, flush=True)


def config3(n=2 ** 18):
    P = oracle.ellipse_perimeter(2.0, 1.0)
    k = 2 * np.pi * 8 / P
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.combined_field_system(curve, k)
    (tree, cm), tc = timed(lambda: sk.bie.compress_system(system, 1e-9, 64))
    fi, tf = timed(lambda: sk.factor(cm))
    rng = np.random.default_rng(0)
    B = rng.standard_normal((n, 4)) + 1j * rng.standard_normal((n, 4))
    report(f"config3 N={n}", tree, sk.bie.BieSource(system, tree.perm), cm, fi, B, tc, tf)


def config4(n=40000):
    pts = sk.PointSet(oracle.fib_sphere(n), None, np.full(n, 4 * np.pi / n))
    tree = sk.build_tree(pts, 64)
    src = sk.KernelSource(sk.KernelSpec("laplace", 3), pts, tree.perm, diag=1.0)
    cm, tc = timed(lambda: sk.compress_source(src, tree, 1e-6))
    fi, tf = timed(lambda: sk.factor(cm))
    B = np.random.default_rng(0).standard_normal((n, 1))
    report(f"config4 N={n}", tree, src, cm, fi, B, tc, tf)


def profile_big(n=40000):
    """Attribute config-4 compress time to the big-box pieces (synchronising)."""
    import collections
    from paper_1110_3105_b200 import _bigbox, skel as skmod
    acc = collections.defaultdict(float)
    cnt = collections.Counter()

    def wrap(name, fn):
        def f(*a, **k):
            torch.cuda.synchronize()
            t = time.perf_counter()
            r = fn(*a, **k)
            torch.cuda.synchronize()
            acc[name] += time.perf_counter() - t
            cnt[name] += 1
            return r
        return f
    _bigbox._norm_estimate = wrap("norm_est", _bigbox._norm_estimate)
    _bigbox._randomized = wrap("randomized(total)", _bigbox._randomized)
    _bigbox.run_boxes = wrap("run_boxes(total)", _bigbox.run_boxes)
    _bigbox.SketchStream.sketch = wrap("sketch_wait", _bigbox.SketchStream.sketch)
    from paper_1110_3105_b200 import _native
    Lb = _native.lib()
    for nm in ("skel_gemm_tn", "skel_big_target", "skel_big_output", "skel_big_probe",
               "skel_big_interp", "skel_gemv", "skel_factor_big", "skel_dense_inverse_big"):
        setattr(Lb, nm, wrap(nm, getattr(Lb, nm)))
    orig = _bigbox._cpqr

    def cp(L, W, m, n, ld, eps, min_rank, resume, state, field, st):
        torch.cuda.synchronize()
        t = time.perf_counter()
        orig(L, W, m, n, ld, eps, min_rank, resume, state, field, st)
        torch.cuda.synchronize()
        key = "cpqr_full" if m > 4000 else "cpqr_sketch"
        acc[key] += time.perf_counter() - t
        cnt[key] += 1
        acc[key + "_steps"] += _bigbox._rank_of(state)
    _bigbox._cpqr = cp
    _profile.reset()
    _profile.enabled = True
    config4(n)
    _profile.enabled = False
    for r in _profile.records:
        if r.kind in ("level", "id_level", "assemble_D", "id_big", "factor_level"):
            m = {k: (v.size if hasattr(v, "size") else v) for k, v in r.meta.items()}
            print(f"  {r.kind:12s} {r.ms():9.2f} ms  {m}")
    for k in sorted(acc, key=lambda k: -acc[k]):
        print(f"  {k:20s} {acc[k]:8.3f} s  x{cnt[k]}")


if __name__ == "__main__" and sys.argv[1] == "prof":
    profile_big(int(sys.argv[2]) if len(sys.argv) > 2 else 40000)
    sys.exit(0)

if __name__ == "__main__":
    which = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else None
    for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
        if which == "3":
            config3(n or 2 ** 18)
        else:
            config4(n or 40000)
