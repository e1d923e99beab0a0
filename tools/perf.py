"""Developer timing probe (not the bench contract): per-phase timings of
compress / factor / solve at a given N, plus per-level device spans."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, time
import numpy as np
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import _profile

LEVELS_SHOWN = tuple(int(x) for x in __import__("os").environ.get("PERF_LEVELS", "0,1,2").split(","))


def run(n, eps, R, reps=4, detail=True):
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    best = None
    for rep in range(reps):
        last = rep == reps - 1
        _profile.reset(); _profile.enabled = last and detail
        torch.cuda.synchronize(); t0 = time.perf_counter()
        tree = sk.build_tree(system.points, 64)
        for li in range(tree.depth): tree.cover_neighbors(li)
        t1 = time.perf_counter()
        src = sk.bie.BieSource(system, tree.perm)
        cm = sk.compress_source(src, tree, eps)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        fi = sk.factor(cm)
        torch.cuda.synchronize(); t3 = time.perf_counter()
        if not _profile.enabled and rep > 0 and (best is None or t3 - t0 < best[3] - best[0]):
            best = (t0, t1, t2, t3)
        _profile.enabled = False
    if best is not None:
        t0, t1, t2, t3 = best
    B = torch.randn(n, R, dtype=torch.float64, device="cuda")
    for _ in range(2): sk.solve_device(fi, B)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    for _ in range(5): X = sk.solve_device(fi, B)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    tsv = (t5 - t4) / 5
    print(f"N={n} eps={eps:g} tree+nbrs {t1-t0:.4f}s compress {t2-t1:.4f}s factor {t3-t2:.4f}s "
          f"solve(R={R}) {tsv*1e3:.3f} ms -> {n*R/tsv:.3e} N*RHS/s  S={tuple(cm.S_dev.shape)} "
          f"factor bytes {fi.factor_bytes()/n:.0f} B/pt", flush=True)
    if detail:
        lv = [r for r in _profile.records if r.kind == "level"]
        idl = [r for r in _profile.records if r.kind == "id_level"]
        for r in lv:
            li = r.meta["level"]
            ks = [x for x in idl if x.meta["level"] == li]
            kms = sum(x.ms() for x in ks)
            print(f"  level {li:2d}: span {r.ms():7.3f} ms  id-kernels(sum) {kms:7.3f} ms  launches {len(ks)} "
                  f"boxes {sum(x.meta['sel'].size for x in ks)}  GF/s {sum(x.flops for x in ks)/max(kms,1e-9)/1e6:8.1f}")
        for x in idl:
            if x.meta["level"] in LEVELS_SHOWN:
                print(f"     L{x.meta['level']} bucket boxes {x.meta['sel'].size:6d} max_m {x.meta['max_m']:4d} "
                      f"max_n {x.meta['max_n']:3d} max_w {x.meta['max_w']:6d}  {x.ms():8.3f} ms")
        fl = [r for r in _profile.records if r.kind == "factor_level"]
        print(f"  factor kernels sum {sum(x.ms() for x in fl):.3f} ms over {len(fl)} launches")
        for li in sorted(set(x.meta["level"] for x in fl)):
            xs = [x for x in fl if x.meta["level"] == li]
            t0 = min(xs, key=lambda x: 0).start
            span = max(x.start.elapsed_time(x.end) for x in xs)
            print(f"    factor L{li}: launches {len(xs)} max-launch {span:.3f} ms  sum {sum(x.ms() for x in xs):.3f} ms "
                  f"GF/s {sum(x.flops for x in xs)/max(sum(x.ms() for x in xs),1e-9)/1e6:.1f}")
    return cm, fi

if __name__ == "__main__":
    for arg in sys.argv[1:]:
        n, eps, R = arg.split(",")
        run(int(n), float(eps), int(R))
