"""Developer timing probe (not the bench contract): per-phase CUDA-event
timings of compress / factor / solve at a given N."""
import sys, time
import numpy as np
import torch
import paper_1110_3105_b200 as sk

def run(n, eps, R, reps=2):
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    for rep in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        tree = sk.build_tree(system.points, 64)
        for li in range(tree.depth): tree.cover_neighbors(li)
        t1 = time.perf_counter()
        src = sk.bie.BieSource(system, tree.perm)
        cm = sk.compress_source(src, tree, eps)
        torch.cuda.synchronize(); t2 = time.perf_counter()
        fi = sk.factor(cm)
        torch.cuda.synchronize(); t3 = time.perf_counter()
    B = torch.randn(n, R, dtype=torch.float64, device="cuda")
    for _ in range(2): sk.solve_device(fi, B)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    for _ in range(5): X = sk.solve_device(fi, B)
    torch.cuda.synchronize(); t5 = time.perf_counter()
    tsv = (t5 - t4) / 5
    print(f"N={n} eps={eps:g} tree+nbrs {t1-t0:.4f}s compress {t2-t1:.4f}s factor {t3-t2:.4f}s "
          f"solve(R={R}) {tsv*1e3:.3f} ms -> {n*R/tsv:.3e} N*RHS/s  S={tuple(cm.S_dev.shape)} "
          f"factor bytes {fi.factor_bytes()/n:.0f} B/pt", flush=True)
    return cm, fi

if __name__ == "__main__":
    for arg in sys.argv[1:]:
        n, eps, R = arg.split(",")
        run(int(n), float(eps), int(R))
