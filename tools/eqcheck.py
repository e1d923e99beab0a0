"""Developer probe: after compression, every box must have kr == kc
(equalize_ranks).  Prints the mismatching boxes with their target shapes.

    python tools/eqcheck.py [log2N] [eps] [reps]
"""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import sys, warnings  # noqa: E401
import numpy as np
import torch
import paper_1110_3105_b200 as sk
from paper_1110_3105_b200 import skel

warnings.simplefilter("ignore")
n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 20)
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-12
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
curve = sk.bie.ellipse(2.0, 1.0, n)
system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
tree = sk.build_tree(system.points, 64)
src = sk.bie.BieSource(system, tree.perm)
for rep in range(reps):
    cm = skel.compress_source(src, tree, eps, eager_factor=False)
    torch.cuda.synchronize()
    bad = 0
    for li, lv in enumerate(cm.levels):
        kr, kc = lv.kr_counts, lv.kc_counts
        nr, nc = lv.row_dof_counts, lv.col_dof_counts
        idx = np.nonzero(kr != kc)[0]
        bad += idx.size
        for a in idx[:5]:
            noff, nidx = tree.cover_neighbors(li)
            nb = nidx[noff[a]:noff[a + 1]]
            print(f"rep {rep} level {li} box {a}: nr={nr[a]} nc={nc[a]} kr={kr[a]} kc={kc[a]} "
                  f"m_row={int(nc[nb].sum())}+pxy m_col={int(nr[nb].sum())}+pxy", flush=True)
        if (nr != nc).any():
            print(f"rep {rep} level {li}: {(nr != nc).sum()} boxes with nr != nc", flush=True)
    print(f"rep {rep}: N={n} eps={eps:g}: {bad} boxes with kr != kc", flush=True)
