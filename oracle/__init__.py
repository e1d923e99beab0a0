"""CPU oracle for the recursive-skeletonization factor / solve path.

TEST INFRASTRUCTURE ONLY.  This package is a plain numpy/scipy restatement of
the reference algorithm (skelkit 0.1.0, ``/root/reference/pkg/src/skelkit``),
written from the reference's behaviour, not copied from it.  Every function
cites the reference file:line it restates.

Who may use it:
  * ``tests/`` (as the checker for the CUDA path),
  * ``__graft_entry__.smoke()`` (as the checker),
  * ``bench.py`` (the ``cpu_baseline`` leg and ``--impl reference``).

The product package ``paper_1110_3105_b200`` never imports this package; it
fails loudly when its CUDA library is missing.

Pinning: the oracle is pinned against golden vectors generated from the live
reference in this container (``tests/golden/make_golden.py``, fixtures in
``tests/golden/*.npz``), see ``tests/test_oracle_golden.py``.
"""

from .geometry import (Tree, build_tree, cover_children, ellipse, fib_sphere,
                       level_neighbors, proxy_unit_points)
from .entries import eval_block, ellipse_perimeter
from .lowrank import cpqr, id_fixed, id_randomized
from .sources import BieSource, CfieSource, KernelSource
from .rskel import (OracleCompressed, OracleFactored, apply, compress,
                    dense_matvec, factor, solve)

__all__ = [
    "Tree", "build_tree", "cover_children", "ellipse", "fib_sphere",
    "level_neighbors", "proxy_unit_points", "eval_block", "ellipse_perimeter",
    "cpqr", "id_fixed", "id_randomized", "BieSource", "CfieSource",
    "KernelSource", "OracleCompressed", "OracleFactored", "apply", "compress",
    "dense_matvec", "factor", "solve",
]
