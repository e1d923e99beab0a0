"""paper_1110_3105_b200: recursive-skeletonization factor / multi-RHS solve
(Ho & Greengard, arXiv 1110.3105) on NVIDIA B200 (sm_100a).

Drop-in for the factor/solve path of the reference package ``skelkit``: the
same public names and argument meanings (compress, compress_source, factor,
solve, apply, bie.compress_system / solve_dirichlet, ...), backed by
hand-written CUDA kernels in ``libskel_sm100.so`` (C ABI:
include/skel_b200.h).  PyTorch is used only for device buffers and streams.
There is no CPU fallback.
"""

from . import bie  # noqa: F401
from .errors import (AccuracyWarning, InvalidInput, NotConverged, RefusedTooLarge,
                     SingularBlock, SkelkitError)
from .geom import OrthTree, PointSet, build_tree, level_neighbors, neighbors
from .container import load_compressed, load_factored, save_compressed, save_factored
from .embedding import SparseEmbedding, assemble_embedding, export_matrix_market
from .kernels import KernelSpec, bessel_h0, eval_block
from .krylov import gmres
from .lowrank import (InterpDecomp, id_fixed_precision, id_fixed_precision_batched,
                      id_fixed_precision_large, id_randomized, id_rows)
from .skel import (CompressedLevel, CompressedMatrix, CompressedNode, KernelSource, ProxyConfig,
                   apply, compress, compress_source, proxy_points)
from .solver import FactoredInverse, factor, solve, solve_device

__version__ = "0.1.0"

__all__ = [
    "AccuracyWarning", "InvalidInput", "NotConverged", "RefusedTooLarge", "SingularBlock",
    "SkelkitError", "OrthTree", "PointSet", "build_tree", "level_neighbors", "neighbors",
    "KernelSpec", "eval_block", "InterpDecomp", "id_fixed_precision",
    "id_fixed_precision_batched", "id_fixed_precision_large", "id_randomized", "id_rows", "CompressedLevel", "CompressedMatrix",
    "CompressedNode", "KernelSource", "ProxyConfig", "apply", "compress", "compress_source",
    "proxy_points", "FactoredInverse", "factor", "solve", "solve_device", "__version__",
    "bessel_h0", "save_compressed", "load_compressed", "save_factored", "load_factored",
    "SparseEmbedding", "assemble_embedding", "export_matrix_market", "gmres",
]
