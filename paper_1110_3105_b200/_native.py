"""ctypes binding of libskel_sm100.so (the C ABI declared in include/skel_b200.h).

The library is REQUIRED: there is no CPU fallback.  Importing the package
works without a GPU (so the host-side tree builder and symbol checks can run
on a CPU box), but every compute entry point raises when CUDA is absent.
"""

import ctypes
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SKEL_LIB: developer A/B of two builds of the same library (tools/); no fallback either way
LIB_PATH = os.environ.get("SKEL_LIB") or os.path.join(_HERE, "libskel_sm100.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "skel_b200.h")

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_vp = ctypes.c_void_p

SRC_BIE, SRC_KERNEL, SRC_CFIE, SRC_NTRACE = 0, 1, 2, 3
EQ_LAPLACE, EQ_HELMHOLTZ = 0, 1
LAYER_SINGLE, LAYER_DOUBLE = 0, 1


class SkelSource(ctypes.Structure):
    _fields_ = [
        ("x", c_vp), ("y", c_vp), ("z", c_vp),
        ("nx", c_vp), ("ny", c_vp), ("nz", c_vp),
        ("w", c_vp), ("curv", c_vp), ("orig", c_vp),
        ("n", c_i64), ("dim", c_i32), ("kind", c_i32), ("equation", c_i32),
        ("layer", c_i32), ("curvature_limit", c_i32), ("kr10", c_i32),
        ("k", c_f64), ("identity_coef", c_f64), ("diag", c_f64), ("wscale", c_f64),
        ("coincide_tol", c_f64),
        ("grp", c_vp), ("grp_start", c_vp), ("grp_size", c_vp),
    ]


class SkelLevel(ctypes.Structure):
    _fields_ = [
        ("nbox", c_i32), ("level", c_i32), ("equalize", c_i32), ("n_unit", c_i32),
        ("eps", c_f64),
        ("rdof_off", c_vp), ("rdofs", c_vp), ("cdof_off", c_vp), ("cdofs", c_vp),
        ("child_off", c_vp), ("prev_kr", c_vp), ("prev_kc", c_vp),
        ("nbr_off", c_vp), ("nbr", c_vp),
        ("box_c", c_vp), ("box_r", c_vp), ("pxy_begin", c_vp), ("pxy_count", c_vp),
        ("pxy_unit", c_vp),
        ("d_off", c_vp), ("l_off", c_vp), ("r_off", c_vp),
        ("D", c_vp), ("L", c_vp), ("R", c_vp),
        ("rskel", c_vp), ("cskel", c_vp), ("kr", c_vp), ("kc", c_vp), ("flags", c_vp),
        ("scratch", c_vp), ("scratch_bytes", c_i64), ("debug_skip", c_i32),
    ]


class SkelFactorLevel(ctypes.Structure):
    _fields_ = [
        ("nbox", c_i32), ("level", c_i32), ("regularize", c_f64),
        ("n", c_vp), ("k", c_vp),
        ("d_off", c_vp), ("l_off", c_vp), ("r_off", c_vp),
        ("D", c_vp), ("L", c_vp), ("R", c_vp),
        ("child_off", c_vp), ("prev_lam_off", c_vp), ("prev_lam", c_vp), ("prev_k", c_vp),
        ("dd_off", c_vp), ("ld_off", c_vp), ("rd_off", c_vp), ("lam_off", c_vp),
        ("Dd", c_vp), ("Ld", c_vp), ("Rd", c_vp), ("Lam", c_vp),
        ("status", c_vp), ("rcond_d", c_vp), ("rcond_m", c_vp),
        ("scratch", c_vp), ("scratch_bytes", c_i64),
        ("order", c_vp), ("nrun", c_i32),
    ]


_P = ctypes.POINTER
_SIGS = {
    "skel_id_level": [_P(SkelSource), _P(SkelLevel), c_vp, c_i32, c_i32, c_i32, c_i64, c_i32, c_vp],
    "skel_assemble_D": [_P(SkelSource), _P(SkelLevel), c_vp, c_i32, c_i32, c_i32, c_vp],
    "skel_assemble_S": [_P(SkelSource), c_vp, c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_i32, c_vp],
    "skel_eval_block": [_P(SkelSource), c_vp, c_i32, c_vp, c_i32, c_vp, c_i32, c_vp],
    "skel_id_batched": [c_vp, c_vp, c_vp, c_vp, c_i32, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp,
                        c_vp, c_vp, c_vp, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp],
    "skel_pivoted_qr_batched": [c_vp, c_vp, c_vp, c_vp, c_i32, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp,
                                c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp, c_i64, c_i32, c_i32, c_vp],
    "skel_factor_level": [_P(SkelFactorLevel), c_i32, c_i32, c_i32, c_vp],
    "skel_dense_inverse": [c_vp, c_vp, c_vp, c_i32, c_f64, c_vp, c_vp, c_i32, c_vp, c_vp],
    "skel_sweep_up_ex": [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32,
                         c_i32, c_i32, c_vp, c_vp],
    "skel_sweep_down_ex": [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                           c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp],
    "skel_sweep_up_rows": [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32,
                           c_i32, c_i32, c_vp, c_vp, c_vp],
    "skel_sweep_down_rows": [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp,
                             c_vp, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp],
    "skel_dense_apply": [c_vp, c_i32, c_i32, c_vp, c_vp, c_i32, c_i32, c_vp],
    "skel_permute_rows": [c_vp, c_i64, c_vp, c_vp, c_i32, c_i32, c_i32, c_vp],
    "skel_compact_i32": [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "skel_dense_matvec": [_P(SkelSource), c_vp, c_vp, c_i32, c_i32, c_vp],
    "skel_tree_build": [c_vp, c_i64, c_i32, c_i64, _P(c_vp)],
    "skel_perm_mean": [c_vp, c_vp, c_i64, _P(c_f64)],
    "skel_check_points": [c_vp, c_vp, c_i64, c_i32],
    "skel_tree_sizes": [c_vp, _P(c_i64), _P(c_i32)],
    "skel_tree_nodes": [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp],
    "skel_tree_cover": [c_vp, c_i32, _P(c_i64), c_vp],
    "skel_tree_neighbors": [c_vp, c_i32, c_vp, _P(c_i64), c_vp],
    "skel_tree_perm_ptr": [c_vp, c_vp],
    "skel_tree_free": [c_vp],
    "skel_device_query": [_P(c_i32), _P(c_i32), _P(c_i32), _P(c_i32)],
    "skel_fp64_probe": [c_i32, c_i32, c_vp, _P(c_f64), c_vp],
    "skel_big_state_bytes": [c_i32],
    "skel_big_target": [_P(SkelSource), _P(SkelLevel), c_i32, c_i32, c_vp, c_vp, c_i32, c_i32, c_i32,
                        c_vp, c_i64, c_i32, c_vp],
    "skel_cpqr_big": [c_vp, c_i32, c_i32, c_i64, c_f64, c_i32, c_i32, c_vp, c_i32, c_vp],
    "skel_big_interp": [c_vp, c_i32, c_i64, c_vp, c_i32, c_i32, c_vp],
    "skel_big_output": [_P(SkelLevel), c_i32, c_i32, c_vp, c_i64, c_vp, c_i32, c_i32, c_vp],
    "skel_gemm_tn": [c_i32, c_i32, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i32, c_vp],
    "skel_gemv": [c_i32, c_i32, c_i32, c_vp, c_i64, c_vp, c_vp, c_i32, c_vp],
    "skel_big_probe": [c_i32, c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_vp],
    "skel_gj_scratch_bytes": [c_i32],
    "skel_factor_big_bytes": [c_i32, c_i32, c_i32],
    "skel_dense_lu": [c_vp, c_i32, c_vp, c_vp, c_i32, c_vp, c_vp],
    "skel_bessel_h0": [c_vp, c_i64, c_vp, c_vp],
    "skel_plan_id_level": [c_i64] + [c_vp] * 6 + [c_i32, c_i64, c_vp, c_i32, c_vp, c_i32, c_i64, c_i64,
                                                  c_i64] + [c_vp] * 14,
    "skel_plan_factor_level": [c_i64] + [c_vp] * 5 + [c_i32, c_i64, c_vp, c_i32, c_i64, c_i64, c_vp,
                                                      c_i32] + [c_vp] * 17,
    "skel_lu_inverse": [c_vp, c_vp, c_i32, c_vp, c_i32, c_vp],
    "skel_factor_big": [_P(SkelFactorLevel), c_i32, c_i32, c_i32, c_i64, c_i64, c_i64, c_i64, c_vp,
                        c_i64, c_i32, c_vp],
    "skel_dense_inverse_big": [c_vp, c_i32, c_f64, c_vp, c_i32, c_vp, c_vp],
}
_RESTYPE_I64 = {"skel_big_state_bytes", "skel_gj_scratch_bytes", "skel_factor_big_bytes"}

_lib = None

# entry points that launch kernels (the tree builder / queries run on the host)
_LAUNCHING = {"skel_id_level", "skel_assemble_D", "skel_assemble_S", "skel_eval_block", "skel_id_batched",
              "skel_pivoted_qr_batched",
              "skel_factor_level", "skel_dense_inverse", "skel_sweep_up_ex",
              "skel_sweep_down_ex", "skel_dense_apply", "skel_permute_rows",
              "skel_compact_i32", "skel_dense_matvec", "skel_fp64_probe", "skel_big_target",
              "skel_cpqr_big", "skel_big_interp", "skel_big_output", "skel_gemm_tn", "skel_gemv",
              "skel_big_probe", "skel_dense_inverse_big", "skel_factor_big", "skel_dense_lu",
              "skel_lu_inverse", "skel_bessel_h0", "skel_sweep_up_rows", "skel_sweep_down_rows"}
launch_count = [0]


class _CountingLib:
    """Wraps the CDLL so every launching entry point is counted (bench.py
    reports ``gpu_launches`` from this)."""

    def __init__(self, cdll):
        self._cdll = cdll
        for name in _SIGS:
            fn = getattr(cdll, name)
            if name in _LAUNCHING:
                setattr(self, name, self._wrap(name, fn))
            else:
                setattr(self, name, fn)
        self.skel_version = cdll.skel_version

    @staticmethod
    def _wrap(name, fn):
        def call(*args):
            n = 1
            if name == "skel_dense_matvec":
                n = max(1, (int(args[3]) + 3) // 4)
            elif name == "skel_id_level":
                n = 1 if int(args[3]) > 0 else 0
            launch_count[0] += n
            return fn(*args)
        call.__name__ = name
        return call


class NativeError(RuntimeError):
    """A CUDA or argument error reported by libskel_sm100.so."""


def lib():
    """Load the sm_100a library (once).  Fails loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = c_i64 if name in _RESTYPE_I64 else c_i32
        L.skel_version.restype = ctypes.c_char_p
        L.skel_version.argtypes = []
        _lib = _CountingLib(L)
    return _lib


def header_symbols():
    """Function names declared in include/skel_b200.h."""
    with open(HEADER_PATH) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|int)\s+(skel_\w+)\s*\(", text, re.M)))


def check(rc, what):
    if rc != 0:
        raise NativeError(f"{what} failed with status {rc}"
                          + (" (invalid argument / scratch too small)" if rc < 0 else
                             " (CUDA error code)"))


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1110_3105_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return torch


def ptr(t):
    """Raw device/host pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return c_vp(t.data_ptr())


def stream_ptr():
    import torch
    return c_vp(torch.cuda.current_stream().cuda_stream)


_DTYPES = {}


def torch_dtype(field):
    import torch
    return torch.complex128 if field == 1 else torch.float64


def field_of(dtype):
    return 1 if np.issubdtype(np.dtype(dtype), np.complexfloating) else 0


def to_host(t):
    """Device tensor -> numpy through a (cached) pinned host block: a DMA
    copy instead of the pageable staging path."""
    torch = require_cuda()
    h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()
