"""Interpolative decompositions on the GPU (drop-in for the deterministic
path of skelkit/lowrank.py): the same CTA-cooperative CPQR routine the
compression kernel uses (csrc/cpqr.cuh), exposed for explicit matrices."""

import warnings
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InvalidInput


@dataclass
class InterpDecomp:
    """A ~ A[:, skel] @ proj; skel in pivot order, proj[:, skel] == I."""
    skel: np.ndarray
    proj: np.ndarray
    rank: int
    achieved_error: float

    @property
    def k(self):
        return self.rank


def _as_matrix(A):
    A = np.asarray(A)
    if A.dtype.kind not in "fc":
        A = A.astype(np.float64)
    if A.ndim != 2:
        raise InvalidInput("expected a 2D matrix")
    if not np.all(np.isfinite(A)):
        raise InvalidInput("matrix has non-finite entries")
    return A


def id_fixed_precision_batched(mats, eps, min_ranks=None):
    """Column IDs of several matrices in one launch (one CTA per matrix)."""
    torch = _native.require_cuda()
    if not 0 < eps < 1:
        raise InvalidInput("eps must lie in (0, 1)")
    mats = [_as_matrix(A) for A in mats]
    cplx = any(A.dtype.kind == "c" for A in mats)
    dt = np.complex128 if cplx else np.float64
    field = int(cplx)
    nb = len(mats)
    ms = np.array([A.shape[0] for A in mats], dtype=np.int32)
    ns = np.array([A.shape[1] for A in mats], dtype=np.int32)
    a_off = np.concatenate([[0], np.cumsum(ms.astype(np.int64) * ns)]).astype(np.int64)
    flat = np.concatenate([np.asarray(A, dtype=dt).ravel(order="F") for A in mats]) if nb else np.zeros(0, dt)
    s_off = np.concatenate([[0], np.cumsum(ns.astype(np.int64))]).astype(np.int64)
    p_off = np.concatenate([[0], np.cumsum(ns.astype(np.int64) ** 2)]).astype(np.int64)
    mr = np.zeros(nb, dtype=np.int32) if min_ranks is None else np.asarray(min_ranks, dtype=np.int32)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    dA, dao, dm, dn, dmr = up(flat), up(a_off), up(ms), up(ns), up(mr)
    rank = torch.zeros(nb, dtype=torch.int32, device=dev)
    skel = torch.zeros(max(int(s_off[-1]), 1), dtype=torch.int32, device=dev)
    proj = torch.zeros(max(int(p_off[-1]), 1), dtype=_native.torch_dtype(field), device=dev)
    big = torch.zeros(nb, dtype=torch.float64, device=dev)
    ratio = torch.zeros(nb, dtype=torch.float64, device=dev)
    dso, dpo = up(s_off), up(p_off)
    max_m = int(ms.max()) if nb else 1
    max_n = int(ns.max()) if nb else 1
    # real targets use an even leading dimension inside the kernel
    need = nb * (max_m + (0 if cplx else max_m % 2)) * max_n * (16 if cplx else 8)
    scratch = torch.empty(max(need // 8, 1), dtype=torch.float64, device=dev)
    p = _native.ptr
    _native.check(_native.lib().skel_id_batched(
        p(dA), p(dao), p(dm), p(dn), nb, float(eps), p(dmr), p(rank), p(skel), p(dso), p(proj),
        p(dpo), p(big), p(ratio), field, p(scratch), scratch.numel() * 8, max_m, max_n,
        _native.stream_ptr()), "skel_id_batched")
    rank, skel, proj, big = rank.cpu().numpy(), skel.cpu().numpy(), proj.cpu().numpy(), big.cpu().numpy()
    ratio = ratio.cpu().numpy()
    out = []
    for b in range(nb):
        k, n = int(rank[b]), int(ns[b])
        P = proj[p_off[b]:p_off[b] + k * n].reshape(k, n).astype(dt)
        if big[b] > 2.0:
            warnings.warn(f"interpolation matrix entries reach {big[b]:.3g} (> 2); "
                          "pivoting quality degraded on this block", stacklevel=3)
        out.append(InterpDecomp(skel=skel[s_off[b]:s_off[b] + k].astype(np.int64), proj=P,
                                rank=k, achieved_error=float(ratio[b])))
    return out


def id_fixed_precision(A, eps, min_rank=0) -> InterpDecomp:
    """Column ID to relative precision eps by CPQR (lowrank.py:136-161)."""
    if not 0 < eps < 1:
        raise InvalidInput("eps must lie in (0, 1)")
    return id_fixed_precision_batched([A], eps, [min_rank])[0]


def id_rows(A, eps, min_rank=0) -> InterpDecomp:
    """Row ID: A ~ proj.T @ A[skel, :] (plain transpose, lowrank.py:164-166)."""
    return id_fixed_precision(np.asarray(A).T, eps, min_rank=min_rank)


def pivoted_qr(A, eps, min_rank=0):
    """Column-pivoted Householder QR stopped at relative pivot size eps, but not
    before min_rank columns (lowrank.py:48-119), on the GPU (the CPQR of
    csrc/cpqr.cuh through ``skel_pivoted_qr_batched``).

    Returns (piv, R, rank, trailing_ratio) as the reference does: the whole
    pivot permutation, the rank x n upper-trapezoidal factor with its columns
    in pivot order, the number of completed steps and the first rejected pivot
    magnitude over the leading one."""
    torch = _native.require_cuda()
    A = _as_matrix(A)
    m, n = A.shape
    cplx = A.dtype.kind == "c"
    dt = np.complex128 if cplx else np.float64
    if m == 0 or n == 0:
        return np.arange(n), np.zeros((0, n), dtype=dt), 0, 0.0
    field = int(cplx)
    dev = torch.device("cuda")
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
    tdt = _native.torch_dtype(field)
    dA = up(np.asarray(A, dtype=dt).ravel(order="F"))
    zero = up(np.zeros(1, dtype=np.int64))
    dm, dn = up(np.array([m], np.int32)), up(np.array([n], np.int32))
    dmr = up(np.array([min_rank], np.int32))
    rank = torch.zeros(1, dtype=torch.int32, device=dev)
    piv = torch.zeros(n, dtype=torch.int32, device=dev)
    rfac = torch.zeros(min(m, n) * n, dtype=tdt, device=dev)
    proj = torch.zeros(n * n, dtype=tdt, device=dev)
    big = torch.zeros(1, dtype=torch.float64, device=dev)
    ratio = torch.zeros(1, dtype=torch.float64, device=dev)
    need = (m + (0 if cplx else m % 2)) * n * (16 if cplx else 8)
    scratch = torch.empty(max(need // 8, 1), dtype=torch.float64, device=dev)
    p = _native.ptr
    _native.check(_native.lib().skel_pivoted_qr_batched(
        p(dA), p(zero), p(dm), p(dn), 1, float(eps), p(dmr), p(rank), p(piv), p(zero), p(rfac),
        p(zero), p(proj), p(zero), p(big), p(ratio), field, p(scratch), scratch.numel() * 8, m, n,
        _native.stream_ptr()), "skel_pivoted_qr_batched")
    r = int(rank.cpu()[0])
    R = rfac.cpu().numpy()[:r * n].reshape(r, n).astype(dt)
    return piv.cpu().numpy().astype(np.int64), R, r, float(ratio.cpu()[0])


def _big_side(A):
    """Upload an explicit matrix as a big-box side (column-major target)."""
    from . import _bigbox
    torch = _native.require_cuda()
    A = _as_matrix(A)
    m, n = A.shape
    field = int(A.dtype.kind == "c")
    tdt = _native.torch_dtype(field)
    sd = _bigbox._Side(torch, m, n, tdt)
    sd.W.copy_(torch.from_numpy(np.ascontiguousarray(A.T, dtype=np.complex128 if field else np.float64)
                                ).reshape(-1).to("cuda"))
    return torch, sd, field, tdt


def _big_result(sd, field, min_rank):
    """InterpDecomp from a big-box CPQR state (interp already applied)."""
    n = sd.n
    st = sd.state_out
    hdr = st[:4].cpu().view(_i32()).numpy()
    r, pad = int(hdr[0]), int(hdr[2])
    raw = st.cpu().numpy().view(np.uint8)
    piv = raw[256 + 24 * n:256 + 28 * n].view(np.int32).astype(np.int64)
    p0 = float(raw[16:24].view(np.float64)[0])         # BigState.p0
    bigP = float(raw[32:40].view(np.float64)[0])       # BigState.bigP
    trail = float(raw[40:48].view(np.float64)[0])      # BigState.pad0: first rejected pivot
    W = sd.W_out.cpu().numpy().reshape(n, sd.ld_out)          # row q = column q of the target
    dt = np.complex128 if field else np.float64
    K = r + pad
    P = np.zeros((K, n), dtype=dt)
    for s in range(K):
        P[s, piv[s]] = 1.0
    for q in range(K, n):
        P[:r, piv[q]] = W[piv[q], :r]
    if bigP > 2.0:
        warnings.warn(f"interpolation matrix entries reach {bigP:.3g} (> 2); "
                      "pivoting quality degraded on this block", stacklevel=3)
    ratio = trail / p0 if p0 > 0.0 else 0.0
    if sd.kind == "rand":
        ratio = sd.worst                       # worst probe error (lowrank.py:219-231)
    return InterpDecomp(skel=piv[:K].copy(), proj=P, rank=K, achieved_error=float(ratio))


def _i32():
    import torch
    return torch.int32


def id_fixed_precision_large(A, eps, min_rank=0) -> InterpDecomp:
    """id_fixed_precision for matrices too large for one CTA: the whole-GPU
    cooperative CPQR of csrc/big.cu (same pivot / stop rules)."""
    from . import _bigbox
    if not 0 < eps < 1:
        raise InvalidInput("eps must lie in (0, 1)")
    torch, sd, field, _ = _big_side(A)
    L = _native.lib()
    st = _native.stream_ptr()
    _bigbox._cpqr(L, sd.W, sd.m, sd.n, sd.m, eps, min_rank, 0, sd.state, field, st)
    _native.check(L.skel_big_interp(_native.ptr(sd.W), sd.n, sd.m, _native.ptr(sd.state), min_rank,
                                    field, st), "skel_big_interp")
    return _big_result(sd, field, min_rank)


def id_randomized(A, eps, oversampling=10, seed=0) -> InterpDecomp:
    """Randomized ID (lowrank.py:186-231): Gaussian sketch with doubling,
    5-probe check and deterministic fallback, on the GPU; the random numbers
    are drawn from numpy's default_rng(seed) in the reference's order."""
    from . import _bigbox
    if not 0 < eps < 1:
        raise InvalidInput("eps must lie in (0, 1)")
    if oversampling < 4:
        raise InvalidInput("oversampling must be >= 4")
    torch, sd, field, tdt = _big_side(A)
    L = _native.lib()
    st = _native.stream_ptr()
    _bigbox._randomized(torch, L, sd, eps, seed, field, tdt, st, oversampling=int(oversampling))
    if sd.kind == "fixed":
        _native.check(L.skel_big_interp(_native.ptr(sd.W), sd.n, sd.m, _native.ptr(sd.state), 0,
                                        field, st), "skel_big_interp")
    return _big_result(sd, field, 0)
