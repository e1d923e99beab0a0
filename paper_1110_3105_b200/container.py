"""The reference's binary container ("SKLC", skel.py:428-511 and
solver.py:439-529), byte-compatible in both directions, for compressed
matrices and factored inverses.

Layout (little endian):

  magic  b"SKLC"
  u16 version (1), u8 kind (1 compressed / 2 factored), u8 field (0 real / 1 complex)
  i64 N, u32 levels, f64 eps (0.0 for a factored inverse)
  array perm
  per level: u32 node count, then per node
      compressed: u8 has_children, array children, row_skel, col_skel, D, L, R
      factored:   array Dd, Ld, Rd
  compressed: array S          factored: array lu, array piv (Shat = P L U)

  array = u8 dtype code (0 float64, 1 complex128, 2 int64), u8 ndim,
          i64[ndim] shape, raw C-order bytes

Loading puts the blocks straight into device slabs (the GPU solve / apply
paths never see the host copies); saving reads the device blocks back.  The
factored container carries Shat as LU factors: a GPU-factored inverse is
saved with the LU of its Shat computed on the device (skel_dense_lu) and a
loaded one gets its explicit Shat^-1 from the stored factors on the device
(skel_lu_inverse).
"""

import io
import struct

import numpy as np

from . import _native
from .errors import InvalidInput

MAGIC = b"SKLC"
VERSION = 1
_CODES = {np.dtype(np.float64): 0, np.dtype(np.complex128): 1, np.dtype(np.int64): 2}
_DTYPES = {v: k for k, v in _CODES.items()}


def write_array(f, a):
    a = np.ascontiguousarray(a)
    if a.dtype not in _CODES:
        raise InvalidInput(f"unsupported array dtype {a.dtype} for the container")
    f.write(struct.pack("<BB", _CODES[a.dtype], a.ndim))
    f.write(struct.pack(f"<{a.ndim}q", *a.shape))
    f.write(a.tobytes())


def read_array(f):
    hdr = f.read(2)
    if len(hdr) != 2:
        raise InvalidInput("truncated container")
    code, ndim = struct.unpack("<BB", hdr)
    if code not in _DTYPES:
        raise InvalidInput(f"unknown array dtype code {code}")
    shape = struct.unpack(f"<{ndim}q", f.read(8 * ndim))
    dt = _DTYPES[code]
    nbytes = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    buf = f.read(nbytes)
    if len(buf) != nbytes:
        raise InvalidInput("truncated container")
    return np.frombuffer(buf, dtype=dt).reshape(shape).copy()


def _header(f, kind, field, n, nlev, eps):
    f.write(MAGIC)
    f.write(struct.pack("<HBB", VERSION, kind, field))
    f.write(struct.pack("<qId", int(n), int(nlev), float(eps)))


def _read_header(f, want_kind=None):
    if f.read(4) != MAGIC:
        raise InvalidInput("not a skelkit container")
    version, kind, field = struct.unpack("<HBB", f.read(4))
    if version != VERSION:
        raise InvalidInput(f"unsupported container version {version}")
    if want_kind is not None and kind != want_kind:
        raise InvalidInput("not a factored-inverse container" if want_kind == 2
                           else "not a skelkit compressed-matrix container")
    n, nlev, eps = struct.unpack("<qId", f.read(20))
    return kind, field, n, nlev, eps


# ---------------------------------------------------------------------------
# compressed matrix

def serialize_compressed(cm) -> bytes:
    f = io.BytesIO()
    _header(f, 1, cm.field, cm.n, cm.nlevels, cm.eps)
    write_array(f, np.asarray(cm.perm, dtype=np.int64))
    dt = cm.dtype
    for lv in cm.levels:
        nodes = lv.nodes
        f.write(struct.pack("<I", len(nodes)))
        for nd in nodes:
            has = nd.children is not None
            f.write(struct.pack("<B", 1 if has else 0))
            write_array(f, np.asarray(nd.children if has else np.empty(0), dtype=np.int64))
            write_array(f, np.asarray(nd.row_skel, dtype=np.int64))
            write_array(f, np.asarray(nd.col_skel, dtype=np.int64))
            write_array(f, np.asarray(nd.D, dtype=dt))
            write_array(f, np.asarray(nd.L, dtype=dt))
            write_array(f, np.asarray(nd.R, dtype=dt))
    write_array(f, np.asarray(cm.S, dtype=dt))
    return f.getvalue()


def deserialize_compressed(data: bytes):
    from .skel import CompressedLevel, CompressedMatrix, CompressedNode
    f = io.BytesIO(data)
    _, field, n, nlev, eps = _read_header(f)
    perm = read_array(f)
    levels = []
    for _ in range(nlev):
        (count,) = struct.unpack("<I", f.read(4))
        nodes = []
        for _ in range(count):
            (has,) = struct.unpack("<B", f.read(1))
            ch = read_array(f)
            rs, cs = read_array(f), read_array(f)
            D, L, R = read_array(f), read_array(f), read_array(f)
            nodes.append(CompressedNode(row_skel=rs, col_skel=cs, D=D, L=L, R=R,
                                        children=ch if has else None))
        levels.append(CompressedLevel(nodes))
    S = read_array(f)
    return CompressedMatrix(levels, S, n, eps, perm, "complex" if field else "real")


def save_compressed(cm, path):
    with open(path, "wb") as fh:
        fh.write(serialize_compressed(cm))


def load_compressed(path):
    with open(path, "rb") as fh:
        return deserialize_compressed(fh.read())


# ---------------------------------------------------------------------------
# factored inverse

def parse_factored(data: bytes):
    """Host view of a factored container: (field, n, perm, levels, lu, piv)
    with levels = [[(Dd, Ld, Rd), ...], ...] (no device needed)."""
    f = io.BytesIO(data)
    _, field, n, nlev, _eps = _read_header(f, want_kind=2)
    perm = read_array(f)
    levels = []
    for _ in range(nlev):
        (count,) = struct.unpack("<I", f.read(4))
        levels.append([(read_array(f), read_array(f), read_array(f)) for _ in range(count)])
    lu = read_array(f)
    piv = read_array(f)
    return field, n, perm, levels, lu, piv


def emit_factored(field, n, perm, levels, lu, piv) -> bytes:
    f = io.BytesIO()
    _header(f, 2, field, n, len(levels), 0.0)
    write_array(f, np.asarray(perm, dtype=np.int64))
    for nodes in levels:
        f.write(struct.pack("<I", len(nodes)))
        for Dd, Ld, Rd in nodes:
            write_array(f, Dd)
            write_array(f, Ld)
            write_array(f, Rd)
    write_array(f, lu)
    write_array(f, np.asarray(piv, dtype=np.int64))
    return f.getvalue()


def serialize_factored(fi) -> bytes:
    dt = fi.dtype
    levels = [[(np.asarray(nd.Dd, dtype=dt), np.asarray(nd.Ld, dtype=dt), np.asarray(nd.Rd, dtype=dt))
               for nd in lv.nodes] for lv in fi.levels]
    S_lu = fi.S_lu
    if S_lu is None:
        lu, piv = np.zeros((0, 0), dtype=dt), np.zeros(0, dtype=np.int64)
    else:
        lu, piv = S_lu
    return emit_factored(fi.field, fi.n, fi.perm, levels, np.asarray(lu, dtype=dt), piv)


def deserialize_factored(data: bytes):
    from .solver import FactoredInverse, factored_level_from_host
    torch = _native.require_cuda()
    field, n, perm, levels, lu, piv = parse_factored(data)
    flevels = [factored_level_from_host(nodes, field) for nodes in levels]
    S_inv = None
    if lu.size:
        K = lu.shape[0]
        tdt = _native.torch_dtype(field)
        dlu = torch.from_numpy(np.ascontiguousarray(lu)).to("cuda")
        dpiv = torch.from_numpy(piv.astype(np.int32)).to("cuda")
        S_inv = torch.empty((K, K), dtype=tdt, device="cuda")
        _native.check(_native.lib().skel_lu_inverse(_native.ptr(dlu), _native.ptr(dpiv), K,
                                                    _native.ptr(S_inv), field, _native.stream_ptr()),
                      "skel_lu_inverse")
    fi = FactoredInverse(flevels, None, S_inv, n, perm, "complex" if field else "real", [])
    if lu.size:
        fi._S_lu = (lu, piv.astype(np.int32))
    return fi


def save_factored(fi, path):
    with open(path, "wb") as fh:
        fh.write(serialize_factored(fi))


def load_factored(path):
    with open(path, "rb") as fh:
        return deserialize_factored(fh.read())
