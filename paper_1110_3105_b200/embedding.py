"""Sparse multilevel embedding of a compressed matrix and its Matrix Market
export (reference solver.py:34-140, 414-433, 532-560).

The embedding is the block-sparse system the telescoping factorization is
equivalent to -- an independent cross-check with any sparse solver.  Unknowns
are ordered [x, y1, z1, ..., yL, zL] (x in tree order), equations
[b-rows, z1-coupling, y1-coupling, ...]; entries are grouped into labelled
blocks "D<l>", "L<l>", "R<l>", "I:z<l>", "I:y<l>" and "S" in the reference's
order (levels ascending, nodes in cover order, row-major non-zeros inside a
block), so ``to_coo`` returns the reference's arrays entry for entry.

The blocks are read back from the device slabs of a GPU-compressed matrix
in one copy per slab and expanded with vectorised index arithmetic.
"""

from dataclasses import dataclass

import numpy as np

from .errors import InvalidInput


@dataclass
class SparseEmbedding:
    m: int
    n: int
    dtype: np.dtype
    blocks: dict
    perm: np.ndarray

    def to_coo(self):
        parts = list(self.blocks.values())
        if not parts:
            z = np.zeros(0, dtype=np.int64)
            return z, z.copy(), np.zeros(0, dtype=self.dtype)
        return (np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
                np.concatenate([p[2] for p in parts]))

    def to_dense(self):
        A = np.zeros((self.m, self.m), dtype=self.dtype)
        r, c, v = self.to_coo()
        A[r, c] = v
        return A

    def rhs(self, b):
        b = np.asarray(b)
        if b.shape[0] != self.n:
            raise InvalidInput("rhs length mismatch")
        out = np.zeros((self.m,) + b.shape[1:], dtype=np.result_type(self.dtype, b.dtype))
        out[:self.n] = b[self.perm]
        return out

    def extract_x(self, sol):
        out = np.empty_like(sol[:self.n])
        out[self.perm] = sol[:self.n]
        return out

    @property
    def nnz(self):
        return int(sum(len(p[0]) for p in self.blocks.values()))


def _level_blocks(lv, dtype):
    """(nr, nc, kr, kc, D, L, R) of one level: counts per node and the blocks
    as tight concatenations (row-major per node)."""
    if lv.dev is not None and lv._nodes is None:
        d = lv.dev
        nr, nc, kr, kc = d.nr, d.nc, d.kr, d.kc
        D = d.D.cpu().numpy()[:int((nr * nc).sum())]
        Lcap = d.L.cpu().numpy()
        Rcap = d.R.cpu().numpy()
        # L lives as nr x kr inside an nr x nr slot, R as kc x nc in nc x nc
        def tight(cap, off, cnt):
            if cnt.sum() == 0:
                return np.zeros(0, dtype=dtype)
            base = np.repeat(off[:-1], cnt)
            loc = np.arange(int(cnt.sum())) - np.repeat(np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
            return cap[base + loc]
        L = tight(Lcap, d.l_off, nr * kr)
        R = tight(Rcap, d.r_off, kc * nc)
        return nr, nc, kr, kc, D.astype(dtype, copy=False), L, R
    nodes = lv.nodes
    nr = np.array([nd.D.shape[0] for nd in nodes], dtype=np.int64)
    nc = np.array([nd.D.shape[1] for nd in nodes], dtype=np.int64)
    kr = np.array([nd.L.shape[1] for nd in nodes], dtype=np.int64)
    kc = np.array([nd.R.shape[0] for nd in nodes], dtype=np.int64)
    cat = lambda xs: (np.concatenate([np.asarray(x, dtype=dtype).ravel() for x in xs])  # noqa: E731
                      if xs else np.zeros(0, dtype=dtype))
    return nr, nc, kr, kc, cat([nd.D for nd in nodes]), cat([nd.L for nd in nodes]), cat([nd.R for nd in nodes])


def _block_coo(vals, rows_per, cols_per, r_base, c_base):
    """Row-major coordinates of consecutive blocks (rows_per[a] x cols_per[a]
    at (r_base[a], c_base[a])), non-zeros only, node order preserved."""
    sizes = rows_per * cols_per
    tot = int(sizes.sum())
    if tot == 0:
        return None
    box = np.repeat(np.arange(sizes.size), sizes)
    loc = np.arange(tot) - np.repeat(np.concatenate([[0], np.cumsum(sizes)[:-1]]), sizes)
    w = cols_per[box]
    r = r_base[box] + loc // np.maximum(w, 1)
    c = c_base[box] + loc % np.maximum(w, 1)
    nz = np.flatnonzero(vals[:tot])
    if nz.size == 0:
        return None
    return r[nz].astype(np.int64), c[nz].astype(np.int64), vals[nz]


def assemble_embedding(cm) -> SparseEmbedding:
    """Coordinate-form multilevel embedding of ``cm`` (solver.py:91-140)."""
    n = cm.n
    dtype = np.dtype(cm.dtype)
    blocks = {}
    S = np.asarray(cm.S)

    def put(label, coo):
        if coo is not None:
            blocks[label] = coo

    if cm.nlevels == 0:
        put("S", _block_coo(S.ravel(), np.array([S.shape[0]]), np.array([S.shape[1]]),
                            np.array([0]), np.array([0])))
        return SparseEmbedding(m=n, n=n, dtype=dtype, blocks=blocks, perm=np.asarray(cm.perm))
    per = [_level_blocks(lv, dtype) for lv in cm.levels]
    Kr = [int(x[2].sum()) for x in per]
    Kc = [int(x[3].sum()) for x in per]
    col_off, row_off = [0, n], [0, n]
    for a, b in zip(Kr, Kc):
        col_off += [col_off[-1] + a, col_off[-1] + a + b]
        row_off += [row_off[-1] + b, row_off[-1] + b + a]
    m = col_off[-1]
    for li, (nr, nc, kr, kc, D, L, R) in enumerate(per):
        l1 = li + 1
        dl_rows = 0 if li == 0 else row_off[2 * li]
        dl_cols = 0 if li == 0 else col_off[2 * li]
        y_cols, z_cols = col_off[2 * li + 1], col_off[2 * li + 2]
        r_rows = row_off[2 * li + 1]
        rdo = np.concatenate([[0], np.cumsum(nr)])[:-1]
        cdo = np.concatenate([[0], np.cumsum(nc)])[:-1]
        kro = np.concatenate([[0], np.cumsum(kr)])[:-1]
        kco = np.concatenate([[0], np.cumsum(kc)])[:-1]
        put(f"D{l1}", _block_coo(D, nr, nc, dl_rows + rdo, dl_cols + cdo))
        put(f"L{l1}", _block_coo(L, nr, kr, dl_rows + rdo, y_cols + kro))
        put(f"R{l1}", _block_coo(R, kc, nc, r_rows + kco, dl_cols + cdo))
        iz = np.arange(Kc[li], dtype=np.int64)
        blocks[f"I:z{l1}"] = (r_rows + iz, z_cols + iz, np.full(Kc[li], -1.0, dtype=dtype))
        iy = np.arange(Kr[li], dtype=np.int64)
        blocks[f"I:y{l1}"] = (row_off[2 * li + 2] + iy, y_cols + iy, np.full(Kr[li], -1.0, dtype=dtype))
    L_ = cm.nlevels
    put("S", _block_coo(S.ravel(), np.array([S.shape[0]]), np.array([S.shape[1]]),
                        np.array([row_off[2 * L_]]), np.array([col_off[2 * L_]])))
    return SparseEmbedding(m=m, n=n, dtype=dtype, blocks=blocks, perm=np.asarray(cm.perm))


def export_matrix_market(se: SparseEmbedding, path):
    """Coordinate Matrix Market file: 1-based indices, entries sorted by
    (column, row), 17 significant digits (solver.py:414-433)."""
    r, c, v = se.to_coo()
    order = np.lexsort((r, c))
    r, c, v = r[order] + 1, c[order] + 1, v[order]
    cplx = np.issubdtype(se.dtype, np.complexfloating)
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate {'complex' if cplx else 'real'} general\n")
        f.write(f"{se.m} {se.m} {len(v)}\n")
        if cplx:
            f.writelines(f"{a} {b} {x.real:.17g} {x.imag:.17g}\n" for a, b, x in zip(r, c, v))
        else:
            f.writelines(f"{a} {b} {x:.17g}\n" for a, b, x in zip(r, c, v))


def read_matrix_market(path):
    """Coordinate-format reader: ((m, n), rows, cols, vals), 0-based."""
    with open(path) as f:
        head = f.readline()
        if not head.startswith("%%MatrixMarket matrix coordinate"):
            raise InvalidInput("unsupported Matrix Market header")
        cplx = "complex" in head
        line = f.readline()
        while line.startswith("%"):
            line = f.readline()
        m, n, nnz = (int(t) for t in line.split())
        data = np.loadtxt(f, ndmin=2, max_rows=nnz) if nnz else np.zeros((0, 4 if cplx else 3))
    rows = data[:, 0].astype(np.int64) - 1
    cols = data[:, 1].astype(np.int64) - 1
    vals = data[:, 2] + 1j * data[:, 3] if cplx else data[:, 2].astype(np.float64)
    return (m, n), rows, cols, vals
