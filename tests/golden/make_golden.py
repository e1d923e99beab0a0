"""Generate golden fixtures from the LIVE reference (skelkit 0.1.0).

Run in the build container only (the reference is not present on GPU boxes):

    python tests/golden/make_golden.py

Imports ``skelkit`` from /root/reference/pkg/src, drives it through its public
API on seeded inputs, and writes small .npz fixtures next to this script.  The
oracle (oracle/) is pinned against these in tests/test_oracle_golden.py and
the CUDA path is compared against them in tests/test_gpu_parity.py.

Config-3 (CFIE) and config-4 (3D sphere, unit diagonal) sources are composed
from reference pieces exactly as SURVEY.md App. B describes; they live here
(test harness), not in the reference.
"""

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import skelkit  # noqa: E402
from skelkit import bie, geom  # noqa: E402
from skelkit.kernels import KernelSpec, eval_block  # noqa: E402
from skelkit.lowrank import id_fixed_precision  # noqa: E402
from skelkit.skel import KernelSource, compress_source  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def pack_cm(cm, tree):
    """Flatten a CompressedMatrix into CSR-style arrays."""
    out = {"perm": tree.perm, "S": cm.S, "nlevels": np.array(cm.nlevels)}
    for li, lv in enumerate(cm.levels):
        out[f"L{li}_kr"] = lv.kr_counts
        out[f"L{li}_kc"] = lv.kc_counts
        out[f"L{li}_nr"] = lv.row_dof_counts
        out[f"L{li}_nc"] = lv.col_dof_counts
        out[f"L{li}_row_skel"] = np.concatenate([nd.row_skel for nd in lv.nodes])
        out[f"L{li}_col_skel"] = np.concatenate([nd.col_skel for nd in lv.nodes])
    return out


def pack_blocks(cm, fi=None):
    out = {}
    for li, lv in enumerate(cm.levels):
        out[f"L{li}_D"] = np.concatenate([nd.D.ravel() for nd in lv.nodes])
        out[f"L{li}_L"] = np.concatenate([nd.L.ravel() for nd in lv.nodes])
        out[f"L{li}_R"] = np.concatenate([nd.R.ravel() for nd in lv.nodes])
        if fi is not None:
            fl = fi.levels[li]
            out[f"L{li}_Dd"] = np.concatenate([f.Dd.ravel() for f in fl.nodes])
            out[f"L{li}_Ld"] = np.concatenate([f.Ld.ravel() for f in fl.nodes])
            out[f"L{li}_Rd"] = np.concatenate([f.Rd.ravel() for f in fl.nodes])
            out[f"L{li}_Lam"] = np.concatenate([f.Lam.ravel() for f in fl.nodes])
    return out


def neighbor_csr(tree):
    out = {}
    for li in range(len(tree.levels)):
        nb = geom.level_neighbors(tree, li)
        out[f"N{li}_off"] = np.concatenate([[0], np.cumsum([len(x) for x in nb])])
        out[f"N{li}_idx"] = np.array([b for x in nb for b in x], dtype=np.int64)
        out[f"C{li}"] = np.array(tree.levels[li])
    nodes = tree.nodes
    out["node_center"] = np.array([nd.center for nd in nodes])
    out["node_hw"] = np.array([nd.halfwidth for nd in nodes])
    out["node_lo"] = np.array([nd.lo for nd in nodes])
    out["node_hi"] = np.array([nd.hi for nd in nodes])
    out["node_depth"] = np.array([nd.depth for nd in nodes])
    return out


def ellipse_case(n, eps, nrhs, full=False, neighbors=False):
    curve = bie.ellipse(2.0, 1.0, n)
    system = bie.discretize_dirichlet(curve, KernelSpec("laplace", 2))
    tree, cm = bie.compress_system(system, eps, 64)
    fi = skelkit.factor(cm)
    B = np.random.default_rng(0).standard_normal((n, nrhs))
    X = skelkit.solve(fi, B)
    out = pack_cm(cm, tree)
    out.update({"X": X, "eps": np.array(eps), "n": np.array(n),
                "warnings": np.array(len(fi.warnings))})
    if full:
        out.update(pack_blocks(cm, fi))
        out["Y_apply"] = skelkit.apply(cm, X)
    if neighbors:
        out.update(neighbor_csr(tree))
    if n <= 4096:
        A = system.matrix()
        out["resid"] = np.array(np.linalg.norm(A @ X - B) / np.linalg.norm(B))
    return out


class CfieSource:
    """Config 3 composed from reference pieces."""

    def __init__(self, curve, perm, k):
        self.perm = np.asarray(perm)
        self.n = curve.n
        self.k = k
        self.dtype = np.complex128
        self.wavenumber = k
        self.pts = curve.point_set()
        self.tpts = self.pts.subset(self.perm)
        self.dl = KernelSpec("helmholtz", 2, "double", k)
        self.sl = KernelSpec("helmholtz", 2, "single", k)
        self.wscale = float(np.mean(self.tpts.weights))

    def block(self, rows, cols):
        oi, oj = self.perm[rows], self.perm[cols]
        tgt = self.pts.subset(oi)
        src = self.pts.subset(oj)
        srcw = skelkit.PointSet(src.coords, None, src.weights)
        G = eval_block(self.dl, tgt, src) - 1j * self.k * eval_block(self.sl, tgt, srcw)
        d = np.abs(oi[:, None] - oj[None, :])
        d = np.minimum(d, self.n - d)
        near = (d >= 1) & (d <= bie.KR10_GAMMA.size)
        G = G * np.where(near, 1.0 + bie.KR10_GAMMA[np.minimum(d, 10) - 1], 1.0)
        return G + np.where(oi[:, None] == oj[None, :], 0.5, 0.0)

    def proxy_row_block(self, rows, pxy):
        return self.wscale * eval_block(self.sl, self.tpts.subset(rows), pxy)

    def proxy_col_block(self, cols, pxy):
        s = self.tpts.subset(cols)
        return eval_block(self.sl, pxy, skelkit.PointSet(s.coords, None, s.weights))


class DiagOneSource(KernelSource):
    """Config 4: 3D Laplace single layer with area weights, unit diagonal."""

    def block(self, rows, cols):
        G = super().block(rows, cols)
        return G + np.where(np.asarray(rows)[:, None] == np.asarray(cols)[None, :], 1.0, 0.0)


def cfie_case(n, eps, nrhs):
    per = perimeter()
    k = 2 * np.pi * 8 / per
    curve = bie.ellipse(2.0, 1.0, n)
    tree = geom.build_tree(curve.point_set(), 64)
    src = CfieSource(curve, tree.perm, k)
    cm = compress_source(src, tree, eps)
    fi = skelkit.factor(cm)
    rng = np.random.default_rng(0)
    B = rng.standard_normal((n, nrhs)) + 1j * rng.standard_normal((n, nrhs))
    X = skelkit.solve(fi, B)
    out = pack_cm(cm, tree)
    idx = np.arange(n)
    A = src.block(idx, idx)[np.argsort(tree.perm)][:, np.argsort(tree.perm)]
    out.update({"X": X, "eps": np.array(eps), "n": np.array(n), "k": np.array(k),
                "resid": np.array(np.linalg.norm(A @ X - B) / np.linalg.norm(B))})
    return out


def sphere_points(n):
    i = np.arange(n) + 0.5
    z = 1.0 - 2.0 * i / n
    rho = np.sqrt(np.clip(1 - z * z, 0, None))
    th = np.pi * (3 - np.sqrt(5.0)) * i
    return np.column_stack([rho * np.cos(th), rho * np.sin(th), z])


def sphere_case(n, eps, nrhs, full=False):
    pts = skelkit.PointSet(sphere_points(n), None, np.full(n, 4 * np.pi / n))
    tree = geom.build_tree(pts, 64)
    src = DiagOneSource(KernelSpec("laplace", 3), pts, tree.perm)
    cm = compress_source(src, tree, eps)
    fi = skelkit.factor(cm)
    B = np.random.default_rng(0).standard_normal((n, nrhs))
    X = skelkit.solve(fi, B)
    out = pack_cm(cm, tree)
    out["S_shape"] = np.array(out.pop("S").shape)   # S is 1240^2: keep fixtures small
    out.update(neighbor_csr(tree))
    out.update({"X": X, "eps": np.array(eps), "n": np.array(n)})
    if full:
        out.update(pack_blocks(cm, fi))
    return out


def sklc_case(n, eps, nrhs):
    """The reference's binary containers (skel.py:428-511, solver.py:439-529)
    of one compressed matrix / factored inverse, plus the solution they give."""
    from skelkit.skel import serialize_compressed
    from skelkit.solver import serialize_factored
    curve = bie.ellipse(2.0, 1.0, n)
    system = bie.discretize_dirichlet(curve, KernelSpec("laplace", 2))
    tree, cm = bie.compress_system(system, eps, 64)
    fi = skelkit.factor(cm)
    B = np.random.default_rng(0).standard_normal((n, nrhs))
    X = skelkit.solve(fi, B)
    import os
    import tempfile
    se = skelkit.assemble_embedding(cm)
    r, c, v = se.to_coo()
    fd, path = tempfile.mkstemp(suffix=".mtx")
    os.close(fd)
    skelkit.export_matrix_market(se, path)
    with open(path, "rb") as fh:
        mm = fh.read()
    os.unlink(path)
    # a small GMRES case (solver.py:328-408): diagonally shifted random system
    rng = np.random.default_rng(5)
    G = rng.standard_normal((60, 60)) / np.sqrt(60) + 2.0 * np.eye(60)
    gb = rng.standard_normal(60)
    gx, gits = skelkit.gmres(G, gb, tol=1e-12)
    return {"cm_bytes": np.frombuffer(serialize_compressed(cm), dtype=np.uint8),
            "fi_bytes": np.frombuffer(serialize_factored(fi), dtype=np.uint8),
            "X": X, "Y_apply": skelkit.apply(cm, X), "n": np.array(n), "eps": np.array(eps),
            "emb_m": np.array(se.m), "emb_rows": r, "emb_cols": c, "emb_vals": v,
            "emb_labels": np.array(list(se.blocks.keys())),
            "mm_bytes": np.frombuffer(mm, dtype=np.uint8),
            "gmres_A": G, "gmres_b": gb, "gmres_x": gx, "gmres_iters": np.array(gits)}


def scattering_case(n, k):
    """Two sound-hard trefoils (bie.py:305-459): system entries (a sample),
    plane-wave data, block-preconditioned GMRES, scattered field."""
    curves = [bie.trefoil(n, center=(-0.6, 0.0), scale=1.0), bie.trefoil(n, center=(0.6, 0.1), scale=0.8)]
    sysm = bie.scattering_system(curves, k)
    A = sysm.matrix()
    rng = np.random.default_rng(9)
    ii = rng.integers(0, A.shape[0], 3000)
    jj = rng.integers(0, A.shape[0], 3000)
    diag = np.arange(A.shape[0])
    b = sysm.rhs_plane_wave()
    facs = sysm.precond_blocks(1e-8, 32)
    x, its = skelkit.gmres(A, b, tol=1e-10, precond=sysm.precond_apply(facs))
    tg = np.array([[3.0, 0.5], [-2.5, -1.0], [0.0, 2.5]])
    return {"ii": ii, "jj": jj, "A_sample": A[ii, jj], "A_diag": A[diag, diag],
            "A_row0": A[0], "A_row_last": A[-1], "rhs": b, "x": x, "iters": np.array(its),
            "field_targets": tg, "field": sysm.scattered_field(x, tg), "n": np.array(n),
            "k": np.array(k), "ranks": np.array([f_.levels[0].nodes[0].Ld.shape[1] if f_.levels else 0
                                                  for f_ in facs])}


def perimeter(m=4096):
    t = 2 * np.pi * np.arange(m) / m
    return float(np.sum(np.sqrt((2 * np.sin(t)) ** 2 + np.cos(t) ** 2)) * 2 * np.pi / m)


def kernel_kats():
    rng = np.random.default_rng(11)
    out = {}
    for dim in (2, 3):
        tgt = rng.standard_normal((17, dim))
        src = rng.standard_normal((13, dim))
        src[:3] = tgt[:3]                      # coincident pairs
        nrm = rng.standard_normal((13, dim))
        nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
        w = rng.random(13) + 0.5
        kap = rng.random(13)
        out[f"d{dim}_tgt"], out[f"d{dim}_src"] = tgt, src
        out[f"d{dim}_nrm"], out[f"d{dim}_w"], out[f"d{dim}_kap"] = nrm, w, kap
        for eq, k in (("laplace", 0.0), ("helmholtz", 3.7)):
            for layer in ("single", "double"):
                spec = KernelSpec(eq, dim, layer, k)
                S = skelkit.PointSet(src, nrm if layer == "double" else None, w)
                out[f"d{dim}_{eq}_{layer}"] = eval_block(spec, skelkit.PointSet(tgt), S)
        spec = KernelSpec("laplace", 2, "double", 0.0, "curvature_limit") if dim == 2 else None
        if spec is not None:
            S = skelkit.PointSet(src, nrm, w, kap)
            out["d2_laplace_double_curv"] = eval_block(spec, skelkit.PointSet(tgt), S)
    return out


def lowrank_kats():
    rng = np.random.default_rng(7)
    out = {}
    cases = []
    for i, (m, n, prof) in enumerate([(200, 40, "geometric"), (300, 64, "algebraic"),
                                      (120, 90, "step"), (64, 64, "random"),
                                      (500, 30, "geometric"), (40, 100, "algebraic")]):
        k = min(m, n)
        s = {"geometric": 0.6 ** np.arange(k), "algebraic": 1.0 / (1 + np.arange(k)) ** 3,
             "step": np.where(np.arange(k) < k // 4, 1.0, 1e-12),
             "random": np.abs(rng.standard_normal(k)) + 1e-3}[prof]
        U, _ = np.linalg.qr(rng.standard_normal((m, k)))
        V, _ = np.linalg.qr(rng.standard_normal((n, k)))
        cases.append((U * s) @ V.T)
    Z = rng.standard_normal((60, 3)) + 1j * rng.standard_normal((60, 3))
    cases.append(Z @ (rng.standard_normal((3, 25)) + 1j * rng.standard_normal((3, 25))))
    cases.append(np.array([[1.0, 2.0], [2.0, 4.0]]))
    cases.append(np.zeros((5, 4)))
    cases.append(np.outer(np.arange(1, 9.0), np.ones(6)))   # exact rank 1 (padding)
    for i, A in enumerate(cases):
        out[f"A{i}"] = A
        for j, (eps, mr) in enumerate([(1e-9, 0), (1e-12, 0), (1e-6, 0), (1e-9, 5)]):
            with warnings.catch_warnings():
                warnings.simplefilter("ignore")
                idp = id_fixed_precision(A, eps, min_rank=mr)
            out[f"A{i}_{j}_skel"] = idp.skel
            out[f"A{i}_{j}_proj"] = idp.proj
            out[f"A{i}_{j}_eps"] = np.array(eps)
            out[f"A{i}_{j}_minrank"] = np.array(mr)
    out["ncases"] = np.array(len(cases))
    return out


def main():
    warnings.simplefilter("ignore")
    jobs = {
        "kernels_kat": kernel_kats,
        "lowrank_kat": lowrank_kats,
        "ellipse_1024_1e-9_full": lambda: ellipse_case(1024, 1e-9, 3, full=True, neighbors=True),
        "ellipse_4096_1e-9": lambda: ellipse_case(4096, 1e-9, 4, neighbors=True),
        "ellipse_16384_1e-12": lambda: ellipse_case(16384, 1e-12, 2),
        "cfie_2048_1e-9": lambda: cfie_case(2048, 1e-9, 2),
        "sphere_2000_1e-6": lambda: sphere_case(2000, 1e-6, 1),
        # randomized IDs (m > max(4096, 4n + 256)) at the coarse levels
        "sphere_10000_1e-6": lambda: sphere_case(10000, 1e-6, 1),
        "sklc_ellipse_512_1e-6": lambda: sklc_case(512, 1e-6, 2),
        "scattering_2x256_k3": lambda: scattering_case(256, 3.0),
    }
    only = sys.argv[1:]
    for name, fn in jobs.items():
        if only and name not in only:
            continue
        data = fn()
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **data)
        print(f"{name}: {os.path.getsize(path) / 1e3:.1f} kB")


if __name__ == "__main__":
    main()
