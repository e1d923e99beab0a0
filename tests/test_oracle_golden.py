"""Pin the CPU oracle (oracle/) against golden vectors produced by the live
reference (tests/golden/make_golden.py).  Bit-exact where the reference's own
arithmetic is reproduced op for op."""

import numpy as np
import pytest

import oracle
from oracle.lowrank import id_fixed


def _unpack_skels(g, li, nb):
    kr, kc = g[f"L{li}_kr"], g[f"L{li}_kc"]
    return kr, kc


def _check_compressed(oc, g, blocks=False):
    assert len(oc.levels) == int(g["nlevels"])
    for li, lv in enumerate(oc.levels):
        np.testing.assert_array_equal(lv.kr, g[f"L{li}_kr"])
        np.testing.assert_array_equal(lv.kc, g[f"L{li}_kc"])
        np.testing.assert_array_equal(np.concatenate(lv.row_skel), g[f"L{li}_row_skel"])
        np.testing.assert_array_equal(np.concatenate(lv.col_skel), g[f"L{li}_col_skel"])
        if blocks:
            np.testing.assert_array_equal(np.concatenate([d.ravel() for d in lv.D]), g[f"L{li}_D"])
            np.testing.assert_array_equal(np.concatenate([d.ravel() for d in lv.L]), g[f"L{li}_L"])
            np.testing.assert_array_equal(np.concatenate([d.ravel() for d in lv.R]), g[f"L{li}_R"])
    if "S" in g:
        np.testing.assert_array_equal(oc.S, g["S"])


@pytest.mark.parametrize("name", ["ellipse_1024_1e-9_full", "ellipse_4096_1e-9"])
def test_tree_and_neighbors_ellipse(golden, name):
    g = golden(name)
    n = int(g["n"])
    T = oracle.build_tree(oracle.ellipse(2.0, 1.0, n)["xy"], 64)
    np.testing.assert_array_equal(T.perm, g["perm"])
    np.testing.assert_array_equal(T.center, g["node_center"])
    np.testing.assert_array_equal(T.hw, g["node_hw"])
    for li in range(len(T.covers)):
        np.testing.assert_array_equal(T.covers[li], g[f"C{li}"])
        off, idx = oracle.level_neighbors(T, li)
        np.testing.assert_array_equal(off, g[f"N{li}_off"])
        np.testing.assert_array_equal(idx, g[f"N{li}_idx"])


def test_tree_and_neighbors_sphere(golden):
    g = golden("sphere_2000_1e-6")
    T = oracle.build_tree(oracle.fib_sphere(2000), 64)
    np.testing.assert_array_equal(T.perm, g["perm"])
    for li in range(len(T.covers)):
        np.testing.assert_array_equal(T.covers[li], g[f"C{li}"])
        off, idx = oracle.level_neighbors(T, li)
        np.testing.assert_array_equal(off, g[f"N{li}_off"])
        np.testing.assert_array_equal(idx, g[f"N{li}_idx"])


def test_kernel_kats(golden):
    g = golden("kernels_kat")
    for dim in (2, 3):
        tgt, src = g[f"d{dim}_tgt"], g[f"d{dim}_src"]
        nrm, w = g[f"d{dim}_nrm"], g[f"d{dim}_w"]
        for eq, k in (("laplace", 0.0), ("helmholtz", 3.7)):
            for layer in ("single", "double"):
                got = oracle.eval_block(eq, dim, layer, k, tgt, src,
                                        nrm if layer == "double" else None, w)
                np.testing.assert_allclose(got, g[f"d{dim}_{eq}_{layer}"], rtol=1e-15, atol=0)
    got = oracle.eval_block("laplace", 2, "double", 0.0, g["d2_tgt"], g["d2_src"], g["d2_nrm"],
                            g["d2_w"], g["d2_kap"], "curvature_limit")
    np.testing.assert_array_equal(got, g["d2_laplace_double_curv"])


def test_lowrank_kats(golden):
    g = golden("lowrank_kat")
    for i in range(int(g["ncases"])):
        A = g[f"A{i}"]
        for j in range(4):
            skel, P, rank, _ = id_fixed(A, float(g[f"A{i}_{j}_eps"]), int(g[f"A{i}_{j}_minrank"]))
            np.testing.assert_array_equal(skel, g[f"A{i}_{j}_skel"])
            np.testing.assert_array_equal(P, g[f"A{i}_{j}_proj"])


def _ellipse_run(n, eps, nrhs):
    cur = oracle.ellipse(2.0, 1.0, n)
    T = oracle.build_tree(cur["xy"], 64)
    src = oracle.BieSource(cur, T.perm)
    oc = oracle.compress(src, T, eps)
    of = oracle.factor(oc)
    B = np.random.default_rng(0).standard_normal((n, nrhs))
    return src, oc, of, B, oracle.solve(of, B)


def test_ellipse_1024_full_pipeline(golden):
    g = golden("ellipse_1024_1e-9_full")
    src, oc, of, B, X = _ellipse_run(1024, 1e-9, 3)
    _check_compressed(oc, g, blocks=True)
    for li in range(len(oc.levels)):
        for key, arrs in (("Dd", of.Dd), ("Ld", of.Ld), ("Rd", of.Rd), ("Lam", of.Lam)):
            np.testing.assert_array_equal(np.concatenate([a.ravel() for a in arrs[li]]),
                                          g[f"L{li}_{key}"])
    np.testing.assert_array_equal(X, g["X"])
    np.testing.assert_array_equal(oracle.apply(oc, X), g["Y_apply"])
    res = np.linalg.norm(oracle.dense_matvec(src, X) - B) / np.linalg.norm(B)
    assert res == pytest.approx(float(g["resid"]), rel=1e-3)


def test_ellipse_4096_config1(golden):
    g = golden("ellipse_4096_1e-9")
    src, oc, of, B, X = _ellipse_run(4096, 1e-9, 4)
    _check_compressed(oc, g)
    np.testing.assert_array_equal(X, g["X"])


@pytest.mark.slow
def test_ellipse_16384_eps12(golden):
    g = golden("ellipse_16384_1e-12")
    src, oc, of, B, X = _ellipse_run(16384, 1e-12, 2)
    _check_compressed(oc, g)
    np.testing.assert_array_equal(X, g["X"])


@pytest.mark.slow
def test_cfie_2048(golden):
    g = golden("cfie_2048_1e-9")
    n = 2048
    cur = oracle.ellipse(2.0, 1.0, n)
    T = oracle.build_tree(cur["xy"], 64)
    k = 2 * np.pi * 8 / oracle.ellipse_perimeter()
    assert k == float(g["k"])
    src = oracle.CfieSource(cur, T.perm, k)
    oc = oracle.compress(src, T, 1e-9)
    _check_compressed(oc, g)
    rng = np.random.default_rng(0)
    B = rng.standard_normal((n, 2)) + 1j * rng.standard_normal((n, 2))
    np.testing.assert_array_equal(oracle.solve(oracle.factor(oc), B), g["X"])


@pytest.mark.slow
def test_sphere_2000(golden):
    g = golden("sphere_2000_1e-6")
    n = 2000
    T = oracle.build_tree(oracle.fib_sphere(n), 64)
    src = oracle.KernelSource("laplace", 3, "single", oracle.fib_sphere(n), T.perm,
                              weights=np.full(n, 4 * np.pi / n), diag=1.0)
    oc = oracle.compress(src, T, 1e-6)
    _check_compressed(oc, g)
    assert oc.S.shape == tuple(g["S_shape"])
    B = np.random.default_rng(0).standard_normal((n, 1))
    X = oracle.solve(oracle.factor(oc), B)
    np.testing.assert_allclose(X, g["X"], rtol=0, atol=1e-12 * np.abs(g["X"]).max())
