"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; the native tree / neighbour builder equals the oracle (and
hence the reference); host-side API validation."""

import numpy as np
import pytest

import oracle


def test_library_exports_header_symbols():
    from paper_1110_3105_b200 import _native
    lib = _native.lib()
    syms = _native.header_symbols()
    assert len(syms) >= 15
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert b"sm_100a" in lib.skel_version()


@pytest.mark.parametrize("n,dim", [(1024, 2), (4096, 2), (65536, 2), (5000, 3), (20000, 3)])
def test_native_tree_equals_oracle(n, dim):
    import paper_1110_3105_b200 as sk
    X = oracle.ellipse(2.0, 1.0, n)["xy"] if dim == 2 else oracle.fib_sphere(n)
    T = sk.build_tree(sk.PointSet(X), 64)
    O = oracle.build_tree(X, 64)
    np.testing.assert_array_equal(T.perm, O.perm)
    np.testing.assert_array_equal(T.center, O.center)
    np.testing.assert_array_equal(T.hw, O.hw)
    assert len(T.levels) == len(O.covers)
    for li in range(len(T.levels)):
        np.testing.assert_array_equal(T.levels[li], O.covers[li])
        off, idx = T.cover_neighbors(li)
        o2, i2 = oracle.level_neighbors(O, li)
        np.testing.assert_array_equal(off, o2)
        np.testing.assert_array_equal(idx, i2)
        if li:
            np.testing.assert_array_equal(T.cover_children(li), oracle.cover_children(O, li))


@pytest.mark.parametrize("n,dim", [(2 ** 20, 2), (300000, 3)])
def test_native_tree_equals_oracle_large(n, dim):
    """Sizes where the native build runs its parallel split passes (ranges of
    >= 2^17 points) on the persistent worker pool: perm, nodes and covers
    identical to the oracle."""
    import paper_1110_3105_b200 as sk
    X = oracle.ellipse(2.0, 1.0, n)["xy"] if dim == 2 else oracle.fib_sphere(n)
    T = sk.build_tree(sk.PointSet(X), 64)
    O = oracle.build_tree(X, 64)
    np.testing.assert_array_equal(T.perm, O.perm)
    np.testing.assert_array_equal(T.center, O.center)
    np.testing.assert_array_equal(T.hw, O.hw)
    assert len(T.levels) == len(O.covers)
    for li in range(len(T.levels)):
        np.testing.assert_array_equal(T.levels[li], O.covers[li])


def test_native_tree_matches_golden(golden):
    import paper_1110_3105_b200 as sk
    g = golden("sphere_2000_1e-6")
    T = sk.build_tree(sk.PointSet(oracle.fib_sphere(2000)), 64)
    np.testing.assert_array_equal(T.perm, g["perm"])
    for li in range(T.depth):
        off, idx = T.cover_neighbors(li)
        np.testing.assert_array_equal(off, g[f"N{li}_off"])
        np.testing.assert_array_equal(idx, g[f"N{li}_idx"])
    assert sk.level_neighbors(T, 0)[0] == list(g["N0_idx"][g["N0_off"][0]:g["N0_off"][1]])


def test_tree_edge_cases():
    import paper_1110_3105_b200 as sk
    # identical points do not recurse forever (geom.py _MAX_DEPTH)
    T = sk.build_tree(sk.PointSet(np.zeros((100, 2))), 8)
    assert T.n_points == 100
    # split-plane tie goes to the upper child
    X = np.array([[0.0, 0.0], [1.0, 1.0], [0.5, 0.5], [0.25, 0.75]])
    T = sk.build_tree(sk.PointSet(X), 1)
    O = oracle.build_tree(X, 1)
    np.testing.assert_array_equal(T.perm, O.perm)
    # single point
    T = sk.build_tree(sk.PointSet(np.array([[3.0, 4.0]])), 64)
    assert T.depth == 1


def test_host_validation():
    import paper_1110_3105_b200 as sk
    with pytest.raises(sk.InvalidInput):
        sk.PointSet(np.zeros((3, 4)))
    with pytest.raises(sk.InvalidInput):
        sk.PointSet(np.array([[np.nan, 0.0]]))
    with pytest.raises(sk.InvalidInput):
        sk.KernelSpec("stokes", 2)
    with pytest.raises(sk.InvalidInput):
        sk.KernelSpec("helmholtz", 2)
    with pytest.raises(sk.InvalidInput):
        sk.bie.discretize_dirichlet(sk.bie.ellipse(2, 1, 64), sk.KernelSpec("helmholtz", 2, "double", 3.0),
                                    quad="plain_trapezoid")
    with pytest.raises(sk.InvalidInput):
        sk.ProxyConfig(n_proxy=4).resolve(2)


def test_proxy_points_match_oracle():
    import paper_1110_3105_b200 as sk
    T = sk.build_tree(sk.PointSet(oracle.ellipse(2.0, 1.0, 512)["xy"]), 64)
    node = T.nodes[3]
    P = sk.proxy_points(node, sk.ProxyConfig(), 2).coords
    ref = node.center + oracle.geometry.proxy_radius(node.halfwidth, 2) * oracle.proxy_unit_points(64, 2)
    np.testing.assert_array_equal(P, ref)


def test_level_planner_matches_numpy():
    """csrc/plan.cpp (host bookkeeping of a level) == the numpy formulation:
    target heights, offsets, big-box selection, size buckets and order."""
    from paper_1110_3105_b200 import _plan
    from paper_1110_3105_b200._staging import size_buckets
    rng = np.random.default_rng(0)
    p = 5000
    nr = rng.integers(0, 70, p)
    nc = nr.copy()
    noff = np.concatenate([[0], np.cumsum(rng.integers(1, 9, p))])
    nidx = rng.integers(0, p, noff[-1])
    neff = np.full(p, 64)
    W = (18 << 10, 27 << 10, 35 << 10, 46 << 10, 64 << 10, 100 << 10, 214 << 10)
    M = (64, 128, 192, 256, 384, 512, 768)
    pl = _plan.plan_id_level(nr, nc, noff, nidx, neff, None, 8, 232448, W, M, 512, 4096, 400)
    m0 = np.array([nc[nidx[noff[a]:noff[a + 1]]].sum() for a in range(p)]) + 64
    np.testing.assert_array_equal(pl.m0, m0)
    np.testing.assert_array_equal(pl.rdof_off, np.concatenate([[0], np.cumsum(nr)]))
    np.testing.assert_array_equal(pl.d_off, np.concatenate([[0], np.cumsum(nr * nc)]))
    need_m = np.maximum(pl.m0, pl.m1)
    need_m += need_m % 2                  # real targets: even leading dimension
    need_n = np.maximum(np.maximum(nr, nc), 1)
    wb = need_m * need_n * 8
    cls = np.searchsorted(np.asarray(W), wb) * 16 + np.searchsorted(np.asarray(M), need_m)
    cls = np.where(pl.big, -1, cls)
    ref = size_buckets(cls, wb)
    assert len(ref) == len(pl.buckets)
    for a, b in zip(ref, pl.buckets):
        np.testing.assert_array_equal(a, b)
    # factor plan: offsets, solve buckets grouped by size class
    kr = np.minimum(nr, rng.integers(0, 30, p))
    fp = _plan.plan_factor_level(nr, nc, kr, kr, None, 8, 232448,
                                 (24 << 10, 48 << 10, 80 << 10, 112 << 10, 160 << 10, 224 << 10),
                                 768, 400, (24, 40, 56, 72, 96, 128))
    np.testing.assert_array_equal(fp.dd_off, np.concatenate([[0], np.cumsum(nr * nr)]))
    np.testing.assert_array_equal(fp.ld_off, np.concatenate([[0], np.cumsum(nr * kr)]))
    scls = np.searchsorted(np.asarray((24, 40, 56, 72, 96, 128)), nr)
    for a, b in zip(size_buckets(np.where(nr > 0, scls, -1)), fp.sbuckets):
        np.testing.assert_array_equal(a, b)


def test_perm_mean_matches_numpy_bitwise():
    """The native mean(w[perm]) (proxy weight scale, bie.py:251) reproduces
    numpy's pairwise summation order bit for bit, with no gathered copy."""
    from paper_1110_3105_b200.bie import perm_mean
    rng = np.random.default_rng(11)
    for n in list(range(1, 260)) + [1023, 4096, 4097, 65543, 2 ** 20 + 5]:
        w = rng.standard_normal(n) * rng.uniform(0.1, 10.0) + 2.0
        perm = rng.permutation(n)
        assert perm_mean(w, perm) == float(np.mean(w[perm])), n


def test_native_point_checks_match_numpy_rules():
    """PointSet's native finiteness / unit-normal pass decides exactly as the
    reference's numpy expressions (geom.py:42-49), including NaN normals
    (which compare false there) and rows at the 1e-12 threshold."""
    import ctypes
    from paper_1110_3105_b200 import _native
    L = _native.lib()
    rng = np.random.default_rng(2)
    for d in (2, 3):
        for trial in range(60):
            n = 500
            v = rng.standard_normal((n, d))
            v /= np.linalg.norm(v, axis=1, keepdims=True)
            k = rng.integers(0, n, 3)
            v[k] *= 1 + rng.uniform(-2e-12, 2e-12, (3, 1))
            if trial % 7 == 0:
                v[k[0], 0] = np.nan
            ref = bool(np.any(np.abs(np.linalg.norm(v, axis=1) - 1.0) > 1e-12))
            c = rng.standard_normal((n, d))
            if trial % 11 == 0:
                c[k[1], d - 1] = np.inf
            rc = L.skel_check_points(c.ctypes.data_as(ctypes.c_void_p),
                                     v.ctypes.data_as(ctypes.c_void_p), n, d)
            want = -3 if not np.isfinite(c).all() else (-4 if ref else 0)
            assert rc == want, (d, trial, rc, want)
