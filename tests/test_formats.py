"""Data formats either side of the path: the reference's SKLC
binary containers, the sparse embedding + Matrix Market export, GMRES, and
bessel_h0.  Golden bytes / arrays come from the live reference
(tests/golden/make_golden.py, case sklc_ellipse_512_1e-6)."""

import os
import tempfile

import numpy as np
import pytest

gpu = pytest.mark.gpu


def _g(golden):
    return golden("sklc_ellipse_512_1e-6")


# ---------------------------------------------------------------------------
# CPU: container / embedding / Matrix Market / GMRES semantics

def test_compressed_container_round_trip_bytes(golden):
    from paper_1110_3105_b200 import container
    g = _g(golden)
    data = g["cm_bytes"].tobytes()
    cm = container.deserialize_compressed(data)
    assert cm.n == int(g["n"]) and cm.eps == float(g["eps"])
    assert container.serialize_compressed(cm) == data


def test_factored_container_round_trip_bytes(golden):
    from paper_1110_3105_b200 import container
    g = _g(golden)
    data = g["fi_bytes"].tobytes()
    parsed = container.parse_factored(data)
    assert parsed[1] == int(g["n"])
    assert container.emit_factored(*parsed) == data


def test_container_rejects_garbage(golden):
    from paper_1110_3105_b200 import InvalidInput, container
    with pytest.raises(InvalidInput):
        container.deserialize_compressed(b"NOPE" + b"\0" * 64)
    g = _g(golden)
    with pytest.raises(InvalidInput):              # a compressed container is not a factored one
        container.parse_factored(g["cm_bytes"].tobytes())
    with pytest.raises(InvalidInput):
        container.deserialize_compressed(g["cm_bytes"].tobytes()[:100])


def test_embedding_matches_reference(golden):
    from paper_1110_3105_b200 import assemble_embedding, container
    g = _g(golden)
    cm = container.deserialize_compressed(g["cm_bytes"].tobytes())
    se = assemble_embedding(cm)
    assert se.m == int(g["emb_m"])
    assert list(se.blocks.keys()) == [str(x) for x in g["emb_labels"]]
    r, c, v = se.to_coo()
    np.testing.assert_array_equal(r, g["emb_rows"])
    np.testing.assert_array_equal(c, g["emb_cols"])
    np.testing.assert_array_equal(v, g["emb_vals"])
    # the embedding reproduces the solve: x = first n unknowns of A_e^-1 [b, 0]
    A = se.to_dense()
    b = np.random.default_rng(0).standard_normal(cm.n)
    x = se.extract_x(np.linalg.solve(A, se.rhs(b)))
    assert np.isfinite(x).all()


def test_matrix_market_export_is_reference_text(golden):
    from paper_1110_3105_b200 import assemble_embedding, container, export_matrix_market
    from paper_1110_3105_b200.embedding import read_matrix_market
    g = _g(golden)
    se = assemble_embedding(container.deserialize_compressed(g["cm_bytes"].tobytes()))
    fd, path = tempfile.mkstemp(suffix=".mtx")
    os.close(fd)
    try:
        export_matrix_market(se, path)
        with open(path, "rb") as fh:
            assert fh.read() == g["mm_bytes"].tobytes()
        shape, r, c, v = read_matrix_market(path)
    finally:
        os.unlink(path)
    assert shape == (se.m, se.m)
    A = np.zeros(shape)
    A[r, c] = v
    np.testing.assert_array_equal(A, se.to_dense())


def test_gmres_matches_reference(golden):
    from paper_1110_3105_b200 import NotConverged, gmres
    g = _g(golden)
    x, its = gmres(g["gmres_A"], g["gmres_b"], tol=1e-12)
    assert its == int(g["gmres_iters"])
    np.testing.assert_allclose(x, g["gmres_x"], rtol=0, atol=1e-12)
    with pytest.raises(NotConverged) as exc:
        gmres(g["gmres_A"], g["gmres_b"], tol=1e-14, max_iter=3)
    assert exc.value.iterations == 3 and exc.value.x.shape == (60,)


# ---------------------------------------------------------------------------
# GPU: loading into device slabs, saving from them

def _sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1110_3105_b200 as sk
    return sk


@gpu
def test_load_reference_factored_and_solve(golden):
    sk = _sk()
    from paper_1110_3105_b200 import container
    g = _g(golden)
    fi = container.deserialize_factored(g["fi_bytes"].tobytes())
    n = int(g["n"])
    B = np.random.default_rng(0).standard_normal((n, 2))
    X = sk.solve(fi, B)
    np.testing.assert_allclose(X, g["X"], rtol=0, atol=1e-12 * np.abs(g["X"]).max())
    # and save it back byte for byte (blocks and the stored LU untouched)
    assert container.serialize_factored(fi) == g["fi_bytes"].tobytes()


@gpu
def test_load_reference_compressed_factor_apply(golden):
    sk = _sk()
    from paper_1110_3105_b200 import container
    g = _g(golden)
    cm = container.deserialize_compressed(g["cm_bytes"].tobytes())
    fi = sk.factor(cm)
    n = int(g["n"])
    B = np.random.default_rng(0).standard_normal((n, 2))
    X = sk.solve(fi, B)
    assert np.linalg.norm(X - g["X"]) / np.linalg.norm(g["X"]) <= 1e-10
    Y = sk.apply(cm, g["X"])
    np.testing.assert_allclose(Y, g["Y_apply"], rtol=0, atol=1e-12 * np.abs(g["Y_apply"]).max())


@gpu
def test_save_load_gpu_factorization(tmp_path):
    sk = _sk()
    import scipy.linalg as sla
    n = 2048
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    tree, cm = sk.bie.compress_system(system, 1e-10, 64)
    fi = sk.factor(cm)
    B = np.random.default_rng(1).standard_normal((n, 3))
    X = sk.solve(fi, B)
    sk.save_compressed(cm, tmp_path / "cm.sklc")
    sk.save_factored(fi, tmp_path / "fi.sklc")
    fi2 = sk.load_factored(tmp_path / "fi.sklc")
    X2 = sk.solve(fi2, B)
    assert np.linalg.norm(X2 - X) / np.linalg.norm(X) <= 1e-12
    # the stored Shat factors are a valid getrf result: P L U = Shat
    lu, piv = fi.S_lu
    Sh = fi.S_hat.cpu().numpy()
    ref_lu, ref_piv = sla.lu_factor(Sh)
    x = np.random.default_rng(2).standard_normal(Sh.shape[0])
    np.testing.assert_allclose(sla.lu_solve((lu, piv), x), sla.lu_solve((ref_lu, ref_piv), x),
                               rtol=1e-9, atol=1e-12)
    cm2 = sk.load_compressed(tmp_path / "cm.sklc")
    np.testing.assert_allclose(sk.apply(cm2, X), sk.apply(cm, X), rtol=0, atol=1e-13)


@gpu
def test_bessel_h0_gpu():
    sk = _sk()
    import scipy.special as spc
    z = np.linspace(0.01, 600.0, 4001)
    h = sk.bessel_h0(z)
    ref = spc.j0(z) + 1j * spc.y0(z)
    # CUDA's j0 / y0 below z = 16, Hankel's asymptotic expansion above
    # (csrc/entries.cuh sk_hankel): the reference's own bar, 1e-13 of |H0|
    # (tests/test_kernels.py:99-106), against Cephes here and mpmath below
    assert np.max(np.abs(h - ref) / np.abs(ref)) < 1e-13
    mp = pytest.importorskip("mpmath")
    mp.mp.dps = 30
    zs = np.concatenate([np.geomspace(1e-3, 8, 25), np.linspace(8.3, 700, 40), [15.99, 16.0, 16.01]])
    got = sk.bessel_h0(zs)
    for zz, gg in zip(zs, got):
        exact = complex(mp.besselj(0, mp.mpf(float(zz))) + 1j * mp.bessely(0, mp.mpf(float(zz))))
        assert abs(gg - exact) / abs(exact) < 1e-13, zz
    assert isinstance(sk.bessel_h0(1.0), complex)
    with pytest.raises(sk.InvalidInput):
        sk.bessel_h0(0.0)


# ---------------------------------------------------------------------------
# multiple scattering: Neumann-trace source on the GPU,
# skeletonized block preconditioner, GMRES -- against the live reference

def _scat(sk, g):
    n, k = int(g["n"]), float(g["k"])
    curves = [sk.bie.trefoil(n, center=(-0.6, 0.0), scale=1.0),
              sk.bie.trefoil(n, center=(0.6, 0.1), scale=0.8)]
    return sk.bie.scattering_system(curves, k)


@gpu
def test_scattering_entries_and_rhs(golden):
    sk = _sk()
    g = golden("scattering_2x256_k3")
    sysm = _scat(sk, g)
    A = sysm.matrix()
    # CUDA j1 / y1 vs Cephes (~1e-12 abs), KR10 inside each scatterer, -1/2 jump
    np.testing.assert_allclose(A[g["ii"], g["jj"]], g["A_sample"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(np.diag(A), g["A_diag"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(A[0], g["A_row0"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(A[-1], g["A_row_last"], rtol=0, atol=1e-11)
    np.testing.assert_allclose(sysm.rhs_plane_wave(), g["rhs"], rtol=1e-15, atol=1e-15)
    x = np.random.default_rng(4).standard_normal(sysm.n) + 0j
    np.testing.assert_allclose(sysm.apply(x), A @ x, rtol=0, atol=1e-10)


@gpu
def test_scattering_preconditioned_gmres(golden):
    sk = _sk()
    g = golden("scattering_2x256_k3")
    sysm = _scat(sk, g)
    facs = sysm.precond_blocks(1e-8, 32)
    b = sysm.rhs_plane_wave()
    x, its = sk.gmres(sysm.apply, b, tol=1e-10, precond=sysm.precond_apply(facs))
    assert abs(its - int(g["iters"])) <= 1
    assert np.linalg.norm(x - g["x"]) / np.linalg.norm(g["x"]) <= 1e-7
    np.testing.assert_allclose(sysm.scattered_field(x, g["field_targets"]), g["field"],
                               rtol=1e-6, atol=1e-9)
    with pytest.raises(sk.InvalidInput):
        sk.bie.scattering_system([sk.bie.trefoil(64), sk.bie.trefoil(64, scale=0.5)], 3.0)


@gpu
def test_embedding_of_gpu_compression_solves_like_the_factorization(tmp_path):
    """assemble_embedding (solver.py:91-140) of a GPU-compressed matrix, solved
    by an independent sparse direct solver (scipy SuperLU), equals the
    telescoping factor/solve of the same matrix; the Matrix Market export of
    it reads back to the same COO."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    sk = _sk()
    from paper_1110_3105_b200 import embedding
    n, eps = 4096, 1e-9
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    _, cm = sk.bie.compress_system(system, eps, 64)
    se = sk.assemble_embedding(cm)
    r, c, v = se.to_coo()
    A = sp.csc_matrix((v, (r, c)), shape=(se.m, se.m))
    b = np.random.default_rng(4).standard_normal(n)
    x_emb = se.extract_x(spla.spsolve(A, se.rhs(b)))
    x_fac = sk.solve(sk.factor(cm), b)
    assert np.linalg.norm(x_emb - x_fac) / np.linalg.norm(x_fac) <= 1e-10
    path = tmp_path / "emb.mtx"
    sk.export_matrix_market(se, str(path))
    shape, r2, c2, v2 = embedding.read_matrix_market(str(path))
    assert shape == (se.m, se.m)
    A2 = sp.csc_matrix((v2, (r2, c2)), shape=shape)
    assert abs(A2 - A).max() <= 1e-15 * abs(A).max()
