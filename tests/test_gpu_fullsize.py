"""Parity at the BASELINE sizes against golden fixtures produced by the LIVE
reference (tests/golden/make_golden_full.py):

  * config 2: 2D Laplace DL ellipse, N = 2^20, eps = 1e-12, 16 RHS;
  * config 5: the same factorization, 1024 RHS (the R >= 64 DMMA sweeps),
    first 64 columns compared through a Gaussian sketch;
  * config 3: CFIE (complex128), N = 2^18, eps = 1e-9, 4 RHS;
  * config 4: 3D sphere SL, unit diagonal, N = 40000, eps = 1e-6.

Every test reports SURVEY 8(d)'s correctness numbers -- the per-box rank
delta histogram, the number of boxes whose row / column skeleton SETS differ
from the reference (exact up to 64-bit hash collisions), ||x - x_ref|| /
||x_ref||, and the relative residual ||A x - b|| / ||b|| of BOTH solutions
against the exact operator (K6, on-the-fly dense matvec) -- printed and
written to gpurun_out/parity_<config>.json.

Bars (BASELINE north_star): ranks within +-2 per box; solution within
10 eps_ID of the reference.  SURVEY F3: at eps = 1e-12 a 1-ulp perturbation of
the ID targets already flips a few skeleton sets in the reference itself and
moves its solution by 3e-11 .. 2.3e-10 (> 10 eps), so for configs 2 / 5 the
solution bar is replaced by: GPU residual <= 2 x the reference's own residual
(measured with the same K6 operator), and the measured error is reported.
"""

import json
import os
import sys

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
from skelhash import skel_set_hash  # noqa: E402

gpu = pytest.mark.gpu
ROOT = os.path.dirname(HERE)


def _sk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs CUDA")
    import paper_1110_3105_b200 as sk
    return sk


def parity_report(cm, g):
    """Per-box rank deltas and differing skeleton sets vs the reference."""
    hist = {}
    diff_r = diff_c = nbox = 0
    worst = 0
    for li in range(int(g["nlevels"])):
        lv = cm.levels[li]
        kr, kc = lv.kr_counts, lv.kc_counts
        dr = kr - g[f"L{li}_kr"].astype(np.int64)
        dc = kc - g[f"L{li}_kc"].astype(np.int64)
        for d in np.concatenate([dr, dc]):
            hist[int(d)] = hist.get(int(d), 0) + 1
        worst = max(worst, int(np.abs(dr).max(initial=0)), int(np.abs(dc).max(initial=0)))
        rs, cs = lv.skeleton_arrays()
        diff_r += int((skel_set_hash(rs, kr) != g[f"L{li}_row_hash"]).sum())
        diff_c += int((skel_set_hash(cs, kc) != g[f"L{li}_col_hash"]).sum())
        nbox += kr.size
    return {"boxes": nbox, "rank_delta_hist": dict(sorted(hist.items())), "max_rank_delta": worst,
            "row_skel_sets_differing": diff_r, "col_skel_sets_differing": diff_c}


def _resid(sk, src, x, b):
    y = sk.bie.dense_matvec(src, x.reshape(-1, 1))
    return float(np.linalg.norm(y - b.reshape(-1, 1)) / np.linalg.norm(b))


def _emit(name, rep):
    print(f"\nparity[{name}] " + json.dumps(rep))
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, f"parity_{name}.json"), "w") as f:
            json.dump(rep, f, indent=1)


@gpu
def test_config2_and_5_full_size_parity(golden):
    """N = 2^20, eps = 1e-12 (BASELINE configs 2 and 5) vs the live reference."""
    import torch
    sk = _sk()
    g = golden("full_c2_ellipse_1048576_1e-12")
    n, eps = 1 << 20, 1e-12
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    tree, cm = sk.bie.compress_system(system, eps, 64)
    assert cm.nlevels == int(g["nlevels"])
    fi = sk.factor(cm)
    rep = parity_report(cm, g)
    rep["S_shape"] = list(cm.S_shape())
    rep["S_shape_ref"] = g["S_shape"].tolist()
    B = np.random.default_rng(0).standard_normal((n, 16))
    X = sk.solve(fi, B)
    x0, xr = X[:, 0], g["X0"]
    rep["rel_err_x"] = float(np.linalg.norm(x0 - xr) / np.linalg.norm(xr))
    rep["colnorm_rel_dev"] = float(np.abs(np.linalg.norm(X, axis=0) / g["X_colnorm"] - 1).max())
    src = sk.bie.BieSource(system, tree.perm)
    rep["residual_gpu"] = _resid(sk, src, x0, B[:, 0])
    rep["residual_ref"] = _resid(sk, src, xr, B[:, 0])
    # config 5: the seeded 1024-RHS block, every column through the DMMA
    # pipe sweeps; the first 64 columns against the reference via the sketch
    del X, B
    B5 = np.random.default_rng(0).standard_normal((n, 1024))
    Bd = torch.from_numpy(B5).cuda()
    del B5
    X5 = sk.solve_device(fi, Bd)
    del Bd
    Om = torch.from_numpy(np.random.default_rng(1).standard_normal((n, 8))).cuda()
    sk5 = (Om.T @ X5[:, :64]).cpu().numpy()
    cn5 = torch.linalg.norm(X5[:, :64], dim=0).cpu().numpy()
    del X5, Om
    torch.cuda.empty_cache()
    rep["c5_sketch_rel_err"] = float(np.linalg.norm(sk5 - g["c5_sketch"]) /
                                     np.linalg.norm(g["c5_sketch"]))
    rep["c5_colnorm_rel_dev"] = float(np.abs(cn5 / g["c5_colnorm"] - 1).max())
    _emit("config2_n1048576", rep)
    assert rep["max_rank_delta"] <= 2
    assert rep["residual_gpu"] <= 2 * rep["residual_ref"] + 1e-14
    assert rep["residual_gpu"] <= 1e-10
    assert rep["rel_err_x"] <= 1e-9            # measured value is in the report
    assert rep["c5_sketch_rel_err"] <= 1e-9
    assert rep["c5_colnorm_rel_dev"] <= 1e-9


@gpu
def test_config3_full_size_parity(golden):
    """CFIE, complex128, N = 2^18, eps = 1e-9 (BASELINE config 3)."""
    sk = _sk()
    g = golden("full_c3_cfie_262144_1e-9")
    n, eps = 1 << 18, 1e-9
    k = float(g["k"])
    assert abs(k - 2 * np.pi * 8 / oracle.ellipse_perimeter(2.0, 1.0)) < 1e-12
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.combined_field_system(curve, k)
    tree, cm = sk.bie.compress_system(system, eps, 64)
    fi = sk.factor(cm)
    rep = parity_report(cm, g)
    rep["S_shape"], rep["S_shape_ref"] = list(cm.S_shape()), g["S_shape"].tolist()
    rng = np.random.default_rng(0)
    B = rng.standard_normal((n, 4)) + 1j * rng.standard_normal((n, 4))
    X = sk.solve(fi, B)
    x0, xr = X[:, 0], g["X0"]
    rep["rel_err_x"] = float(np.linalg.norm(x0 - xr) / np.linalg.norm(xr))
    rep["colnorm_rel_dev"] = float(np.abs(np.linalg.norm(X, axis=0) / g["X_colnorm"] - 1).max())
    src = sk.bie.BieSource(system, tree.perm)
    rep["residual_gpu"] = _resid(sk, src, x0, B[:, 0])
    rep["residual_ref"] = _resid(sk, src, xr, B[:, 0])
    _emit("config3_n262144", rep)
    assert rep["max_rank_delta"] <= 2
    assert rep["rel_err_x"] <= 10 * eps
    assert rep["residual_gpu"] <= 2 * rep["residual_ref"] + 1e-12


@gpu
def test_config4_full_size_parity(golden):
    """3D sphere single layer, unit diagonal, N = 40000, eps = 1e-6 (BASELINE
    config 4; its coarse levels take the randomized ID, whose sketch draws are
    the reference's numpy draws)."""
    sk = _sk()
    g = golden("full_c4_sphere_40000_1e-6")
    n, eps = 40000, 1e-6
    pts = sk.PointSet(oracle.fib_sphere(n), None, np.full(n, 4 * np.pi / n))
    tree = sk.build_tree(pts, 64)
    src = sk.KernelSource(sk.KernelSpec("laplace", 3), pts, tree.perm, diag=1.0)
    cm = sk.compress_source(src, tree, eps)
    fi = sk.factor(cm)
    rep = parity_report(cm, g)
    rep["S_shape"], rep["S_shape_ref"] = list(cm.S_shape()), g["S_shape"].tolist()
    B = np.random.default_rng(0).standard_normal((n, 1))
    X = sk.solve(fi, B)
    xr = g["X"][:, 0]
    rep["rel_err_x"] = float(np.linalg.norm(X[:, 0] - xr) / np.linalg.norm(xr))
    rep["residual_gpu"] = _resid(sk, src, X[:, 0], B[:, 0])
    rep["residual_ref"] = _resid(sk, src, xr, B[:, 0])
    _emit("config4_n40000", rep)
    assert rep["max_rank_delta"] <= 2
    assert rep["rel_err_x"] <= 10 * eps
    assert rep["residual_gpu"] <= 2 * rep["residual_ref"] + 1e-12


@gpu
@pytest.mark.parametrize("R", [64, 1024])
def test_config5_shape_many_rhs_vs_oracle(R):
    """The R >= 64 DMMA-pipe sweeps against the ORACLE's solve (solver.py:
    279-318 restated) on the oracle's own factorization of the same system,
    every column, at N = 4096 / eps = 1e-12."""
    sk = _sk()
    import torch
    n, eps = 4096, 1e-12
    curve = sk.bie.ellipse(2.0, 1.0, n)
    system = sk.bie.discretize_dirichlet(curve, sk.KernelSpec("laplace", 2))
    tree, cm = sk.bie.compress_system(system, eps, 64)
    fi = sk.factor(cm)
    B = np.random.default_rng(R).standard_normal((n, R))
    X = sk.solve_device(fi, torch.from_numpy(B).cuda()).cpu().numpy()
    oc = oracle.ellipse(2.0, 1.0, n)
    T = oracle.build_tree(oc["xy"], 64)
    osrc = oracle.BieSource(oc, T.perm)
    Xo = oracle.solve(oracle.factor(oracle.compress(osrc, T, eps)), B)
    err = np.linalg.norm(X - Xo, axis=0) / np.linalg.norm(Xo, axis=0)
    # eps = 1e-12: SURVEY F3 pivot flips; the solutions agree far below the
    # discretisation error and every column is checked
    assert err.max() <= 1e-9, err.max()
