"""Oracle matrix entries.  TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Restates:
  * eval_block            kernels.py:82-161 (Green's functions, coincident
                          policy, source-weight column scaling)
  * BieSystem.block       bie.py:158-172 (KR10 reweighting, identity term)
  * KR10 table            bie.py:31-42 (numbers are the published
                          Kapur-Rokhlin order-10 weights)
"""

import numpy as np
from scipy import special as sp

COINCIDENT_RTOL = 1e-14   # kernels.py:24

KR10_GAMMA = np.array([
    7.832432020568779e+00, -4.565161670374749e+01, 1.452168846354677e+02,
    -2.901348302886379e+02, 3.870862162579900e+02, -3.523821383570681e+02,
    2.172421547519342e+02, -8.707796087382991e+01, 2.053584266072635e+01,
    -2.166984103403823e+00,
])


def _span(t, s):
    ext = [1.0]
    for c in (t, s):
        if c.shape[0]:
            ext.append(float(np.ptp(c, axis=0).max()))
            ext.append(float(np.abs(c).max()))
    return max(ext)


def eval_block(equation, dim, layer, k, tgt, src, src_normals=None,
               src_weights=None, src_curv=None, self_interaction="zero"):
    """Dense block G(x_i, y_j) or dG/dnu_y (kernels.py:82-161).

    Conventions (kernels.py:3-11): 2D Laplace -log r/(2pi); 3D 1/(4 pi r);
    2D Helmholtz (i/4) H0(kr); 3D exp(ikr)/(4 pi r).  Double layer is the
    normal derivative at the source.  Columns scaled by source weights.
    """
    tgt = np.asarray(tgt, dtype=np.float64)
    src = np.asarray(src, dtype=np.float64)
    diff = tgt[:, None, :] - src[None, :, :]
    r = np.sqrt(np.sum(diff * diff, axis=2))
    same = r < COINCIDENT_RTOL * _span(tgt, src)
    rs = np.where(same, 1.0, r)
    helm = equation == "helmholtz"
    if layer == "single":
        if not helm:
            G = -np.log(rs) / (2 * np.pi) if dim == 2 else 1.0 / (4 * np.pi * rs)
        elif dim == 2:
            G = 0.25j * (sp.j0(k * rs) + 1j * sp.y0(k * rs))
        else:
            G = np.exp(1j * k * rs) / (4 * np.pi * rs)
    else:
        ndot = -np.einsum("ijk,jk->ij", diff, src_normals)
        if not helm:
            G = -ndot / (2 * np.pi * rs * rs) if dim == 2 else -ndot / (4 * np.pi * rs ** 3)
        elif dim == 2:
            G = -0.25j * k * (sp.j1(k * rs) + 1j * sp.y1(k * rs)) * ndot / rs
        else:
            G = np.exp(1j * k * rs) * (1j * k * rs - 1.0) / (4 * np.pi * rs * rs) * ndot / rs
    if same.any():
        if self_interaction == "zero":
            G = np.where(same, np.zeros(1, dtype=G.dtype), G)
        else:
            lim = -np.asarray(src_curv) / (4 * np.pi)
            G = np.where(same, np.broadcast_to(lim, G.shape[1:])[None, :], G)
    if src_weights is not None:
        G = G * np.asarray(src_weights)[None, :]
    return G


def cyclic_distance(i, j, n):
    """bie.py:130-132."""
    d = np.abs(np.asarray(i)[:, None] - np.asarray(j)[None, :])
    return np.minimum(d, n - d)


def kr10_factor(i, j, n):
    """(1 + gamma_d) for cyclic distance d in [1, 10], else 1 (bie.py:164-168)."""
    d = cyclic_distance(i, j, n)
    near = (d >= 1) & (d <= KR10_GAMMA.size)
    return np.where(near, 1.0 + KR10_GAMMA[np.clip(d, 1, KR10_GAMMA.size) - 1], 1.0)


def ellipse_perimeter(a=2.0, b=1.0, m=4096):
    """Trapezoid rule on the periodic speed |x'(t)| (spectrally accurate);
    used to pick the config-3 wavenumber."""
    t = 2 * np.pi * np.arange(m) / m
    return float(np.sum(np.sqrt((a * np.sin(t)) ** 2 + (b * np.cos(t)) ** 2)) * 2 * np.pi / m)
