// entries.cuh -- on-the-fly matrix entries of the supported matrix sources.
//
// Restates, per entry, the reference's block evaluators:
//   eval_block                kernels.py:82-161
//   BieSystem.block           bie.py:158-172 (KR10 bie.py:31-42,164-168)
//   _BieSource proxy blocks   bie.py:256-262 (row proxies * wscale, col proxies
//                             weighted, single layer)
//   KernelSource blocks       skel.py:113-124
// The float64 Laplace entries use explicitly rounded operations in numpy's
// evaluation order (no FMA contraction), so they reproduce the reference's
// values bit for bit wherever libm agrees.
#pragma once

#include "common.cuh"

struct Pt {
  double x, y, z, nx, ny, nz, w, kap;
  int64_t o;
};

__device__ __forceinline__ Pt load_pt(const SkelSource& S, int64_t i) {
  Pt p;
  p.x = __ldg(S.x + i);
  p.y = __ldg(S.y + i);
  p.z = S.z ? __ldg(S.z + i) : 0.0;
  p.nx = S.nx ? __ldg(S.nx + i) : 0.0;
  p.ny = S.ny ? __ldg(S.ny + i) : 0.0;
  p.nz = S.nz ? __ldg(S.nz + i) : 0.0;
  p.w = S.w ? __ldg(S.w + i) : 1.0;
  p.kap = S.curv ? __ldg(S.curv + i) : 0.0;
  p.o = S.orig ? __ldg(S.orig + i) : i;
  return p;
}

__constant__ double c_kr10[10] = {
    7.832432020568779e+00, -4.565161670374749e+01, 1.452168846354677e+02,
    -2.901348302886379e+02, 3.870862162579900e+02, -3.523821383570681e+02,
    2.172421547519342e+02, -8.707796087382991e+01, 2.053584266072635e+01,
    -2.166984103403823e+00};

// sqrt(sum(diff*diff)) as numpy evaluates it (kernels.py:108-109)
__device__ __forceinline__ double sk_dist(const SkelSource& S, double dx, double dy, double dz) {
  double r2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  if (S.dim == 3) r2 = __dadd_rn(r2, __dmul_rn(dz, dz));
  return __dsqrt_rn(r2);
}

// (y - x) . nu_y  (the reference's -ndot, kernels.py:132)
__device__ __forceinline__ double sk_ndot_neg(const SkelSource& S, double dx, double dy, double dz,
                                              const Pt& s) {
  double e = __dadd_rn(__dmul_rn(dx, s.nx), __dmul_rn(dy, s.ny));
  if (S.dim == 3) e = __dadd_rn(e, __dmul_rn(dz, s.nz));
  return e;  // = einsum(diff, nu); reference ndot = -e, numerator -ndot = e
}

__device__ __forceinline__ double kr10_factor(const SkelSource& S, int64_t oi, int64_t oj) {
  int64_t nn = S.n;
  if (S.grp) {
    const int g = __ldg(S.grp + oi);
    if (g != __ldg(S.grp + oj)) return 1.0;
    const int64_t b = __ldg(S.grp_start + g);
    oi -= b;
    oj -= b;
    nn = __ldg(S.grp_size + g);
  }
  int64_t d = oi > oj ? oi - oj : oj - oi;
  int64_t d2 = nn - d;
  if (d2 < d) d = d2;
  if (d >= 1 && d <= 10) return __dadd_rn(1.0, c_kr10[d - 1]);
  return 1.0;
}

// ---- Green's functions (unweighted) ---------------------------------------
// Laplace single layer
__device__ __forceinline__ double lap_sl(const SkelSource& S, double r) {
  if (S.dim == 2) return __ddiv_rn(-log(r), SKEL_TWO_PI);
  return __ddiv_rn(1.0, __dmul_rn(SKEL_FOUR_PI, r));
}
// Laplace double layer dG/dnu_y given e = (x-y).nu_y ... see sk_ndot_neg
__device__ __forceinline__ double lap_dl(const SkelSource& S, double e, double r) {
  if (S.dim == 2) return __ddiv_rn(e, __dmul_rn(__dmul_rn(SKEL_TWO_PI, r), r));
  return __ddiv_rn(e, __dmul_rn(SKEL_FOUR_PI, pow(r, 3.0)));
}
// Hankel function H_NU^(1)(z) = J_NU + i Y_NU, NU in {0, 1} (kernels.py:65-75 uses
// scipy's Cephes j0/y0/j1/y1, ~1e-15 of |H| everywhere).  CUDA's j0/y0/j1/y1 hold
// <= 7e-15 of |H| up to z = 16 but lose up to 9e-12 beyond (measured against
// mpmath, tools/h0acc.py), so from 16 on Hankel's asymptotic expansion is summed:
//   H ~ sqrt(2/(pi z)) e^{i(z - NU pi/2 - pi/4)} sum_k i^k a_k / z^k,
//   a_k = a_{k-1} (4 NU^2 - (2k-1)^2) / (8k),
// to its smallest term (< e^{-2z} <= 1.3e-14, <= 1.6e-15 of |H| measured); the phase
// factor is applied as e^{iz} times the exact constant, no reduced argument.
template <int NU>
__device__ __forceinline__ void sk_hankel(double z, double& re, double& im) {
  if (z < 16.0) {
    re = NU == 0 ? j0(z) : j1(z);
    im = NU == 0 ? y0(z) : y1(z);
    return;
  }
  const double mu = 4.0 * NU * NU;
  const double iz = 1.0 / (8.0 * z);
  double pr = 1.0, pi = 0.0, cr = 1.0, ci = 0.0;
  for (int k = 1; k < 64; ++k) {
    const double t = 2.0 * k - 1.0;
    const double f = (mu - t * t) * iz / k;
    if (fabs(f) >= 1.0) break;
    const double nr = -ci * f, ni = cr * f;      // c *= i f
    cr = nr;
    ci = ni;
    pr += cr;
    pi += ci;
    if (fabs(cr) + fabs(ci) < 1e-18) break;
  }
  double sn, cs;
  sincos(z, &sn, &cs);
  const double amp = sqrt(0.63661977236758134308 / z) * 0.70710678118654752440;
  const double er = NU == 0 ? (cs + sn) * amp : (sn - cs) * amp;
  const double ei = NU == 0 ? (sn - cs) * amp : -(cs + sn) * amp;
  re = er * pr - ei * pi;
  im = er * pi + ei * pr;
}

// Helmholtz single layer: 2D (i/4) H0(kr), 3D exp(ikr)/(4 pi r)
__device__ __forceinline__ zc helm_sl(const SkelSource& S, double r) {
  double kr = S.k * r;
  if (S.dim == 2) {
    double hj, hy;
    sk_hankel<0>(kr, hj, hy);
    return zc(-0.25 * hy, 0.25 * hj);
  }
  double sn, cs;
  sincos(kr, &sn, &cs);
  double den = SKEL_FOUR_PI * r;
  return zc(cs / den, sn / den);
}
// Helmholtz double layer given the reference's ndot (= -e)
__device__ __forceinline__ zc helm_dl(const SkelSource& S, double e, double r) {
  double ndot = -e;
  double kr = S.k * r;
  if (S.dim == 2) {
    // (-0.25j * k) * (J1 + i Y1) * ndot / r   (kernels.py:141)
    double a = 0.25 * S.k;
    double hj, hy;
    sk_hankel<1>(kr, hj, hy);
    zc h = zc(a * hy, -a * hj);
    return zc(h.re * ndot / r, h.im * ndot / r);
  }
  // exp(ikr) (ikr - 1) / (4 pi r^2) * ndot / r  (kernels.py:143-144)
  double sn, cs;
  sincos(kr, &sn, &cs);
  zc ex(cs, sn);
  zc g = ex * zc(-1.0, kr);
  double den = SKEL_FOUR_PI * r * r;
  g = zc(g.re / den, g.im / den);
  return zc(g.re * ndot / r, g.im * ndot / r);
}

template <class T> __device__ __forceinline__ T as_T(double v);
template <> __device__ __forceinline__ double as_T<double>(double v) { return v; }
template <> __device__ __forceinline__ zc as_T<zc>(double v) { return zc(v); }
template <class T> __device__ __forceinline__ T from_zc(zc v);
template <> __device__ __forceinline__ double from_zc<double>(zc v) { return v.re; }
template <> __device__ __forceinline__ zc from_zc<zc>(zc v) { return v; }

// ---- system entry A(t, s) -------------------------------------------------
template <class T>
__device__ __forceinline__ T entry_A(const SkelSource& S, const Pt& t, const Pt& s) {
  double dx = __dsub_rn(t.x, s.x), dy = __dsub_rn(t.y, s.y), dz = __dsub_rn(t.z, s.z);
  double r = sk_dist(S, dx, dy, dz);
  bool same = r < S.coincide_tol;
  bool helm = S.equation == SKEL_EQ_HELMHOLTZ;
  T g;
  if (S.kind == SKEL_SRC_NTRACE) {
    // -(ik/4) H1(kr) (x - y).nu_x / r * w_y  (bie.py:305-323)
    zc v(0.0);
    if (!same) v = helm_dl(S, -__dadd_rn(__dmul_rn(dx, t.nx), __dmul_rn(dy, t.ny)), r);
    g = from_zc<T>(zc(v.re * s.w, v.im * s.w));
  } else if (S.kind == SKEL_SRC_CFIE) {
    zc v(0.0);
    if (!same) {
      double e = sk_ndot_neg(S, dx, dy, dz, s);
      zc dl = helm_dl(S, e, r);
      zc sl = helm_sl(S, r);
      dl = zc(dl.re * s.w, dl.im * s.w);
      sl = zc(sl.re * s.w, sl.im * s.w);
      // dl - 1j*k*sl
      v = zc(dl.re - (-S.k * sl.im), dl.im - S.k * sl.re);
    }
    g = from_zc<T>(v);
  } else {
    bool dbl = S.kind == SKEL_SRC_BIE || S.layer == SKEL_LAYER_DOUBLE;
    if (same) {
      if (dbl && S.curvature_limit && !helm)
        g = as_T<T>(__dmul_rn(__ddiv_rn(-s.kap, SKEL_FOUR_PI), s.w));
      else
        g = as_T<T>(0.0);
    } else if (!helm) {
      double v;
      if (dbl) v = lap_dl(S, sk_ndot_neg(S, dx, dy, dz, s), r);
      else v = lap_sl(S, r);
      g = as_T<T>(S.w ? __dmul_rn(v, s.w) : v);
    } else {
      zc v = dbl ? helm_dl(S, sk_ndot_neg(S, dx, dy, dz, s), r) : helm_sl(S, r);
      if (S.w) v = zc(v.re * s.w, v.im * s.w);
      g = from_zc<T>(v);
    }
  }
  if (S.kr10) g = g * kr10_factor(S, t.o, s.o);
  if (t.o == s.o) {
    double add = (S.kind == SKEL_SRC_KERNEL) ? S.diag : S.identity_coef;
    g = g + as_T<T>(add);
  }
  return g;
}

// single-layer proxy interaction, unweighted (kernels.py SL branch)
template <class T>
__device__ __forceinline__ T proxy_G(const SkelSource& S, double dx, double dy, double dz) {
  double r = sk_dist(S, dx, dy, dz);
  if (r < S.coincide_tol) return as_T<T>(0.0);
  if (S.equation == SKEL_EQ_HELMHOLTZ) return from_zc<T>(helm_sl(S, r));
  return as_T<T>(lap_sl(S, r));
}

// row proxy: wscale * G_SL(x_t, pxy)   (bie.py:256-257, skel.py:116-118)
template <class T>
__device__ __forceinline__ T entry_proxy_row(const SkelSource& S, const Pt& t, double px,
                                             double py, double pz) {
  const double dx = __dsub_rn(t.x, px), dy = __dsub_rn(t.y, py), dz = __dsub_rn(t.z, pz);
  if (S.kind == SKEL_SRC_NTRACE) {
    // Neumann trace of the proxy's single-layer field, unweighted (bie.py:342-344)
    const double r = sk_dist(S, dx, dy, dz);
    if (r < S.coincide_tol) return as_T<T>(0.0);
    return from_zc<T>(helm_dl(S, -__dadd_rn(__dmul_rn(dx, t.nx), __dmul_rn(dy, t.ny)), r));
  }
  T g = proxy_G<T>(S, dx, dy, dz);
  return g * S.wscale;
}

// column proxy: G_SL(pxy, y_s) * w_s   (bie.py:259-262, skel.py:120-124)
template <class T>
__device__ __forceinline__ T entry_proxy_col(const SkelSource& S, double px, double py,
                                             double pz, const Pt& s) {
  T g = proxy_G<T>(S, __dsub_rn(px, s.x), __dsub_rn(py, s.y), __dsub_rn(pz, s.z));
  if (S.w) g = g * s.w;
  return g;
}
