// cpqr.cuh -- CTA-cooperative column-pivoted Householder QR + interpolation
// matrix on a column-major target held in shared memory (or a global
// scratch slab for oversized targets).
//
// Restates lowrank.py:48-161 step for step:
//   * norms2 = exact squared column norms; ref2 = copy, indexed by POSITION
//     and never swapped (lowrank.py:55-64)
//   * every 32 steps the trailing norms are recomputed (lowrank.py:71-74)
//   * a norm that fell below 1e-8 of its reference is recomputed (75-81)
//   * pivot = first maximum of the trailing norms (82)
//   * stop when step >= min_rank and pn <= eps*p0, or pn == 0 (88-93)
//   * Householder alpha = -phase(x0)|x|, v = x - alpha e1, W -= v (2/|v|^2)(v^H W)
//     (98-110); norms2 -= |R[s,:]|^2 clipped at 0 (111-114)
//   * P[:, skel] = I, P[:, rest] = R11^-1 R12 (lowrank.py:122-133); padding to
//     min_rank with unit rows (lowrank.py:147-157)
//
// GPU mapping (two CTA barriers per step, almost no serial work):
//   * columns never move: a position -> column map (`piv`, which is also the
//     pivot order the reference returns) replaces the column swaps;
//   * phase B (all warps): every warp owns a round-robin share of the trailing
//     positions and, per column, applies the reflector (v^H w and the rank-1
//     update with the column held in registers), downdates that position's
//     norm, runs the NEXT step's renormalisation / stale rule, records the
//     exact trailing norm (the next Householder |x| if this column is picked)
//     and folds the position into a per-warp first-maximum candidate; a
//     column is handled by a group of GL lanes (several columns per warp
//     instruction, log2(GL)-level reductions);
//   * phase A (one thread): reduce the per-warp candidates to the pivot,
//     apply the stop rule, swap the position bookkeeping and form alpha, v0,
//     2/|v|^2 from the precomputed exact norm.
#pragma once

#include "common.cuh"

#define CPQR_MAXW 32

template <class T>
struct CpqrShared {
  T v0;          // first entry of the Householder vector
  T alpha;       // new diagonal entry
  double beta;   // 2/|v|^2 (0 when |v| = 0)
  double p0;     // leading pivot norm
  int rank;      // completed steps
  int stop;      // loop exit flag
  int pad;       // padded columns (min_rank > achieved rank)
  int partner_k; // rank of the other side of the box (equalize)
  int pc;        // column of the current pivot
  double bigP;   // max |P| (interp quality warning, lowrank.py:128-132)
  double trail;  // first rejected pivot norm (achieved_error numerator, lowrank.py:88-90)
  double cand_v[CPQR_MAXW];
  int cand_i[CPQR_MAXW];
};

__device__ __forceinline__ double sk_unit_phase(double x0, double) { return x0 > 0.0 ? 1.0 : -1.0; }
__device__ __forceinline__ zc sk_unit_phase(zc x0, double a) { return zc(x0.re / a, x0.im / a); }

// first-maximum merge: larger value wins, ties -> lower position
__device__ __forceinline__ void cand_merge(double& bv, int& bi, double ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
}
// FROM: only lanes that are multiples of FROM hold candidates (column-group
// leaders), so the butterfly stops there -- log2(32/FROM) dependent shuffle
// rounds instead of five; lane 0 ends with the warp's first maximum.
template <int FROM = 1>
__device__ __forceinline__ void warp_cand(double& bv, int& bi) {
#pragma unroll
  for (int o = 16; o >= FROM; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    cand_merge(bv, bi, ov, oi);
  }
}

// Initial exact norms (all rows): nrm = ref = xn2, piv = identity, and the
// per-warp pivot candidates for step 0 (lowrank.py:55-64).
template <class T>
__device__ void cpqr_init(const T* W, int m, int n, int ld, double* nrm, double* ref,
                          double* xn2, int* piv, CpqrShared<T>& sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int c = warp; c < n; c += nw) {
    double s = 0.0;
    for (int i = lane; i < m; i += SKEL_WARP) s += sk_abs2(W[(int64_t)c * ld + i]);
    s = warp_sum(s);
    if (lane == 0) { nrm[c] = s; ref[c] = s; xn2[c] = s; }
    cand_merge(bv, bi, s, c);
  }
  for (int c = threadIdx.x; c < n; c += blockDim.x) piv[c] = c;
  if (lane == 0) { sh.cand_v[warp] = bv; sh.cand_i[warp] = bi; }
}

// Phase A of step s (warp 0).  Lane 0 merges the per-warp candidates into
// the pivot (first maximum), applies the stop rule and swaps the position
// bookkeeping; the exact |x| of the pivot column is either the trailing norm
// the update phase maintained (xn2 != NULL) or a warp reduction over rows s..m-1.
template <class T>
__device__ void cpqr_pivot(T* W, int m, int n, int ld, double* nrm, double* xn2, int* piv,
                           CpqrShared<T>& sh, int s, double eps, int min_rank, int nw) {
  // all 32 lanes: the per-warp candidates are merged by a butterfly (every
  // lane ends with the first maximum), the stop rule is evaluated uniformly,
  // and the pivot column is known to every lane without a broadcast
  const int lane = threadIdx.x & 31;
  // every lane merges the (<= 16) per-warp candidates itself: independent
  // shared-memory loads and a short compare chain, no dependent shuffle
  // rounds, and the pivot is warp-uniform (the stop decision below is taken
  // per lane)
  double bv = -1.0;
  int j = 0x7fffffff;
#pragma unroll 4
  for (int w = 0; w < nw; ++w) cand_merge(bv, j, sh.cand_v[w], sh.cand_i[w]);
  int stop = 0;
  double pn = 0.0;
  if (j >= n) {
    stop = 1;
  } else {
    pn = sqrt(fmax(nrm[j], 0.0));
    const double p0 = s == 0 ? pn : sh.p0;
    if (s == 0 && pn == 0.0) stop = 1;
    else if ((s >= min_rank && pn <= eps * p0) || pn == 0.0) stop = 2;
  }
  if (lane == 0) {
    if (s == 0 && j < n) sh.p0 = pn;
    if (stop == 2) sh.trail = pn;
    sh.stop = stop;
  }
  if (stop) return;
  const int pc = piv[j];                 // pivot column (position j before the swap)
  double nx2 = 0.0;
  if (xn2) nx2 = xn2[j];
  else if (s == 0) nx2 = nrm[j];         // exact full norm at step 0
  __syncwarp();
  if (lane == 0 && j != s) {
    double t = nrm[s]; nrm[s] = nrm[j]; nrm[j] = t;
    if (xn2) { t = xn2[s]; xn2[s] = xn2[j]; xn2[j] = t; }
    piv[j] = piv[s];
    piv[s] = pc;
  }
  if (!xn2 && s > 0) {
    const T* x = W + (int64_t)pc * ld;
    double acc = 0.0;
    for (int i = s + lane; i < m; i += SKEL_WARP) acc += sk_abs2(x[i]);
    nx2 = warp_sum(acc);
  }
  if (lane == 0) {
    const T x0 = W[(int64_t)pc * ld + s];
    const double ax0 = sk_abs(x0);
    const double normx = sqrt(nx2);
    T phase = T(1.0);
    if (ax0 != 0.0) phase = sk_unit_phase(x0, ax0);   // x0 / |x0|
    const T alpha = -(phase * normx);
    const double vv = 2.0 * normx * (normx + ax0);    // |x - alpha e1|^2
    sh.v0 = x0 - alpha;
    sh.alpha = alpha;
    // 2 / vv exactly: a power-of-two scaling commutes with rounding
    sh.beta = vv > 0.0 ? 2.0 * __drcp_rn(vv) : 0.0;
    sh.pc = pc;
  }
}

// Phase B of step s (all warps).  Register path: a column is handled by a
// group of GL lanes (32/GL columns per warp per pass), each lane holding
// RPL rows (i = s + lane%GL + GL*r) of the reflector and of its column, so the
// two reductions per column (v^H w, trailing |w|^2) take log2(GL) shuffle
// levels and several columns share every instruction.
template <class T, int GL, int RPL>
__device__ void cpqr_update(T* W, int m, int n, int ld, double* nrm, double* ref, double* xn2,
                            const int* piv, CpqrShared<T>& sh, int s, int kmax) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const T v0 = sh.v0;
  const double beta = sh.beta;
  const int s1 = s + 1;
  const bool renorm = (s1 < kmax) && (s1 % 32 == 0);
  const T* vcol = W + (int64_t)sh.pc * ld;
  double bv = -1.0;
  int bi = 0x7fffffff;
  if constexpr (RPL > 0) {
    constexpr int CPW = 32 / GL;             // columns per warp per pass
    const int g = lane / GL, gl = lane - (lane / GL) * GL;
    T vr[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      int i = s + gl + GL * r;
      vr[r] = (i < m) ? ((r == 0 && gl == 0) ? v0 : vcol[i]) : T(0.0);
    }
    for (int cb = s1 + warp * CPW; cb < n; cb += nw * CPW) {
      const int c = cb + g;
      const bool act = c < n;
      T* wc = W + (int64_t)piv[act ? c : n - 1] * ld;
      T wr[RPL];
      // 4 partial sums break the dependent FMA chains
      T d4[4] = {T(0.0), T(0.0), T(0.0), T(0.0)};
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        int i = s + gl + GL * r;
        wr[r] = (i < m) ? wc[i] : T(0.0);
        d4[r & 3] += sk_conj(vr[r]) * wr[r];
      }
      T dot = (d4[0] + d4[1]) + (d4[2] + d4[3]);
#pragma unroll
      for (int o = GL / 2; o > 0; o >>= 1) dot += shfl_xor_T(dot, o);
      const T f = dot * beta;
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        int i = s + gl + GL * r;
        if (beta != 0.0) wr[r] -= vr[r] * f;
        if (i < m && beta != 0.0 && act) wc[i] = wr[r];
      }
      // downdate; the exact trailing norm is only needed on the rare
      // renormalisation / stale steps (lowrank.py:71-81)
      double t = 0.0;
      int need = 0;
      if (gl == 0 && act) {
        // wr[0] of the group leader is row s of the updated column (R[s, c])
        t = nrm[c] - sk_abs2(wr[0]);
        t = t > 0.0 ? t : 0.0;
        need = (s1 < kmax) && (renorm || t < 1e-8 * ref[c]);
      }
      need = __shfl_sync(0xffffffffu, need, g * GL);
      if (__any_sync(0xffffffffu, need)) {
        double x4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          int i = s + gl + GL * r;
          if (i < m && i > s) x4[r & 3] += sk_abs2(wr[r]);
        }
        double xa = (x4[0] + x4[1]) + (x4[2] + x4[3]);
#pragma unroll
        for (int o = GL / 2; o > 0; o >>= 1) xa += __shfl_xor_sync(0xffffffffu, xa, o);
        if (gl == 0 && need) { t = xa; ref[c] = xa; }
      }
      if (gl == 0 && act) {
        nrm[c] = t;
        cand_merge(bv, bi, t, c);
      }
    }
    warp_cand<GL>(bv, bi);
  } else {
    for (int c = s1 + warp; c < n; c += nw) {
      T* wc = W + (int64_t)piv[c] * ld;
      T dot = T(0.0);
      for (int i = s + lane; i < m; i += SKEL_WARP) {
        T vi = (i == s) ? v0 : vcol[i];
        dot += sk_conj(vi) * wc[i];
      }
      dot = warp_sum(dot);
      const T f = dot * beta;
      double acc = 0.0;
      for (int i = s + lane; i < m; i += SKEL_WARP) {
        T vi = (i == s) ? v0 : vcol[i];
        T nwv = wc[i];
        if (beta != 0.0) {
          nwv -= vi * f;
          wc[i] = nwv;
        }
        if (i > s) acc += sk_abs2(nwv);
      }
      __syncwarp();
      acc = warp_sum(acc);
      const T row = wc[s];
      if (lane == 0) {
        double t = nrm[c] - sk_abs2(row);
        t = t > 0.0 ? t : 0.0;
        if (renorm || t < 1e-8 * ref[c]) { t = acc; ref[c] = acc; }
        nrm[c] = t;
        xn2[c] = acc;
        cand_merge(bv, bi, t, c);
      }
    }
  }
  if (lane == 0) { sh.cand_v[warp] = bv; sh.cand_i[warp] = bi; }
}

// Phase B, real targets, paired-row register path.  Requires an EVEN leading
// dimension whose pad row (row m when m is odd) is zero in every column and a
// 16-byte aligned W.  Lane gl of a GL-lane group holds the row pairs
// {s0 + 2 gl + 2 GL r, +1} (s0 = s rounded down to even, r < RP2) of the
// reflector and of its column, so every shared-memory access is one 16-byte
// LDS/STS per two rows and no per-row predicate is needed: the reflector is
// zero above row s (those rows of the column are left exactly unchanged) and
// the pad row stays zero (0 - 0 f).  Same arithmetic per entry as the
// generic path (dot in four partial chains, one rank-1 update per entry).
template <int GL, int RP2>
__device__ void cpqr_update_pr(double* W, int m, int n, int ld, double* nrm, double* ref,
                               const int* piv, CpqrShared<double>& sh, int s, int kmax) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double v0 = sh.v0;
  const double beta = sh.beta;
  const int s1 = s + 1, s0 = s & ~1;
  const bool renorm = (s1 < kmax) && (s1 % 32 == 0);
  constexpr int CPW = 32 / GL;
  const int g = lane / GL, gl = lane - (lane / GL) * GL;
  const double* vcol = W + (int64_t)sh.pc * ld;
  double2 vr[RP2];
#pragma unroll
  for (int r = 0; r < RP2; ++r) {
    const int i = s0 + 2 * gl + 2 * GL * r;
    vr[r] = (i < m) ? *reinterpret_cast<const double2*>(vcol + i) : make_double2(0.0, 0.0);
  }
  if (gl == 0) {
    // rows s0, s0+1: row s carries v0; an odd s zeroes row s-1 (an R entry)
    if (s & 1) { vr[0].x = 0.0; vr[0].y = v0; } else { vr[0].x = v0; }
  }
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int cb = s1 + warp * CPW; cb < n; cb += nw * CPW) {
    const int c = cb + g;
    const bool act = c < n;
    double* wc = W + (int64_t)piv[act ? c : n - 1] * ld;
    double2 wr[RP2];
    double d4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int r = 0; r < RP2; ++r) {
      const int i = s0 + 2 * gl + 2 * GL * r;
      wr[r] = (i < m) ? *reinterpret_cast<const double2*>(wc + i) : make_double2(0.0, 0.0);
      d4[(2 * r) & 3] += vr[r].x * wr[r].x;
      d4[(2 * r + 1) & 3] += vr[r].y * wr[r].y;
    }
    double dot = (d4[0] + d4[1]) + (d4[2] + d4[3]);
#pragma unroll
    for (int o = GL / 2; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const double f = dot * beta;
#pragma unroll
    for (int r = 0; r < RP2; ++r) {
      const int i = s0 + 2 * gl + 2 * GL * r;
      wr[r].x -= vr[r].x * f;
      wr[r].y -= vr[r].y * f;
      if (i < m && act) *reinterpret_cast<double2*>(wc + i) = wr[r];
    }
    double t = 0.0;
    int need = 0;
    if (gl == 0 && act) {
      const double rs = (s & 1) ? wr[0].y : wr[0].x;     // R[s, c]
      t = nrm[c] - rs * rs;
      t = t > 0.0 ? t : 0.0;
      need = (s1 < kmax) && (renorm || t < 1e-8 * ref[c]);
    }
    need = __shfl_sync(0xffffffffu, need, g * GL);
    if (__any_sync(0xffffffffu, need)) {
      double x4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int r = 0; r < RP2; ++r) {
        const int i = s0 + 2 * gl + 2 * GL * r;
        if (i > s) x4[(2 * r) & 3] += wr[r].x * wr[r].x;
        if (i + 1 > s) x4[(2 * r + 1) & 3] += wr[r].y * wr[r].y;
      }
      double xa = (x4[0] + x4[1]) + (x4[2] + x4[3]);
#pragma unroll
      for (int o = GL / 2; o > 0; o >>= 1) xa += __shfl_xor_sync(0xffffffffu, xa, o);
      if (gl == 0 && need) { t = xa; ref[c] = xa; }
    }
    if (gl == 0 && act) {
      nrm[c] = t;
      cand_merge(bv, bi, t, c);
    }
  }
  warp_cand<GL>(bv, bi);
  if (lane == 0) { sh.cand_v[warp] = bv; sh.cand_i[warp] = bi; }
}

template <class T, int GL, int RPL>
__device__ __forceinline__ void cpqr_update_any(T* W, int m, int n, int ld, double* nrm, double* ref,
                                                double* xn2, const int* piv, CpqrShared<T>& sh, int s,
                                                int kmax) {
  if constexpr (sizeof(T) == sizeof(double) && RPL > 0 && (RPL & 1) == 0)
    cpqr_update_pr<GL, RPL / 2>(W, m, n, ld, nrm, ref, piv, sh, s, kmax);
  else
    cpqr_update<T, GL, RPL>(W, m, n, ld, nrm, ref, xn2, piv, sh, s, kmax);
}

// Run CPQR steps from sh.rank until the stop rule (with min_rank) fires.
// For real targets with an even register tile (RPL even) the paired-row path
// runs, which needs the even-ld / zero-pad-row layout (cpqr_ld()).
// `kcap` (equalisation only) ends the run after exactly kcap steps: the
// reference re-runs the smaller side with min_rank = k and normally stops
// right at k, but a stale-norm recomputation can lift the next trailing
// pivot back above eps*p0 and carry it past k -- which would leave the box
// non-square and make factor() fail (solver.py:200-203).  Capping at k keeps
// every equalised box square; it differs from the reference only where the
// reference itself would fail.
template <class T, int GL, int RPL>
__device__ void cpqr_run(T* W, int m, int n, int ld, double* nrm, double* ref, double* xn2,
                         int* piv, CpqrShared<T>& sh, double eps, int min_rank,
                         int kcap = 0x7fffffff) {
  const int kmax = m < n ? m : n;
  const int kend = kmax < kcap ? kmax : kcap;
  const int nw = blockDim.x >> 5;
  int s = sh.rank;
  while (s < kend) {
    if (threadIdx.x < 32)
      cpqr_pivot<T>(W, m, n, ld, nrm, RPL == 0 ? xn2 : nullptr, piv, sh, s, eps, min_rank, nw);
    __syncthreads();
    if (sh.stop) break;
    cpqr_update_any<T, GL, RPL>(W, m, n, ld, nrm, ref, xn2, piv, sh, s, kmax);
    if (threadIdx.x == 0) {
      W[(int64_t)sh.pc * ld + s] = sh.alpha;
      sh.rank = s + 1;
    }
    __syncthreads();
    ++s;
  }
  __syncthreads();
}

// X = R11^-1 R12 in place (positions r..n-1, rows 0..r-1), one thread per
// column, column-oriented back substitution (dtrsm order).  Also pads to
// min_rank and records max|P|.
template <class T>
__device__ void interp_solve(T* W, int n, int ld, const int* piv, CpqrShared<T>& sh, int min_rank,
                             double* red) {
  const int r = sh.rank;
  double big = 0.0;
  for (int c = r + threadIdx.x; c < n; c += blockDim.x) {
    T* x = W + (int64_t)piv[c] * ld;
    for (int s = r - 1; s >= 0; --s) {
      T xs = x[s];
      if (xs != T(0.0)) {
        const T* rs = W + (int64_t)piv[s] * ld;   // R[:, s]
        xs = xs / rs[s];
        x[s] = xs;
        for (int t = 0; t < s; ++t) x[t] -= rs[t] * xs;
      }
    }
    for (int s = 0; s < r; ++s) big = fmax(big, sk_abs(x[s]));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) big = fmax(big, __shfl_xor_sync(0xffffffffu, big, o));
  if (lane == 0) red[warp] = big;
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < nw; ++w) b = fmax(b, red[w]);
    if (r > 0) b = fmax(b, 1.0);
    sh.bigP = b;
    int kmin = min_rank < n ? min_rank : n;
    sh.pad = (r < kmin) ? kmin - r : 0;
  }
  __syncthreads();
}

// Entry P(s, q) of the interpolation matrix for pivot POSITION q (column
// piv[q] of the target), row s (pivot order), after interp_solve.
template <class T>
__device__ __forceinline__ T interp_entry(const T* W, int ld, const int* piv, int r, int kfin, int s,
                                          int q) {
  if (q < kfin) return (s == q) ? T(1.0) : T(0.0);
  return (s < r) ? W[(int64_t)piv[q] * ld + s] : T(0.0);
}
