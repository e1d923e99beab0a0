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
// GPU mapping: warp 0 runs the serial part of a step (argmax, swap,
// Householder vector); then every warp owns a strided set of trailing
// columns and, per column, computes v^H w, applies the reflector and
// downdates that column's norm -- fusing the next step's renormalisation /
// stale checks into the same pass so a step costs two CTA barriers.
// With RPL > 0 the reflector and the column slice live in registers
// (RPL = max rows per lane), so each element is read and written once.
#pragma once

#include "common.cuh"

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
  double bigP;   // max |P| (interp quality warning, lowrank.py:128-132)
};

__device__ __forceinline__ double sk_unit_phase(double x0, double) { return x0 > 0.0 ? 1.0 : -1.0; }
__device__ __forceinline__ zc sk_unit_phase(zc x0, double a) { return zc(x0.re / a, x0.im / a); }

// squared norm of rows [r0, m) of column c, warp-cooperative
template <class T>
__device__ __forceinline__ double col_norm2(const T* W, int ld, int c, int r0, int m, int lane) {
  double s = 0.0;
  for (int i = r0 + lane; i < m; i += SKEL_WARP) s += sk_abs2(W[(int64_t)c * ld + i]);
  return warp_sum(s);
}

// Initial exact norms (all rows), nrm = ref (lowrank.py:55-64).
template <class T>
__device__ void cpqr_init(const T* W, int m, int n, int ld, double* nrm, double* ref, int* piv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < n; c += nw) {
    double s = col_norm2(W, ld, c, 0, m, lane);
    if (lane == 0) {
      nrm[c] = s;
      ref[c] = s;
    }
  }
  for (int c = threadIdx.x; c < n; c += blockDim.x) piv[c] = c;
}

// Serial part of step s on warp 0.  Returns via sh.
template <class T>
__device__ void cpqr_pivot_step(T* W, int m, int n, int ld, double* nrm, int* piv,
                                CpqrShared<T>& sh, int s, double eps, int min_rank) {
  const int lane = threadIdx.x & 31;
  // first maximum of nrm[s:]
  double best = -1.0;
  int bj = n;
  for (int c = s + lane; c < n; c += SKEL_WARP) {
    double v = nrm[c];
    if (v > best) { best = v; bj = c; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, best, o);
    int oj = __shfl_xor_sync(0xffffffffu, bj, o);
    if (ov > best || (ov == best && oj < bj)) { best = ov; bj = oj; }
  }
  double pn = sqrt(fmax(best, 0.0));
  int stop = 0;
  if (s == 0) {
    if (lane == 0) sh.p0 = pn;
    if (pn == 0.0) stop = 1;
  }
  double p0 = (s == 0) ? pn : sh.p0;
  if (!stop && s >= min_rank && pn <= eps * p0) stop = 1;
  if (!stop && pn == 0.0) stop = 1;
  if (stop) {
    if (lane == 0) sh.stop = 1;
    return;
  }
  if (bj != s) {
    for (int i = lane; i < m; i += SKEL_WARP) {
      T a = W[(int64_t)s * ld + i];
      W[(int64_t)s * ld + i] = W[(int64_t)bj * ld + i];
      W[(int64_t)bj * ld + i] = a;
    }
    if (lane == 0) {
      double t = nrm[s]; nrm[s] = nrm[bj]; nrm[bj] = t;
      int p = piv[s]; piv[s] = piv[bj]; piv[bj] = p;
    }
  }
  __syncwarp();
  // Householder vector of x = W[s:, s]
  double s1 = 0.0;
  for (int i = s + 1 + lane; i < m; i += SKEL_WARP) s1 += sk_abs2(W[(int64_t)s * ld + i]);
  s1 = warp_sum(s1);
  if (lane == 0) {
    T x0 = W[(int64_t)s * ld + s];
    double ax0 = sk_abs(x0);
    double normx = sqrt(s1 + sk_abs2(x0));
    T phase = T(1.0);
    if (ax0 != 0.0) phase = sk_unit_phase(x0, ax0);   // x0 / |x0|
    T alpha = -(phase * normx);
    T v0 = x0 - alpha;
    double vv = s1 + sk_abs2(v0);
    sh.v0 = v0;
    sh.alpha = alpha;
    sh.beta = vv > 0.0 ? 2.0 / vv : 0.0;
    sh.stop = 0;
  }
}

// Parallel part of step s: apply the reflector to columns s+1..n-1, downdate
// norms, and run step s+1's renormalisation / stale recompute.
template <class T, int RPL>
__device__ void cpqr_update(T* W, int m, int n, int ld, double* nrm, double* ref,
                            const CpqrShared<T>& sh, int s, int kmax) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const T v0 = sh.v0;
  const double beta = sh.beta;
  const int s1 = s + 1;
  const bool renorm = (s1 < kmax) && (s1 % 32 == 0);
  const bool check = (s1 < kmax);
  const T* vcol = W + (int64_t)s * ld;
  if constexpr (RPL > 0) {
    T vr[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
      int i = s + lane + SKEL_WARP * r;
      vr[r] = (i < m) ? ((r == 0 && lane == 0) ? v0 : vcol[i]) : T(0.0);
    }
    for (int c = s1 + warp; c < n; c += nw) {
      T* wc = W + (int64_t)c * ld;
      T wr[RPL];
      T dot = T(0.0);
#pragma unroll
      for (int r = 0; r < RPL; ++r) {
        int i = s + lane + SKEL_WARP * r;
        wr[r] = (i < m) ? wc[i] : T(0.0);
        dot += sk_conj(vr[r]) * wr[r];
      }
      dot = warp_sum(dot);
      if (beta != 0.0) {
        T f = dot * beta;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          int i = s + lane + SKEL_WARP * r;
          if (i < m) {
            wr[r] -= vr[r] * f;
            wc[i] = wr[r];
          }
        }
      }
      T row = shfl(wr[0], 0);
      double nv = 0.0;
      if (check) {
        double acc = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
          int i = s + lane + SKEL_WARP * r;
          if (i < m && i > s) acc += sk_abs2(wr[r]);
        }
        nv = acc;  // reduced lazily below (only if needed)
      }
      if (lane == 0) {
        double t = nrm[c] - sk_abs2(row);
        nrm[c] = t > 0.0 ? t : 0.0;
      }
      __syncwarp();
      if (check) {
        bool need = renorm || (nrm[c] < 1e-8 * ref[c]);
        if (need) {
          double full = warp_sum(nv);
          if (lane == 0) { nrm[c] = full; ref[c] = full; }
        }
      }
      __syncwarp();
    }
  } else {
    for (int c = s1 + warp; c < n; c += nw) {
      T* wc = W + (int64_t)c * ld;
      T dot = T(0.0);
      for (int i = s + lane; i < m; i += SKEL_WARP) {
        T vi = (i == s) ? v0 : vcol[i];
        dot += sk_conj(vi) * wc[i];
      }
      dot = warp_sum(dot);
      double acc = 0.0;
      T row = wc[s];
      if (beta != 0.0) {
        T f = dot * beta;
        for (int i = s + lane; i < m; i += SKEL_WARP) {
          T vi = (i == s) ? v0 : vcol[i];
          T nwv = wc[i] - vi * f;
          wc[i] = nwv;
          if (i > s) acc += sk_abs2(nwv);
        }
        __syncwarp();
        row = wc[s];
      } else {
        for (int i = s + 1 + lane; i < m; i += SKEL_WARP) acc += sk_abs2(wc[i]);
      }
      if (lane == 0) {
        double t = nrm[c] - sk_abs2(row);
        nrm[c] = t > 0.0 ? t : 0.0;
      }
      __syncwarp();
      if (check) {
        bool need = renorm || (nrm[c] < 1e-8 * ref[c]);
        if (need) {
          double full = warp_sum(acc);
          if (lane == 0) { nrm[c] = full; ref[c] = full; }
        }
      }
      __syncwarp();
    }
  }
}

// Run CPQR steps from sh.rank until the stop rule (with min_rank) fires.
template <class T, int RPL>
__device__ void cpqr_run(T* W, int m, int n, int ld, double* nrm, double* ref, int* piv,
                         CpqrShared<T>& sh, double eps, int min_rank) {
  const int kmax = m < n ? m : n;
  const int warp = threadIdx.x >> 5;
  int s = sh.rank;
  while (s < kmax) {
    if (warp == 0) cpqr_pivot_step<T>(W, m, n, ld, nrm, piv, sh, s, eps, min_rank);
    __syncthreads();
    if (sh.stop) break;
    cpqr_update<T, RPL>(W, m, n, ld, nrm, ref, sh, s, kmax);
    if (threadIdx.x == 0) {
      W[(int64_t)s * ld + s] = sh.alpha;
      sh.rank = s + 1;
    }
    __syncthreads();
    ++s;
  }
  __syncthreads();
}

// X = R11^-1 R12 in place (columns r..n-1, rows 0..r-1), one thread per
// column, column-oriented back substitution (dtrsm order).  Also pads to
// min_rank and records max|P|.
template <class T>
__device__ void interp_solve(T* W, int n, int ld, CpqrShared<T>& sh, int min_rank,
                             double* red) {
  const int r = sh.rank;
  double big = 0.0;
  for (int c = r + threadIdx.x; c < n; c += blockDim.x) {
    T* x = W + (int64_t)c * ld;
    for (int s = r - 1; s >= 0; --s) {
      T xs = x[s];
      if (xs != T(0.0)) {
        xs = xs / W[(int64_t)s * ld + s];
        x[s] = xs;
        for (int t = 0; t < s; ++t) x[t] -= W[(int64_t)s * ld + t] * xs;
      }
    }
    for (int s = 0; s < r; ++s) big = fmax(big, sk_abs(x[s]));
  }
  // block max
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
// piv[q] of the original target), row s (pivot order), after interp_solve.
template <class T>
__device__ __forceinline__ T interp_entry(const T* W, int ld, int r, int kfin, int s, int q) {
  if (q < kfin) return (s == q) ? T(1.0) : T(0.0);
  return (s < r) ? W[(int64_t)q * ld + s] : T(0.0);
}
