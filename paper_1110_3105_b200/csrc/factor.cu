// factor.cu -- K3 + K4: batched per-box telescoping factorization and the
// dense top-level inverse.
//
// Reference work replaced: factor / factor_node (solver.py:187-276), the
// per-box LAPACK getrf/getrs calls (solver.py:210,243,252-256), _rcond1
// (solver.py:179-184) and the top `_lu(Shat)` (solver.py:269-274).
//
// One CTA per box; every operand of the box lives in shared memory:
//   A  (n x n)  D_eff -> D^-1 (Gauss-Jordan, partial pivoting) -> Dd
//   Lb (n x k)  L -> Ld = X Lam
//   Rb (k x n)  R -> Rd = Lam RD
//   X  (n x k)  D^-1 L
//   Y  (k x n)  R D^-1
//   M  (k x k)  R X -> Lam = M^-1
// Gauss-Jordan with row pivoting chooses the same pivots as getrf (the rows
// below the diagonal see the same Schur complements), so exact-zero pivots
// (SingularBlock, solver.py:211-212) are detected identically.
#include "common.cuh"

template <class T>
__device__ __forceinline__ void cp_async_block_one(T* dst, const T* src) {
  constexpr int W = sizeof(T) / 8;
#pragma unroll
  for (int w = 0; w < W; ++w)
    cp_async8(reinterpret_cast<double*>(dst) + w, reinterpret_cast<const double*>(src) + w);
}

// 1/x correctly rounded (the reciprocal is the only division of a GJ step)
__device__ __forceinline__ double fac_recip(double x) { return __drcp_rn(x); }
__device__ __forceinline__ zc fac_recip(zc x) { return zc(1.0) / x; }

// first-maximum merge (ties -> lower index), LAPACK i?amax order
__device__ __forceinline__ void fac_cmerge(double& bv, int& bi, double ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
}
#define cmerge fac_cmerge

template <class T>
struct FacShared {
  int status;
  int piv_row;
  double amax;
  double red[32];
  int red_i[32];
};

// 1-norm (max column abs sum) of a row-major p x q matrix
template <class T>
__device__ double sm_norm1(const T* A, int lda, int p, int q, FacShared<T>& sh) {
  double best = 0.0;
  for (int j = threadIdx.x; j < q; j += blockDim.x) {
    double s = 0.0;
    for (int i = 0; i < p; ++i) s += sk_abs(A[(int64_t)i * lda + j]);
    best = fmax(best, s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = best;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, sh.red[w]);
  __syncthreads();
  return r;
}

// In-place Gauss-Jordan inverse of a row-major p x p matrix with partial
// pivoting (pivot = first maximum |a| as LAPACK's i?amax).  Two barriers per
// step: warp 0 finds the pivot and stages the pivot column and the two rows
// being exchanged; then every thread updates an independent (row, column)
// tile (row exchange, scaling and elimination fused).
// scratch: 3p entries (colk, rowp, rowk), ipiv: p ints.  Returns 1 on an
// exactly zero pivot (SingularBlock).
template <class T>
__device__ int sm_invert(T* A, int lda, int p, T* scratch, int* ipiv, FacShared<T>& sh) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  T* colk = scratch;
  T* rowp = scratch + p;
  T* rowk = scratch + 2 * p;
  for (int kk = 0; kk < p; ++kk) {
    if (warp == 0) {
      double best = -1.0;
      int bi = p;
      for (int i = kk + lane; i < p; i += 32) {
        double v = sk_pivabs(A[(int64_t)i * lda + kk]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (best > 0.0) {
        const int pr = bi;
        const T inv = T(1.0) / A[(int64_t)pr * lda + kk];
        for (int i = lane; i < p; i += 32) {
          // pivot column after the exchange of rows kk and pr
          colk[i] = (i == pr) ? A[(int64_t)kk * lda + kk] : A[(int64_t)i * lda + kk];
        }
        __syncwarp();
        for (int j = lane; j < p; j += 32) {
          // the scaled pivot row (its column kk holds 1/pivot), and the
          // exchange done in place: row pr takes old row kk
          const T vp = A[(int64_t)pr * lda + j];
          const T vk = A[(int64_t)kk * lda + j];
          rowp[j] = (j == kk) ? inv : vp * inv;
          if (pr != kk) A[(int64_t)pr * lda + j] = vk;
        }
      }
      if (lane == 0) {
        sh.piv_row = bi;
        sh.amax = best;
        ipiv[kk] = bi;
      }
    }
    __syncthreads();
    if (sh.amax == 0.0) return 1;
    // eliminate column kk everywhere (rows already exchanged, pivot row
    // scaled in rowp with 1/pivot in its column kk): a_ij -= a_ik * r_j, and
    // column kk becomes -a_ik / pivot (in-place inverse)
    {
      // flat (row, column) walk: every thread gets ~p^2 / nt elements
      const int di = nt / p, dj = nt - (nt / p) * p;
      int i = tid / p, j = tid - (tid / p) * p;
      for (int e = tid; e < p * p; e += nt) {
        T* Aij = A + (int64_t)i * lda + j;
        const T r = rowp[j];
        if (i == kk) {
          *Aij = r;
        } else {
          const T a = (j == kk) ? T(0.0) : *Aij;
          *Aij = a - colk[i] * r;
        }
        i += di;
        j += dj;
        if (j >= p) { j -= p; ++i; }
      }
    }
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, last first: rows are
  // independent, so each thread replays the whole sequence on its own rows
  // (one barrier instead of one per column)
  for (int i = tid; i < p; i += nt) {
    T* Ai = A + (int64_t)i * lda;
    for (int kk = p - 1; kk >= 0; --kk) {
      const int pr = ipiv[kk];
      if (pr != kk) {
        const T t = Ai[kk];
        Ai[kk] = Ai[pr];
        Ai[pr] = t;
      }
    }
  }
  __syncthreads();
  return 0;
}

// Gauss-Jordan inverse, same pivots and the same per-entry arithmetic as
// sm_invert (bit-identical result), restructured so no step has a
// single-warp serial phase:
//   (1) every thread merges the per-warp pivot candidates of column kk
//       (written during the previous step's elimination) and forms 1/pivot;
//   (2) all threads stage the scaled pivot row, the old row kk (it moves to
//       row pr) and column kk after the exchange;            -- barrier
//   (3) warp w eliminates rows i = w (mod warps), lanes over columns (the
//       pivot row in CPL registers per lane), the lane that owns column kk+1
//       folds the new |a_i,kk+1| (rows > kk) into the warp's candidate for
//       the next step.                                          -- barrier
// Two barriers per step as before, but the pivot search rides on the
// elimination and the row exchange is a staged copy (no warp-0 column scan,
// no flat (i, j) index walk).  p <= 32 * CPL.
template <class T, int CPL>
__device__ int sm_invert_rows(T* A, int lda, int p, T* scratch, int* ipiv, FacShared<T>& sh) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  T* rowp = scratch;
  T* rowk = scratch + p;
  T* colk = scratch + 2 * p;
  {
    double bv = -1.0;
    int bi = p;
    for (int i = tid; i < p; i += nt) cmerge(bv, bi, sk_pivabs(A[(int64_t)i * lda]), i);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      cmerge(bv, bi, ov, oi);
    }
    if (lane == 0) { sh.red[warp] = bv; sh.red_i[warp] = bi; }
  }
  __syncthreads();
  for (int kk = 0; kk < p; ++kk) {
    // per-warp candidates: lanes < nw load one each, a log2(nw)-round
    // butterfly, then lane 0's result is broadcast (warp-uniform pivot)
    double best = -1.0;
    int pr = p;
    if (lane < nw) { best = sh.red[lane]; pr = sh.red_i[lane]; }
    for (int o = 1; o < nw; o <<= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, pr, o);
      cmerge(best, pr, ov, oi);
    }
    best = __shfl_sync(0xffffffffu, best, 0);
    pr = __shfl_sync(0xffffffffu, pr, 0);
    if (!(best > 0.0) || pr >= p) return 1;          // exact zero pivot (uniform)
    const T inv = fac_recip(A[(int64_t)pr * lda + kk]);
    const T akk = A[(int64_t)kk * lda + kk];
    for (int j = tid; j < p; j += nt) {
      const T vp = A[(int64_t)pr * lda + j];
      rowp[j] = (j == kk) ? inv : vp * inv;
      rowk[j] = A[(int64_t)kk * lda + j];
      colk[j] = (j == pr) ? akk : A[(int64_t)j * lda + kk];
    }
    if (tid == 0) ipiv[kk] = pr;
    __syncthreads();
    T rp[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
      const int j = lane + 32 * c;
      rp[c] = j < p ? rowp[j] : T(0.0);
    }
    const int jn = kk + 1;
    double bv = -1.0;
    int bi = p;
    for (int i = warp; i < p; i += nw) {
      T* Ai = A + (int64_t)i * lda;
      if (i == kk) {
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
          const int j = lane + 32 * c;
          if (j < p) Ai[j] = rp[c];
        }
        continue;
      }
      const T* src = (i == pr) ? rowk : Ai;
      const T f = colk[i];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int j = lane + 32 * c;
        if (j < p) {
          const T a = (j == kk) ? T(0.0) : src[j];
          Ai[j] = a - f * rp[c];
        }
      }
      // the owner lane of column kk+1 re-reads its own fresh store
      if (lane == (jn & 31) && jn < p && i > kk) cmerge(bv, bi, sk_pivabs(Ai[jn]), i);
    }
    if (jn < p && lane == (jn & 31)) { sh.red[warp] = bv; sh.red_i[warp] = bi; }
    __syncthreads();
  }
  for (int i = tid; i < p; i += nt) {
    T* Ai = A + (int64_t)i * lda;
    for (int kk = p - 1; kk >= 0; --kk) {
      const int pr = ipiv[kk];
      if (pr != kk) {
        const T t = Ai[kk];
        Ai[kk] = Ai[pr];
        Ai[pr] = t;
      }
    }
  }
  __syncthreads();
  return 0;
}

template <class T>
__device__ int sm_invert_any(T* A, int lda, int p, T* scratch, int* ipiv, FacShared<T>& sh) {
  if (p <= 32) return sm_invert_rows<T, 1>(A, lda, p, scratch, ipiv, sh);
  if (p <= 64) return sm_invert_rows<T, 2>(A, lda, p, scratch, ipiv, sh);
  if (p <= 96) return sm_invert_rows<T, 3>(A, lda, p, scratch, ipiv, sh);
  if (p <= 128) return sm_invert_rows<T, 4>(A, lda, p, scratch, ipiv, sh);
  return sm_invert<T>(A, lda, p, scratch, ipiv, sh);
}

// Top-level variant (k_dense_inverse only -- instantiating these in k_factor_level costs
// that kernel 5-12 % through its 64-register cap): real blocks that still fit shared memory
// (p <= 168: the 2^20 top level, K = 160) also take the row-parallel elimination; same
// pivots and arithmetic, 0.88 -> 0.64 ms at K = 160.  Wider blocks run out of a global
// scratch slab, where the flat walk of sm_invert is the faster one.
template <class T>
__device__ int sm_invert_top(T* A, int lda, int p, T* scratch, int* ipiv, FacShared<T>& sh) {
  if constexpr (sizeof(T) == sizeof(double)) {
    if (p > 128 && p <= 160) return sm_invert_rows<T, 5>(A, lda, p, scratch, ipiv, sh);
    if (p > 160 && p <= 168) return sm_invert_rows<T, 6>(A, lda, p, scratch, ipiv, sh);
  }
  return sm_invert_any<T>(A, lda, p, scratch, ipiv, sh);
}

// ---------------------------------------------------------------------------
// Register-resident Gauss-Jordan inverse with panel look-ahead (real blocks,
// 8-warp CTAs, p <= 32 * RPL and p <= 8 * CW).  Same pivots and the same
// per-entry arithmetic as sm_invert / sm_invert_rows (a - f * r with the
// scaled pivot row, 1/pivot by __drcp_rn): the result is bit-identical.
//
// Layout: warp w owns the CW contiguous columns [w CW, (w+1) CW), lane l the
// rows l, l + 32, ...: the whole matrix lives in registers (RPL x CW doubles
// per thread) for the duration of the inversion.  A Gauss-Jordan step needs,
// besides a warp's own columns, only the pivot row index and column kk (the
// multipliers): the warp that owns a panel of CW columns therefore runs its
// CW steps ALONE, ahead of everybody (pivot search by a warp butterfly, pivot
// row entries by shuffles: no shared memory, no CTA barrier), publishing per
// step the pivot row index and the raw column kk; after one barrier the other
// seven warps replay the CW steps on their own columns.  Two CTA barriers per
// CW steps instead of two per step, no per-step shared-memory traffic for the
// matrix, and the row exchange is a register patch on two lanes.
//   pubf: CW * p doubles (raw column kk of each step of the current panel)
//   sh.red_i[u]: pivot row of step u; sh.piv_row < 0: exact zero pivot
// One Gauss-Jordan step on a warp's own columns.  UO >= 0: this warp owns
// column kk = column slot UO of its tile (compile-time), fr = that column.
// KS / PS: register slots (row / 32) of rows kk and pr, compile-time so the
// two special rows are patched with two predicated moves per column (PS < 0:
// pr == kk, no exchange): row kk <- r, row pr <- old row kk - akk r (the
// exchange of sm_invert); every other entry is t - f r.
template <int RPL, int CW, int UO, int KS, int PS>
__device__ __forceinline__ void gj_la_step_v(double (&t)[RPL][CW], int lane, int kk, int pr,
                                             const double (&fr)[RPL], double pivv, double akk) {
  const double inv = fac_recip(pivv);
  const bool isk = lane == (kk & 31);
  const bool isp = PS >= 0 && lane == (pr & 31);
#pragma unroll
  for (int c = 0; c < CW; ++c) {
    const double vp = __shfl_sync(0xffffffffu, t[PS >= 0 ? PS : KS][c], pr & 31);   // A[pr][j]
    const double rp = (c == UO) ? inv : vp * inv;
    double pv = 0.0;
    if constexpr (PS >= 0) {
      double vk = __shfl_sync(0xffffffffu, t[KS][c], kk & 31);                       // A[kk][j]
      if (c == UO) vk = 0.0;
      pv = vk - akk * rp;                                      // row pr after the exchange
    }
#pragma unroll
    for (int a = 0; a < RPL; ++a) {
      const double aa = (c == UO) ? 0.0 : t[a][c];
      t[a][c] = aa - fr[a] * rp;
    }
    if constexpr (PS >= 0) {
      if (isp) t[PS][c] = pv;
    }
    if (isk) t[KS][c] = rp;
  }
}

template <int RPL, int CW, int UO>
__device__ __forceinline__ void gj_la_step(double (&t)[RPL][CW], int lane, int kk, int pr,
                                           const double (&fr)[RPL], double pivv, double akk) {
  // kk, pr are CTA-uniform: the slot dispatch is a uniform branch
  if constexpr (RPL == 1) {
    if (pr == kk) gj_la_step_v<RPL, CW, UO, 0, -1>(t, lane, kk, pr, fr, pivv, akk);
    else gj_la_step_v<RPL, CW, UO, 0, 0>(t, lane, kk, pr, fr, pivv, akk);
  } else {
    static_assert(RPL <= 2, "slot dispatch covers two row slots");
    const int ks = kk >> 5, ps = pr >> 5;
    if (pr == kk) {
      if (ks == 0) gj_la_step_v<RPL, CW, UO, 0, -1>(t, lane, kk, pr, fr, pivv, akk);
      else gj_la_step_v<RPL, CW, UO, 1, -1>(t, lane, kk, pr, fr, pivv, akk);
    } else if (ks == 0) {
      if (ps == 0) gj_la_step_v<RPL, CW, UO, 0, 0>(t, lane, kk, pr, fr, pivv, akk);
      else gj_la_step_v<RPL, CW, UO, 0, 1>(t, lane, kk, pr, fr, pivv, akk);
    } else {
      // pr >= kk >= 32: both rows live in slot 1
      gj_la_step_v<RPL, CW, UO, 1, 1>(t, lane, kk, pr, fr, pivv, akk);
    }
  }
}

// Pivot search of one column held one row per (lane, slot): first maximum of
// |x| over rows kk <= i < p (LAPACK i?amax order), by two 32-bit warp
// reductions on the bit pattern of |x| (monotone for non-negative doubles)
// and a ballot for the lowest row.  Returns p when the column is exactly zero
// (or all NaN, which the comparison-based search never selects either).
template <int RPL>
__device__ __forceinline__ int gj_la_pivot(const double (&col)[RPL], int lane, int kk, int p) {
  unsigned long long key = 0ull;
  int slot = 0;
#pragma unroll
  for (int a = 0; a < RPL; ++a) {
    const int i = lane + 32 * a;
    const double v = fabs(col[a]);
    unsigned long long k = (i >= kk && i < p && v == v) ? (unsigned long long)__double_as_longlong(v) : 0ull;
    if (k > key) { key = k; slot = a; }
  }
  const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
  const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
  const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
  if ((mh | ml) == 0u) return p;
  const bool hit = hi == mh && lo == ml;
  int best = p;
#pragma unroll
  for (int a = 0; a < RPL; ++a) {
    const unsigned b = __ballot_sync(0xffffffffu, hit && slot == a);
    if (best == p && b) best = 32 * a + (__ffs(b) - 1);
  }
  return best;
}

// The panel owner's CW steps, unrolled at compile time (the pivot column of
// step U is column slot U of the owner's tile).
template <int RPL, int CW, int U>
__device__ __forceinline__ void gj_la_owner(double (&t)[RPL][CW], int lane, int kk0, int nst, int p,
                                            double* pubf, int* ipiv, FacShared<double>& sh) {
  if constexpr (U < CW) {
    if (U >= nst) return;
    const int kk = kk0 + U;
    double col[RPL];
#pragma unroll
    for (int a = 0; a < RPL; ++a) col[a] = t[a][U];
    const int pr = gj_la_pivot<RPL>(col, lane, kk, p);
    if (pr >= p) {                                  // exact zero pivot (warp-uniform)
      if (lane == 0) sh.piv_row = -1;
      return;
    }
#pragma unroll
    for (int a = 0; a < RPL; ++a) {
      const int i = lane + 32 * a;
      if (i < p) pubf[U * p + i] = col[a];
    }
    if (lane == 0) { sh.red_i[U] = pr; ipiv[kk] = pr; }
    // pivot and old diagonal entry of column kk, from their owner lanes
    double psel = col[0], ksel = col[0];
#pragma unroll
    for (int a = 1; a < RPL; ++a) {
      psel = (a == (pr >> 5)) ? col[a] : psel;
      ksel = (a == (kk >> 5)) ? col[a] : ksel;
    }
    const double pivv = __shfl_sync(0xffffffffu, psel, pr & 31);
    const double akk = __shfl_sync(0xffffffffu, ksel, kk & 31);
    gj_la_step<RPL, CW, U>(t, lane, kk, pr, col, pivv, akk);
    gj_la_owner<RPL, CW, U + 1>(t, lane, kk0, nst, p, pubf, ipiv, sh);
  }
}

template <int RPL, int CW>
__device__ int sm_invert_la(double* A, int lda, int p, double* pubf, int* ipiv, FacShared<double>& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int j0 = warp * CW;
  double t[RPL][CW];
#pragma unroll
  for (int a = 0; a < RPL; ++a) {
    const int i = lane + 32 * a;
#pragma unroll
    for (int c = 0; c < CW; ++c)
      t[a][c] = (i < p && j0 + c < p) ? A[(int64_t)i * lda + j0 + c] : 0.0;
  }
  if (tid == 0) sh.piv_row = 0;
  __syncthreads();
  const int npanel = (p + CW - 1) / CW;
  for (int P = 0; P < npanel; ++P) {
    const int kk0 = P * CW;
    const int nst = (p - kk0) < CW ? (p - kk0) : CW;
    if (warp == P) gj_la_owner<RPL, CW, 0>(t, lane, kk0, nst, p, pubf, ipiv, sh);
    __syncthreads();
    if (sh.piv_row < 0) return 1;
    if (warp != P) {
      for (int u = 0; u < nst; ++u) {
        const int kk = kk0 + u;
        const int pr = sh.red_i[u];
        const double* fu = pubf + u * p;
        double fr[RPL];
#pragma unroll
        for (int a = 0; a < RPL; ++a) {
          const int i = lane + 32 * a;
          fr[a] = i < p ? fu[i] : 0.0;
        }
        gj_la_step<RPL, CW, -1>(t, lane, kk, pr, fr, fu[pr], fu[kk]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < RPL; ++a) {
    const int i = lane + 32 * a;
#pragma unroll
    for (int c = 0; c < CW; ++c)
      if (i < p && j0 + c < p) A[(int64_t)i * lda + j0 + c] = t[a][c];
  }
  __syncthreads();
  // undo the row interchanges as column interchanges, last first
  for (int i = tid; i < p; i += blockDim.x) {
    double* Ai = A + (int64_t)i * lda;
    for (int kk = p - 1; kk >= 0; --kk) {
      const int pr = ipiv[kk];
      if (pr != kk) {
        const double tt = Ai[kk];
        Ai[kk] = Ai[pr];
        Ai[pr] = tt;
      }
    }
  }
  __syncthreads();
  return 0;
}

// pub_cap: doubles available at `pub` for the look-ahead path (0 = use the
// barrier-per-step kernels with the 3p scratch)
template <class T>
__device__ int sm_invert_fast(T* A, int lda, int p, T* scratch, T* pub, int64_t pub_cap, int* ipiv,
                              FacShared<T>& sh) {
  if constexpr (sizeof(T) == sizeof(double)) {
    if (blockDim.x == 256) {
      if (p <= 32 && pub_cap >= 4 * (int64_t)p)
        return sm_invert_la<1, 4>(reinterpret_cast<double*>(A), lda, p, reinterpret_cast<double*>(pub),
                                  ipiv, sh);
      if (p <= 64 && pub_cap >= 8 * (int64_t)p)
        return sm_invert_la<2, 8>(reinterpret_cast<double*>(A), lda, p, reinterpret_cast<double*>(pub),
                                  ipiv, sh);
    }
  }
  return sm_invert_any<T>(A, lda, p, scratch, ipiv, sh);
}

// C (p x q) = [C -] A (p x r) B (r x q), row-major in shared memory, on the
// FP64 tensor pipe: each warp owns 8 x 8 output tiles and runs the k-loop as
// mma.sync.m8n8k4.f64 (A fragment A[i0+g][k0+t], B fragment B[k0+t][j0+g],
// accumulator C[i0+g][j0+2t .. +1]); edges are zero-filled in the fragment
// loads, so p, q, r need no padding.
__device__ __forceinline__ void fac_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool SUB>
__device__ void sm_gemm_dmma(double* C, int ldc, const double* A, int lda, const double* B, int ldb,
                             int p, int q, int r) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int tp = (p + 7) >> 3, tq = (q + 7) >> 3;
  for (int tile = warp; tile < tp * tq; tile += nw) {
    const int i0 = (tile / tq) * 8, j0 = (tile % tq) * 8;
    const int ia = i0 + g, jb = j0 + g;
    double d0 = 0.0, d1 = 0.0;
    const double* ar = A + (int64_t)(ia < p ? ia : 0) * lda;
    for (int k0 = 0; k0 < r; k0 += 4) {
      const int k = k0 + t;
      const double av = (ia < p && k < r) ? ar[k] : 0.0;
      const double bv = (jb < q && k < r) ? B[(int64_t)k * ldb + jb] : 0.0;
      fac_dmma(d0, d1, av, bv);
    }
    const int jc = j0 + 2 * t;
    if (ia < p) {
      double* c = C + (int64_t)ia * ldc;
      if (jc < q) c[jc] = SUB ? c[jc] - d0 : d0;
      if (jc + 1 < q) c[jc + 1] = SUB ? c[jc + 1] - d1 : d1;
    }
  }
}

// C (p x q, ldc) = [C -] A (p x r) * B (r x q), row-major, TS x TS register
// tiles (the caller picks TS so that enough threads get a tile).
template <class T, bool SUB, int TS>
__device__ void sm_gemm_t(T* C, int ldc, const T* A, int lda, const T* B, int ldb, int p, int q,
                          int r) {
  const int tp = (p + TS - 1) / TS, tq = (q + TS - 1) / TS;
  for (int t = threadIdx.x; t < tp * tq; t += blockDim.x) {
    const int i0 = (t / tq) * TS, j0 = (t % tq) * TS;
    T acc[TS][TS];
#pragma unroll
    for (int a = 0; a < TS; ++a)
#pragma unroll
      for (int b = 0; b < TS; ++b) acc[a][b] = T(0.0);
    for (int s = 0; s < r; ++s) {
      T av[TS], bv[TS];
#pragma unroll
      for (int a = 0; a < TS; ++a) av[a] = (i0 + a < p) ? A[(int64_t)(i0 + a) * lda + s] : T(0.0);
#pragma unroll
      for (int b = 0; b < TS; ++b) bv[b] = (j0 + b < q) ? B[(int64_t)s * ldb + j0 + b] : T(0.0);
#pragma unroll
      for (int a = 0; a < TS; ++a)
#pragma unroll
        for (int b = 0; b < TS; ++b) acc[a][b] += av[a] * bv[b];
    }
#pragma unroll
    for (int a = 0; a < TS; ++a)
#pragma unroll
      for (int b = 0; b < TS; ++b)
        if (i0 + a < p && j0 + b < q) {
          T* c = C + (int64_t)(i0 + a) * ldc + j0 + b;
          if (SUB) *c = *c - acc[a][b];
          else *c = acc[a][b];
        }
  }
}

template <class T, bool SUB>
__device__ void sm_gemm(T* C, int ldc, const T* A, int lda, const T* B, int ldb, int p, int q,
                        int r) {
  if constexpr (sizeof(T) == sizeof(double)) {
    // real blocks: DMMA (the dense block contractions of solver.py:243-261)
    sm_gemm_dmma<SUB>(reinterpret_cast<double*>(C), ldc, reinterpret_cast<const double*>(A), lda,
                      reinterpret_cast<const double*>(B), ldb, p, q, r);
    return;
  }
  const int nt = blockDim.x;
  if (((p + 3) >> 2) * ((q + 3) >> 2) >= nt) sm_gemm_t<T, SUB, 4>(C, ldc, A, lda, B, ldb, p, q, r);
  else if (((p + 1) >> 1) * ((q + 1) >> 1) >= nt / 2) sm_gemm_t<T, SUB, 2>(C, ldc, A, lda, B, ldb, p, q, r);
  else sm_gemm_t<T, SUB, 1>(C, ldc, A, lda, B, ldb, p, q, r);
}

template <class T>
__device__ void copy_out(T* dst, const T* src, int64_t cnt) {
  for (int64_t e = threadIdx.x; e < cnt; e += blockDim.x) dst[e] = src[e];
}

template <class T>
static __host__ __device__ inline size_t fac_elems(int n, int k) {
  // A and M are held with odd leading dimensions (n | 1, k | 1: the row-per-
  // lane register loads of sm_invert_la are then bank-conflict free)
  return (size_t)n * n + 4 * (size_t)n * k + (size_t)k * k + 4 * (size_t)n + (size_t)k;
}

// global (contiguous rows of q) <-> shared (row stride ld) block copies
template <class T>
__device__ __forceinline__ void cp_async_block_2d(T* dst, int ld, const T* src, int p, int q) {
  constexpr int W = sizeof(T) / 8;
  for (int e = threadIdx.x; e < p * q; e += blockDim.x) {
    const int i = e / q, j = e - i * q;
#pragma unroll
    for (int w = 0; w < W; ++w)
      cp_async8(reinterpret_cast<double*>(dst + (int64_t)i * ld + j) + w,
                reinterpret_cast<const double*>(src + e) + w);
  }
}
template <class T>
__device__ void copy_out_2d(T* dst, const T* src, int ld, int p, int q) {
  for (int e = threadIdx.x; e < p * q; e += blockDim.x) {
    const int i = e / q, j = e - i * q;
    dst[e] = src[(int64_t)i * ld + j];
  }
}

template <class T, bool GW, int NT>
// (real, 256 threads: capped at 64 registers for 4 CTAs / SM -- no spills)
__global__ void __launch_bounds__(NT, ((NT == 256 && sizeof(T) == sizeof(double)) ? 4 : 1))
    k_factor_level(const SkelFactorLevel F, int max_n, int max_k) {
  extern __shared__ __align__(16) unsigned char smem[];
  FacShared<T>& sh = *reinterpret_cast<FacShared<T>*>(smem);
  int* ipiv = reinterpret_cast<int*>(smem + 512);
  const size_t hdr = 512 + ((sizeof(int) * (size_t)max_n + 15) / 16) * 16;
  T* base = GW ? reinterpret_cast<T*>(F.scratch) + (size_t)blockIdx.x * fac_elems<T>(max_n, max_k)
               : reinterpret_cast<T*>(smem + hdr);
  const int a = F.order ? F.order[blockIdx.x] : blockIdx.x;
  const int n = F.n[a], k = F.k[a];
  if (n == 0) {
    if (threadIdx.x == 0) { F.status[a] = 0; F.rcond_d[a] = 1.0; F.rcond_m[a] = 1.0; }
    return;
  }
  const int lda = n | 1, ldm = k | 1;
  T* A = base;
  T* Lb = A + (size_t)n * lda;
  T* Rb = Lb + (size_t)n * k;
  T* X = Rb + (size_t)k * n;
  T* Y = X + (size_t)n * k;
  T* M = Y + (size_t)k * n;
  T* colk = M + (size_t)k * ldm;

  const T* D = reinterpret_cast<const T*>(F.D) + F.d_off[a];
  const T* Lg = reinterpret_cast<const T*>(F.L) + F.l_off[a];
  const T* Rg = reinterpret_cast<const T*>(F.R) + F.r_off[a];
  if constexpr (!GW) {
    cp_async_block_2d<T>(A, lda, D, n, n);
    cp_async_block<T>(Lb, Lg, (int64_t)n * k);
    cp_async_block<T>(Rb, Rg, (int64_t)n * k);
    cp_async_commit();
    cp_async_wait<0>();
  } else {
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) A[(int64_t)(e / n) * lda + e % n] = D[e];
    for (int64_t e = threadIdx.x; e < (int64_t)n * k; e += blockDim.x) {
      Lb[e] = Lg[e];
      Rb[e] = Rg[e];
    }
  }
  __syncthreads();
  if (F.child_off) {
    // children's Lambda on the diagonal blocks (solver.py:226-233)
    const int64_t c0 = F.child_off[a], c1 = F.child_off[a + 1];
    int ro = 0;
    for (int64_t c = c0; c < c1; ++c) {
      const int kc = F.prev_k[c];
      const T* lam = reinterpret_cast<const T*>(F.prev_lam) + F.prev_lam_off[c];
      for (int e = threadIdx.x; e < kc * kc; e += blockDim.x) {
        int i = e / kc, j = e - i * kc;
        if constexpr (!GW) cp_async_block_one(A + (int64_t)(ro + i) * lda + ro + j, lam + e);
        else A[(int64_t)(ro + i) * lda + ro + j] = lam[e];
      }
      ro += kc;
    }
    if constexpr (!GW) {
      cp_async_commit();
      cp_async_wait<0>();
    }
  }
  __syncthreads();
  if (F.regularize != 0.0) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) A[(int64_t)i * lda + i] += T(F.regularize);
    __syncthreads();
  }
  double nA = sm_norm1<T>(A, lda, n, n, sh);
  // look-ahead publication buffer: X is not live before X = D^-1 L
  int bad = sm_invert_fast<T>(A, lda, n, colk, X, (int64_t)n * k, ipiv, sh);
  if (bad) {
    if (threadIdx.x == 0) { F.status[a] = 1; F.rcond_d[a] = 0.0; F.rcond_m[a] = 0.0; }
    return;
  }
  double nAi = sm_norm1<T>(A, lda, n, n, sh);
  const double rcd = (nA * nAi > 0.0) ? 1.0 / (nA * nAi) : 0.0;
  T* Dd = reinterpret_cast<T*>(F.Dd) + F.dd_off[a];
  if (k == 0) {
    copy_out_2d<T>(Dd, A, lda, n, n);
    if (threadIdx.x == 0) { F.status[a] = 0; F.rcond_d[a] = rcd; F.rcond_m[a] = 1.0; }
    return;
  }
  sm_gemm<T, false>(X, k, A, lda, Lb, k, n, k, n);    // X = D^-1 L
  sm_gemm<T, false>(Y, n, Rb, n, A, lda, k, n, n);    // Y = R D^-1
  __syncthreads();
  sm_gemm<T, false>(M, ldm, Rb, n, X, k, k, k, n);    // M = R X
  __syncthreads();
  double nM = sm_norm1<T>(M, ldm, k, k, sh);
  if (F.regularize != 0.0) {
    for (int i = threadIdx.x; i < k; i += blockDim.x) M[(int64_t)i * ldm + i] += T(F.regularize);
    __syncthreads();
  }
  // L is dead between X = D^-1 L and Ld = X Lam: its slot is the publication buffer
  bad = sm_invert_fast<T>(M, ldm, k, colk, Lb, (int64_t)n * k, ipiv, sh);
  if (bad) {
    if (threadIdx.x == 0) { F.status[a] = 2; F.rcond_d[a] = rcd; F.rcond_m[a] = 0.0; }
    return;
  }
  double nMi = sm_norm1<T>(M, ldm, k, k, sh);
  sm_gemm<T, false>(Rb, n, M, ldm, Y, n, k, n, k);    // Rd = Lam RD
  sm_gemm<T, false>(Lb, k, X, k, M, ldm, n, k, k);    // Ld = X Lam
  __syncthreads();
  sm_gemm<T, true>(A, lda, X, k, Rb, n, n, n, k);     // Dd = D^-1 - X Rd
  __syncthreads();
  copy_out_2d<T>(Dd, A, lda, n, n);
  copy_out<T>(reinterpret_cast<T*>(F.Ld) + F.ld_off[a], Lb, (int64_t)n * k);
  copy_out<T>(reinterpret_cast<T*>(F.Rd) + F.rd_off[a], Rb, (int64_t)k * n);
  copy_out_2d<T>(reinterpret_cast<T*>(F.Lam) + F.lam_off[a], M, ldm, k, k);
  if (threadIdx.x == 0) {
    F.status[a] = 0;
    F.rcond_d[a] = rcd;
    F.rcond_m[a] = (nM * nMi > 0.0) ? 1.0 / (nM * nMi) : 0.0;
  }
}

template <class T>
static int factor_level_impl(const SkelFactorLevel* F, int max_n, int max_k, cudaStream_t st) {
  const int nrun = F->order ? F->nrun : F->nbox;
  if (nrun <= 0) return 0;
  if (max_n < 1) max_n = 1;
  size_t hdr = 512 + ((sizeof(int) * (size_t)max_n + 15) / 16) * 16;
  size_t need = hdr + fac_elems<T>(max_n, max_k) * sizeof(T);
  // few boxes (upper levels): per-box latency is the critical path -> 1024 threads
  const bool wide = nrun < skel_sm_count();
  if (need <= (size_t)skel_smem_optin()) {
    if (wide) {
      auto kern = k_factor_level<T, false, 1024>;
      SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
      kern<<<nrun, 1024, need, st>>>(*F, max_n, max_k);
    } else {
      auto kern = k_factor_level<T, false, 256>;
      SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
      kern<<<nrun, 256, need, st>>>(*F, max_n, max_k);
    }
  } else {
    if (!F->scratch || (size_t)F->scratch_bytes < (size_t)nrun * fac_elems<T>(max_n, max_k) * sizeof(T))
      return -2;
    auto kern = k_factor_level<T, true, 256>;
    SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hdr));
    kern<<<nrun, 256, hdr, st>>>(*F, max_n, max_k);
  }
  return skel_last_error();
}

// dense K x K inverse on one CTA (top level: Shat = S + blockdiag(Lam))
template <class T, bool GW>
__global__ void __launch_bounds__(1024) k_dense_inverse(T* Ag, int K, double reg, int32_t* status,
                                                        double* rcond, T* scratch) {
  extern __shared__ __align__(16) unsigned char smem[];
  FacShared<T>& sh = *reinterpret_cast<FacShared<T>*>(smem);
  int* ipiv = reinterpret_cast<int*>(smem + 512);
  size_t hdr = 512 + ((sizeof(int) * (size_t)K + 15) / 16) * 16;
  T* A = GW ? scratch : reinterpret_cast<T*>(smem + hdr);
  T* colk = GW ? scratch + (size_t)K * K : A + (size_t)K * K;   // 3K scratch
  for (int64_t e = threadIdx.x; e < (int64_t)K * K; e += blockDim.x) A[e] = Ag[e];
  __syncthreads();
  if (reg != 0.0) {
    for (int i = threadIdx.x; i < K; i += blockDim.x) A[(int64_t)i * K + i] += T(reg);
    __syncthreads();
  }
  double nA = sm_norm1<T>(A, K, K, K, sh);
  int bad = sm_invert_top<T>(A, K, K, colk, ipiv, sh);
  if (bad) {
    if (threadIdx.x == 0) { *status = 1; *rcond = 0.0; }
    return;
  }
  double nAi = sm_norm1<T>(A, K, K, K, sh);
  for (int64_t e = threadIdx.x; e < (int64_t)K * K; e += blockDim.x) Ag[e] = A[e];
  if (threadIdx.x == 0) {
    *status = 0;
    *rcond = (nA * nAi > 0.0) ? 1.0 / (nA * nAi) : 0.0;
  }
}

template <class T>
static int dense_inverse_impl(void* A, int K, double reg, int32_t* status, double* rcond,
                              void* scratch, cudaStream_t st) {
  if (K <= 0) return 0;
  size_t hdr = 512 + ((sizeof(int) * (size_t)K + 15) / 16) * 16;
  size_t need = hdr + ((size_t)K * K + 3 * K) * sizeof(T);
  if (need <= (size_t)skel_smem_optin()) {
    auto kern = k_dense_inverse<T, false>;
    SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need));
    kern<<<1, 1024, need, st>>>((T*)A, K, reg, status, rcond, (T*)scratch);
  } else {
    if (!scratch) return -2;
    auto kern = k_dense_inverse<T, true>;
    SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hdr));
    kern<<<1, 1024, hdr, st>>>((T*)A, K, reg, status, rcond, (T*)scratch);
  }
  return skel_last_error();
}

extern "C" {

int skel_factor_level(const SkelFactorLevel* fl, int32_t max_n, int32_t max_k, int32_t field,
                      void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) return factor_level_impl<double>(fl, max_n, max_k, st);
  return factor_level_impl<zc>(fl, max_n, max_k, st);
}

int skel_dense_inverse(void* A, void* lu, int32_t* ipiv, int32_t K, double regularize,
                       int32_t* status, double* rcond, int32_t field, void* scratch, void* stream) {
  (void)lu;
  (void)ipiv;
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) return dense_inverse_impl<double>(A, K, regularize, status, rcond, scratch, st);
  return dense_inverse_impl<zc>(A, K, regularize, status, rcond, scratch, st);
}

}  // extern "C"
