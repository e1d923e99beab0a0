// big.cu -- the "big box" path: interpolative decompositions and dense
// inverses too large for one CTA (3D coarse levels, BASELINE config 4; the
// top-level Shat of large 3D problems).  Every kernel here spreads ONE box
// over the whole GPU:
//
//   * k_big_target     one side's proxy-compressed target (t_row.T or t_col,
//                      skel.py:349-368) assembled into a global column-major
//                      slab, 2D grid over (row tiles, column chunks);
//   * k_cpqr_big       cooperative (grid-synchronised) column-pivoted QR with
//                      the exact pivot / norm / stop rules of lowrank.py:48-119
//                      (the same state machine as cpqr.cuh, two grid barriers
//                      per step, one warp per trailing column);
//   * k_big_interp     P = R11^-1 R12 (lowrank.py:122-133), one thread/column;
//   * k_big_output     sorted skeletons + L / R into the level slabs
//                      (skel.py:384-391);
//   * k_gemm_tn / k_gemv / k_probe_*  the Gaussian sketch Y = Omega A, the
//                      power-iteration norm estimate and the 5-probe check of
//                      id_randomized (lowrank.py:169-231; the random numbers
//                      come from the host with the reference's generator);
//   * k_gj_coop        cooperative Gauss-Jordan inverse with partial pivoting
//                      (the top-level Shat, solver.py:269-274).
#include <cooperative_groups.h>

#include "cpqr.cuh"
#include "entries.cuh"

namespace cg = cooperative_groups;

template <class T>
struct BigState {
  int rank, stop, pad, pc;
  double p0, beta, bigP, pad0;
  T v0, alpha;
};

static inline size_t big_state_hdr() { return 256; }

template <class T>
struct BigView {
  BigState<T>* st;
  double* nrm;
  double* ref;
  double* xn2;
  int* piv;
};

template <class T>
__host__ __device__ inline BigView<T> big_view(void* buf, int n) {
  BigView<T> v;
  unsigned char* p = reinterpret_cast<unsigned char*>(buf);
  v.st = reinterpret_cast<BigState<T>*>(p);
  v.nrm = reinterpret_cast<double*>(p + 256);
  v.ref = v.nrm + n;
  v.xn2 = v.ref + n;
  v.piv = reinterpret_cast<int*>(v.xn2 + n);
  return v;
}

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }
__device__ __forceinline__ zc ldcg(const zc* p) {
  double2 v = __ldcg(reinterpret_cast<const double2*>(p));
  return zc(v.x, v.y);
}
__device__ __forceinline__ int ldcg(const int* p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// target assembly: rows = neighbour dofs (nbr_pref/nbr_box) then proxies
template <class T>
__global__ void __launch_bounds__(128)
    k_big_target(const SkelSource S, const SkelLevel L, int a, int side, const int32_t* nbr_box,
                 const int32_t* nbr_pref, int nnb, int m, T* W, int64_t ld) {
  __shared__ Pt cp[64];
  const int64_t r0 = L.rdof_off[a], c0 = L.cdof_off[a];
  const int n = side == 0 ? (int)(L.rdof_off[a + 1] - r0) : (int)(L.cdof_off[a + 1] - c0);
  const int32_t* mydofs = side == 0 ? L.rdofs + r0 : L.cdofs + c0;
  const int j0 = blockIdx.y * 64;
  const int jn = min(64, n - j0);
  if (jn <= 0) return;
  for (int j = threadIdx.x; j < jn; j += blockDim.x) cp[j] = load_pt(S, mydofs[j0 + j]);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int m_nbr = nbr_pref[nnb];
  if (i < m_nbr) {
    int lo = 0, hi = nnb;             // last q with nbr_pref[q] <= i
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (nbr_pref[mid] <= i) lo = mid; else hi = mid;
    }
    const int b = nbr_box[lo];
    const int off = i - nbr_pref[lo];
    const int32_t idx = side == 0 ? L.cdofs[L.cdof_off[b] + off] : L.rdofs[L.rdof_off[b] + off];
    const Pt rp = load_pt(S, idx);
    if (side == 0) {
      for (int j = 0; j < jn; ++j) W[(int64_t)(j0 + j) * ld + i] = entry_A<T>(S, cp[j], rp);
    } else {
      for (int j = 0; j < jn; ++j) W[(int64_t)(j0 + j) * ld + i] = entry_A<T>(S, rp, cp[j]);
    }
  } else {
    const int dim = S.dim;
    const int pr = L.pxy_begin[a] + (i - m_nbr);
    const double rr = L.box_r[a];
    const double px = __dadd_rn(L.box_c[(int64_t)a * dim + 0], __dmul_rn(rr, L.pxy_unit[(int64_t)pr * dim + 0]));
    const double py = __dadd_rn(L.box_c[(int64_t)a * dim + 1], __dmul_rn(rr, L.pxy_unit[(int64_t)pr * dim + 1]));
    const double pz = dim == 3 ? __dadd_rn(L.box_c[(int64_t)a * dim + 2], __dmul_rn(rr, L.pxy_unit[(int64_t)pr * dim + 2])) : 0.0;
    if (side == 0) {
      for (int j = 0; j < jn; ++j) W[(int64_t)(j0 + j) * ld + i] = entry_proxy_row<T>(S, cp[j], px, py, pz);
    } else {
      for (int j = 0; j < jn; ++j) W[(int64_t)(j0 + j) * ld + i] = entry_proxy_col<T>(S, px, py, pz, cp[j]);
    }
  }
}

// ---------------------------------------------------------------------------
// cooperative CPQR

__device__ __forceinline__ void cmerge(double& bv, int& bi, double ov, int oi) {
  if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
}

// exact initial norms (lowrank.py:55-64), piv = identity, state reset
template <class T>
__global__ void k_cpqr_big_init(const T* W, int m, int n, int64_t ld, void* buf) {
  BigView<T> v = big_view<T>(buf, n);
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  for (int c = gw; c < n; c += tw) {
    const T* x = W + (int64_t)c * ld;
    double s = 0.0;
    for (int i = lane; i < m; i += 32) s += sk_abs2(x[i]);
    s = warp_sum(s);
    if (lane == 0) { v.nrm[c] = s; v.ref[c] = s; v.xn2[c] = s; v.piv[c] = c; }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    v.st->rank = 0; v.st->stop = 0; v.st->pad = 0; v.st->pc = 0;
    v.st->p0 = 0.0; v.st->beta = 0.0; v.st->bigP = 0.0; v.st->pad0 = 0.0;
  }
}

// One grid barrier per step.  Every CTA redundantly reduces the per-CTA
// pivot candidates of the previous step (first maximum by position), applies
// the stop rule and forms the reflector; the position -> column map is
// double-buffered (CTA 0 writes the swapped copy for the next step) so no CTA
// reads an entry another CTA is rewriting.  Phase B: one warp per trailing
// position -- reflector, norm downdate / stale / renorm rules, exact
// trailing norm, next-step candidate.
template <class T>
__global__ void __launch_bounds__(256)
    k_cpqr_big(T* W, int m, int n, int64_t ld, double eps, int min_rank, void* buf, int vsmem,
               int* pivb, double* cand_v, int* cand_i, int kcap) {
  cg::grid_group grid = cg::this_grid();
  BigView<T> v = big_view<T>(buf, n);
  extern __shared__ __align__(16) unsigned char cp_smem[];
  T* vs = reinterpret_cast<T*>(cp_smem);        // the reflector, when it fits
  __shared__ double sv[8];
  __shared__ int si[8];
  __shared__ double red_v;
  __shared__ int red_i;
  const int G = gridDim.x;
  const int kmax = m < n ? m : n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int tw = (gridDim.x * blockDim.x) >> 5;
  int s = ldcg(&v.st->rank);
  double p0 = ldcg(&v.st->p0);
  if (blockIdx.x == 0 && threadIdx.x == 0) v.st->pad0 = 0.0;   // set again at a rule stop
  int* pcur = v.piv;
  int* pnext = pivb;
  // candidates for the first step: every CTA scans nrm[s..n) itself
  {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int c = s + threadIdx.x; c < n; c += blockDim.x) cmerge(bv, bi, ldcg(v.nrm + c), c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      cmerge(bv, bi, ov, oi);
    }
    if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0;
      int j = 0x7fffffff;
      for (int w = 0; w < nwb; ++w) cmerge(b, j, sv[w], si[w]);
      red_v = b;
      red_i = j;
    }
    __syncthreads();
  }
  double bsel = red_v;
  int jsel = red_i;
  int par = 0;
  const int kend = kmax < kcap ? kmax : kcap;     // equalisation: exactly min_rank steps
  while (s < kend) {
    // ---- pivot + stop rule (identical on every CTA)
    const int j = jsel;
    int stop = 0;
    double pn = 0.0;
    if (j >= n) {
      stop = 1;
    } else {
      pn = sqrt(fmax(bsel, 0.0));
      if (s == 0) {
        p0 = pn;
        if (pn == 0.0) stop = 1;
      }
      if (!stop && ((s >= min_rank && pn <= eps * p0) || pn == 0.0)) stop = 2;
    }
    if (stop) {
      // first rejected pivot norm: achieved_error numerator (lowrank.py:88-90)
      if (blockIdx.x == 0 && threadIdx.x == 0) v.st->pad0 = stop == 2 ? pn : 0.0;
      break;
    }
    const int pc = ldcg(pcur + j);           // pivot column
    const int ps_old = ldcg(pcur + s);
    const double nrm_s_old = ldcg(v.nrm + s);
    const double nx2 = ldcg(v.xn2 + j);
    const T x0 = ldcg(W + (int64_t)pc * ld + s);
    const double ax0 = sk_abs(x0);
    const double normx = sqrt(nx2);
    T phase = T(1.0);
    if (ax0 != 0.0) phase = sk_unit_phase(x0, ax0);
    const T alpha = -(phase * normx);
    const double vv = 2.0 * normx * (normx + ax0);
    const T v0 = x0 - alpha;
    const double beta = vv > 0.0 ? 2.0 / vv : 0.0;
    if (blockIdx.x == 0) {
      // next step's position -> column map, with positions s and j swapped
      for (int c = threadIdx.x; c < n; c += blockDim.x) {
        int col = ldcg(pcur + c);
        if (c == s) col = pc;
        else if (c == j) col = ps_old;
        pnext[c] = col;
      }
      if (threadIdx.x == 0 && s == 0) v.st->p0 = p0;
    }
    // ---- phase B
    const int s1 = s + 1;
    const bool renorm = (s1 < kmax) && (s1 % 32 == 0);
    const T* vcol = W + (int64_t)pc * ld;
    if (vsmem) {
      for (int i = s + threadIdx.x; i < m; i += blockDim.x) vs[i] = (i == s) ? v0 : ldcg(vcol + i);
      __syncthreads();
    }
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int c = s1 + gw; c < n; c += tw) {
      const int col = (c == j) ? ps_old : ldcg(pcur + c);
      T* wc = W + (int64_t)col * ld;
      // U rows per lane per pass (all loads of a pass issued before any use:
      // the trailing matrix lives in L2 / HBM, so the pass is load-latency
      // bound), 4 partial sums
      constexpr int U = sizeof(T) == sizeof(double) ? 16 : 8;
      T d4[4] = {T(0.0), T(0.0), T(0.0), T(0.0)};
      for (int i0 = s; i0 < m; i0 += 32 * U) {
        T wv[U], vq[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + lane + 32 * u;
          wv[u] = i < m ? ldcg(wc + i) : T(0.0);
          vq[u] = i < m ? (vsmem ? vs[i] : ((i == s) ? v0 : ldcg(vcol + i))) : T(0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) d4[u & 3] += sk_conj(vq[u]) * wv[u];
      }
      T dot = (d4[0] + d4[1]) + (d4[2] + d4[3]);
      dot = warp_sum(dot);
      const T f = dot * beta;
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
      T row = T(0.0);
      for (int i0 = s; i0 < m; i0 += 32 * U) {
        T wv[U], vq[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + lane + 32 * u;
          wv[u] = i < m ? ldcg(wc + i) : T(0.0);
          vq[u] = i < m ? (vsmem ? vs[i] : ((i == s) ? v0 : ldcg(vcol + i))) : T(0.0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + lane + 32 * u;
          if (i < m) {
            T w = wv[u];
            if (beta != 0.0) {
              w -= vq[u] * f;
              wc[i] = w;
            }
            if (i > s) a4[u & 3] += sk_abs2(w);
            if (i == s) row = w;
          }
        }
      }
      double acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
      acc = warp_sum(acc);
      row = shfl(row, 0);
      double t = ((c == j) ? nrm_s_old : ldcg(v.nrm + c)) - sk_abs2(row);
      t = t > 0.0 ? t : 0.0;
      if (renorm || t < 1e-8 * ldcg(v.ref + c)) {
        t = acc;
        if (lane == 0) v.ref[c] = acc;
      }
      if (lane == 0) {
        v.nrm[c] = t;
        v.xn2[c] = acc;
      }
      cmerge(bv, bi, t, c);
    }
    if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
    __syncthreads();
    par ^= 1;
    if (threadIdx.x == 0) {
      double b = -1.0;
      int jj = 0x7fffffff;
      for (int w = 0; w < nwb; ++w) cmerge(b, jj, sv[w], si[w]);
      cand_v[par * 4096 + blockIdx.x] = b;
      cand_i[par * 4096 + blockIdx.x] = jj;
    }
    grid.sync();
    // every CTA has read x0 of this step: the diagonal entry can be written
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      W[(int64_t)pc * ld + s] = alpha;
      v.st->rank = s + 1;
    }
    // ---- reduce the candidates for the next step (warp 0 of every CTA)
    if (wid == 0) {
      double b = -1.0;
      int jj = 0x7fffffff;
      for (int q = lane; q < G; q += 32)
        cmerge(b, jj, ldcg(cand_v + par * 4096 + q), ldcg(cand_i + par * 4096 + q));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, b, o);
        int oi = __shfl_xor_sync(0xffffffffu, jj, o);
        cmerge(b, jj, ov, oi);
      }
      if (lane == 0) { red_v = b; red_i = jj; }
    }
    __syncthreads();
    bsel = red_v;
    jsel = red_i;
    int* t = pcur; pcur = pnext; pnext = t;
    ++s;
  }
  // the final map must live in v.piv
  if (pcur != v.piv) {
    grid.sync();
    if (blockIdx.x == 0)
      for (int c = threadIdx.x; c < n; c += blockDim.x) v.piv[c] = ldcg(pcur + c);
  }
}

// P = R11^-1 R12 in place (rows 0..r-1 of the non-pivot columns), max|P|,
// padding count to min_rank (lowrank.py:122-161).  One warp per column, the
// column staged in shared memory; the back substitution runs in the same
// (dtrsm, column-oriented) order as cpqr.cuh's interp_solve, with the
// x[t] -= R[t,s] x[s] updates of one step spread over the lanes.
template <class T>
__global__ void __launch_bounds__(128) k_big_interp(T* W, int n, int64_t ld, void* buf, int min_rank) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BigView<T> v = big_view<T>(buf, n);
  const int r = v.st->rank;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T* xs = reinterpret_cast<T*>(smem_raw) + (size_t)wid * (r > 0 ? r : 1);
  const int c = r + blockIdx.x * (blockDim.x >> 5) + wid;
  double big = 0.0;
  if (c < n && r > 0) {
    T* x = W + (int64_t)v.piv[c] * ld;
    for (int t = lane; t < r; t += 32) xs[t] = x[t];
    __syncwarp();
    for (int s = r - 1; s >= 0; --s) {
      T xv = xs[s];
      if (xv != T(0.0)) {
        const T* rs = W + (int64_t)v.piv[s] * ld;   // R[:, s]
        xv = xv / rs[s];
        __syncwarp();
        if (lane == 0) xs[s] = xv;
        for (int t = lane; t < s; t += 32) xs[t] -= rs[t] * xv;
      }
      __syncwarp();
    }
    for (int t = lane; t < r; t += 32) {
      x[t] = xs[t];
      big = fmax(big, sk_abs(xs[t]));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) big = fmax(big, __shfl_xor_sync(0xffffffffu, big, o));
  if (lane == 0 && big > 0.0)
    atomicMax(reinterpret_cast<unsigned long long*>(&v.st->bigP), (unsigned long long)__double_as_longlong(big));
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int kmin = min_rank < n ? min_rank : n;
    v.st->pad = (r < kmin) ? kmin - r : 0;
  }
}

template <class T>
__device__ __forceinline__ T big_interp_entry(const T* W, int64_t ld, const int* piv, int r, int kfin,
                                              int s, int q) {
  if (q < kfin) return (s == q) ? T(1.0) : T(0.0);
  return (s < r) ? W[(int64_t)piv[q] * ld + s] : T(0.0);
}

// sorted skeletons and L (n x K) / R (K x n) into the level slabs, k into
// kr / kc, the |P| > 2 warning flag (skel.py:384-391, lowrank.py:128-132)
template <class T>
__global__ void k_big_output(const SkelLevel L, int a, int side, const T* W, int64_t ld, const void* buf,
                             int n) {
  extern __shared__ int pos[];
  BigView<T> v = big_view<T>(const_cast<void*>(buf), n);
  const int r = v.st->rank;
  const int K = r + v.st->pad;
  const int* piv = v.piv;
  for (int s = threadIdx.x; s < K; s += blockDim.x) {
    const int ps = piv[s];
    int c = 0;
    for (int t = 0; t < K; ++t) c += piv[t] < ps;
    pos[s] = c;
  }
  __syncthreads();
  const int64_t r0 = L.rdof_off[a], c0 = L.cdof_off[a];
  const int32_t* mydofs = side == 0 ? L.rdofs + r0 : L.cdofs + c0;
  int32_t* skel = side == 0 ? L.rskel + r0 : L.cskel + c0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = tid; s < K; s += nt) skel[pos[s]] = mydofs[piv[s]];
  const int64_t tot = (int64_t)n * K;
  if (side == 0) {
    T* Lo = reinterpret_cast<T*>(L.L) + L.l_off[a];
    for (int64_t e = tid; e < tot; e += nt) {
      const int q = (int)(e / K), s = (int)(e - (int64_t)q * K);
      Lo[(int64_t)piv[q] * K + pos[s]] = big_interp_entry<T>(W, ld, piv, r, K, s, q);
    }
  } else {
    T* Ro = reinterpret_cast<T*>(L.R) + L.r_off[a];
    for (int64_t e = tid; e < tot; e += nt) {
      const int s = (int)(e / n), q = (int)(e - (int64_t)s * n);
      Ro[(int64_t)pos[s] * n + piv[q]] = big_interp_entry<T>(W, ld, piv, r, K, s, q);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    (side == 0 ? L.kr : L.kc)[a] = K;
    if (v.st->bigP > 2.0) atomicOr(L.flags + a, 1 << side);
  }
}

// ---------------------------------------------------------------------------
// sketch / probes of id_randomized

// Y (m x n, ld ldy) = X^T A, X k x m (ld ldx), A k x n (ld lda), column-major
template <class T>
__global__ void __launch_bounds__(256)
    k_gemm_tn(int m, int n, int k, const T* __restrict__ X, int64_t ldx, const T* __restrict__ A,
              int64_t lda, T* Y, int64_t ldy) {
  __shared__ T xs[16][65];
  __shared__ T as[16][65];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  T acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int w = 0; w < 4; ++w) acc[u][w] = T(0.0);
  for (int i0 = 0; i0 < k; i0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int ii = e & 15, cc = e >> 4;
      const int i = i0 + ii;
      xs[ii][cc] = (i < k && r0 + cc < m) ? X[(int64_t)(r0 + cc) * ldx + i] : T(0.0);
      as[ii][cc] = (i < k && c0 + cc < n) ? A[(int64_t)(c0 + cc) * lda + i] : T(0.0);
    }
    __syncthreads();
#pragma unroll
    for (int ii = 0; ii < 16; ++ii) {
      T xr[4], ar[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { xr[u] = xs[ii][ty * 4 + u]; ar[u] = as[ii][tx * 4 + u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] += xr[u] * ar[w];
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int r = r0 + ty * 4 + u, c = c0 + tx * 4 + w;
      if (r < m && c < n) Y[(int64_t)c * ldy + r] = acc[u][w];
    }
}

// DMMA (mma.sync m8n8k4 f64) version of k_gemm_tn for real data: 64 x 64 CTA
// tile, 4 warps of 32 x 32, K staged 16 deep in shared memory with cp.async
// (double-buffered).  Both operands are contiguous along K in global memory
// and in shared memory (row stride 20 doubles: conflict-free fragment loads).
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

#define TN_LDS 20
__global__ void __launch_bounds__(128)
    k_gemm_tn_dmma(int m, int n, int k, const double* __restrict__ X, int64_t ldx,
                   const double* __restrict__ A, int64_t lda, double* Y, int64_t ldy) {
  __shared__ __align__(16) double xs[2][64 * TN_LDS];
  __shared__ __align__(16) double as[2][64 * TN_LDS];
  const int r0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wr = (wid >> 1) * 32, wc = (wid & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  auto stage = [&](int buf, int k0) {
    for (int e = threadIdx.x; e < 64 * 16; e += 128) {
      const int kk = e & 15, rr = e >> 4;
      const int i = k0 + kk;
      double* dx = &xs[buf][rr * TN_LDS + kk];
      double* da = &as[buf][rr * TN_LDS + kk];
      if (i < k && r0 + rr < m) cp_async8(dx, X + (int64_t)(r0 + rr) * ldx + i); else *dx = 0.0;
      if (i < k && c0 + rr < n) cp_async8(da, A + (int64_t)(c0 + rr) * lda + i); else *da = 0.0;
    }
    cp_async_commit();
  };
  const int nk = (k + 15) / 16;
  stage(0, 0);
  for (int t = 0; t < nk; ++t) {
    const int buf = t & 1;
    if (t + 1 < nk) {
      stage(buf ^ 1, (t + 1) * 16);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
#pragma unroll
    for (int k4 = 0; k4 < 16; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) af[a] = xs[buf][(wr + a * 8 + (lane >> 2)) * TN_LDS + k4 + (lane & 3)];
#pragma unroll
      for (int b = 0; b < 4; ++b) bf[b] = as[buf][(wc + b * 8 + (lane >> 2)) * TN_LDS + k4 + (lane & 3)];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) dmma884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = r0 + wr + a * 8 + (lane >> 2);
        const int c = c0 + wc + b * 8 + 2 * (lane & 3) + h;
        if (r < m && c < n) Y[(int64_t)c * ldy + r] = acc[a][b][h];
      }
}

// y = A x (trans 0: thread per row) or y = A^H x (trans 1: warp per column)
template <class T>
__global__ void k_gemv(int trans, int m, int n, const T* __restrict__ A, int64_t lda,
                       const T* __restrict__ x, T* y) {
  if (trans == 0) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    T s = T(0.0);
    for (int j = 0; j < n; ++j) s += A[(int64_t)j * lda + i] * x[j];
    y[i] = s;
  } else {
    const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (j >= n) return;
    T s = T(0.0);
    for (int i = lane; i < m; i += 32) s += sk_conj(A[(int64_t)j * lda + i]) * x[i];
    s = warp_sum(s);
    if (lane == 0) y[j] = s;
  }
}

// u = P v for the interpolation matrix of a CPQR state (P[:, piv[s]] = e_s,
// P[:, piv[q]] = X[:, q] for q >= r), length r
template <class T>
__global__ void k_probe_pv(const T* W, int n, int64_t ld, const void* buf, const T* vin, T* u) {
  BigView<T> v = big_view<T>(const_cast<void*>(buf), n);
  const int r = v.st->rank;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= r) return;
  T acc = vin[v.piv[s]];
  for (int q = r; q < n; ++q) acc += W[(int64_t)v.piv[q] * ld + s] * vin[v.piv[q]];
  u[s] = acc;
}

// z = A v - A[:, skel] u  (skel = piv[:r] of the sketch's CPQR state)
template <class T>
__global__ void k_probe_z(int m, int n, const T* __restrict__ A, int64_t lda, const void* buf,
                          const T* vin, const T* u, T* z) {
  BigView<T> v = big_view<T>(const_cast<void*>(buf), n);
  const int r = v.st->rank;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  T s1 = T(0.0), s2 = T(0.0);
  for (int j = 0; j < n; ++j) s1 += A[(int64_t)j * lda + i] * vin[j];
  for (int q = 0; q < r; ++q) s2 += A[(int64_t)v.piv[q] * lda + i] * u[q];
  z[i] = s1 - s2;
}

// ---------------------------------------------------------------------------
// cooperative Gauss-Jordan inverse, partial pivoting, row-major n x n in place
// (the reference LU-factors Shat, solver.py:269-274; the explicit inverse
// turns the top solve into one GEMM)

template <class T>
__global__ void __launch_bounds__(256)
    k_gj_coop(T* A, int n, double regularize, int32_t* status, double* part_v, int* part_i,
              T* colc, int* swaps, const int32_t* skip) {
  // Two grid barriers per column: (1) after the row swap / pivot-row scaling,
  // (2) after the elimination, which also produces the next column's pivot
  // candidates over each CTA's own rows.
  cg::grid_group grid = cg::this_grid();
  if (skip && *skip) return;           // an earlier step of the same box failed
  extern __shared__ __align__(16) unsigned char gj_smem[];
  T* prow = reinterpret_cast<T*>(gj_smem);
  __shared__ double sv[8];
  __shared__ int si[8];
  __shared__ double red_v;
  __shared__ int red_i;
  const int G = gridDim.x;
  const int rpc = (n + G - 1) / G;
  const int r0 = min(n, (int)blockIdx.x * rpc), r1 = min(n, r0 + rpc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  auto block_cand = [&](double bv, int bi, int slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      cmerge(bv, bi, ov, oi);
    }
    if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0;
      int j = 0x7fffffff;
      for (int w = 0; w < nwb; ++w) cmerge(b, j, sv[w], si[w]);
      part_v[slot * 4096 + blockIdx.x] = b;
      part_i[slot * 4096 + blockIdx.x] = j;
    }
  };
  {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
      if (regularize != 0.0) A[(int64_t)r * n + r] += T(regularize);
      cmerge(bv, bi, sk_pivabs(A[(int64_t)r * n]), r);
    }
    block_cand(bv, bi, 0);
  }
  grid.sync();
  int par = 0;
  for (int c = 0; c < n; ++c) {
    // pivot: first max of |A[r][c]| over r >= c (LAPACK i?amax order)
    if (wid == 0) {
      double b = -1.0;
      int jj = 0x7fffffff;
      for (int q = lane; q < G; q += 32) cmerge(b, jj, ldcg(part_v + par * 4096 + q), ldcg(part_i + par * 4096 + q));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, b, o);
        int oi = __shfl_xor_sync(0xffffffffu, jj, o);
        cmerge(b, jj, ov, oi);
      }
      if (lane == 0) { red_v = b; red_i = jj; }
    }
    __syncthreads();
    const double b = red_v;
    const int p = red_i;
    if (p >= n || b == 0.0) {
      if (gt == 0) *status = 1;
      return;                        // uniform across the grid
    }
    const T apc = ldcg(A + (int64_t)p * n + c);
    const T inv = T(1.0) / apc;
    // swap rows c <-> p and scale the pivot row (column c excluded: it is
    // rewritten whole below); save column c as it reads after the swap
    for (int64_t j = gt; j < n; j += nt) {
      if (j == c) continue;
      const T vp = ldcg(A + (int64_t)p * n + j);
      const T vc = ldcg(A + (int64_t)c * n + j);
      if (p != c) A[(int64_t)p * n + j] = vc;
      A[(int64_t)c * n + j] = vp * inv;
    }
    for (int64_t r = gt; r < n; r += nt) {
      T v = (r == p) ? ldcg(A + (int64_t)c * n + c) : ldcg(A + r * n + c);
      if (r == c) v = apc;
      colc[r] = v;
    }
    if (gt == 0) swaps[c] = p;
    grid.sync();
    // eliminate column c from the CTA's rows (in-place inverse columns), the
    // scaled pivot row staged in shared memory; candidates for column c + 1
    for (int j = threadIdx.x; j < n; j += blockDim.x) prow[j] = ldcg(A + (int64_t)c * n + j);
    __syncthreads();
    double bv = -1.0;
    int bi = 0x7fffffff;
    const int cn = c + 1;
    for (int r = r0 + wid; r < r1; r += nwb) {
      T* Ar = A + (int64_t)r * n;
      if (r == c) {
        if (lane == 0) Ar[c] = inv;
        continue;
      }
      const T f = ldcg(colc + r);
      for (int j0 = 0; j0 < n; j0 += 128) {
        T av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + lane + 32 * u;
          av[u] = j < n ? ldcg(Ar + j) : T(0.0);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + lane + 32 * u;
          if (j < n) {
            T nv;
            if (j == c) nv = -(f * inv);
            else nv = av[u] - f * prow[j];
            Ar[j] = nv;
            if (j == cn && r >= cn) cmerge(bv, bi, sk_pivabs(nv), r);
          }
        }
      }
    }
    par ^= 1;
    if (cn < n) block_cand(bv, bi, par);
    grid.sync();
  }
}

// Cooperative LU with partial pivoting, row-major n x n in place, LAPACK
// getrf conventions (unit-lower L below the diagonal, U on and above, piv[c]
// = the row interchanged with row c, 0-based as scipy.linalg.lu_factor
// returns it) -- the reference stores Shat as lu_factor output
// (solver.py:269-274) and its container keeps (lu, piv).
template <class T>
__global__ void __launch_bounds__(256)
    k_lu_coop(T* A, int n, int32_t* status, double* part_v, int* part_i, T* colc, int* piv) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char lu_smem[];
  T* prow = reinterpret_cast<T*>(lu_smem);
  __shared__ double sv[8];
  __shared__ int si[8];
  __shared__ double red_v;
  __shared__ int red_i;
  const int G = gridDim.x;
  const int rpc = (n + G - 1) / G;
  const int r0 = min(n, (int)blockIdx.x * rpc), r1 = min(n, r0 + rpc);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  auto block_cand = [&](double bv, int bi, int slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      cmerge(bv, bi, ov, oi);
    }
    if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0;
      int j = 0x7fffffff;
      for (int w = 0; w < nwb; ++w) cmerge(b, j, sv[w], si[w]);
      part_v[slot * 4096 + blockIdx.x] = b;
      part_i[slot * 4096 + blockIdx.x] = j;
    }
  };
  {
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) cmerge(bv, bi, sk_pivabs(A[(int64_t)r * n]), r);
    block_cand(bv, bi, 0);
  }
  grid.sync();
  int par = 0;
  for (int c = 0; c < n; ++c) {
    if (wid == 0) {
      double b = -1.0;
      int jj = 0x7fffffff;
      for (int q = lane; q < G; q += 32) cmerge(b, jj, ldcg(part_v + par * 4096 + q), ldcg(part_i + par * 4096 + q));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, b, o);
        int oi = __shfl_xor_sync(0xffffffffu, jj, o);
        cmerge(b, jj, ov, oi);
      }
      if (lane == 0) { red_v = b; red_i = jj; }
    }
    __syncthreads();
    const double b = red_v;
    const int p = red_i;
    if (p >= n || b == 0.0) {
      if (gt == 0) *status = 1;
      return;
    }
    // interchange rows c and p (whole rows, as getrf; column c is handled
    // through colc and rewritten below), save column c as it reads after
    for (int64_t j = gt; j < n; j += nt) {
      if (p != c && j != c) {
        const T vp = ldcg(A + (int64_t)p * n + j);
        const T vc = ldcg(A + (int64_t)c * n + j);
        A[(int64_t)p * n + j] = vc;
        A[(int64_t)c * n + j] = vp;
      }
    }
    for (int64_t r = gt; r < n; r += nt) {
      T v = (r == p) ? ldcg(A + (int64_t)c * n + c) : ldcg(A + r * n + c);
      if (r == c) v = ldcg(A + (int64_t)p * n + c);
      colc[r] = v;
    }
    if (gt == 0) piv[c] = p;
    grid.sync();
    // multipliers and the rank-1 update of the trailing block (own rows > c)
    for (int j = threadIdx.x; j < n; j += blockDim.x) prow[j] = ldcg(A + (int64_t)c * n + j);
    __syncthreads();
    const T pv = ldcg(colc + c);
    const T inv = T(1.0) / pv;
    if (gt == 0) A[(int64_t)c * n + c] = pv;
    double bv = -1.0;
    int bi = 0x7fffffff;
    const int cn = c + 1;
    for (int r = max(r0, c + 1) + wid; r < r1; r += nwb) {
      T* Ar = A + (int64_t)r * n;
      const T l = ldcg(colc + r) * inv;
      if (lane == 0) Ar[c] = l;
      for (int j = c + 1 + lane; j < n; j += 32) {
        const T nv = ldcg(Ar + j) - l * prow[j];
        Ar[j] = nv;
        if (j == cn) cmerge(bv, bi, sk_pivabs(nv), r);
      }
    }
    par ^= 1;
    if (cn < n) block_cand(bv, bi, par);
    grid.sync();
  }
}

// inverse from getrf factors: one warp per right-hand side e_j (row
// interchanges, unit-lower forward, upper backward substitution; getrs order)
template <class T>
__global__ void k_lu_inverse(const T* __restrict__ LU, const int* __restrict__ piv, int n, T* inv) {
  extern __shared__ __align__(16) unsigned char li_smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int j = blockIdx.x * (blockDim.x >> 5) + wid;
  if (j >= n) return;
  T* x = reinterpret_cast<T*>(li_smem) + (size_t)wid * n;
  for (int i = lane; i < n; i += 32) x[i] = (i == j) ? T(1.0) : T(0.0);
  __syncwarp();
  if (lane == 0)
    for (int i = 0; i < n; ++i) {
      const int p = piv[i];
      if (p != i) { T t = x[i]; x[i] = x[p]; x[p] = t; }
    }
  __syncwarp();
  for (int i = 1; i < n; ++i) {
    const T* li = LU + (int64_t)i * n;
    T s = T(0.0);
    for (int t = lane; t < i; t += 32) s += li[t] * x[t];
    s = warp_sum(s);
    if (lane == 0) x[i] -= s;
    __syncwarp();
  }
  for (int i = n - 1; i >= 0; --i) {
    const T* ui = LU + (int64_t)i * n;
    T s = T(0.0);
    for (int t = i + 1 + lane; t < n; t += 32) s += ui[t] * x[t];
    s = warp_sum(s);
    if (lane == 0) x[i] = (x[i] - s) / ui[i];
    __syncwarp();
  }
  for (int i = lane; i < n; i += 32) inv[(int64_t)i * n + j] = x[i];
}

// undo the row interchanges on the inverse's columns (reverse order)
template <class T>
__global__ void k_gj_unswap(T* A, int n, const int* swaps, const int32_t* status,
                            const int32_t* skip) {
  // skipped (skip set: an earlier step of the box failed) or singular runs
  // leave `swaps` unwritten: never read it then
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n || *status || (skip && *skip)) return;
  T* row = A + r * n;
  for (int c = n - 1; c >= 0; --c) {
    const int p = swaps[c];
    if (p != c) { T t = row[c]; row[c] = row[p]; row[p] = t; }
  }
}

// ---------------------------------------------------------------------------
// big-box factor_node (solver.py:224-262) over the whole GPU: D_eff gather,
// cooperative inverses of D and M = R D^-1 L, row-major GEMMs for the rest

// C (m x n) = alpha A (m x k) B (k x n) + beta Cin, row-major; skipped when *flag
template <class T>
__global__ void __launch_bounds__(256)
    k_gemm_rm(int m, int n, int k, double alpha, const T* __restrict__ A, int64_t lda,
              const T* __restrict__ B, int64_t ldb, double beta, const T* Cin, int64_t ldcin, T* C,
              int64_t ldc, const int32_t* flag, int nflag) {
  if (flag) {
    for (int q = 0; q < nflag; ++q)
      if (flag[q]) return;
  }
  __shared__ T as[16][65];
  __shared__ T bs[16][65];
  const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  T acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int w = 0; w < 4; ++w) acc[u][w] = T(0.0);
  for (int k0 = 0; k0 < k; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e & 15, rr = e >> 4;         // A: 64 rows x 16 k (k fastest)
      const int i = r0 + rr, kq = k0 + kk;
      as[kk][rr] = (i < m && kq < k) ? A[(int64_t)i * lda + kq] : T(0.0);
      const int cc = e & 63, kb = e >> 6;         // B: 16 k x 64 cols (cols fastest)
      const int j = c0 + cc, kr = k0 + kb;
      bs[kb][cc] = (j < n && kr < k) ? B[(int64_t)kr * ldb + j] : T(0.0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      T ar[4], br[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { ar[u] = as[kk][ty * 4 + u]; br[u] = bs[kk][tx * 4 + u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[u][w] += ar[u] * br[w];
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const int i = r0 + ty * 4 + u, j = c0 + tx * 4 + w;
      if (i < m && j < n) {
        T v = acc[u][w] * alpha;
        if (beta != 0.0) v += Cin[(int64_t)i * ldcin + j] * beta;
        C[(int64_t)i * ldc + j] = v;
      }
    }
}

// A = D (+ children Lambda on the diagonal blocks) (+ regularize I); also
// copies L, R of the box into the workspace
template <class T>
__global__ void k_fb_gather(const SkelFactorLevel F, int a, int n, int k, T* A, T* Lw, T* Rw) {
  const T* D = reinterpret_cast<const T*>(F.D) + F.d_off[a];
  const T* Lg = reinterpret_cast<const T*>(F.L) + F.l_off[a];
  const T* Rg = reinterpret_cast<const T*>(F.R) + F.r_off[a];
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = tid; e < (int64_t)n * n; e += nt) A[e] = D[e];
  for (int64_t e = tid; e < (int64_t)n * k; e += nt) { Lw[e] = Lg[e]; Rw[e] = Rg[e]; }
}

template <class T>
__global__ void k_fb_diag(const SkelFactorLevel F, int a, int n, T* A) {
  // children Lambda blocks (solver.py:226-233) and regularize; one block per child
  if (F.child_off) {
    const int64_t c0 = F.child_off[a], c1 = F.child_off[a + 1];
    int ro = 0;
    for (int64_t c = c0; c < c1; ++c) {
      const int kc = F.prev_k[c];
      if (c - c0 == blockIdx.x) {
        const T* lam = reinterpret_cast<const T*>(F.prev_lam) + F.prev_lam_off[c];
        for (int e = threadIdx.x; e < kc * kc; e += blockDim.x) {
          const int i = e / kc, j = e - i * kc;
          A[(int64_t)(ro + i) * n + ro + j] = lam[e];
        }
      }
      ro += kc;
    }
  }
}

template <class T>
__global__ void k_add_diag(T* A, int n, double reg, const int32_t* flag) {
  if (flag && *flag) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) A[(int64_t)i * n + i] += T(reg);
}

// column abs sums of a row-major m x n matrix (atomic partial sums per 64 rows)
template <class T>
__global__ void k_colabs(const T* A, int m, int n, double* colsum, const int32_t* flag) {
  if (flag && *flag) return;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int i0 = blockIdx.y * 64, i1 = min(m, i0 + 64);
  double s = 0.0;
  for (int i = i0; i < i1; ++i) s += sk_abs(A[(int64_t)i * n + j]);
  atomicAdd(colsum + j, s);
}

// status / rcond of the box from the column sums (slots: 0 nA, 1 nAi, 2 nM, 3 nMi)
__global__ void k_fb_finish(const SkelFactorLevel F, int a, int n, int k, const double* cs,
                            const int32_t* stD, const int32_t* stM) {
  __shared__ double mx[4];
  if (threadIdx.x < 4) mx[threadIdx.x] = 0.0;
  __syncthreads();
  const int len[4] = {n, n, k, k};
  for (int q = 0; q < 4; ++q) {
    double v = 0.0;
    for (int j = threadIdx.x; j < len[q]; j += blockDim.x) v = fmax(v, cs[(int64_t)q * n + j]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0)
      atomicMax(reinterpret_cast<unsigned long long*>(mx + q), (unsigned long long)__double_as_longlong(v));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double nA = mx[0], nAi = mx[1], nM = mx[2], nMi = mx[3];
    if (*stD) { F.status[a] = 1; F.rcond_d[a] = 0.0; F.rcond_m[a] = 0.0; return; }
    const double rcd = (nA * nAi > 0.0) ? 1.0 / (nA * nAi) : 0.0;
    if (*stM) { F.status[a] = 2; F.rcond_d[a] = rcd; F.rcond_m[a] = 0.0; return; }
    F.status[a] = 0;
    F.rcond_d[a] = rcd;
    F.rcond_m[a] = k == 0 ? 1.0 : ((nM * nMi > 0.0) ? 1.0 / (nM * nMi) : 0.0);
  }
}

template <class T>
__global__ void k_copy_flag(T* dst, const T* src, int64_t cnt, const int32_t* flag) {
  if (flag && (flag[0] || flag[1])) return;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = tid; e < cnt; e += nt) dst[e] = src[e];
}

// ---------------------------------------------------------------------------
// launchers

template <class K>
static int coop_grid(K kernel, int threads, size_t smem) {
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, smem);
  if (per < 1) per = 1;
  if (per > 2) per = 2;
  return per * skel_sm_count();
}

template <class T>
static int cpqr_big_impl(void* W, int m, int n, int64_t ld, double eps, int min_rank, int resume,
                         void* state, cudaStream_t st) {
  // resume bit 0: continue a previous run; bit 1: equalisation -- stop after
  // exactly min_rank steps (see cpqr_run in cpqr.cuh)
  const int kcap = (resume & 2) ? min_rank : 0x7fffffff;
  if (!(resume & 1)) {
    int blocks = (n * 32 + 255) / 256;
    if (blocks < 1) blocks = 1;
    k_cpqr_big_init<T><<<blocks, 256, 0, st>>>((const T*)W, m, n, ld, state);
    SKEL_TRY(cudaGetLastError());
  }
  if (m <= 0 || n <= 0) return 0;
  size_t smem = sizeof(T) * (size_t)m;
  int vsmem = smem <= (size_t)skel_smem_optin() - 1024;
  if (!vsmem) smem = 0;
  SKEL_TRY(cudaFuncSetAttribute(k_cpqr_big<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = coop_grid(k_cpqr_big<T>, 256, smem);
  if (grid > 4096) grid = 4096;
  // scratch behind the state: second position map + 2 x 4096 candidates
  unsigned char* extra = (unsigned char*)state + 256 + (size_t)n * (3 * sizeof(double) + sizeof(int));
  extra = (unsigned char*)(((uintptr_t)extra + 15) / 16 * 16);
  int* pivb = (int*)extra;
  double* cand_v = (double*)(extra + (((size_t)n * sizeof(int) + 15) / 16) * 16);
  int* cand_i = (int*)(cand_v + 2 * 4096);
  T* Wp = (T*)W;
  int kc = kcap;
  void* args[] = {&Wp, &m, &n, &ld, &eps, &min_rank, &state, &vsmem, &pivb, &cand_v, &cand_i, &kc};
  SKEL_TRY(cudaLaunchCooperativeKernel((const void*)k_cpqr_big<T>, grid, 256, args, smem, st));
  return 0;
}

template <class T>
static int gj_impl(void* A, int n, double regularize, int32_t* status, void* scratch, cudaStream_t st,
                   const int32_t* skip = nullptr) {
  const size_t smem = sizeof(T) * (size_t)(n > 0 ? n : 1);
  SKEL_TRY(cudaFuncSetAttribute(k_gj_coop<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int grid = coop_grid(k_gj_coop<T>, 256, smem);
  if (grid > 4096) grid = 4096;
  unsigned char* p = (unsigned char*)scratch;
  double* part_v = (double*)p;                       // 2 x 4096 (double-buffered)
  int* part_i = (int*)(p + 2 * 4096 * sizeof(double));
  T* colc = (T*)(p + 2 * 4096 * (sizeof(double) + sizeof(int)));
  int* swaps = (int*)((unsigned char*)colc + (size_t)n * 16);
  T* Ap = (T*)A;
  void* args[] = {&Ap, &n, &regularize, &status, &part_v, &part_i, &colc, &swaps, &skip};
  SKEL_TRY(cudaLaunchCooperativeKernel((const void*)k_gj_coop<T>, grid, 256, args, smem, st));
  k_gj_unswap<T><<<(n + 127) / 128, 128, 0, st>>>(Ap, n, swaps, status, skip);
  return skel_last_error();
}

template <class T>
static int gemm_rm(int m, int n, int k, double alpha, const T* A, int64_t lda, const T* B, int64_t ldb,
                   double beta, const T* Cin, int64_t ldcin, T* C, int64_t ldc, const int32_t* flag,
                   int nflag, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  dim3 grid((n + 63) / 64, (m + 63) / 64);
  k_gemm_rm<T><<<grid, 256, 0, st>>>(m, n, k, alpha, A, lda, B, ldb, beta, Cin, ldcin, C, ldc, flag,
                                     nflag);
  return skel_last_error();
}

template <class T>
static int factor_big_impl(const SkelFactorLevel* F, int a, int n, int k, int64_t dd_off,
                           int64_t ld_off, int64_t rd_off, int64_t lam_off, void* work, int64_t wbytes,
                           cudaStream_t st) {
  // workspace: flags(2 int, padded) | colsums 4n doubles | gj scratch | A n^2 | L nk | R kn | X nk | Y kn | M k^2
  unsigned char* p = (unsigned char*)work;
  int32_t* flags = (int32_t*)p;                        // [0] D singular, [1] Lambda singular
  double* cs = (double*)(p + 64);
  unsigned char* gjs = p + 64 + 4 * (size_t)n * sizeof(double);
  const size_t gjb = ((size_t)skel_gj_scratch_bytes(n) + 255) / 256 * 256;
  T* A = (T*)(gjs + gjb);
  T* Lw = A + (size_t)n * n;
  T* Rw = Lw + (size_t)n * k;
  T* X = Rw + (size_t)k * n;
  T* Y = X + (size_t)n * k;
  T* M = Y + (size_t)k * n;
  const size_t need = (size_t)((unsigned char*)(M + (size_t)k * k) - p);
  if ((size_t)wbytes < need) return -2;
  SKEL_TRY(cudaMemsetAsync(work, 0, 64 + 4 * (size_t)n * sizeof(double), st));
  const int sms = skel_sm_count();
  k_fb_gather<T><<<2 * sms, 256, 0, st>>>(*F, a, n, k, A, Lw, Rw);
  if (F->child_off) k_fb_diag<T><<<8, 256, 0, st>>>(*F, a, n, A);
  if (F->regularize != 0.0) k_add_diag<T><<<(n + 255) / 256, 256, 0, st>>>(A, n, F->regularize, nullptr);
  dim3 gcs((n + 127) / 128, (n + 63) / 64);
  k_colabs<T><<<gcs, 128, 0, st>>>(A, n, n, cs, nullptr);
  int rc = gj_impl<T>(A, n, 0.0, flags, gjs, st);
  if (rc) return rc;
  k_colabs<T><<<gcs, 128, 0, st>>>(A, n, n, cs + n, flags);
  T* Dd = reinterpret_cast<T*>(F->Dd);
  if (k > 0) {
    if ((rc = gemm_rm<T>(n, k, n, 1.0, A, n, Lw, k, 0.0, nullptr, 0, X, k, flags, 1, st))) return rc;   // X = D^-1 L
    if ((rc = gemm_rm<T>(k, n, n, 1.0, Rw, n, A, n, 0.0, nullptr, 0, Y, n, flags, 1, st))) return rc;   // Y = R D^-1
    if ((rc = gemm_rm<T>(k, k, n, 1.0, Rw, n, X, k, 0.0, nullptr, 0, M, k, flags, 1, st))) return rc;   // M = R X
    dim3 gm((k + 127) / 128, (k + 63) / 64);
    k_colabs<T><<<gm, 128, 0, st>>>(M, k, k, cs + 2 * n, flags);
    if (F->regularize != 0.0) k_add_diag<T><<<(k + 255) / 256, 256, 0, st>>>(M, k, F->regularize, flags);
    if ((rc = gj_impl<T>(M, k, 0.0, flags + 1, gjs, st, flags))) return rc;
    k_colabs<T><<<gm, 128, 0, st>>>(M, k, k, cs + 3 * n, flags);
    T* Rd = reinterpret_cast<T*>(F->Rd) + rd_off;
    T* Ld = reinterpret_cast<T*>(F->Ld) + ld_off;
    // Rd = Lam Y, Ld = X Lam, Dd = D^-1 - X Rd (the flag covers both singular cases)
    if ((rc = gemm_rm<T>(k, n, k, 1.0, M, k, Y, n, 0.0, nullptr, 0, Rd, n, flags, 2, st))) return rc;
    if ((rc = gemm_rm<T>(n, k, k, 1.0, X, k, M, k, 0.0, nullptr, 0, Ld, k, flags, 2, st))) return rc;
    if ((rc = gemm_rm<T>(n, n, k, -1.0, X, k, Rd, n, 1.0, A, n, Dd + dd_off, n, flags, 2, st))) return rc;
    k_copy_flag<T><<<sms, 256, 0, st>>>(reinterpret_cast<T*>(F->Lam) + lam_off, M, (int64_t)k * k, flags);
  } else {
    k_copy_flag<T><<<sms, 256, 0, st>>>(Dd + dd_off, A, (int64_t)n * n, flags);
  }
  k_fb_finish<<<1, 256, 0, st>>>(*F, a, n, k, cs, flags, flags + 1);
  return skel_last_error();
}

extern "C" {

int64_t skel_big_state_bytes(int32_t n) {
  return 256 + (int64_t)n * (3 * sizeof(double) + sizeof(int)) + 16 + ((int64_t)n * 4 + 15) / 16 * 16 +
         2 * 4096 * (int64_t)(sizeof(double) + sizeof(int)) + 64;
}

int skel_big_target(const SkelSource* src, const SkelLevel* lv, int32_t box, int32_t side,
                    const int32_t* nbr_box, const int32_t* nbr_pref, int32_t nnb, int32_t m,
                    int32_t n, void* W, int64_t ld, int32_t field, void* stream) {
  if (m <= 0 || n <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((m + 127) / 128, (n + 63) / 64);
  if (field == 0)
    k_big_target<double><<<grid, 128, 0, st>>>(*src, *lv, box, side, nbr_box, nbr_pref, nnb, m,
                                                (double*)W, ld);
  else
    k_big_target<zc><<<grid, 128, 0, st>>>(*src, *lv, box, side, nbr_box, nbr_pref, nnb, m, (zc*)W, ld);
  return skel_last_error();
}

int skel_cpqr_big(void* W, int32_t m, int32_t n, int64_t ld, double eps, int32_t min_rank,
                  int32_t resume, void* state, int32_t field, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  return field == 0 ? cpqr_big_impl<double>(W, m, n, ld, eps, min_rank, resume, state, st)
                    : cpqr_big_impl<zc>(W, m, n, ld, eps, min_rank, resume, state, st);
}

int skel_big_interp(void* W, int32_t n, int64_t ld, void* state, int32_t min_rank, int32_t field,
                    void* stream) {
  // the rank lives on the device: size the staging for r <= n
  cudaStream_t st = (cudaStream_t)stream;
  const size_t col = (size_t)(n > 0 ? n : 1) * (field ? 16 : 8);
  int wpb = (int)((size_t)skel_smem_optin() / col);
  if (wpb > 4) wpb = 4;
  if (wpb < 1) return -2;
  int blocks = (n + wpb - 1) / wpb;
  if (blocks < 1) blocks = 1;
  const size_t smem = wpb * col;
  if (field == 0) {
    SKEL_TRY(cudaFuncSetAttribute(k_big_interp<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_big_interp<double><<<blocks, 32 * wpb, smem, st>>>((double*)W, n, ld, state, min_rank);
  } else {
    SKEL_TRY(cudaFuncSetAttribute(k_big_interp<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_big_interp<zc><<<blocks, 32 * wpb, smem, st>>>((zc*)W, n, ld, state, min_rank);
  }
  return skel_last_error();
}

int skel_big_output(const SkelLevel* lv, int32_t box, int32_t side, const void* W, int64_t ld,
                    const void* state, int32_t n, int32_t field, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const size_t smem = sizeof(int) * (size_t)(n > 0 ? n : 1);
  const int blocks = 2 * skel_sm_count();
  if (field == 0) {
    SKEL_TRY(cudaFuncSetAttribute(k_big_output<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_big_output<double><<<blocks, 256, smem, st>>>(*lv, box, side, (const double*)W, ld, state, n);
  } else {
    SKEL_TRY(cudaFuncSetAttribute(k_big_output<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_big_output<zc><<<blocks, 256, smem, st>>>(*lv, box, side, (const zc*)W, ld, state, n);
  }
  return skel_last_error();
}

int skel_gemm_tn(int32_t m, int32_t n, int32_t k, const void* X, int64_t ldx, const void* A,
                 int64_t lda, void* Y, int64_t ldy, int32_t field, void* stream) {
  if (m <= 0 || n <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((m + 63) / 64, (n + 63) / 64);
  if (field == 0)
    k_gemm_tn_dmma<<<grid, 128, 0, st>>>(m, n, k, (const double*)X, ldx, (const double*)A, lda,
                                         (double*)Y, ldy);
  else
    k_gemm_tn<zc><<<grid, 256, 0, st>>>(m, n, k, (const zc*)X, ldx, (const zc*)A, lda, (zc*)Y, ldy);
  return skel_last_error();
}

int skel_gemv(int32_t trans, int32_t m, int32_t n, const void* A, int64_t lda, const void* x, void* y,
              int32_t field, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int rows = trans == 0 ? m : n * 32;
  const int blocks = (rows + 255) / 256;
  if (blocks <= 0) return 0;
  if (field == 0)
    k_gemv<double><<<blocks, 256, 0, st>>>(trans, m, n, (const double*)A, lda, (const double*)x, (double*)y);
  else
    k_gemv<zc><<<blocks, 256, 0, st>>>(trans, m, n, (const zc*)A, lda, (const zc*)x, (zc*)y);
  return skel_last_error();
}

int skel_big_probe(int32_t m, int32_t n, const void* A, int64_t lda, const void* Ysk, int64_t ldy,
                   const void* state, const void* v, void* u, void* z, int32_t field, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int bu = (n + 127) / 128, bz = (m + 127) / 128;
  if (field == 0) {
    k_probe_pv<double><<<bu, 128, 0, st>>>((const double*)Ysk, n, ldy, state, (const double*)v, (double*)u);
    k_probe_z<double><<<bz, 128, 0, st>>>(m, n, (const double*)A, lda, state, (const double*)v,
                                          (const double*)u, (double*)z);
  } else {
    k_probe_pv<zc><<<bu, 128, 0, st>>>((const zc*)Ysk, n, ldy, state, (const zc*)v, (zc*)u);
    k_probe_z<zc><<<bz, 128, 0, st>>>(m, n, (const zc*)A, lda, state, (const zc*)v, (const zc*)u, (zc*)z);
  }
  return skel_last_error();
}

int64_t skel_gj_scratch_bytes(int32_t n) {
  return 2 * 4096 * (int64_t)(sizeof(double) + sizeof(int)) + (int64_t)n * (16 + sizeof(int)) + 256;
}

// Shat^-1 in place for big K (status 1: exact zero pivot).  The caller zeroes
// *status first.
int skel_dense_inverse_big(void* A, int32_t n, double regularize, int32_t* status, int32_t field,
                           void* scratch, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  return field == 0 ? gj_impl<double>(A, n, regularize, status, scratch, st)
                    : gj_impl<zc>(A, n, regularize, status, scratch, st);
}

int64_t skel_factor_big_bytes(int32_t n, int32_t k, int32_t field) {
  const int64_t el = field ? 16 : 8;
  const int64_t gjb = (skel_gj_scratch_bytes(n) + 255) / 256 * 256;
  return 64 + 4 * (int64_t)n * 8 + gjb + el * ((int64_t)n * n + 4 * (int64_t)n * k + (int64_t)k * k) + 256;
}

// factor_node of ONE big box over the whole GPU (status / rcond / outputs as
// skel_factor_level); the box's output offsets are passed by the host.
int skel_factor_big(const SkelFactorLevel* F, int32_t box, int32_t n, int32_t k, int64_t dd_off,
                    int64_t ld_off, int64_t rd_off, int64_t lam_off, void* work, int64_t work_bytes,
                    int32_t field, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  return field == 0 ? factor_big_impl<double>(F, box, n, k, dd_off, ld_off, rd_off, lam_off, work,
                                              work_bytes, st)
                    : factor_big_impl<zc>(F, box, n, k, dd_off, ld_off, rd_off, lam_off, work,
                                          work_bytes, st);
}

// LU with partial pivoting of a row-major n x n matrix in place (getrf
// conventions, 0-based piv); *status (zeroed by the caller) = 1 on an exact
// zero pivot.  scratch: skel_gj_scratch_bytes(n).
int skel_dense_lu(void* A, int32_t n, int32_t* piv, int32_t* status, int32_t field, void* scratch,
                  void* stream) {
  if (n <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  auto run = [&](auto kern, size_t el) -> int {
    const size_t smem = el * (size_t)n;
    SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int grid = coop_grid(kern, 256, smem);
    if (grid > 4096) grid = 4096;
    unsigned char* p = (unsigned char*)scratch;
    double* part_v = (double*)p;
    int* part_i = (int*)(p + 2 * 4096 * sizeof(double));
    void* colc = (void*)(p + 2 * 4096 * (sizeof(double) + sizeof(int)));
    void* Ap = A;
    void* args[] = {&Ap, &n, &status, &part_v, &part_i, &colc, &piv};
    SKEL_TRY(cudaLaunchCooperativeKernel((const void*)kern, grid, 256, args, smem, st));
    return 0;
  };
  return field == 0 ? run(k_lu_coop<double>, 8) : run(k_lu_coop<zc>, 16);
}

// inv (row-major n x n) = A^-1 from skel_dense_lu / getrf factors.
int skel_lu_inverse(const void* lu, const int32_t* piv, int32_t n, void* inv, int32_t field, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const size_t col = (size_t)n * (field ? 16 : 8);
  int wpb = (int)((size_t)skel_smem_optin() / col);
  if (wpb > 8) wpb = 8;
  if (wpb < 1) return -2;
  const size_t smem = wpb * col;
  const int blocks = (n + wpb - 1) / wpb;
  if (field == 0) {
    SKEL_TRY(cudaFuncSetAttribute(k_lu_inverse<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_lu_inverse<double><<<blocks, 32 * wpb, smem, st>>>((const double*)lu, piv, n, (double*)inv);
  } else {
    SKEL_TRY(cudaFuncSetAttribute(k_lu_inverse<zc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_lu_inverse<zc><<<blocks, 32 * wpb, smem, st>>>((const zc*)lu, piv, n, (zc*)inv);
  }
  return skel_last_error();
}

}  // extern "C"
