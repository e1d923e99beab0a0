// id_level.cuh -- K1 + K2: fused proxy-target assembly and CPQR interpolative
// decomposition for every box of one cover, both sides, on one 2-CTA cluster
// per box.  Also the explicit batched ID, top-level S assembly, dense block
// evaluation and the on-the-fly dense matvec (K6).
//
// Reference work replaced: build_node (skel.py:341-391), _run_id (414-422),
// id_fixed_precision / pivoted_qr / _proj_from_qr (lowrank.py:48-161),
// S assembly (skel.py:399-408), eval_block (kernels.py:82-161),
// BieSystem.matrix() @ x (bie.py:174-176).
//
// Cluster (2,1,1): CTA 0 runs the row ID on t_row.T, CTA 1 the column ID on
// t_col.  Equalisation (skel.py:377-382) needs both ranks: each CTA stores its
// rank into the partner's shared memory (DSMEM) and the smaller side simply
// continues its own CPQR to k = max(kr, kc) -- identical to the reference's
// re-run with min_rank = k because the CPQR is a deterministic state machine
// whose first steps do not depend on min_rank.
#pragma once
#include <cooperative_groups.h>
#include <cstdlib>

#include "cpqr.cuh"
#include "entries.cuh"

namespace cg = cooperative_groups;

#define SKEL_MAX_NBR 256
#define SKEL_MAX_CHILD 8

struct LevelSmemHdr {
  int nbr_pref[SKEL_MAX_NBR + 1];
  int nbr_box[SKEL_MAX_NBR];
  int rsplit[SKEL_MAX_CHILD + 1];
  int csplit[SKEL_MAX_CHILD + 1];
  int nch;
  int err;
  double red[32];
};

static __host__ __device__ inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

template <class T>
static __host__ __device__ inline size_t level_smem_fixed(int max_n) {
  size_t s = align_up(sizeof(CpqrShared<T>), 16);
  s += align_up(sizeof(LevelSmemHdr), 16);
  s += align_up(sizeof(Pt) * (size_t)max_n, 16);
  s += align_up(3 * sizeof(double) * (size_t)max_n, 16);
  s += align_up(2 * sizeof(int) * (size_t)max_n, 16);
  s += align_up(6 * sizeof(double) * (size_t)max_n, 16);   // fast-path column SoA
  return s;
}

__device__ __forceinline__ int find_run(const int* pref, int cnt, int i) {
  int q = 0;
  while (q + 1 < cnt && pref[q + 1] <= i) ++q;
  return q;
}

// Fast K1 for the 2D Laplace double-layer BIE (BASELINE configs 1/2/5):
// per-source constants hoisted (n.w/(2 pi), curvature limit), r^2 instead of
// sqrt(r)^2, log(r^2)/(4 pi) for the single-layer proxies, four entries per
// iteration for ILP.  Differs from numpy's evaluation order by a few ulps.
static __device__ __noinline__ void assemble_bie_lap2(const SkelSource& S, const SkelLevel& L, int a,
                                               int side, int n, int m, int m_nbr, int nnb_c,
                                               const int* nbr_pref, const int* nbr_box,
                                               const int32_t* mydofs, const Pt* cp, double* fsoa,
                                               int max_n, double* W, int ld) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const double inv2pi = 1.0 / SKEL_TWO_PI, inv4pi = 1.0 / SKEL_FOUR_PI;
  const double tol2 = S.coincide_tol * S.coincide_tol;
  const double ic = S.identity_coef;
  double* fx = fsoa;
  double* fy = fsoa + max_n;
  double* fa = fsoa + 2 * max_n;   // side 1 sources: nx w / 2pi
  double* fb = fsoa + 3 * max_n;   //                 ny w / 2pi
  double* fc = fsoa + 4 * max_n;   //                 curvature limit * w
  double* fw = fsoa + 5 * max_n;   //                 -w / 4pi (column proxies)
  for (int j = tid; j < n; j += nt) {
    const Pt q = cp[j];
    fx[j] = q.x;
    fy[j] = q.y;
    fa[j] = q.nx * q.w * inv2pi;
    fb[j] = q.ny * q.w * inv2pi;
    fc[j] = (-q.kap * inv4pi) * q.w;
    fw[j] = -q.w * inv4pi;
  }
  __syncthreads();
  const int pb = L.pxy_begin[a];
  const double rr = L.box_r[a];
  const double cx = L.box_c[(int64_t)a * 2], cy = L.box_c[(int64_t)a * 2 + 1];
  const double rowp = -S.wscale * inv4pi;
  for (int i = tid; i < m; i += nt) {
    double* Wi = W + i;
    if (i < m_nbr) {
      int q = find_run(nbr_pref, nnb_c + 1, i);
      int b = nbr_box[q];
      int off = i - nbr_pref[q];
      const int32_t idx = side == 0 ? L.cdofs[L.cdof_off[b] + off] : L.rdofs[L.rdof_off[b] + off];
      const double px = __ldg(S.x + idx), py = __ldg(S.y + idx);
      if (side == 0) {
        // row point is the SOURCE, box points are targets: t_row.T[i][j] = A(rd_j, nbr_i)
        const double w = __ldg(S.w + idx);
        const double sa = __ldg(S.nx + idx) * w * inv2pi, sb = __ldg(S.ny + idx) * w * inv2pi;
        const double sc = (-__ldg(S.curv + idx) * inv4pi) * w;
        int j = 0;
        for (; j + 3 < n; j += 4) {
          double v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double dx = fx[j + u] - px, dy = fy[j + u] - py;
            const double r2 = dx * dx + dy * dy;
            double e = (dx * sa + dy * sb) / r2;
            if (r2 < tol2) e = sc;
            if (mydofs[j + u] == idx) e += ic;
            v[u] = e;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) Wi[(int64_t)(j + u) * ld] = v[u];
        }
        for (; j < n; ++j) {
          const double dx = fx[j] - px, dy = fy[j] - py;
          const double r2 = dx * dx + dy * dy;
          double e = (dx * sa + dy * sb) / r2;
          if (r2 < tol2) e = sc;
          if (mydofs[j] == idx) e += ic;
          Wi[(int64_t)j * ld] = e;
        }
      } else {
        // row point is the TARGET, box points are sources: t_col[i][j] = A(nbr_i, cd_j)
        int j = 0;
        for (; j + 3 < n; j += 4) {
          double v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double dx = px - fx[j + u], dy = py - fy[j + u];
            const double r2 = dx * dx + dy * dy;
            double e = (dx * fa[j + u] + dy * fb[j + u]) / r2;
            if (r2 < tol2) e = fc[j + u];
            if (mydofs[j + u] == idx) e += ic;
            v[u] = e;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) Wi[(int64_t)(j + u) * ld] = v[u];
        }
        for (; j < n; ++j) {
          const double dx = px - fx[j], dy = py - fy[j];
          const double r2 = dx * dx + dy * dy;
          double e = (dx * fa[j] + dy * fb[j]) / r2;
          if (r2 < tol2) e = fc[j];
          if (mydofs[j] == idx) e += ic;
          Wi[(int64_t)j * ld] = e;
        }
      }
    } else {
      const int pr = pb + (i - m_nbr);
      const double px = __dadd_rn(cx, __dmul_rn(rr, L.pxy_unit[(int64_t)pr * 2]));
      const double py = __dadd_rn(cy, __dmul_rn(rr, L.pxy_unit[(int64_t)pr * 2 + 1]));
      int j = 0;
      for (; j + 3 < n; j += 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double dx = fx[j + u] - px, dy = fy[j + u] - py;
          const double r2 = dx * dx + dy * dy;
          // row proxy: wscale * (-log r / 2pi); column proxy: -log r / 2pi * w_j
          const double g = log(r2);
          v[u] = r2 < tol2 ? 0.0 : (side == 0 ? g * rowp : g * fw[j + u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) Wi[(int64_t)(j + u) * ld] = v[u];
      }
      for (; j < n; ++j) {
        const double dx = fx[j] - px, dy = fy[j] - py;
        const double r2 = dx * dx + dy * dy;
        const double g = log(r2);
        Wi[(int64_t)j * ld] = r2 < tol2 ? 0.0 : (side == 0 ? g * rowp : g * fw[j]);
      }
    }
  }
}

template <class T, int GL, int RPL, bool GW, int NT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT)
    k_id_level(const SkelSource S, const SkelLevel L, const int32_t* __restrict__ order,
               int64_t max_w, int max_n) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* p = smem;
  CpqrShared<T>& sh = *reinterpret_cast<CpqrShared<T>*>(p);
  p += align_up(sizeof(CpqrShared<T>), 16);
  LevelSmemHdr& hd = *reinterpret_cast<LevelSmemHdr*>(p);
  p += align_up(sizeof(LevelSmemHdr), 16);
  Pt* cp = reinterpret_cast<Pt*>(p);
  p += align_up(sizeof(Pt) * (size_t)max_n, 16);
  double* nrm = reinterpret_cast<double*>(p);
  double* ref = nrm + max_n;
  double* xn2 = ref + max_n;
  p += align_up(3 * sizeof(double) * (size_t)max_n, 16);
  int* piv = reinterpret_cast<int*>(p);
  int* pos = piv + max_n;
  p += align_up(2 * sizeof(int) * (size_t)max_n, 16);
  double* fsoa = reinterpret_cast<double*>(p);
  p += align_up(6 * sizeof(double) * (size_t)max_n, 16);
  T* W = GW ? reinterpret_cast<T*>(L.scratch) + (size_t)blockIdx.x * max_w
            : reinterpret_cast<T*>(p);

  const int side = blockIdx.x & 1;
  const int a = order[blockIdx.x >> 1];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (L.debug_skip == 3) { if (tid == 0) (side == 0 ? L.kr : L.kc)[a] = 0; return; }
  const bool eq = L.equalize != 0;

  const int64_t r0 = L.rdof_off[a], c0 = L.cdof_off[a];
  const int nr = (int)(L.rdof_off[a + 1] - r0), nc = (int)(L.cdof_off[a + 1] - c0);
  const int n = side == 0 ? nr : nc;
  const int32_t* mydofs = side == 0 ? L.rdofs + r0 : L.cdofs + c0;
  const int64_t nb0 = L.nbr_off[a];
  const int nnb = (int)(L.nbr_off[a + 1] - nb0);
  const int npx = L.pxy_count[a];

  if (tid == 0) {
    sh.rank = 0; sh.stop = 0; sh.p0 = 0.0; sh.pad = 0; sh.bigP = 0.0; sh.partner_k = 0; sh.trail = 0.0;
    hd.err = nnb > SKEL_MAX_NBR;
    int acc = 0;
    hd.nbr_pref[0] = 0;
    for (int q = 0; q < nnb && q < SKEL_MAX_NBR; ++q) {
      int b = L.nbr[nb0 + q];
      hd.nbr_box[q] = b;
      int cnt = side == 0 ? (int)(L.cdof_off[b + 1] - L.cdof_off[b])
                          : (int)(L.rdof_off[b + 1] - L.rdof_off[b]);
      acc += cnt;
      hd.nbr_pref[q + 1] = acc;
    }
    int nch = 0;
    hd.rsplit[0] = 0; hd.csplit[0] = 0;
    if (L.child_off) {
      int64_t ch0 = L.child_off[a], ch1 = L.child_off[a + 1];
      nch = (int)(ch1 - ch0);
      if (nch > SKEL_MAX_CHILD) { hd.err = 1; nch = SKEL_MAX_CHILD; }
      for (int q = 0; q < nch; ++q) {
        hd.rsplit[q + 1] = hd.rsplit[q] + L.prev_kr[ch0 + q];
        hd.csplit[q + 1] = hd.csplit[q] + L.prev_kc[ch0 + q];
      }
    }
    hd.nch = nch;
  }
  for (int j = tid; j < n; j += nt) cp[j] = load_pt(S, mydofs[j]);
  __syncthreads();
  // cluster arrive only AFTER sh.partner_k was initialised (release
  // semantics): the partner's DSMEM rank store (after its wait, below) can
  // then never be overwritten by this CTA's initialisation
  if (eq) asm volatile("barrier.cluster.arrive.aligned;\n" ::: "memory");
  const int nnb_c = nnb < SKEL_MAX_NBR ? nnb : SKEL_MAX_NBR;
  const int m_nbr = hd.nbr_pref[nnb_c];
  const int m = m_nbr + npx;
  // real targets: even leading dimension with a zero pad row (cpqr_update_pr)
  const int ld = sizeof(T) == sizeof(double) ? ((m + 1) & ~1) : m;

  // ---- K1: assemble the proxy-compressed target, column-major ----------
  const bool fast = sizeof(T) == sizeof(double) && S.kind == SKEL_SRC_BIE &&
                    S.equation == SKEL_EQ_LAPLACE && S.dim == 2 && !S.kr10 && S.curvature_limit;
  if (fast && n > 0) {
    assemble_bie_lap2(S, L, a, side, n, m, m_nbr, nnb_c, hd.nbr_pref, hd.nbr_box, mydofs, cp,
                      fsoa, max_n, reinterpret_cast<double*>(W), ld);
  } else if (n > 0) {
    const int pb = L.pxy_begin[a];
    const double rr = L.box_r[a];
    const int dim = S.dim;
    for (int i = tid; i < m; i += nt) {
      if (i < m_nbr) {
        int q = find_run(hd.nbr_pref, nnb_c + 1, i);
        int b = hd.nbr_box[q];
        int off = i - hd.nbr_pref[q];
        int32_t idx = side == 0 ? L.cdofs[L.cdof_off[b] + off] : L.rdofs[L.rdof_off[b] + off];
        Pt rp = load_pt(S, idx);
        if (side == 0) {
          for (int j = 0; j < n; ++j) W[(int64_t)j * ld + i] = entry_A<T>(S, cp[j], rp);
        } else {
          for (int j = 0; j < n; ++j) W[(int64_t)j * ld + i] = entry_A<T>(S, rp, cp[j]);
        }
      } else {
        int pr = pb + (i - m_nbr);
        // proxy point c + r*u (skel.py:87-96), rounded as numpy does
        double px = __dadd_rn(L.box_c[(int64_t)a * dim + 0], __dmul_rn(rr, L.pxy_unit[(int64_t)pr * dim + 0]));
        double py = __dadd_rn(L.box_c[(int64_t)a * dim + 1], __dmul_rn(rr, L.pxy_unit[(int64_t)pr * dim + 1]));
        double pz = dim == 3 ? __dadd_rn(L.box_c[(int64_t)a * dim + 2], __dmul_rn(rr, L.pxy_unit[(int64_t)pr * dim + 2])) : 0.0;
        if (side == 0) {
          for (int j = 0; j < n; ++j) W[(int64_t)j * ld + i] = entry_proxy_row<T>(S, cp[j], px, py, pz);
        } else {
          for (int j = 0; j < n; ++j) W[(int64_t)j * ld + i] = entry_proxy_col<T>(S, px, py, pz, cp[j]);
        }
      }
    }
  }
  if (ld > m)
    for (int j = tid; j < n; j += nt) W[(int64_t)j * ld + m] = T(0.0);
  __syncthreads();

  // ---- K2: CPQR ID ---------------------------------------------------------
  if (L.debug_skip == 1) { if (tid == 0) (side == 0 ? L.kr : L.kc)[a] = 0; return; }
  cpqr_init<T>(W, m, n, ld, nrm, ref, xn2, piv, sh);
  __syncthreads();
  if (L.debug_skip == 2) { if (tid == 0) (side == 0 ? L.kr : L.kc)[a] = 0; return; }
  cpqr_run<T, GL, RPL>(W, m, n, ld, nrm, ref, xn2, piv, sh, L.eps, 0);
  if (L.debug_skip == 4) { if (tid == 0) (side == 0 ? L.kr : L.kc)[a] = 0; return; }
  int min_rank = 0;
  if (eq) {
    cg::cluster_group cl = cg::this_cluster();
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    if (tid == 0) {
      int* remote = cl.map_shared_rank(&sh.partner_k, side ^ 1);
      *remote = sh.rank;
    }
    cl.sync();
    const int k = sh.rank > sh.partner_k ? sh.rank : sh.partner_k;
    if (sh.rank < k) {
      min_rank = k;
      cpqr_run<T, GL, RPL>(W, m, n, ld, nrm, ref, xn2, piv, sh, L.eps, k, k);
    }
  }
  if (L.debug_skip == 5) { if (tid == 0) (side == 0 ? L.kr : L.kc)[a] = 0; return; }
  interp_solve<T>(W, n, ld, piv, sh, min_rank, hd.red);
  if (L.debug_skip == 6) { if (tid == 0) (side == 0 ? L.kr : L.kc)[a] = 0; return; }
  const int r = sh.rank;
  const int K = r + sh.pad;
  for (int s = tid; s < K; s += nt) {
    int ps = piv[s], c = 0;
    for (int t = 0; t < K; ++t) c += piv[t] < ps;
    pos[s] = c;
  }
  __syncthreads();

  // ---- outputs: sorted skeletons, L (n x K) or R (K x n) ------------------
  int32_t* skel = side == 0 ? L.rskel + r0 : L.cskel + c0;
  for (int s = tid; s < K; s += nt) skel[pos[s]] = mydofs[piv[s]];
  if (side == 0) {
    T* Lo = reinterpret_cast<T*>(L.L) + L.l_off[a];
    for (int e = tid; e < n * K; e += nt) {
      int q = e / K, s = e - q * K;
      Lo[(int64_t)piv[q] * K + pos[s]] = interp_entry<T>(W, ld, piv, r, K, s, q);
    }
  } else {
    T* Ro = reinterpret_cast<T*>(L.R) + L.r_off[a];
    for (int e = tid; e < n * K; e += nt) {
      int s = e / n, q = e - s * n;
      Ro[(int64_t)pos[s] * n + piv[q]] = interp_entry<T>(W, ld, piv, r, K, s, q);
    }
  }
  if (tid == 0) {
    (side == 0 ? L.kr : L.kc)[a] = K;
    int f = (sh.bigP > 2.0 ? (1 << side) : 0) | (hd.err ? 8 : 0);
    if (f) atomicOr(L.flags + a, f);
  }
}

// D = A(rd, cd) with the children's diagonal blocks zeroed (skel.py:344-348).
// One CTA (or, for few big boxes, gridDim.y CTAs splitting the rows) per box;
// column points staged in shared memory in chunks of `chunk`, each warp owns
// a row and reads its point once from global memory.
template <class T>
__global__ void __launch_bounds__(128) k_assemble_D(const SkelSource S, const SkelLevel L, int chunk,
                                                    const int32_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char smem[];
  Pt* cpp = reinterpret_cast<Pt*>(smem);
  __shared__ int rsplit[SKEL_MAX_CHILD + 1], csplit[SKEL_MAX_CHILD + 1], nch_s;
  const int a = order ? order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t r0 = L.rdof_off[a], c0 = L.cdof_off[a];
  const int nr = (int)(L.rdof_off[a + 1] - r0), nc = (int)(L.cdof_off[a + 1] - c0);
  if (nr == 0 || nc == 0) return;
  if (tid == 0) {
    int nch = 0;
    rsplit[0] = 0; csplit[0] = 0;
    if (L.child_off) {
      const int64_t ch0 = L.child_off[a];
      nch = (int)(L.child_off[a + 1] - ch0);
      if (nch > SKEL_MAX_CHILD) nch = SKEL_MAX_CHILD;
      for (int q = 0; q < nch; ++q) {
        rsplit[q + 1] = rsplit[q] + L.prev_kr[ch0 + q];
        csplit[q + 1] = csplit[q] + L.prev_kc[ch0 + q];
      }
    }
    nch_s = nch;
  }
  T* D = reinterpret_cast<T*>(L.D) + L.d_off[a];
  const bool fast = sizeof(T) == sizeof(double) && S.kind == SKEL_SRC_BIE &&
                    S.equation == SKEL_EQ_LAPLACE && S.dim == 2 && !S.kr10 && S.curvature_limit;
  const double inv2pi = 1.0 / SKEL_TWO_PI, inv4pi = 1.0 / SKEL_FOUR_PI;
  const double tol2 = S.coincide_tol * S.coincide_tol;
  const int nw = nt / 32, wid = tid / 32, lane = tid & 31;
  for (int j0 = 0; j0 < nc; j0 += chunk) {
    const int jn = min(chunk, nc - j0);
    __syncthreads();
    for (int j = tid; j < jn; j += nt) cpp[j] = load_pt(S, L.cdofs[c0 + j0 + j]);
    __syncthreads();
    const int nch = nch_s;
    for (int i = blockIdx.y * nw + wid; i < nr; i += nw * gridDim.y) {
      const int ci = nch > 0 ? find_run(rsplit, nch + 1, i) : -1;
      const Pt tp = load_pt(S, L.rdofs[r0 + i]);
      for (int jj = lane; jj < jn; jj += 32) {
        const int j = j0 + jj;
        T v = T(0.0);
        const bool zero = nch > 0 && ci == find_run(csplit, nch + 1, j);
        if (!zero) {
          const Pt& sp = cpp[jj];
          if (fast) {
            const double dx = tp.x - sp.x, dy = tp.y - sp.y;
            const double r2 = dx * dx + dy * dy;
            double e = (dx * (sp.nx * sp.w * inv2pi) + dy * (sp.ny * sp.w * inv2pi)) / r2;
            if (r2 < tol2) e = (-sp.kap * inv4pi) * sp.w;
            if (tp.o == sp.o) e += S.identity_coef;
            v = as_T<T>(e);
          } else {
            v = entry_A<T>(S, tp, sp);
          }
        }
        D[(int64_t)i * nc + j] = v;
      }
    }
  }
}

// explicit batched ID (id_fixed_precision), one CTA per matrix
template <class T, int GL, int RPL, bool GW>
__global__ void __launch_bounds__(128)
    k_id_batched(const T* __restrict__ A, const int64_t* a_off, const int32_t* mm,
                 const int32_t* nn, double eps, const int32_t* min_rank_arr, int32_t* rank_out,
                 int32_t* skel_out, const int64_t* skel_off, T* proj, const int64_t* proj_off,
                 double* bigP_out, double* ratio_out, T* scratch, int max_m, int max_n, T* rfac,
                 const int64_t* rfac_off) {
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* p = smem;
  CpqrShared<T>& sh = *reinterpret_cast<CpqrShared<T>*>(p);
  p += align_up(sizeof(CpqrShared<T>), 16);
  double* red = reinterpret_cast<double*>(p);
  p += align_up(32 * sizeof(double), 16);
  double* nrm = reinterpret_cast<double*>(p);
  double* ref = nrm + max_n;
  double* xn2 = ref + max_n;
  p += align_up(3 * sizeof(double) * (size_t)max_n, 16);
  int* piv = reinterpret_cast<int*>(p);
  p += align_up(sizeof(int) * (size_t)max_n, 16);
  T* W = GW ? scratch + (size_t)blockIdx.x * max_m * max_n : reinterpret_cast<T*>(p);
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const int m = mm[b], n = nn[b];
  const int ld = sizeof(T) == sizeof(double) ? ((m + 1) & ~1) : (m > 0 ? m : 1);
  const int min_rank = min_rank_arr ? min_rank_arr[b] : 0;
  if (tid == 0) { sh.rank = 0; sh.stop = 0; sh.p0 = 0.0; sh.pad = 0; sh.bigP = 0.0; sh.trail = 0.0; }
  const T* src = A + a_off[b];
  for (int64_t e = tid; e < (int64_t)ld * n; e += nt) {
    const int j = (int)(e / ld), i = (int)(e - (int64_t)j * ld);
    W[e] = i < m ? src[(int64_t)j * m + i] : T(0.0);
  }
  __syncthreads();
  cpqr_init<T>(W, m, n, ld, nrm, ref, xn2, piv, sh);
  __syncthreads();
  cpqr_run<T, GL, RPL>(W, m, n, ld, nrm, ref, xn2, piv, sh, eps, min_rank);
  if (rfac) {
    // pivoted_qr (lowrank.py:48-119): the rank x n upper-trapezoidal factor with
    // columns in pivot order, taken before the interpolation solve overwrites R12
    T* Rf = rfac + rfac_off[b];
    const int rr = sh.rank;
    for (int e = tid; e < rr * n; e += nt) {
      const int s = e / n, q = e - s * n;
      Rf[e] = q >= s ? W[(int64_t)piv[q] * ld + s] : T(0.0);
    }
    __syncthreads();
  }
  interp_solve<T>(W, n, ld, piv, sh, min_rank, red);
  const int r = sh.rank, K = r + sh.pad;
  int32_t* sk = skel_out + skel_off[b];
  // with the R factor requested the whole pivot permutation is returned
  for (int s = tid; s < (rfac ? n : K); s += nt) sk[s] = piv[s];
  T* P = proj + proj_off[b];
  for (int e = tid; e < n * K; e += nt) {
    int s = e / n, q = e - s * n;
    P[(int64_t)s * n + piv[q]] = interp_entry<T>(W, ld, piv, r, K, s, q);
  }
  if (tid == 0) {
    rank_out[b] = rfac ? r : K;     // pivoted_qr reports the completed CPQR steps
    bigP_out[b] = sh.bigP;
    if (ratio_out) ratio_out[b] = sh.p0 > 0.0 ? sh.trail / sh.p0 : 0.0;
  }
}

// ---- S / dense blocks / dense matvec --------------------------------------
template <class T>
__global__ void k_assemble_S(const SkelSource S, const int32_t* rows, const int32_t* rbox, int Kr,
                             const int32_t* cols, const int32_t* cbox, int Kc, T* out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)Kr * Kc) return;
  int i = (int)(e / Kc), j = (int)(e - (int64_t)i * Kc);
  T v = T(0.0);
  if (rbox[i] != cbox[j]) v = entry_A<T>(S, load_pt(S, rows[i]), load_pt(S, cols[j]));
  out[e] = v;
}

template <class T>
__global__ void k_eval_block(const SkelSource S, const int32_t* rows, int m, const int32_t* cols,
                             int n, T* out) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)m * n) return;
  int i = (int)(e / n), j = (int)(e - (int64_t)i * n);
  out[e] = entry_A<T>(S, load_pt(S, rows[i]), load_pt(S, cols[j]));
}

// y = A x, thread per row, source tiles staged in shared memory; RB columns
// of x per pass.
template <class T, int RB>
__global__ void __launch_bounds__(256) k_dense_matvec(const SkelSource S, const T* __restrict__ x,
                                                      T* __restrict__ y, int R, int c0) {
  __shared__ Pt sp[256];
  __shared__ T sx[256 * RB];
  const int64_t N = S.n;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  Pt tp;
  if (i < N) tp = load_pt(S, i);
  T acc[RB];
#pragma unroll
  for (int c = 0; c < RB; ++c) acc[c] = T(0.0);
  for (int64_t j0 = 0; j0 < N; j0 += 256) {
    int64_t j = j0 + threadIdx.x;
    if (j < N) {
      sp[threadIdx.x] = load_pt(S, j);
#pragma unroll
      for (int c = 0; c < RB; ++c) sx[threadIdx.x * RB + c] = (c0 + c < R) ? x[j * R + c0 + c] : T(0.0);
    }
    __syncthreads();
    int cnt = (N - j0) < 256 ? (int)(N - j0) : 256;
    if (i < N) {
      for (int q = 0; q < cnt; ++q) {
        T v = entry_A<T>(S, tp, sp[q]);
#pragma unroll
        for (int c = 0; c < RB; ++c) acc[c] += v * sx[q * RB + c];
      }
    }
    __syncthreads();
  }
  if (i < N) {
#pragma unroll
    for (int c = 0; c < RB; ++c)
      if (c0 + c < R) y[i * R + c0 + c] = acc[c];
  }
}

// ---------------------------------------------------------------------------
// host launchers
template <class T, int GL, int RPL, bool GW>
static int launch_id_level(const SkelSource* src, const SkelLevel* lv, const int32_t* order,
                           int nrun, int64_t max_w, int max_n, size_t smem, cudaStream_t st) {
  // few boxes (upper levels): the per-box CPQR latency is the critical path,
  // so give each box-side more warps.  The per-column arithmetic (tile) is
  // unchanged -- results must not depend on how many boxes share a launch
  // (sharded runs are bit-identical to unsharded ones) -- so real tiles,
  // which need more than the 128 registers a 512-thread CTA allows, get 8
  // warps and complex ones 16.
  static const bool no_wide = getenv("SKEL_ID_NOWIDE") != nullptr;   // developer A/B switch
  if (2 * nrun < 2 * skel_sm_count() && !no_wide) {
    constexpr int NTW = sizeof(T) == sizeof(double) && RPL > 0 ? 256 : 512;
    auto kern = k_id_level<T, GL, RPL, GW, NTW>;
    SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<2 * nrun, NTW, smem, st>>>(*src, *lv, order, max_w, max_n);
  } else {
    auto kern = k_id_level<T, GL, RPL, GW, 128>;
    SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<2 * nrun, 128, smem, st>>>(*src, *lv, order, max_w, max_n);
  }
  return skel_last_error();
}

// register tile: GL lanes per column, RPL rows per lane (GL * RPL >= max_m).
// Real targets use the paired-row tiles of cpqr_update_pr.  A bucket whose
// target fits the four smallest shared-memory classes (<= 46 KB, 4+ CTAs per
// SM by shared memory) takes the low-register tiles (16 or 32 lanes per
// column, <= 12 rows per lane: 4-5 CTAs per SM by registers); the larger
// classes, which are held to 2-3 CTAs per SM by shared memory anyway, take
// 8 lanes per column (4 columns per warp instruction, fewest instructions per
// entry).  The choice depends only on the bucket's size CLASS (every box of a
// bucket has the same class), so a box gets the same arithmetic in any launch.
#define SKEL_SMALL_W_BYTES (46 << 10)
template <class T, bool GW>
static int dispatch_id_level(const SkelSource* src, const SkelLevel* lv, const int32_t* order,
                             int nrun, int max_m, int64_t max_w, int max_n, size_t smem,
                             cudaStream_t st) {
#define SKEL_L(GL_, RPL_) launch_id_level<T, GL_, RPL_, GW>(src, lv, order, nrun, max_w, max_n, smem, st)
  if constexpr (sizeof(T) == 8) {
    if constexpr (!GW) {
      if ((int64_t)max_w * 8 <= SKEL_SMALL_W_BYTES) {
        if (max_m <= 64) return SKEL_L(16, 4);
        if (max_m <= 128) return SKEL_L(16, 8);
        if (max_m <= 192) return SKEL_L(16, 12);
        if (max_m <= 256) return SKEL_L(32, 8);
        if (max_m <= 384) return SKEL_L(32, 12);
      }
    }
    if (max_m <= 64) return SKEL_L(8, 8);
    if (max_m <= 128) return SKEL_L(8, 16);
    if (max_m <= 192) return SKEL_L(8, 24);
    if (max_m <= 256) return SKEL_L(16, 16);
    if (max_m <= 384) return SKEL_L(16, 24);
    if (max_m <= 512) return SKEL_L(32, 16);
    if (max_m <= 768) return SKEL_L(32, 24);
  } else {
    if (max_m <= 128) return SKEL_L(16, 8);
    if (max_m <= 256) return SKEL_L(32, 8);
    if (max_m <= 384) return SKEL_L(32, 12);
  }
  return SKEL_L(32, 0);
#undef SKEL_L
}

// max_m / max_n bound the bucket's target; max_w (elements) bounds m*n
template <class T>
static int id_level_impl(const SkelSource* src, const SkelLevel* lv, const int32_t* order,
                         int nrun, int max_m, int max_n, int64_t max_w, cudaStream_t st) {
  if (nrun <= 0) return 0;
  if (max_m < 1) max_m = 1;
  if (max_n < 1) max_n = 1;
  if (max_w < 1) max_w = 1;
  size_t fixed = level_smem_fixed<T>(max_n);
  size_t wbytes = (size_t)max_w * sizeof(T);
  size_t optin = (size_t)skel_smem_optin();
  if (fixed + wbytes <= optin)
    return dispatch_id_level<T, false>(src, lv, order, nrun, max_m, max_w, max_n, fixed + wbytes, st);
  if ((size_t)lv->scratch_bytes < (size_t)2 * nrun * wbytes || !lv->scratch) return -2;
  return dispatch_id_level<T, true>(src, lv, order, nrun, max_m, max_w, max_n, fixed, st);
}

template <class T, int GL, int RPL, bool GW>
static int launch_id_batched(const void* A, const int64_t* a_off, const int32_t* m,
                             const int32_t* n, int nmat, double eps, const int32_t* min_rank,
                             int32_t* rank, int32_t* skel, const int64_t* skel_off, void* proj,
                             const int64_t* proj_off, double* bigP, double* ratio, void* scratch,
                             int max_m, int max_n, size_t smem, cudaStream_t st, void* rfac,
                             const int64_t* rfac_off) {
  auto kern = k_id_batched<T, GL, RPL, GW>;
  SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<nmat, 128, smem, st>>>((const T*)A, a_off, m, n, eps, min_rank, rank, skel, skel_off,
                                (T*)proj, proj_off, bigP, ratio, (T*)scratch, max_m, max_n,
                                (T*)rfac, rfac_off);
  return skel_last_error();
}

template <class T>
static int id_batched_impl(const void* A, const int64_t* a_off, const int32_t* m, const int32_t* n,
                           int nmat, double eps, const int32_t* min_rank, int32_t* rank,
                           int32_t* skel, const int64_t* skel_off, void* proj,
                           const int64_t* proj_off, double* bigP, double* ratio, void* scratch,
                           int64_t scratch_bytes, int max_m, int max_n, cudaStream_t st,
                           void* rfac = nullptr, const int64_t* rfac_off = nullptr) {
  if (nmat <= 0) return 0;
  if (max_m < 1) max_m = 1;
  if (max_n < 1) max_n = 1;
  size_t fixed = align_up(sizeof(CpqrShared<T>), 16) + align_up(32 * sizeof(double), 16) +
                 align_up(3 * sizeof(double) * max_n, 16) + align_up(sizeof(int) * max_n, 16);
  if (sizeof(T) == sizeof(double)) max_m = (max_m + 1) & ~1;   // even ld (cpqr_update_pr)
  size_t wbytes = (size_t)max_m * max_n * sizeof(T);
  if (fixed + wbytes <= (size_t)skel_smem_optin()) {
    if (max_m <= 128)
      return launch_id_batched<T, 8, 16, false>(A, a_off, m, n, nmat, eps, min_rank, rank, skel,
                                                skel_off, proj, proj_off, bigP, ratio, scratch, max_m, max_n,
                                                fixed + wbytes, st, rfac, rfac_off);
    return launch_id_batched<T, 32, 0, false>(A, a_off, m, n, nmat, eps, min_rank, rank, skel,
                                          skel_off, proj, proj_off, bigP, ratio, scratch, max_m, max_n,
                                          fixed + wbytes, st, rfac, rfac_off);
  }
  if (!scratch || (size_t)scratch_bytes < (size_t)nmat * wbytes) return -2;
  return launch_id_batched<T, 32, 0, true>(A, a_off, m, n, nmat, eps, min_rank, rank, skel, skel_off,
                                       proj, proj_off, bigP, ratio, scratch, max_m, max_n, fixed, st, rfac,
                                       rfac_off);
}

// complex (field 1) instantiations live in id_level_z.cu (a second
// translation unit, compiled in parallel)
int id_level_zc(const SkelSource* src, const SkelLevel* lv, const int32_t* order, int nrun,
                int max_m, int max_n, int64_t max_w, cudaStream_t st);
int id_batched_zc(const void* A, const int64_t* a_off, const int32_t* m, const int32_t* n, int nmat,
                  double eps, const int32_t* min_rank, int32_t* rank, int32_t* skel,
                  const int64_t* skel_off, void* proj, const int64_t* proj_off, double* bigP,
                  double* ratio, void* scratch, int64_t scratch_bytes, int max_m, int max_n,
                  cudaStream_t st, void* rfac = nullptr, const int64_t* rfac_off = nullptr);
