// solve.cu -- K5: multi-RHS telescoping solve / compressed apply sweeps.
//
// Reference work replaced: solve (solver.py:279-318) and apply
// (skel.py:206-249): per-box GEMMs of the up-sweep (Rd or R), the dense top
// (Shat^-1 or S) and the down-sweep (Dd + Ld or D + L), plus the tree
// permutation gather / scatter (solver.py:288,316-318).
//
// Vectors are row-major (rows of R contiguous values), so a box's segment is
// one contiguous n x R slab.  One CTA per (box, column chunk): the chunk of
// the input segment(s) is staged in shared memory, factor blocks are streamed
// from HBM exactly once per chunk (read-only path), each thread owns one
// output (row, column) pair.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

// Block GEMM of one tree level, per box a and its slice of RHS columns:
//   O[o_off[a] + i, c] = sum_j A_a[i, j] X[x_off[a] + j, c] (+ sum_t B_a[i, t] Y[y_off[a] + t, c])
// A_a (p x q) and B_a (p x r) are contiguous row-major blocks streamed from HBM
// into shared memory ONCE per CTA; the CTA then walks its columns in chunks
// of CB, staging the X / Y chunk with cp.async (double buffered, the next
// chunk's copy overlaps this chunk's FMAs); each thread accumulates a TM x TN
// register tile.  STAGE = false is the fallback for blocks too large for
// shared memory (3D coarse levels): operands are read through L1 directly.

template <class T, int CB>
__device__ __forceinline__ void stage_chunk(T* sX, const T* Xg, int q, int R, int c0, int cb,
                                            const int64_t* rows = nullptr) {
  constexpr int W = sizeof(T) / 8;   // 8-byte words per element
  for (int e = threadIdx.x; e < q * CB * W; e += blockDim.x) {
    const int el = e / W, wd = e - el * W;
    const int j = el / CB, c = el - j * CB;
    double* d = reinterpret_cast<double*>(sX + el) + wd;
    const T* xr = rows ? Xg + rows[j] * R : Xg + (int64_t)j * R;   // rows: gathered segment
    if (c < cb) cp_async8(d, reinterpret_cast<const double*>(xr + c0 + c) + wd);
    else *d = 0.0;
  }
}

template <class T, int TM, int TN, int CB, bool STAGE, bool ROWS = false>
__global__ void __launch_bounds__(128) k_level_gemm(
    const int32_t* __restrict__ pp, const int32_t* __restrict__ qq, const int32_t* __restrict__ rr,
    const int64_t* __restrict__ a_off, const T* __restrict__ A,
    const int64_t* __restrict__ b_off, const T* __restrict__ Bm,
    const int64_t* __restrict__ x_off, const T* __restrict__ X,
    const int64_t* __restrict__ y_off, const T* __restrict__ Y,
    const int64_t* __restrict__ o_off, T* __restrict__ O, int R, int cols_per_cta, int max_q,
    int max_r, const int32_t* __restrict__ order, const int64_t* __restrict__ xrows,
    const int64_t* __restrict__ orows) {
  // xrows / orows (optional): X rows are X[xrows[x_off + j]] and output rows
  // go to O[orows[o_off + i]] -- the solve's tree-order gather / scatter of
  // the right-hand sides fused into the finest level's sweeps
  extern __shared__ __align__(16) unsigned char smem[];
  const int a = order ? order[blockIdx.x] : blockIdx.x;
  const int p = pp[a], q = qq[a], r = rr ? rr[a] : 0;
  if (p == 0) return;
  const int cbeg = blockIdx.y * cols_per_cta;
  const int cend = min(R, cbeg + cols_per_cta);
  if (cbeg >= cend) return;
  const int tid = threadIdx.x, nt = blockDim.x;
  const T* Ag = A + a_off[a];
  const T* Bg = r ? Bm + b_off[a] : nullptr;
  const int64_t* xr = (ROWS && xrows) ? xrows + x_off[a] : nullptr;
  const int64_t* orw = (ROWS && orows) ? orows + o_off[a] : nullptr;
  const T* Xg = xr ? X : X + x_off[a] * R;
  const T* Yg = r ? Y + y_off[a] * R : nullptr;
  T* Og = orw ? O : O + o_off[a] * R;
  T* sA = reinterpret_cast<T*>(smem);
  T* sB = sA + (STAGE ? (size_t)p * q : 0);
  T* const sXY0 = sB + (STAGE ? (size_t)p * r : 0);
  const size_t sxy_stride = (size_t)(max_q + max_r) * CB;
  if (STAGE) {
    // every operand byte goes global -> shared with cp.async: all loads in
    // flight at once instead of one load-to-store round trip per element
    constexpr int W = sizeof(T) / 8;
    for (int e = tid; e < p * q * W; e += nt)
      cp_async8(reinterpret_cast<double*>(sA) + e, reinterpret_cast<const double*>(Ag) + e);
    for (int e = tid; e < p * r * W; e += nt)
      cp_async8(reinterpret_cast<double*>(sB) + e, reinterpret_cast<const double*>(Bg) + e);
    stage_chunk<T, CB>(sXY0, Xg, q, R, cbeg, min(CB, cend - cbeg), xr);
    if (r) stage_chunk<T, CB>(sXY0 + (size_t)q * CB, Yg, r, R, cbeg, min(CB, cend - cbeg));
    cp_async_commit();
  }
  constexpr int NCT = CB / TN;
  const int nrt = (p + TM - 1) / TM;
  int buf = 0;
  for (int c0 = cbeg; c0 < cend; c0 += CB, buf ^= 1) {
    const int cb = min(CB, cend - c0);
    const T* sX = sXY0 + buf * sxy_stride;
    const T* sY = sX + (size_t)q * CB;
    if (STAGE) {
      const int c1 = c0 + CB;
      if (c1 < cend) {
        T* nb = sXY0 + (buf ^ 1) * sxy_stride;
        stage_chunk<T, CB>(nb, Xg, q, R, c1, min(CB, cend - c1), xr);
        if (r) stage_chunk<T, CB>(nb + (size_t)q * CB, Yg, r, R, c1, min(CB, cend - c1));
      }
      cp_async_commit();
      cp_async_wait<1>();
      __syncthreads();
    }
    for (int t = tid; t < nrt * NCT; t += nt) {
      const int rt = t / NCT, ct = t - rt * NCT;
      const int i0 = rt * TM, j0 = ct * TN;
      T acc[TM][TN];
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = T(0.0);
      for (int j = 0; j < q; ++j) {
        T av[TM], xv[TN];
#pragma unroll
        for (int u = 0; u < TM; ++u)
          av[u] = (i0 + u < p) ? (STAGE ? sA[(i0 + u) * q + j] : __ldg_T(Ag + (int64_t)(i0 + u) * q + j)) : T(0.0);
#pragma unroll
        for (int v = 0; v < TN; ++v)
          xv[v] = STAGE ? sX[j * CB + j0 + v]
                        : ((j0 + v < cb) ? __ldg_T((xr ? Xg + xr[j] * R : Xg + (int64_t)j * R) + c0 + j0 + v)
                                         : T(0.0));
#pragma unroll
        for (int u = 0; u < TM; ++u)
#pragma unroll
          for (int v = 0; v < TN; ++v) acc[u][v] += av[u] * xv[v];
      }
      for (int j = 0; j < r; ++j) {
        T av[TM], xv[TN];
#pragma unroll
        for (int u = 0; u < TM; ++u)
          av[u] = (i0 + u < p) ? (STAGE ? sB[(i0 + u) * r + j] : __ldg_T(Bg + (int64_t)(i0 + u) * r + j)) : T(0.0);
#pragma unroll
        for (int v = 0; v < TN; ++v)
          xv[v] = STAGE ? sY[j * CB + j0 + v]
                        : ((j0 + v < cb) ? __ldg_T(Yg + (int64_t)j * R + c0 + j0 + v) : T(0.0));
#pragma unroll
        for (int u = 0; u < TM; ++u)
#pragma unroll
          for (int v = 0; v < TN; ++v) acc[u][v] += av[u] * xv[v];
      }
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v)
          if (i0 + u < p && j0 + v < cb)
            (orw ? Og + orw[i0 + u] * R : Og + (int64_t)(i0 + u) * R)[c0 + j0 + v] = acc[u][v];
    }
    if (STAGE) __syncthreads();   // buffer `buf` is refilled two chunks later
  }
}

// DMMA (mma.sync.m8n8k4.f64) variant for many RHS: [A | B] (p x (q+r)) and
// [X; Y] ((q+r) x CB) are treated as one GEMM; each warp owns 8-row x 32-col
// output tiles (4 accumulators of 8x8), one A fragment and four B fragments
// per k-step of 4.  X/Y chunks are double buffered with cp.async; the chunk
// row stride is CB+8 doubles so a B-fragment load hits every bank pair once.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int CB>
__global__ void __launch_bounds__(128) k_level_dmma(
    const int32_t* __restrict__ pp, const int32_t* __restrict__ qq, const int32_t* __restrict__ rr,
    const int64_t* __restrict__ a_off, const double* __restrict__ A,
    const int64_t* __restrict__ b_off, const double* __restrict__ Bm,
    const int64_t* __restrict__ x_off, const double* __restrict__ X,
    const int64_t* __restrict__ y_off, const double* __restrict__ Y,
    const int64_t* __restrict__ o_off, double* __restrict__ O, int R, int cols_per_cta, int max_p,
    int max_k, const int32_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int LDX = CB + 8;
  const int a = order ? order[blockIdx.x] : blockIdx.x;
  const int p = pp[a], q = qq[a], r = rr ? rr[a] : 0;
  if (p == 0) return;
  const int cbeg = blockIdx.y * cols_per_cta;
  const int cend = min(R, cbeg + cols_per_cta);
  if (cbeg >= cend) return;
  const int K = q + r, Kp = (K + 3) & ~3, P8 = (p + 7) & ~7;
  const int ldA = Kp + 1;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  double* sA = reinterpret_cast<double*>(smem);
  double* sX0 = sA + (((size_t)max_p + 7) & ~(size_t)7) * (max_k + 1);
  const size_t xstride = (size_t)max_k * LDX;
  const double* Ag = A + a_off[a];
  const double* Bg = r ? Bm + b_off[a] : nullptr;
  const double* Xg = X + x_off[a] * R;
  const double* Yg = r ? Y + y_off[a] * R : nullptr;
  double* Og = O + o_off[a] * R;
  for (int e = tid; e < P8 * Kp; e += nt) {
    const int i = e / Kp, j = e - i * Kp;
    double* d = sA + i * ldA + j;
    if (i < p && j < K) cp_async8(d, j < q ? Ag + (int64_t)i * q + j : Bg + (int64_t)i * r + (j - q));
    else *d = 0.0;
  }
  auto stage = [&](double* dst, int c0) {
    const int cb = min(CB, cend - c0);
    for (int e = tid; e < Kp * CB; e += nt) {
      const int j = e / CB, c = e - j * CB;
      double* d = dst + j * LDX + c;
      if (j < K && c < cb) cp_async8(d, j < q ? Xg + (int64_t)j * R + c0 + c : Yg + (int64_t)(j - q) * R + c0 + c);
      else *d = 0.0;
    }
  };
  stage(sX0, cbeg);
  cp_async_commit();
  const int g = lane >> 2, t4 = lane & 3;
  const int ntask = (P8 / 8) * (CB / 32);
  int buf = 0;
  for (int c0 = cbeg; c0 < cend; c0 += CB, buf ^= 1) {
    const int cb = min(CB, cend - c0);
    const double* sX = sX0 + buf * xstride;
    if (c0 + CB < cend) stage(sX0 + (buf ^ 1) * xstride, c0 + CB);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();
    for (int task = warp; task < ntask; task += nt >> 5) {
      const int rt = task / (CB / 32), cg = task - rt * (CB / 32);
      double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
      const double* arow = sA + (rt * 8 + g) * ldA + t4;
      const double* xcol = sX + t4 * LDX + cg * 32 + g;
      for (int k0 = 0; k0 < Kp; k0 += 4) {
        const double av = arow[k0];
        const double* xk = xcol + k0 * LDX;
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma884(acc[u][0], acc[u][1], av, xk[u * 8]);
      }
      const int row = rt * 8 + g;
      if (row < p) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int col = cg * 32 + u * 8 + 2 * t4;
          if (col < cb) Og[(int64_t)row * R + c0 + col] = acc[u][0];
          if (col + 1 < cb) Og[(int64_t)row * R + c0 + col + 1] = acc[u][1];
        }
      }
    }
    __syncthreads();
  }
}

// DMMA variant for few RHS (R <= 8 * NT): one CTA per box, one warp per
// 8-row output tile with NT 8x8 accumulators.  Only the (small) X / Y slab is
// staged in shared memory; the factor blocks A (p x q) and B (p x r) -- the
// bytes that bound the sweep -- go straight from HBM into the A fragments
// (each lane reads 4 consecutive doubles of one row per k-step, the unrolled
// k-loop keeps several loads in flight), so there is no shared-memory round
// trip and no CTA-wide barrier for them.  Slab layout: rows [0, q) = X,
// zero pad to Qp = q rounded up to 4, rows [Qp, Qp + r) = Y, pad to 4;
// row stride 8 * NT + 8 doubles so a B-fragment load touches each bank pair
// exactly twice (the 2-wavefront minimum for 32 doubles).
template <int NT, bool ROWS, bool CPLX = false>
__global__ void __launch_bounds__(256) k_level_dmma_few(
    const int32_t* __restrict__ pp, const int32_t* __restrict__ qq, const int32_t* __restrict__ rr,
    const int64_t* __restrict__ a_off, const double* __restrict__ A,
    const int64_t* __restrict__ b_off, const double* __restrict__ Bm,
    const int64_t* __restrict__ x_off, const double* __restrict__ X,
    const int64_t* __restrict__ y_off, const double* __restrict__ Y,
    const int64_t* __restrict__ o_off, double* __restrict__ O, int R,
    const int32_t* __restrict__ order, const int64_t* __restrict__ xrows,
    const int64_t* __restrict__ orows) {
  // CPLX: complex128 blocks and vectors (interleaved re, im) as the real GEMM
  // [Re | Im] (p x 2q) x X' (2q x 2R), X' rows 2k = (re, im) pairs of X row k
  // and 2k+1 = (-im, re): column pair (2c, 2c+1) of the result is (Re, Im)
  // of A X, already interleaved.  R, offsets and row maps stay in complex
  // units; below every extent is in doubles.
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CW = 8 * NT, LDX = CW + 8, CF = CPLX ? 2 : 1;
  const int a = order ? order[blockIdx.x] : blockIdx.x;
  const int p = pp[a], q = CF * qq[a], r = rr ? CF * rr[a] : 0;
  R *= CF;
  if (p == 0) return;
  const int Qp = (q + 3) & ~3, Rp = (r + 3) & ~3, Kp = Qp + Rp;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  double* sX = reinterpret_cast<double*>(smem);
  const int64_t* xr = (ROWS && xrows) ? xrows + x_off[a] : nullptr;
  const int64_t* orw = (ROWS && orows) ? orows + o_off[a] : nullptr;
  // <= 8 RHS: the box's factor blocks are contiguous slabs, so two threads
  // ask the TMA unit to pull them into L2 now (cp.async.bulk.prefetch.L2)
  // and the A-fragment loads below find them there instead of paying the HBM
  // latency per k-step with only a few loads in flight per warp (measured at
  // N = 2^20: R = 1 / 4 solves -14 % / -13 %; with 16 RHS the same prefetch
  // costs +13 %, so the wider tiles do not issue it)
  if constexpr (NT == 1) {
    if (tid == 0) prefetch_l2_bulk(A + CF * a_off[a], (size_t)p * q * sizeof(double));
    if (tid == 32 && r) prefetch_l2_bulk(Bm + CF * b_off[a], (size_t)p * r * sizeof(double));
  }
  // stage in 16-byte pieces (column pairs; rows are 16-byte aligned for even R)
  constexpr int CP = CW / 2;
  for (int e = tid; e < Kp * CP; e += nt) {
    const int j = e / CP, c = 2 * (e - j * CP);
    double* d = sX + j * LDX + c;
    const double* src = nullptr;
    int par = 0;
    if (j < q) {
      const int kx = j / CF;
      par = j - kx * CF;
      src = (xr ? X + xr[kx] * R : X + (x_off[a] + kx) * R) + c;
    } else if (j >= Qp && j - Qp < r) {
      const int ky = (j - Qp) / CF;
      par = (j - Qp) - ky * CF;
      src = Y + (y_off[a] + ky) * R + c;
    }
    if (CPLX && par) {               // (-im, re) of complex element c / 2
      d[0] = (src && c < R) ? -__ldg(src + 1) : 0.0;
      d[1] = (src && c < R) ? __ldg(src) : 0.0;
    } else if (src && c + 1 < R && !(reinterpret_cast<uintptr_t>(src) & 15)) {
      cp_async16(d, src);
    } else {
      d[0] = (src && c < R) ? __ldg(src) : 0.0;
      d[1] = (src && c + 1 < R) ? __ldg(src + 1) : 0.0;
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int g = lane >> 2, t4 = lane & 3;
  const int ntile = (p + 7) >> 3;
  for (int rt = warp; rt < ntile; rt += nt >> 5) {
    const int row = rt * 8 + g;
    const bool ok = row < p;
    double acc[NT][2];
#pragma unroll
    for (int u = 0; u < NT; ++u) acc[u][0] = acc[u][1] = 0.0;
    const double* arow = A + CF * a_off[a] + (int64_t)(ok ? row : 0) * q;
    const double* xs = sX + t4 * LDX + g;
#pragma unroll 4
    for (int k0 = 0; k0 < Qp; k0 += 4) {
      const double av = (ok && k0 + t4 < q) ? __ldg(arow + k0 + t4) : 0.0;
#pragma unroll
      for (int u = 0; u < NT; ++u) dmma884(acc[u][0], acc[u][1], av, xs[k0 * LDX + u * 8]);
    }
    if (r) {
      const double* brow = Bm + CF * b_off[a] + (int64_t)(ok ? row : 0) * r;
      const double* ys = xs + Qp * LDX;
#pragma unroll 4
      for (int k0 = 0; k0 < Rp; k0 += 4) {
        const double bv = (ok && k0 + t4 < r) ? __ldg(brow + k0 + t4) : 0.0;
#pragma unroll
        for (int u = 0; u < NT; ++u) dmma884(acc[u][0], acc[u][1], bv, ys[k0 * LDX + u * 8]);
      }
    }
    if (ok) {
      double* orow = orw ? O + orw[row] * R : O + (o_off[a] + row) * R;
#pragma unroll
      for (int u = 0; u < NT; ++u) {
        const int col = u * 8 + 2 * t4;
        if (col + 1 < R && !(R & 1)) {
          *reinterpret_cast<double2*>(orow + col) = make_double2(acc[u][0], acc[u][1]);
        } else {
          if (col < R) orow[col] = acc[u][0];
          if (col + 1 < R) orow[col + 1] = acc[u][1];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Few-RHS sweep with the factor blocks staged by the TMA unit (1-D bulk
// copies).  Row-major blocks make the 8 rows of a warp's output tile ONE
// contiguous chunk of A (8 q doubles) and one of B (8 r doubles): lane 0 of
// the warp arms a warp-private mbarrier with the byte count and issues two
// cp.async.bulk copies into the warp's shared-memory buffer (SASS UBLKCP);
// the whole tile's factor bytes are then in flight at once without holding
// registers, and the A fragments come from shared memory.  The X / Y slab is
// staged as in k_level_dmma_few while the bulk copies fly.  Chunks start on
// 8-byte boundaries: a misaligned chunk is fetched from the 16-byte boundary
// below it (`lead` = 1 double of the previous row / block, inside the slab)
// and an odd trailing double comes by a plain load, so no copy reads past
// the slab.  Same DMMA schedule and arithmetic as k_level_dmma_few.
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(b);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
               : "memory");
}

// one chunk (cnt doubles at g, 8-byte aligned) -> dst (16-byte aligned);
// returns the bytes the bulk copy will deliver; dst[lead + i] = g[i]
__device__ __forceinline__ unsigned bulk_chunk(double* dst, const double* g, int cnt, uint64_t* b,
                                               bool issue) {
  const int lead = (int)((reinterpret_cast<uintptr_t>(g) >> 3) & 1);
  const int total = lead + cnt;
  const unsigned bytes = (unsigned)(total & ~1) * 8u;
  if (issue && bytes) bulk_g2s(dst, g - lead, bytes, b);
  return bytes;
}

template <int NT, bool ROWS>
__global__ void __launch_bounds__(256) k_level_bulk_few(
    const int32_t* __restrict__ pp, const int32_t* __restrict__ qq, const int32_t* __restrict__ rr,
    const int64_t* __restrict__ a_off, const double* __restrict__ A,
    const int64_t* __restrict__ b_off, const double* __restrict__ Bm,
    const int64_t* __restrict__ x_off, const double* __restrict__ X,
    const int64_t* __restrict__ y_off, const double* __restrict__ Y,
    const int64_t* __restrict__ o_off, double* __restrict__ O, int R,
    const int32_t* __restrict__ order, const int64_t* __restrict__ xrows,
    const int64_t* __restrict__ orows, int buf_doubles) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int CW = 8 * NT, LDX = CW + 8;
  const int a = order ? order[blockIdx.x] : blockIdx.x;
  const int p = pp[a], q = qq[a], r = rr ? rr[a] : 0;
  if (p == 0) return;
  const int Qp = (q + 3) & ~3, Rp = (r + 3) & ~3, Kp = Qp + Rp;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem) + warp;
  double* wbuf = reinterpret_cast<double*>(smem + 64) + (size_t)warp * buf_doubles;
  double* sX = reinterpret_cast<double*>(smem + 64) + (size_t)nw * buf_doubles;
  if (lane == 0) mbar_init(mbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
  const double* Ab = A + a_off[a];
  const double* Bb = r ? Bm + b_off[a] : nullptr;
  const int ntile = (p + 7) >> 3;
  // issue tile rt's copies (lane 0); every lane gets the chunk geometry
  double tail_v = 0.0;
  int tail_i = -1;
  auto stage = [&](int rt, int& lead_a, int& off_b, int& lead_b) {
    const int row0 = rt * 8, rows = (p - row0) < 8 ? (p - row0) : 8;
    const double* ga = Ab + (int64_t)row0 * q;
    lead_a = (int)((reinterpret_cast<uintptr_t>(ga) >> 3) & 1);
    off_b = (lead_a + rows * q + 1) & ~1;
    lead_b = 0;
    const double* gb = nullptr;
    if (r) {
      gb = Bb + (int64_t)row0 * r;
      lead_b = (int)((reinterpret_cast<uintptr_t>(gb) >> 3) & 1);
    }
    if (lane == 0) {
      unsigned bytes = bulk_chunk(wbuf, ga, rows * q, mbar, false);
      if (r) bytes += bulk_chunk(wbuf + off_b, gb, rows * r, mbar, false);
      mbar_expect_tx(mbar, bytes);
      bulk_chunk(wbuf, ga, rows * q, mbar, true);
      if (r) bulk_chunk(wbuf + off_b, gb, rows * r, mbar, true);
    }
    // odd trailing doubles come by plain loads: lane 1 (A) and lane 2 (B)
    // fetch them now and store them just before the tile is consumed
    tail_v = 0.0;
    tail_i = -1;
    if (lane == 1 && ((lead_a + rows * q) & 1)) {
      tail_i = lead_a + rows * q - 1;
      tail_v = __ldg(ga + rows * q - 1);
    }
    if (lane == 2 && r && ((lead_b + rows * r) & 1)) {
      tail_i = off_b + lead_b + rows * r - 1;
      tail_v = __ldg(gb + rows * r - 1);
    }
  };
  int lead_a = 0, off_b = 0, lead_b = 0;
  if (warp < ntile) stage(warp, lead_a, off_b, lead_b);
  const int64_t* xr = (ROWS && xrows) ? xrows + x_off[a] : nullptr;
  const int64_t* orw = (ROWS && orows) ? orows + o_off[a] : nullptr;
  constexpr int CP = CW / 2;
  for (int e = tid; e < Kp * CP; e += nt) {
    const int j = e / CP, c = 2 * (e - j * CP);
    double* d = sX + j * LDX + c;
    const double* src = nullptr;
    if (j < q) src = (xr ? X + xr[j] * R : X + (x_off[a] + j) * R) + c;
    else if (j >= Qp && j - Qp < r) src = Y + (y_off[a] + (j - Qp)) * R + c;
    if (src && c + 1 < R && !(reinterpret_cast<uintptr_t>(src) & 15)) {
      cp_async16(d, src);
    } else {
      d[0] = (src && c < R) ? __ldg(src) : 0.0;
      d[1] = (src && c + 1 < R) ? __ldg(src + 1) : 0.0;
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int g = lane >> 2, t4 = lane & 3;
  unsigned phase = 0;
  for (int rt = warp; rt < ntile; rt += nw) {
    if (tail_i >= 0) wbuf[tail_i] = tail_v;
    mbar_wait(mbar, phase);
    phase ^= 1;
    __syncwarp();
    const int row = rt * 8 + g;
    const bool ok = row < p;
    double acc[NT][2];
#pragma unroll
    for (int u = 0; u < NT; ++u) acc[u][0] = acc[u][1] = 0.0;
    const double* arow = wbuf + lead_a + (ok ? g : 0) * q;
    const double* xs = sX + t4 * LDX + g;
#pragma unroll 4
    for (int k0 = 0; k0 < Qp; k0 += 4) {
      const double av = (ok && k0 + t4 < q) ? arow[k0 + t4] : 0.0;
#pragma unroll
      for (int u = 0; u < NT; ++u) dmma884(acc[u][0], acc[u][1], av, xs[k0 * LDX + u * 8]);
    }
    if (r) {
      const double* brow = wbuf + off_b + lead_b + (ok ? g : 0) * r;
      const double* ys = xs + Qp * LDX;
#pragma unroll 4
      for (int k0 = 0; k0 < Rp; k0 += 4) {
        const double bv = (ok && k0 + t4 < r) ? brow[k0 + t4] : 0.0;
#pragma unroll
        for (int u = 0; u < NT; ++u) dmma884(acc[u][0], acc[u][1], bv, ys[k0 * LDX + u * 8]);
      }
    }
    __syncwarp();                       // every lane is done with the buffer
    if (rt + nw < ntile) stage(rt + nw, lead_a, off_b, lead_b);
    if (ok) {
      double* orow = orw ? O + orw[row] * R : O + (o_off[a] + row) * R;
#pragma unroll
      for (int u = 0; u < NT; ++u) {
        const int col = u * 8 + 2 * t4;
        if (col + 1 < R && !(R & 1)) {
          *reinterpret_cast<double2*>(orow + col) = make_double2(acc[u][0], acc[u][1]);
        } else {
          if (col < R) orow[col] = acc[u][0];
          if (col + 1 < R) orow[col + 1] = acc[u][1];
        }
      }
    }
  }
}

// Pipelined DMMA variant for many RHS.  One CTA per (box, column range);
// [A | B] is staged in shared memory once (row stride = 4 mod 16 doubles, so
// an A-fragment load is conflict-free).  A warp task is up to MT 8-row tiles
// x 16 columns, columns paired so lane g of n-tile u holds column c0 + 2g + u
// (one 16-byte load feeds both n-tiles; each lane stores 4 consecutive
// outputs).  Each warp streams its X / Y rows through a private NS-stage
// shared-memory ring with 16-byte cp.async: the bytes in flight live in
// shared memory, not registers, so NS - 1 chunks of 16 rows x 16 columns per
// warp are outstanding while the DMMAs of the current chunk issue; every B
// fragment feeds all the task's row tiles.  No CTA-wide barrier after the A
// stage (the ring is warp-private, __syncwarp only).
template <int MT, int NS>
__global__ void __launch_bounds__(256, 2) k_level_dmma_pipe(
    const int32_t* __restrict__ pp, const int32_t* __restrict__ qq, const int32_t* __restrict__ rr,
    const int64_t* __restrict__ a_off, const double* __restrict__ A,
    const int64_t* __restrict__ b_off, const double* __restrict__ Bm,
    const int64_t* __restrict__ x_off, const double* __restrict__ X,
    const int64_t* __restrict__ y_off, const double* __restrict__ Y,
    const int64_t* __restrict__ o_off, double* __restrict__ O, int R, int cols_per_cta,
    const int32_t* __restrict__ order, int a_words) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int CW = 16, KC = 16;       // columns per task, K rows per chunk
  constexpr int RING = NS * KC * CW;    // doubles per warp ring
  const int a = order ? order[blockIdx.x] : blockIdx.x;
  const int p = pp[a], q = qq[a], r = rr ? rr[a] : 0;
  if (p == 0) return;
  const int cbeg = blockIdx.y * cols_per_cta;
  const int cend = min(R, cbeg + cols_per_cta);
  if (cbeg >= cend) return;
  const int Qp = (q + 3) & ~3, Kp = Qp + ((r + 3) & ~3);
  const int ldA = Kp + ((4 - Kp) & 15);
  const int P8 = (p + 7) & ~7;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  double* sA = reinterpret_cast<double*>(smem);
  double* ring = sA + a_words + warp * RING;
  const double* Ag = A + a_off[a];
  const double* Bg = r ? Bm + b_off[a] : nullptr;
  for (int e = tid; e < P8 * Kp; e += nt) {
    const int i = e / Kp, j = e - i * Kp;
    double* d = sA + i * ldA + j;
    if (i < p && j < q) cp_async8(d, Ag + (int64_t)i * q + j);
    else if (i < p && j >= Qp && j - Qp < r) cp_async8(d, Bg + (int64_t)i * r + (j - Qp));
    else *d = 0.0;
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int g = lane >> 2, t4 = lane & 3;
  const int ntile = P8 >> 3, nrb = (ntile + MT - 1) / MT;
  const int ncg = (cend - cbeg + CW - 1) / CW;
  const int nch = (Kp + KC - 1) / KC;
  const double* Xb = X + x_off[a] * R;
  const double* Yb = r ? Y + (y_off[a] - Qp) * R : nullptr;   // row k >= Qp is Y row k - Qp
  double* Og = O + o_off[a] * R;
  const bool even = !(R & 1);
  for (int task = warp; task < nrb * ncg; task += nt >> 5) {
    const int rb = task / ncg, cg = task - rb * ncg;
    const int c0 = cbeg + cg * CW;
    const bool full = c0 + CW <= cend && even;
    // chunk c -> ring slot c % NS: 16 rows x 8 16-byte pieces, 4 per lane
    auto issue = [&](int c) {
      double* slot = ring + (c % NS) * (KC * CW);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int piece = lane + 32 * t, row = piece >> 3, pc = (piece & 7) * 2;
        const int k = c * KC + row;
        const double* src = k < q ? Xb : ((k >= Qp && k - Qp < r) ? Yb : nullptr);
        double* d = slot + row * CW + pc;
        if (src && full) {
          cp_async16(d, src + (int64_t)k * R + c0 + pc);
        } else {
          d[0] = (src && c0 + pc < cend) ? __ldg(src + (int64_t)k * R + c0 + pc) : 0.0;
          d[1] = (src && c0 + pc + 1 < cend) ? __ldg(src + (int64_t)k * R + c0 + pc + 1) : 0.0;
        }
      }
    };
    double acc[MT][2][2];
#pragma unroll
    for (int m = 0; m < MT; ++m) acc[m][0][0] = acc[m][0][1] = acc[m][1][0] = acc[m][1][1] = 0.0;
    auto chunk = [&](auto mc, double (&ac)[MT][2][2], const double* slot, int kc, int ns, int rb_) {
      constexpr int M = decltype(mc)::value;
      const double* arow = sA + (rb_ * MT * 8 + g) * ldA + kc + t4;
      auto step = [&](int s) {
        const double2 b = *reinterpret_cast<const double2*>(slot + 4 * s * CW);
#pragma unroll
        for (int m = 0; m < M; ++m) {
          const double av = arow[m * 8 * ldA + 4 * s];
          dmma884(ac[m][0][0], ac[m][0][1], av, b.x);
          dmma884(ac[m][1][0], ac[m][1][1], av, b.y);
        }
      };
      if (ns == KC / 4) {
#pragma unroll
        for (int s = 0; s < KC / 4; ++s) step(s);
      } else {
#pragma unroll 1
        for (int s = 0; s < ns; ++s) step(s);
      }
    };
#pragma unroll
    for (int c = 0; c < NS - 1; ++c) {
      if (c < nch) issue(c);
      cp_async_commit();
    }
    for (int c = 0; c < nch; ++c) {
      cp_async_wait<NS - 2>();
      __syncwarp();
      const double* slot = ring + (c % NS) * (KC * CW) + t4 * CW + 2 * g;
      const int kc = c * KC;
      const int ns = min(KC / 4, (Kp - kc) >> 2);
      // exact row-tile count and k-step count: a predicated-off DMMA still
      // occupies the FP64 tensor pipe, so nothing here is guarded per step
      switch (min(MT, ntile - rb * MT)) {
        case 1: chunk(std::integral_constant<int, 1>(), acc, slot, kc, ns, rb); break;
        case 2: chunk(std::integral_constant<int, 2>(), acc, slot, kc, ns, rb); break;
        case 3: chunk(std::integral_constant<int, 3>(), acc, slot, kc, ns, rb); break;
        case 4: chunk(std::integral_constant<int, 4>(), acc, slot, kc, ns, rb); break;
        case 5: if constexpr (MT >= 5) chunk(std::integral_constant<int, 5>(), acc, slot, kc, ns, rb); break;
        case 6: if constexpr (MT >= 6) chunk(std::integral_constant<int, 6>(), acc, slot, kc, ns, rb); break;
        case 7: if constexpr (MT >= 7) chunk(std::integral_constant<int, 7>(), acc, slot, kc, ns, rb); break;
        default: if constexpr (MT >= 8) chunk(std::integral_constant<int, 8>(), acc, slot, kc, ns, rb); break;
      }
      __syncwarp();   // every lane is done with slot c % NS before it is refilled
      if (c + NS - 1 < nch) issue(c + NS - 1);
      cp_async_commit();
    }
    cp_async_wait<0>();
    __syncwarp();
    const int col = c0 + 4 * t4;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int row = (rb * MT + m) * 8 + g;
      if (row < p) {
        double* orow = Og + (int64_t)row * R + col;
        if (full) {
          *reinterpret_cast<double2*>(orow) = make_double2(acc[m][0][0], acc[m][1][0]);
          *reinterpret_cast<double2*>(orow + 2) = make_double2(acc[m][0][1], acc[m][1][1]);
        } else {
          if (col < cend) orow[0] = acc[m][0][0];
          if (col + 1 < cend) orow[1] = acc[m][1][0];
          if (col + 2 < cend) orow[2] = acc[m][0][1];
          if (col + 3 < cend) orow[3] = acc[m][1][1];
        }
      }
    }
  }
}

static int dmma_many_mode() {
  static const int mode = [] {
    const char* e = std::getenv("SKEL_SOLVE_DMMA_MANY");
    return e ? std::atoi(e) : 1;
  }();
  return mode;
}

// TMA-staged few-RHS sweeps: measured at N = 2^20 against the direct-load
// kernel, R = 1 / 4: -6 % / -8 % (on top of its L2 prefetch), R = 16: +4 %,
// R = 32: -1 %.  Default: <= 8 RHS.  SKEL_SOLVE_BULK=0 / 1 forces it off / on
// for every width (A/B runs).
static bool bulk_few_enabled(int nt) {
  static const int mode = [] {
    const char* e = std::getenv("SKEL_SOLVE_BULK");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  return mode < 0 ? nt == 1 : mode == 1;
}

static bool dmma_few_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SKEL_SOLVE_DMMA_FEW");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <class T>
static int level_gemm(int nbox, const int32_t* p, const int32_t* q, const int32_t* r,
                      const int64_t* a_off, const void* A, const int64_t* b_off, const void* B,
                      const int64_t* x_off, const void* X, const int64_t* y_off, const void* Y,
                      const int64_t* o_off, void* O, int R, int max_p, int max_q, int max_r,
                      const int32_t* order, cudaStream_t st, const int64_t* xrows = nullptr,
                      const int64_t* orows = nullptr) {
  // nbox = number of CTAs' boxes: order[0..nbox) when order != NULL
  if (nbox <= 0 || R <= 0) return 0;
  const size_t optin = (size_t)skel_smem_optin();
  auto go = [&](auto kern_s, auto kern_g, int CB) -> int {
    // columns per CTA: enough chunks to amortise staging A, enough CTAs to fill the GPU
    int chunks = (R + CB - 1) / CB;
    int per = 1;
    while (per < chunks && (long long)nbox * ((chunks + per * 2 - 1) / (per * 2)) >= 4LL * 148 * 4) per *= 2;
    const int cols = per * CB;
    dim3 grid(nbox, (R + cols - 1) / cols);
    size_t smem = ((size_t)max_p * max_q + (size_t)max_p * max_r +
                   2 * (size_t)(max_q + max_r) * CB) * sizeof(T);
    if (smem <= optin) {
      SKEL_TRY(cudaFuncSetAttribute(kern_s, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern_s<<<grid, 128, smem, st>>>(p, q, r, a_off, (const T*)A, b_off, (const T*)B, x_off,
                                      (const T*)X, y_off, (const T*)Y, o_off, (T*)O, R, cols, max_q,
                                      max_r, order, xrows, orows);
    } else {
      kern_g<<<grid, 128, 0, st>>>(p, q, r, a_off, (const T*)A, b_off, (const T*)B, x_off,
                                   (const T*)X, y_off, (const T*)Y, o_off, (T*)O, R, cols, max_q,
                                   max_r, order, xrows, orows);
    }
    return skel_last_error();
  };
  if constexpr (sizeof(T) != sizeof(double)) {
    // complex, few RHS: the real-ified DMMA kernel (2R real columns)
    if (R >= 1 && R <= 8 && dmma_few_enabled()) {
      const int nt = 2 * R <= 8 ? 1 : 2;
      const int kmax = ((2 * max_q + 3) & ~3) + ((2 * max_r + 3) & ~3);
      const size_t smem = (size_t)kmax * (8 * nt + 8) * sizeof(double);
      const int threads = 32 * std::min(8, std::max(1, (max_p + 7) / 8));
      if (smem <= optin) {
        const bool rows = xrows || orows;
        auto launch = [&](auto kern) -> int {
          SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          kern<<<nbox, threads, smem, st>>>(p, q, r, a_off, (const double*)A, b_off, (const double*)B,
                                            x_off, (const double*)X, y_off, (const double*)Y, o_off,
                                            (double*)O, R, order, xrows, orows);
          return skel_last_error();
        };
        if (nt == 1) return rows ? launch(k_level_dmma_few<1, true, true>) : launch(k_level_dmma_few<1, false, true>);
        return rows ? launch(k_level_dmma_few<2, true, true>) : launch(k_level_dmma_few<2, false, true>);
      }
    }
  }
  if constexpr (sizeof(T) == sizeof(double)) {
    if (R >= 1 && R <= 32 && dmma_few_enabled()) {
      const int nt = R <= 8 ? 1 : (R <= 16 ? 2 : 4);
      const int kmax = ((max_q + 3) & ~3) + ((max_r + 3) & ~3);
      const size_t smem = (size_t)kmax * (8 * nt + 8) * sizeof(double);
      const int threads = 32 * std::min(8, std::max(1, (max_p + 7) / 8));
      if (smem <= optin) {
        const bool rows = xrows || orows;
        auto launch = [&](auto kern) -> int {
          SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
          kern<<<nbox, threads, smem, st>>>(p, q, r, a_off, (const double*)A, b_off, (const double*)B,
                                            x_off, (const double*)X, y_off, (const double*)Y, o_off,
                                            (double*)O, R, order, xrows, orows);
          return skel_last_error();
        };
        // TMA-staged variant: factor blocks by 1-D bulk copies into warp buffers
        const int bufd = (8 * (max_q + max_r) + 4 + 1) & ~1;
        const size_t bsmem = 64 + ((size_t)(threads / 32) * bufd + (size_t)kmax * (8 * nt + 8)) * sizeof(double);
        if (bulk_few_enabled(nt) && bsmem <= optin) {
          auto blaunch = [&](auto kern) -> int {
            SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsmem));
            kern<<<nbox, threads, bsmem, st>>>(p, q, r, a_off, (const double*)A, b_off, (const double*)B,
                                               x_off, (const double*)X, y_off, (const double*)Y, o_off,
                                               (double*)O, R, order, xrows, orows, bufd);
            return skel_last_error();
          };
          if (nt == 1) return rows ? blaunch(k_level_bulk_few<1, true>) : blaunch(k_level_bulk_few<1, false>);
          if (nt == 2) return rows ? blaunch(k_level_bulk_few<2, true>) : blaunch(k_level_bulk_few<2, false>);
          return rows ? blaunch(k_level_bulk_few<4, true>) : blaunch(k_level_bulk_few<4, false>);
        }
        if (nt == 1) return rows ? launch(k_level_dmma_few<1, true>) : launch(k_level_dmma_few<1, false>);
        if (nt == 2) return rows ? launch(k_level_dmma_few<2, true>) : launch(k_level_dmma_few<2, false>);
        return rows ? launch(k_level_dmma_few<4, true>) : launch(k_level_dmma_few<4, false>);
      }
    }
    if (R >= 64 && !xrows && !orows && dmma_many_mode() == 1) {
      const int kp = ((max_q + 3) & ~3) + ((max_r + 3) & ~3);
      {
        int chunks = (R + 31) / 32;
        int per = 1;
        while (per < chunks && (long long)nbox * ((chunks + per * 2 - 1) / (per * 2)) >= 4LL * 148 * 4) per *= 2;
        const int cols = per * 32;
        dim3 grid(nbox, (R + cols - 1) / cols);
        const int tasks = ((max_p + 7) / 8 + 7) / 8 * ((cols + 15) / 16);
        const int threads = 32 * std::min(8, tasks);
        const int aw = (int)((((size_t)max_p + 7) & ~(size_t)7) * (kp + 16));
        const size_t psmem = (size_t)aw * sizeof(double) + (size_t)(threads / 32) * 4 * 16 * 16 * sizeof(double);
        if (psmem <= optin) {
          auto launch = [&](auto kern) -> int {
            SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
            kern<<<grid, threads, psmem, st>>>(p, q, r, a_off, (const double*)A, b_off, (const double*)B,
                                               x_off, (const double*)X, y_off, (const double*)Y, o_off,
                                               (double*)O, R, cols, order, aw);
            return skel_last_error();
          };
          return max_p <= 32 ? launch(k_level_dmma_pipe<4, 4>) : launch(k_level_dmma_pipe<8, 4>);
        }
      }
    }
    if (R >= 64 && !xrows && !orows) {
      constexpr int CB = 32;
      const int maxk = max_q + max_r;
      size_t smem = ((((size_t)max_p + 7) & ~(size_t)7) * (maxk + 1 + 4) +
                     2 * (size_t)(maxk + 4) * (CB + 8)) * sizeof(double);
      if (smem <= optin) {
        int chunks = (R + CB - 1) / CB;
        int per = 1;
        while (per < chunks && (long long)nbox * ((chunks + per * 2 - 1) / (per * 2)) >= 4LL * 148 * 4) per *= 2;
        const int cols = per * CB;
        dim3 grid(nbox, (R + cols - 1) / cols);
        SKEL_TRY(cudaFuncSetAttribute(k_level_dmma<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        k_level_dmma<CB><<<grid, 128, smem, st>>>(p, q, r, a_off, (const double*)A, b_off,
                                                  (const double*)B, x_off, (const double*)X, y_off,
                                                  (const double*)Y, o_off, (double*)O, R, cols, max_p,
                                                  maxk + 4, order);
        return skel_last_error();
      }
    }
  }
  // register tiles picked per RHS count on B200 (the R=16 sweeps are bound
  // by shared-memory load issue: TN > 1 reuses each staged A element)
  const bool rows = xrows || orows;
  if (R <= 2)
    return rows ? go(k_level_gemm<T, 4, 1, 2, true, true>, k_level_gemm<T, 4, 1, 2, false, true>, 2)
                : go(k_level_gemm<T, 4, 1, 2, true>, k_level_gemm<T, 4, 1, 2, false>, 2);
  if (R <= 8)
    return rows ? go(k_level_gemm<T, 4, 1, 8, true, true>, k_level_gemm<T, 4, 1, 8, false, true>, 8)
                : go(k_level_gemm<T, 4, 1, 8, true>, k_level_gemm<T, 4, 1, 8, false>, 8);
  if (R <= 16)
    return rows ? go(k_level_gemm<T, 4, 2, 16, true, true>, k_level_gemm<T, 4, 2, 16, false, true>, 16)
                : go(k_level_gemm<T, 4, 2, 16, true>, k_level_gemm<T, 4, 2, 16, false>, 16);
  if (rows) return -3;                     // row maps: R <= 16 only
  if (R <= 32) return go(k_level_gemm<T, 4, 4, 32, true>, k_level_gemm<T, 4, 4, 32, false>, 32);
  return go(k_level_gemm<T, 4, 4, 64, true>, k_level_gemm<T, 4, 4, 64, false>, 64);
}

// y (K x R) = M (K x Kc) x (Kc x R): one warp per output row, lanes over
// columns; the row of M is read once per warp (broadcast), four partial sums
template <class T>
__global__ void __launch_bounds__(256) k_dense_apply(const T* __restrict__ M, int K, int Kc,
                                                     const T* __restrict__ x, T* __restrict__ y, int R) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= K) return;
  const int lane = threadIdx.x & 31;
  const T* mr = M + (int64_t)i * Kc;
  for (int c = blockIdx.y * 32 + lane; c < R && c < (int)(blockIdx.y + 1) * 32; c += 32) {
    T a0 = T(0.0), a1 = T(0.0), a2 = T(0.0), a3 = T(0.0);
    int j = 0;
    for (; j + 3 < Kc; j += 4) {
      a0 += __ldg_T(mr + j) * x[(int64_t)j * R + c];
      a1 += __ldg_T(mr + j + 1) * x[(int64_t)(j + 1) * R + c];
      a2 += __ldg_T(mr + j + 2) * x[(int64_t)(j + 2) * R + c];
      a3 += __ldg_T(mr + j + 3) * x[(int64_t)(j + 3) * R + c];
    }
    for (; j < Kc; ++j) a0 += __ldg_T(mr + j) * x[(int64_t)j * R + c];
    y[(int64_t)i * R + c] = (a0 + a1) + (a2 + a3);
  }
}

// one row per thread group of R lanes (R <= 32) or one thread per row chunk
template <class T>
__global__ void k_permute(const int64_t* __restrict__ perm, int64_t N, const T* __restrict__ src,
                          T* __restrict__ dst, int R, int scatter) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (i >= N) return;
  const int64_t p = perm[i];
  for (int c = threadIdx.x; c < R; c += blockDim.x) {
    if (scatter) dst[p * R + c] = src[i * R + c];
    else dst[i * R + c] = src[p * R + c];
  }
}

__global__ void k_compact(int nseg, const int64_t* src_off, const int32_t* len, const int64_t* dst_off,
                          const int32_t* src, int32_t* dst) {
  int seg = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (seg >= nseg) return;
  const int lane = threadIdx.x & 31;
  const int L = len[seg];
  const int32_t* s = src + src_off[seg];
  int32_t* d = dst + dst_off[seg];
  for (int t = lane; t < L; t += 32) d[t] = s[t];
}

extern "C" {

int skel_sweep_up_ex(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                     const int64_t* koff, const int64_t* m_off, const void* M, const void* u,
                     void* out, int32_t R, int32_t field, int32_t max_n, int32_t max_k,
                     const int32_t* order, void* stream) {
  return skel_sweep_up_rows(nbox, n, k, noff, koff, m_off, M, u, out, R, field, max_n, max_k, order,
                            nullptr, stream);
}

int skel_sweep_up_rows(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                       const int64_t* koff, const int64_t* m_off, const void* M, const void* u,
                       void* out, int32_t R, int32_t field, int32_t max_n, int32_t max_k,
                       const int32_t* order, const int64_t* urows, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  // out (k x R) = M (k x n) u (n x R); u rows gathered through urows if given
  if (urows && R > 16) return -3;
  if (field == 0)
    return level_gemm<double>(nbox, k, n, nullptr, m_off, M, nullptr, nullptr, noff, u, nullptr,
                              nullptr, koff, out, R, max_k, max_n, 0, order, st, urows, nullptr);
  return level_gemm<zc>(nbox, k, n, nullptr, m_off, M, nullptr, nullptr, noff, u, nullptr, nullptr,
                        koff, out, R, max_k, max_n, 0, order, st, urows, nullptr);
}

int skel_sweep_down_ex(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                       const int64_t* koff, const int64_t* a_off, const void* A,
                       const int64_t* b_off, const void* B, const void* u, const void* v, void* w,
                       int32_t R, int32_t field, int32_t max_n, int32_t max_k,
                       const int32_t* order, void* stream) {
  return skel_sweep_down_rows(nbox, n, k, noff, koff, a_off, A, b_off, B, u, v, w, R, field, max_n,
                              max_k, order, nullptr, nullptr, stream);
}

int skel_sweep_down_rows(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                         const int64_t* koff, const int64_t* a_off, const void* A,
                         const int64_t* b_off, const void* B, const void* u, const void* v, void* w,
                         int32_t R, int32_t field, int32_t max_n, int32_t max_k,
                         const int32_t* order, const int64_t* urows, const int64_t* wrows,
                         void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  // w (n x R) = A (n x n) u (n x R) + B (n x k) v (k x R); u rows gathered
  // through urows, w rows scattered through wrows, if given
  if ((urows || wrows) && R > 16) return -3;
  if (field == 0)
    return level_gemm<double>(nbox, n, n, k, a_off, A, b_off, B, noff, u, koff, v, noff, w, R, max_n,
                              max_n, max_k, order, st, urows, wrows);
  return level_gemm<zc>(nbox, n, n, k, a_off, A, b_off, B, noff, u, koff, v, noff, w, R, max_n, max_n,
                        max_k, order, st, urows, wrows);
}

int skel_dense_apply(const void* M, int32_t K, int32_t Kc, const void* x, void* y, int32_t R,
                     int32_t field, void* stream) {
  if ((int64_t)K * R == 0) return 0;
  dim3 grid((K + 7) / 8, (R + 31) / 32);
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) k_dense_apply<double><<<grid, 256, 0, st>>>((const double*)M, K, Kc, (const double*)x, (double*)y, R);
  else k_dense_apply<zc><<<grid, 256, 0, st>>>((const zc*)M, K, Kc, (const zc*)x, (zc*)y, R);
  return skel_last_error();
}

int skel_permute_rows(const int64_t* perm, int64_t N, const void* src, void* dst, int32_t R,
                      int32_t scatter, int32_t field, void* stream) {
  if (N == 0 || R <= 0) return 0;
  int tx = R >= 32 ? 32 : (R >= 16 ? 16 : (R >= 8 ? 8 : (R >= 4 ? 4 : (R >= 2 ? 2 : 1))));
  dim3 block(tx, 256 / tx);
  int blocks = (int)((N + block.y - 1) / block.y);
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) k_permute<double><<<blocks, block, 0, st>>>(perm, N, (const double*)src, (double*)dst, R, scatter);
  else k_permute<zc><<<blocks, block, 0, st>>>(perm, N, (const zc*)src, (zc*)dst, R, scatter);
  return skel_last_error();
}

int skel_compact_i32(int32_t nseg, const int64_t* src_off, const int32_t* len, const int64_t* dst_off,
                     const int32_t* src, int32_t* dst, void* stream) {
  if (nseg <= 0) return 0;
  int blocks = (nseg + 7) / 8;
  k_compact<<<blocks, 256, 0, (cudaStream_t)stream>>>(nseg, src_off, len, dst_off, src, dst);
  return skel_last_error();
}

}  // extern "C"
