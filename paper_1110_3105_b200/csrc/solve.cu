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
#include "common.cuh"

#define SWEEP_CB 32   // RHS columns per CTA chunk

template <class T>
__global__ void __launch_bounds__(256) k_sweep_up(const int32_t* __restrict__ nn, const int32_t* __restrict__ kk,
                                                  const int64_t* __restrict__ noff, const int64_t* __restrict__ koff,
                                                  const int64_t* __restrict__ m_off, const T* __restrict__ M,
                                                  const T* __restrict__ u, T* __restrict__ out, int R) {
  extern __shared__ __align__(16) unsigned char smem[];
  T* su = reinterpret_cast<T*>(smem);
  const int a = blockIdx.x;
  const int n = nn[a], k = kk[a];
  if (k == 0) return;
  const int c0 = blockIdx.y * SWEEP_CB;
  const int cb = min(SWEEP_CB, R - c0);
  const T* ua = u + noff[a] * R;
  for (int e = threadIdx.x; e < n * cb; e += blockDim.x) {
    int j = e / cb, c = e - j * cb;
    su[e] = ua[(int64_t)j * R + c0 + c];
  }
  __syncthreads();
  const T* Ma = M + m_off[a];
  T* oa = out + koff[a] * R;
  for (int e = threadIdx.x; e < k * cb; e += blockDim.x) {
    int t = e / cb, c = e - t * cb;
    const T* mr = Ma + (int64_t)t * n;
    T acc = T(0.0);
    for (int j = 0; j < n; ++j) acc += __ldg_T(mr + j) * su[j * cb + c];
    oa[(int64_t)t * R + c0 + c] = acc;
  }
}

template <class T>
__global__ void __launch_bounds__(256) k_sweep_down(const int32_t* __restrict__ nn, const int32_t* __restrict__ kk,
                                                    const int64_t* __restrict__ noff, const int64_t* __restrict__ koff,
                                                    const int64_t* __restrict__ a_off, const T* __restrict__ A,
                                                    const int64_t* __restrict__ b_off, const T* __restrict__ B,
                                                    const T* __restrict__ u, const T* __restrict__ v,
                                                    T* __restrict__ w, int R) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int a = blockIdx.x;
  const int n = nn[a], k = kk[a];
  if (n == 0) return;
  const int c0 = blockIdx.y * SWEEP_CB;
  const int cb = min(SWEEP_CB, R - c0);
  T* su = reinterpret_cast<T*>(smem);
  T* sv = su + (size_t)n * cb;
  const T* ua = u + noff[a] * R;
  const T* va = v + koff[a] * R;
  for (int e = threadIdx.x; e < n * cb; e += blockDim.x) {
    int j = e / cb, c = e - j * cb;
    su[e] = ua[(int64_t)j * R + c0 + c];
  }
  for (int e = threadIdx.x; e < k * cb; e += blockDim.x) {
    int j = e / cb, c = e - j * cb;
    sv[e] = va[(int64_t)j * R + c0 + c];
  }
  __syncthreads();
  const T* Aa = A + a_off[a];
  const T* Ba = B + b_off[a];
  T* wa = w + noff[a] * R;
  for (int e = threadIdx.x; e < n * cb; e += blockDim.x) {
    int i = e / cb, c = e - i * cb;
    const T* ar = Aa + (int64_t)i * n;
    T acc = T(0.0);
    for (int j = 0; j < n; ++j) acc += __ldg_T(ar + j) * su[j * cb + c];
    const T* br = Ba + (int64_t)i * k;
    T acc2 = T(0.0);
    for (int t = 0; t < k; ++t) acc2 += __ldg_T(br + t) * sv[t * cb + c];
    wa[(int64_t)i * R + c0 + c] = (k > 0) ? acc + acc2 : acc;
  }
}

template <class T>
__global__ void k_dense_apply(const T* __restrict__ M, int K, int Kc, const T* __restrict__ x,
                              T* __restrict__ y, int R) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)K * R) return;
  int i = (int)(e / R), c = (int)(e - (int64_t)i * R);
  const T* mr = M + (int64_t)i * Kc;
  T acc = T(0.0);
  for (int j = 0; j < Kc; ++j) acc += mr[j] * x[(int64_t)j * R + c];
  y[e] = acc;
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

template <class T>
static int sweep_up_impl(int nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                         const int64_t* koff, const int64_t* m_off, const void* M, const void* u,
                         void* out, int R, int max_n, cudaStream_t st) {
  if (nbox <= 0 || R <= 0) return 0;
  dim3 grid(nbox, (R + SWEEP_CB - 1) / SWEEP_CB);
  size_t smem = (size_t)max_n * SWEEP_CB * sizeof(T);
  auto kern = k_sweep_up<T>;
  SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, 128, smem, st>>>(n, k, noff, koff, m_off, (const T*)M, (const T*)u, (T*)out, R);
  return skel_last_error();
}

template <class T>
static int sweep_down_impl(int nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                           const int64_t* koff, const int64_t* a_off, const void* A,
                           const int64_t* b_off, const void* B, const void* u, const void* v,
                           void* w, int R, int max_nk, cudaStream_t st) {
  if (nbox <= 0 || R <= 0) return 0;
  dim3 grid(nbox, (R + SWEEP_CB - 1) / SWEEP_CB);
  size_t smem = (size_t)max_nk * SWEEP_CB * sizeof(T);
  auto kern = k_sweep_down<T>;
  SKEL_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kern<<<grid, 128, smem, st>>>(n, k, noff, koff, a_off, (const T*)A, b_off, (const T*)B, (const T*)u,
                                (const T*)v, (T*)w, R);
  return skel_last_error();
}

extern "C" {

int skel_sweep_up_ex(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                     const int64_t* koff, const int64_t* m_off, const void* M, const void* u,
                     void* out, int32_t R, int32_t field, int32_t max_n, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) return sweep_up_impl<double>(nbox, n, k, noff, koff, m_off, M, u, out, R, max_n, st);
  return sweep_up_impl<zc>(nbox, n, k, noff, koff, m_off, M, u, out, R, max_n, st);
}

int skel_sweep_down_ex(int32_t nbox, const int32_t* n, const int32_t* k, const int64_t* noff,
                       const int64_t* koff, const int64_t* a_off, const void* A,
                       const int64_t* b_off, const void* B, const void* u, const void* v, void* w,
                       int32_t R, int32_t field, int32_t max_nk, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0)
    return sweep_down_impl<double>(nbox, n, k, noff, koff, a_off, A, b_off, B, u, v, w, R, max_nk, st);
  return sweep_down_impl<zc>(nbox, n, k, noff, koff, a_off, A, b_off, B, u, v, w, R, max_nk, st);
}

int skel_dense_apply(const void* M, int32_t K, int32_t Kc, const void* x, void* y, int32_t R,
                     int32_t field, void* stream) {
  int64_t tot = (int64_t)K * R;
  if (tot == 0) return 0;
  int blocks = (int)((tot + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (field == 0) k_dense_apply<double><<<blocks, 256, 0, st>>>((const double*)M, K, Kc, (const double*)x, (double*)y, R);
  else k_dense_apply<zc><<<blocks, 256, 0, st>>>((const zc*)M, K, Kc, (const zc*)x, (zc*)y, R);
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
