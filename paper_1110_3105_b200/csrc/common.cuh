// common.cuh -- scalar types, warp reductions and launch helpers shared by
// the sm_100a kernels of libskel_sm100.so.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <math.h>

#include "../../include/skel_b200.h"

#define SKEL_WARP 32

// numpy's float64 values of 2*pi and 4*pi (np.pi doubled exactly)
#define SKEL_TWO_PI 6.283185307179586
#define SKEL_FOUR_PI 12.566370614359172

// ---------------------------------------------------------------------------
// complex128 (numpy layout: re, im interleaved)
struct zc {
  double re, im;
  __host__ __device__ zc() : re(0.0), im(0.0) {}
  __host__ __device__ zc(double r) : re(r), im(0.0) {}
  __host__ __device__ zc(double r, double i) : re(r), im(i) {}
};
__device__ __forceinline__ zc operator+(zc a, zc b) { return zc(a.re + b.re, a.im + b.im); }
__device__ __forceinline__ zc operator-(zc a, zc b) { return zc(a.re - b.re, a.im - b.im); }
__device__ __forceinline__ zc operator-(zc a) { return zc(-a.re, -a.im); }
__device__ __forceinline__ zc operator*(zc a, zc b) {
  return zc(a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re);
}
__device__ __forceinline__ zc operator*(zc a, double s) { return zc(a.re * s, a.im * s); }
__device__ __forceinline__ zc operator*(double s, zc a) { return zc(a.re * s, a.im * s); }
__device__ __forceinline__ zc& operator+=(zc& a, zc b) { a.re += b.re; a.im += b.im; return a; }
__device__ __forceinline__ zc& operator-=(zc& a, zc b) { a.re -= b.re; a.im -= b.im; return a; }
__device__ __forceinline__ bool operator==(zc a, zc b) { return a.re == b.re && a.im == b.im; }
__device__ __forceinline__ bool operator!=(zc a, zc b) { return !(a == b); }
__device__ __forceinline__ zc operator/(zc a, zc b) {
  // Smith's algorithm (numpy's complex division is also scaled)
  if (fabs(b.re) >= fabs(b.im)) {
    double r = b.im / b.re, d = b.re + b.im * r;
    return zc((a.re + a.im * r) / d, (a.im - a.re * r) / d);
  } else {
    double r = b.re / b.im, d = b.re * r + b.im;
    return zc((a.re * r + a.im) / d, (a.im * r - a.re) / d);
  }
}

__device__ __forceinline__ double sk_abs2(double a) { return a * a; }
__device__ __forceinline__ double sk_abs2(zc a) { return a.re * a.re + a.im * a.im; }
__device__ __forceinline__ double sk_abs(double a) { return fabs(a); }
__device__ __forceinline__ double sk_abs(zc a) { return hypot(a.re, a.im); }
// |a| as LAPACK's i?amax ranks pivots: |x| real, |re|+|im| complex (dcabs1)
__device__ __forceinline__ double sk_pivabs(double a) { return fabs(a); }
__device__ __forceinline__ double sk_pivabs(zc a) { return fabs(a.re) + fabs(a.im); }
__device__ __forceinline__ double sk_conj(double a) { return a; }
__device__ __forceinline__ zc sk_conj(zc a) { return zc(a.re, -a.im); }
__device__ __forceinline__ double sk_real(double a) { return a; }
__device__ __forceinline__ double sk_real(zc a) { return a.re; }

template <class T> __device__ __forceinline__ T sk_zero() { return T(0.0); }

__device__ __forceinline__ double __ldg_T(const double* p) { return __ldg(p); }
__device__ __forceinline__ zc __ldg_T(const zc* p) {
  double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return zc(v.x, v.y);
}

// ---------------------------------------------------------------------------
// warp reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ zc warp_sum(zc v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.re += __shfl_xor_sync(0xffffffffu, v.re, o);
    v.im += __shfl_xor_sync(0xffffffffu, v.im, o);
  }
  return v;
}
__device__ __forceinline__ double shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double shfl_xor_T(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ zc shfl_xor_T(zc v, int o) {
  return zc(__shfl_xor_sync(0xffffffffu, v.re, o), __shfl_xor_sync(0xffffffffu, v.im, o));
}
__device__ __forceinline__ zc shfl(zc v, int src) {
  return zc(__shfl_sync(0xffffffffu, v.re, src), __shfl_sync(0xffffffffu, v.im, src));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS): global -> shared without a register round trip, so a
// thread keeps all of its staging loads in flight at once
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

// One-instruction bulk prefetch of a contiguous global range into L2 by the
// TMA unit (cp.async.bulk.prefetch.L2, sm_90+): the range is widened to
// 16-byte boundaries (its ends may touch a neighbouring block of the same
// slab, which is harmless for a prefetch) and split in <= 1 MB pieces.
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, size_t bytes) {
  if (bytes == 0) return;
  uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  while (a < e) {
    const uint32_t n = (uint32_t)((e - a) < (1u << 20) ? (e - a) : (1u << 20));
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"(n) : "memory");
    a += n;
  }
}
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// copy `count` elements of T from global to shared (8-byte words, async)
template <class T>
__device__ __forceinline__ void cp_async_block(T* dst, const T* src, int64_t count) {
  constexpr int W = sizeof(T) / 8;
  double* d = reinterpret_cast<double*>(dst);
  const double* s = reinterpret_cast<const double*>(src);
  for (int64_t e = threadIdx.x; e < count * W; e += blockDim.x) cp_async8(d + e, s + e);
}

// ---------------------------------------------------------------------------
// error plumbing
#define SKEL_TRY(expr)                                   \
  do {                                                   \
    cudaError_t _e = (expr);                             \
    if (_e != cudaSuccess) return (int)_e;               \
  } while (0)

static inline int skel_last_error() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

static inline int skel_smem_optin() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return v;
}

static inline int skel_sm_count() {
  int dev = 0, v = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}
