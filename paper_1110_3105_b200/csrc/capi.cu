// capi.cu -- library self-description entry points.
#include "common.cuh"
#include "entries.cuh"

extern "C" {

const char* skel_version(void) { return "skel_b200 0.1.0 sm_100a"; }

int skel_device_query(int32_t* sm_count, int32_t* smem_optin, int32_t* cc_major, int32_t* cc_minor) {
  int dev = 0;
  SKEL_TRY(cudaGetDevice(&dev));
  int v = 0;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  *sm_count = v;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  *smem_optin = v;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMajor, dev));
  *cc_major = v;
  SKEL_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrComputeCapabilityMinor, dev));
  *cc_minor = v;
  return 0;
}

}  // extern "C"

// ---- FP64 peak probes (bench.py's roofline denominator for FP64 kernels;
// MEASURED_PEAKS.json carries only HBM and bf16 figures) --------------------
__global__ void __launch_bounds__(256) k_dfma_probe(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = 1e-3 * (threadIdx.x + c);
  const double b = 0.999999999, d = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = fma(a[c], b, d);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

__global__ void __launch_bounds__(256) k_dmma_probe(double* out, int iters) {
  double acc[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) { acc[c][0] = 1e-3 * c; acc[c][1] = 2e-3 * c; }
  const double av = 1e-3 * (threadIdx.x & 31), bv = 0.5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1])
                   : "d"(av), "d"(bv));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

extern "C" int skel_fp64_probe(int32_t kind, int32_t iters, double* scratch, double* flops,
                               void* stream) {
  int sms = skel_sm_count();
  int blocks = sms * 8, threads = 256;
  cudaStream_t st = (cudaStream_t)stream;
  if (kind == 0) {
    k_dfma_probe<<<blocks, threads, 0, st>>>(scratch, iters);
    *flops = 2.0 * 8.0 * (double)iters * blocks * threads;
  } else {
    k_dmma_probe<<<blocks, threads, 0, st>>>(scratch, iters);
    *flops = 512.0 * 4.0 * (double)iters * blocks * (threads / 32);
  }
  return skel_last_error();
}

// H0^(1)(z) = J0(z) + i Y0(z) elementwise (kernels.py:65-75; sk_hankel<0>, the same
// function the Helmholtz entries use).  out: interleaved complex.
__global__ void k_bessel_h0(const double* __restrict__ z, int64_t n, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = z[i];
  double hj, hy;
  sk_hankel<0>(x, hj, hy);
  out[2 * i] = hj;
  out[2 * i + 1] = hy;
}

extern "C" int skel_bessel_h0(const double* z, int64_t n, double* out, void* stream) {
  if (n <= 0) return 0;
  k_bessel_h0<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(z, n, out);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}
