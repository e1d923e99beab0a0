// Developer probe: DMMA.8x8x4 throughput vs warps/SM, chains/warp, operand reuse.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH, bool DIST>
__global__ void k(double* out, const double* in, int iters) {
  double acc[CH][2];
  double a[CH], b[CH];
  for (int c = 0; c < CH; ++c) { acc[c][0] = acc[c][1] = 0; a[c] = in[(threadIdx.x + c) & 63]; b[c] = in[(threadIdx.x * 3 + c) & 63]; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const double av = DIST ? a[c] : a[0], bv = DIST ? b[c] : b[0];
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(av), "d"(bv));
    }
  }
  double s = 0;
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1.2345) out[0] = s;
}
template <int CH, bool DIST>
void run(int warps_per_block, int blocks_per_sm, double* o, double* in) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<CH, DIST><<<sms * blocks_per_sm, 32 * warps_per_block>>>(o, in, 10);
  cudaEventRecord(e0);
  k<CH, DIST><<<sms * blocks_per_sm, 32 * warps_per_block>>>(o, in, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * CH * iters * (double)sms * blocks_per_sm * warps_per_block;
  printf("chains %2d dist %d warps/SM %3d: %.1f TF/s\n", CH, DIST, warps_per_block * blocks_per_sm, fl / ms / 1e9);
}
int main() {
  double *o, *in; cudaMalloc(&o, 64); cudaMalloc(&in, 64 * 8); double h[64]; for (int i = 0; i < 64; ++i) h[i] = 0.37 + 0.013 * i * ((i & 1) ? -1 : 1); cudaMemcpy(in, h, 512, cudaMemcpyHostToDevice);
  for (int w : {4, 8, 16, 32, 64}) {
    run<4, false>(w < 8 ? w : 8, w < 8 ? 1 : w / 8, o, in);
    run<4, true>(w < 8 ? w : 8, w < 8 ? 1 : w / 8, o, in);
    run<10, true>(w < 8 ? w : 8, w < 8 ? 1 : w / 8, o, in);
    run<16, true>(w < 8 ? w : 8, w < 8 ? 1 : w / 8, o, in);
  }
  return 0;
}
