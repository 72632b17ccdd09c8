// DFMA throughput vs independent chains per thread (ILP) and resident warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters, double a, double b) {
  double x[C];
#pragma unroll
  for (int i = 0; i < C; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 32 / C; ++r)
#pragma unroll
      for (int i = 0; i < C; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
template <int C>
void run(int warps_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d; cudaMalloc(&d, 8);
  int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
  int blocks_per_sm = warps_per_sm * 32 / threads;
  int iters = 2000;
  k<C><<<sms * blocks_per_sm, threads>>>(d, 10, 0.9999, 1e-6);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<C><<<sms * blocks_per_sm, threads>>>(d, iters, 0.9999, 1e-6);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 32 * iters * (double)sms * blocks_per_sm * threads;
  printf("chains %2d warps/SM %2d : %6.2f TF/s\n", C, warps_per_sm, flops / ms / 1e9);
  cudaFree(d);
}
int main() {
  int ws[] = {4, 8, 12, 16, 32};
  for (int w : ws) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); run<16>(w); }
  return 0;
}
