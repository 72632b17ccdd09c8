// FP64 tensor-core (mma.sync m8n8k4 f64, SASS DMMA) throughput on sm_100a, alone and concurrently with
// FP64 CUDA-core FMAs (DFMA): do the two FP64 paths share hardware?
//   mode 0: DMMA only (8 independent accumulator chains per warp)
//   mode 1: DFMA only (8 independent chains per thread)
//   mode 2: both interleaved in every warp (same per-warp counts as modes 0 and 1 together)
//   mode 3: half the warps DMMA, half DFMA
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int MODE>
__global__ void k(double* out, int iters) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double c[8][2], f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { c[i][0] = c[i][1] = 0.0; f[i] = lane * 1e-2 + i; }
  const bool do_mma = MODE == 0 || MODE == 2 || (MODE == 3 && (warp & 1) == 0);
  const bool do_fma = MODE == 1 || MODE == 2 || (MODE == 3 && (warp & 1) == 1);
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    if (do_fma) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], 0.999999, 1e-7);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
float run(double* out, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<blocks, threads>>>(out, 10);
  cudaEventRecord(e0);
  k<MODE><<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  const int iters = 20000;
  for (int wps : {4, 8, 16, 32}) {
    const int blocks = sms * (wps / 4 > 0 ? wps / 4 : 1), threads = 128;
    const double warps = (double)blocks * threads / 32;
    float m0 = run<0>(out, blocks, threads, iters), m1 = run<1>(out, blocks, threads, iters);
    float m2 = run<2>(out, blocks, threads, iters), m3 = run<3>(out, blocks, threads, iters);
    const double mma_fl = warps * iters * 8 * 512.0, fma_fl = warps * 32 * iters * 32 * 2.0;
    printf("warps/SM %2d | DMMA only %6.2f TF/s | DFMA only %6.2f TF/s | both per warp %6.2f ms (%6.2f TF/s; serial sum %6.2f ms) | split warps %6.2f ms (%6.2f TF/s)\n",
           wps, mma_fl / m0 / 1e9, fma_fl / m1 / 1e9, m2, (mma_fl + fma_fl) / m2 / 1e9, m0 + m1, m3,
           (mma_fl + fma_fl) / 2 / m3 / 1e9);
  }
  return 0;
}
