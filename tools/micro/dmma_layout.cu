// Fragment layout and dependent-issue latency of mma.sync m8n8k4 f64 (SASS DMMA) on sm_100a.
// Layout check: A[m][k] = 100 m + k, B[k][n] = 10 k + n (exact in FP64); each lane's claimed fragment
// coordinates are used to load A, B and to check D = A B element by element.
#include <cstdio>
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__global__ void layout(int* bad) {
  const int t = threadIdx.x;
  // claimed: A: row t>>2, col t&3;  B: row (k) t&3, col (n) t>>2;  C: row t>>2, cols 2 (t&3) + {0,1}
  const double a = 100.0 * (t >> 2) + (t & 3), b = 10.0 * (t & 3) + (t >> 2);
  double d0 = 0, d1 = 0;
  dmma(d0, d1, a, b);
  const int m = t >> 2;
  for (int i = 0; i < 2; ++i) {
    const int n = 2 * (t & 3) + i;
    double ref = 0;
    for (int k = 0; k < 4; ++k) ref += (100.0 * m + k) * (10.0 * k + n);
    if ((i ? d1 : d0) != ref) atomicAdd(bad, 1);
  }
}
__global__ void lat(double* out, long long* cyc, int iters) {
  double d0 = 0, d1 = 0, a = threadIdx.x * 1e-3, b = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) dmma(d0, d1, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = d0 + d1;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  int* bad; cudaMallocManaged(&bad, 4); *bad = 0;
  layout<<<1, 32>>>(bad);
  cudaDeviceSynchronize();
  printf("layout mismatches: %d (0 = fragment layout as claimed)\n", *bad);
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 8);
  lat<<<1, 32>>>(o, c, 1000);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 10000);
  cudaDeviceSynchronize();
  printf("dependent DMMA latency: %.1f clk\n", *c / 10000.0);
  return 0;
}
