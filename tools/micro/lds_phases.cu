// LDS.128 / STS.128 wavefront rules on sm_100a: each kernel runs one access pattern many times;
// compare ncu l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum per instruction.
// pattern(lane) -> 16-byte slot index:
//   0 distinct: lane                   1 all same: 0
//   2 lane % 8 (same 8 in every quarter)   3 lane / 8 (quarter-uniform)
//   4 lane % 4                          5 (lane % 8) * 8 (8-way conflict)   6 lane % 16
#include <cstdio>
__device__ __forceinline__ int pat(int p, int l) {
  switch (p) {
    case 0: return l;
    case 1: return 0;
    case 2: return l % 8;
    case 3: return l / 8;
    case 4: return l % 4;
    case 5: return (l % 8) * 8;
    default: return l % 16;
  }
}
template <int P>
__global__ void k(double* out, int iters) {
  __shared__ double2 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_double2(i, -i);
  __syncthreads();
  const int l = threadIdx.x & 31;
  const int a = pat(P, l);
  double acc = 0;
  volatile int z = 0;
  for (int it = 0; it < iters; ++it) {
    double2 v = s[a + (z & it)];
    acc += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  double* o;
  cudaMalloc(&o, 148 * 256 * 8);
  k<0><<<148, 256>>>(o, 1000);
  k<1><<<148, 256>>>(o, 1000);
  k<2><<<148, 256>>>(o, 1000);
  k<3><<<148, 256>>>(o, 1000);
  k<4><<<148, 256>>>(o, 1000);
  k<5><<<148, 256>>>(o, 1000);
  k<6><<<148, 256>>>(o, 1000);
  cudaDeviceSynchronize();
  printf("done\n");
  return 0;
}
