// abc_kernel.cuh -- ABC-model |M|^2 kernel (App. F; include/abc.h), sm_100a, FP64.
//
// One thread per phase-space point, grid-stride over a persistent grid.  The thread loads the incoming
// A-on and the N B-on momenta from the SoA rows (coalesced: consecutive threads read consecutive
// doubles of a row; the outgoing A-on is not needed by the amplitude and is not read), evaluates the
// generated straight-line body (gen/abc.py: CDAG trie or Berends-Giele currents) in registers and
// stores g^(2N) M^2.  Bound: HBM for N <= 4 (8 + 32 (N + 1) bytes against a few hundred flops per
// point), FP64 ALU for the CDAG at N = 6 (720 joins).
#pragma once
#include <cuda_runtime.h>

namespace qed {

constexpr double kMA2 = 1.0 * 1.0;    // m_A^2 (include/abc.h ABC_MASS_A)
constexpr double kMC2 = 1.2 * 1.2;    // m_C^2 (ABC_MASS_C)

struct AbcArgs {
  const double* mom;       // device SoA: mom[(4 j + mu) * n_points + i]
  double* out;             // device: n_points doubles
  long long n_points;
  int part[10];            // particle (row group) of B-on i
  double sg[10];           // +1 incoming B-on (q = +k), -1 outgoing (q = -k)
  double g2n;              // g^(2N)
};

template <int N, class Body>
__global__ void __launch_bounds__(256) abc_kernel(AbcArgs a) {
  const long long n = a.n_points;
  double sg[N];
#pragma unroll
  for (int b = 0; b < N; ++b) sg[b] = a.sg[b];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double pA[4], k[N][4];
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) pA[mu] = __ldg(a.mom + (long long)mu * n + i);
#pragma unroll
    for (int b = 0; b < N; ++b)
#pragma unroll
      for (int mu = 0; mu < 4; ++mu) k[b][mu] = __ldg(a.mom + (long long)(4 * a.part[b] + mu) * n + i);
    const double M = Body::amp(pA, k, sg);
    a.out[i] = a.g2n * M * M;
  }
}

}  // namespace qed
