// qed_kernel_args.h -- launch arguments shared by the runtime (qed_runtime.cu) and the kernels.
#pragma once
#include <stdint.h>

namespace qed {

struct QedEvalArgs {
  const double* mom;          // device, SoA: mom[(4 j + mu) * n_points + i]
  double* out;                // device: n_points doubles, or n_points * 2^(N+2) (per-configuration)
  long long n_points;
  int n_in_ph;                // photons 0..n_in_ph-1 are incoming (q = +k), the rest outgoing (q = -k)
  int e_out_particle;         // particle index of the outgoing electron
  unsigned long long photon_particle;  // 4 bits per photon i: particle index of photon i
  unsigned long long ext_bit; // 4 bits per internal configuration bit: external particle index
  unsigned fixed_mask;        // internal configuration bits fixed by the process spec
  unsigned fixed_val;
  double norm;                // e^(2N) x 1/2 per summed initial particle
  double coupling;            // e^(2N) (per-configuration output, no averaging)
};

}  // namespace qed
