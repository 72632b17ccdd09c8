// qed_mc_args.h -- launch arguments of the fused Monte-Carlo kernel (qed_mc_kernel.cuh).
#pragma once

namespace qed {

struct QedMcArgs {
  double sqrt_s, omega_min;
  unsigned long long seed, first_index, n_points;
  double* partials;  // device, 3 doubles per chunk of `chunk` global indices
  int chunk;
};

}  // namespace qed
