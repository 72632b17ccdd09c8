// qed_eval_kernel.cuh -- the batched |M|^2 kernel for one process size (sm_100a, FP64 CUDA cores).
//
// Instantiated once per photon count N = n+1 by the generated translation units
// csrc/generated/qed_eval_N{N}.cu, which include the lowered node-reduction
// fixpoint of the paper's CDAG (App. C; gen/lower.py) as task
// tables (namespace T = qedgen_N{N}).
//
// Mapping: a group of T::G lanes evaluates one phase-space point (T::PPW = 32/G
// points per warp, independent warps, no __syncthreads).  Lane g owns the 8
// helicity configurations (s, lam_0, s') x fixed (lam_1..lam_{N-1}) = bits of g, and
// accumulates their amplitudes in registers over all (n+1)! diagrams.  Shared
// memory holds one point's external states, propagator constants, interior trie
// nodes and the leaves of the current photon subset (layout in the tables).
//
// Algorithmic work per point: gen/lower.py Plan.flops.
#pragma once
#include "qed_device.cuh"
#include "qed_kernel_args.h"

namespace qed {

template <class T>
__device__ __forceinline__ void stage_externals(double* base, int g, const QedEvalArgs& a) {
  constexpr int N = T::N;
  constexpr int NT = N + 2 + (1 << N) - 2;
  for (int t = g; t < NT; t += T::G) {
    if (t < N) {
      external_eps(base + T::MOM + 4 * ((a.photon_particle >> (4 * t)) & 15), base + T::EPS + 8 * t);
    } else if (t == N) {
      external_u(base + T::MOM, base + T::U);
    } else if (t == N + 1) {
      external_ubar(base + T::MOM + 4 * a.e_out_particle, base + T::UB);
    } else {
      // propagator constants of S(Q_S), Q_S = p + sum_{i in S} q_i, q = +k (in) / -k (out)
      const int m = t - (N + 2) + 1;
      double Q0 = base[T::MOM + 0], Q1 = base[T::MOM + 1], Q2 = base[T::MOM + 2], Q3 = base[T::MOM + 3];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        if ((m >> i) & 1) {
          const double* k = base + T::MOM + 4 * ((a.photon_particle >> (4 * i)) & 15);
          if (i < a.n_in_ph) {
            Q0 += k[0]; Q1 += k[1]; Q2 += k[2]; Q3 += k[3];
          } else {
            Q0 -= k[0]; Q1 -= k[1]; Q2 -= k[2]; Q3 -= k[3];
          }
        }
      }
      const double D = Q0 * Q0 - Q1 * Q1 - Q2 * Q2 - Q3 * Q3 - 1.0;
      const double inv = 1.0 / D;
      double* mk = base + T::MASK + 6 * m;
      reinterpret_cast<double2*>(mk)[0] = make_double2((Q0 + 1.0) * inv, (1.0 - Q0) * inv);
      reinterpret_cast<double2*>(mk)[1] = make_double2(Q1 * inv, Q2 * inv);
      reinterpret_cast<double2*>(mk)[2] = make_double2(Q3 * inv, 0.0);
    }
  }
}

// Join of one photon subset A: acc[s | lam0 << 1 | s' << 2] += sum_{sigma, tau} ubar_tau . phi_sigma
// XIN: photon 0 in A -> hi tile (s, lam0) x ho tile (s'); else hi tile (s) x ho tile (s', lam0).
template <class T, bool XIN>
__device__ __forceinline__ void join_set(const double* __restrict__ base, int hi_base, int ho_base, double (&acc)[16]) {
  constexpr int KH = XIN ? 4 : 2;   // hi tile
  constexpr int KO = XIN ? 2 : 4;   // ho tile
#pragma unroll
  for (int c = 0; c < 4; ++c) {
#pragma unroll
    for (int sg = 0; sg < T::NSIG; ++sg) {
      c2 ph[KH];
#pragma unroll
      for (int k = 0; k < KH; ++k) ph[k] = ld2(base + T::PHI + ((sg * T::NHI + hi_base + k) * 4 + c) * 2);
#pragma unroll
      for (int tu = 0; tu < T::NTAU; ++tu) {
        c2 ub[KO];
#pragma unroll
        for (int m = 0; m < KO; ++m) ub[m] = ld2(base + T::UBL + ((tu * T::NHO + ho_base + m) * 4 + c) * 2);
#pragma unroll
        for (int k = 0; k < KH; ++k) {
#pragma unroll
          for (int m = 0; m < KO; ++m) {
            // config index: s | lam0 << 1 | s' << 2
            const int idx = XIN ? (k | (m << 2)) : (k | ((m >> 1) << 1) | ((m & 1) << 2));
            acc[2 * idx] = fma(ub[m].r, ph[k].r, fma(-ub[m].i, ph[k].i, acc[2 * idx]));
            acc[2 * idx + 1] = fma(ub[m].r, ph[k].i, fma(ub[m].i, ph[k].r, acc[2 * idx + 1]));
          }
        }
      }
    }
  }
}

// Stages 1-3 for the point whose momenta are in base[T::MOM..]: external states,
// propagator constants, interior trie levels, then leaves + joins per photon subset.
// On return lane g holds the amplitudes of its 8 configurations (without e^N).
template <class T>
__device__ __forceinline__ void eval_point(double* base, int g, const QedEvalArgs& a, double (&acc)[16]) {
  constexpr int G = T::G;
  stage_externals<T>(base, g, a);
  __syncwarp();
  T::run_interiors(base, g);
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = 0.0;
  for (int si = 0; si < T::NSETS; ++si) {
    for (int t = g; t < T::NPHI; t += G) task_vs_col(base, T::phi_task(si * T::NPHI + t));
    for (int t = g; t < T::NUB; t += G) task_v_row(base, T::ub_task(si * T::NUB + t));
    __syncwarp();
    int hi_base = 0, ho_base = 0;
    const unsigned inA = T::set_mask(si);
#pragma unroll
    for (int i = 1; i < T::N; ++i) {
      const int lam = (g >> (i - 1)) & 1;
      if ((inA >> i) & 1) hi_base |= lam << T::set_pos(si, i);
      else ho_base |= lam << T::set_pos(si, i);
    }
    if (inA & 1) join_set<T, true>(base, hi_base, ho_base, acc);
    else join_set<T, false>(base, hi_base, ho_base, acc);
    __syncwarp();
  }
}

// internal configuration index of accumulator idx of lane g: s | lam0 << 1 | g << 2 | s' << (N+1)
template <class T>
__device__ __forceinline__ unsigned config_of(int idx, int g) {
  return (idx & 1) | (((idx >> 1) & 1) << 1) | ((unsigned)g << 2) | (((idx >> 2) & 1) << (T::N + 1));
}

// sum over the group's configurations allowed by the spec of |amp|^2, times norm; valid in all lanes
template <class T>
__device__ __forceinline__ double group_msq(const double (&acc)[16], int g, const QedEvalArgs& a) {
  double sum = 0.0;
#pragma unroll
  for (int idx = 0; idx < 8; ++idx) {
    const unsigned h = config_of<T>(idx, g);
    if ((h & a.fixed_mask) == a.fixed_val) sum = fma(acc[2 * idx], acc[2 * idx], fma(acc[2 * idx + 1], acc[2 * idx + 1], sum));
  }
#pragma unroll
  for (int o = T::G / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  return a.norm * sum;
}

template <class T, bool PER_CONFIG>
__global__ void __launch_bounds__(T::WPB * 32) qed_eval_kernel(QedEvalArgs a) {
  extern __shared__ __align__(16) double smem[];
  constexpr int G = T::G;
  constexpr int PPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int g = lane % G;
  const int grp = lane / G;
  double* base = smem + (warp * PPW + grp) * T::STRIDE;
  const long long n = a.n_points;
  const long long warps_total = (long long)gridDim.x * T::WPB;
#pragma unroll 1
  for (long long p0 = ((long long)blockIdx.x * T::WPB + warp) * PPW; p0 < n; p0 += warps_total * PPW) {
    const long long pt = p0 + grp;
    const bool valid = pt < n;
    const long long ptc = valid ? pt : n - 1;
    // stage 0: momenta, SoA layout mom[(4 j + mu) n + i]
    for (int t = g; t < 4 * (T::N + 2); t += G) base[T::MOM + t] = __ldg(a.mom + (long long)t * n + ptc);
    __syncwarp();
    double acc[16];
    eval_point<T>(base, g, a, acc);
    // stage 4: |amp|^2 and the spin/polarisation sum or average
    if (PER_CONFIG) {
      if (valid) {
#pragma unroll
        for (int idx = 0; idx < 8; ++idx) {
          const unsigned h = config_of<T>(idx, g);
          unsigned hx = 0;
#pragma unroll
          for (int b = 0; b < T::N + 2; ++b) hx |= ((h >> b) & 1u) << ((a.ext_bit >> (4 * b)) & 15);
          a.out[pt * (1LL << (T::N + 2)) + hx] = a.coupling * fma(acc[2 * idx], acc[2 * idx], acc[2 * idx + 1] * acc[2 * idx + 1]);
        }
      }
    } else {
      const double msq = group_msq<T>(acc, g, a);
      if (valid && g == 0) a.out[pt] = msq;
    }
  }
}

}  // namespace qed
