// qed_mc_kernel.cuh -- fused Monte-Carlo kernel:
// Philox4x32-10 -> massive RAMBO (CM frame) -> |M|^2 (same eval_point as qed_eval_msq)
// -> weight x cut -> deterministic per-chunk partial sums.  The caller all-reduces the
// chunk vector across ranks (the only collective).
//
// Phase space (the paper gives none; reading R9):
// RAMBO, Kleiss-Stirling-Ellis CPC 40 (1986) 359, rambo.f conventions:
//   q_i: c = 2 r1 - 1, phi = 2 pi r2, q0 = -log(r3 r4), q = q0 (sqrt(1-c^2) cos phi, sqrt(1-c^2) sin phi, c)
//   boost + scale to (sqrt s, 0); mass rescaling sum_i sqrt(m_i^2 + xi^2 p_i0^2) = sqrt s (Newton)
//   w = (2pi)^(4-3K) (pi/2)^(K-1) s^(K-2) / ((K-1)!(K-2)!) xi^(2K-3) sqrt(s) prod(|k_i|/E_i) / sum(|k_i|^2/E_i)
// Random numbers: Philox4x32-10 (Salmon et al., SC'11), key = seed, counter =
// (index_lo, index_hi, particle, draw); uniform u = (53-bit integer + 0.5) 2^-53.
#pragma once
#include "qed_eval_kernel.cuh"
#include "qed_mc_args.h"

namespace qed {


__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const unsigned hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const unsigned hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}

__device__ __forceinline__ double u53(unsigned hi, unsigned lo) {
  const unsigned long long r = ((unsigned long long)hi << 21) | (lo >> 11);
  return ((double)r + 0.5) * 0x1.0p-53;
}

// RAMBO step 1 for particle i: the isotropic massless momentum q_i (Philox draws 4 i .. 4 i + 3) -> q[4]
__device__ __forceinline__ void rambo_massless(unsigned long long idx, int i, const QedMcArgs& m, double* q) {
  const uint2 key = make_uint2((unsigned)m.seed, (unsigned)(m.seed >> 32));
  const uint4 a = philox4x32_10(make_uint4((unsigned)idx, (unsigned)(idx >> 32), (unsigned)i, 0u), key);
  const uint4 b = philox4x32_10(make_uint4((unsigned)idx, (unsigned)(idx >> 32), (unsigned)i, 1u), key);
  const double r1 = u53(a.x, a.y), r2 = u53(a.z, a.w), r3 = u53(b.x, b.y), r4 = u53(b.z, b.w);
  const double c = 2.0 * r1 - 1.0, st = sqrt(1.0 - c * c), f = 2.0 * M_PI * r2;
  const double q0 = -log(r3 * r4);
  double sf, cf;
  sincos(f, &sf, &cf);
  q[0] = q0; q[1] = q0 * st * cf; q[2] = q0 * st * sf; q[3] = q0 * c;
}

// massless K-body volume (2pi)^(4-3K) (pi/2)^(K-1) s^(K-2) / ((K-1)! (K-2)!): one value per launch
template <int K>
__device__ double rambo_volume(double s) {
  double vol = 1.0, fk1 = 1.0, fk2 = 1.0;
#pragma unroll
  for (int i = 0; i < K - 1; ++i) vol *= 0.5 * M_PI;
#pragma unroll
  for (int i = 0; i < K - 2; ++i) vol *= s;
#pragma unroll
  for (int i = 2; i <= K - 1; ++i) fk1 *= i;
#pragma unroll
  for (int i = 2; i <= K - 2; ++i) fk2 *= i;
  vol /= fk1 * fk2;
  return vol * pow(2.0 * M_PI, 4.0 - 3.0 * K);
}

// Massive RAMBO steps 2-4 for K final particles (particle 0 = electron, m = 1; others massless) from the massless
// momenta qin[4 i + mu] (step 1, rambo_massless, one lane per particle), written into mom (particle order e-_in,
// gamma_in, e-_out, gamma_out...); returns the weight (vol = rambo_volume<K>(s)).
// The steps are spread over the lanes of a group of G lanes (lane i: particle i; lanes >= K shadow particle K - 1).
// The per-particle square roots and divisions run in parallel; every sum is gathered with shuffles and accumulated
// in particle order (as the oracle does), so all lanes hold the same xi and weight and take the same Newton exit.  mom is written by lane i (particle i) and lane 0 (beams).
template <int K, int G>
__device__ double rambo_group(const double* qin, const QedMcArgs& m, double vol, double* mom, int g) {
  constexpr int GW = G < 32 ? G : 32;                       // lanes of the group inside this warp
  const int lane = threadIdx.x & 31;
  const int base = lane & ~(GW - 1);
  const unsigned mask = GW == 32 ? 0xffffffffu : (((1u << GW) - 1u) << base);
  const int i = g < K ? g : K - 1;
  double Q[4] = {0, 0, 0, 0};
#pragma unroll
  for (int j = 0; j < K; ++j)
#pragma unroll
    for (int mu = 0; mu < 4; ++mu) Q[mu] += qin[4 * j + mu];
  double q[4];
#pragma unroll
  for (int mu = 0; mu < 4; ++mu) q[mu] = qin[4 * i + mu];
  __syncwarp(mask);   // every lane has read the stage-1 momenta before any lane overwrites them (mom aliases qin)
  const double sqs = m.sqrt_s, s = sqs * sqs;
  const double M = sqrt(Q[0] * Q[0] - Q[1] * Q[1] - Q[2] * Q[2] - Q[3] * Q[3]);
  const double b1 = -Q[1] / M, b2 = -Q[2] / M, b3 = -Q[3] / M;
  const double x = sqs / M, gam = Q[0] / M, aa = 1.0 / (1.0 + gam);
  const double bq = b1 * q[1] + b2 * q[2] + b3 * q[3];
  const double p0 = x * (gam * q[0] + bq);
  const double pv0 = x * (q[1] + b1 * q[0] + aa * bq * b1);
  const double pv1 = x * (q[2] + b2 * q[0] + aa * bq * b2);
  const double pv2 = x * (q[3] + b3 * q[0] + aa * bq * b3);
  const double mi2 = (i == 0) ? 1.0 : 0.0;
  double xi = sqrt(1.0 - 1.0 / s);
  for (int it = 0; it < 50; ++it) {
    const double e = sqrt(mi2 + xi * xi * p0 * p0);
    const double d = xi * p0 * p0 / e;
    double f = -sqs, df = 0.0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      f += __shfl_sync(mask, e, base + j);
      df += __shfl_sync(mask, d, base + j);
    }
    const double dxi = f / df;
    xi -= dxi;
    if (fabs(dxi) <= 1e-15 * xi) break;
  }
  const double kx = xi * pv0, ky = xi * pv1, kz = xi * pv2;
  const double E = sqrt(mi2 + xi * xi * p0 * p0);
  const double kk = sqrt(kx * kx + ky * ky + kz * kz);
  const double r1 = kk / E, r2 = kk * kk / E;
  double prod = 1.0, sum = 0.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    prod *= __shfl_sync(mask, r1, base + j);
    sum += __shfl_sync(mask, r2, base + j);
  }
  if (g < K) {
    double* o = mom + 8 + 4 * g;
    o[0] = E; o[1] = kx; o[2] = ky; o[3] = kz;
  }
  if (g == 0) {
    const double kin = (s - 1.0) / (2.0 * sqs);
    mom[0] = (s + 1.0) / (2.0 * sqs); mom[1] = 0.0; mom[2] = 0.0; mom[3] = -kin;
    mom[4] = kin; mom[5] = 0.0; mom[6] = 0.0; mom[7] = kin;
  }
  double xp = 1.0;
#pragma unroll
  for (int j = 0; j < 2 * K - 3; ++j) xp *= xi;
  return vol * xp * sqs * prod / sum;
}

// RAMBO staging of the fused MC kernel: the block generates RB points per round (one subgroup of SUB >= K lanes
// per point: 4, 8 or 16; at most 8 eval passes), then evaluates them PB at a time.  Per point: the momenta in the eval slot layout
// (4 (N + 2) doubles), the weight and the cut flag.  qed_runtime.cu sizes the shared memory with the same rule.

template <class T, class V>
__global__ void __launch_bounds__(V::WPB * 32, V::MIN_BLOCKS) qed_mc_kernel(QedEvalArgs a, QedMcArgs m) {
  extern __shared__ __align__(16) double smem[];
  constexpr int G = T::G;
  constexpr int PB = V::WPB * 32 / G;     // points per block and eval pass (0 if a point spans several warps)
  constexpr int PBE = PB > 0 ? PB : 1;
  constexpr int K = T::N;                 // final state: electron + n photons = N particles
  constexpr int SUB = K <= 4 ? 4 : K <= 8 ? 8 : 16;   // RAMBO subgroup: one lane per particle
  // points per RAMBO round: one per subgroup, at most 8 eval passes (bounds the staging for the 220 KB n = 8 slot)
  constexpr int RB = V::WPB * 32 / SUB < 8 * PBE ? V::WPB * 32 / SUB : 8 * PBE;
  constexpr int SD = 4 * (T::N + 2) + 2;
  static_assert(RB % PBE == 0, "a RAMBO round covers whole eval passes");
  const int g = threadIdx.x % G;
  const int pb = threadIdx.x / G;
  double* base = smem + pb * T::STRIDE;
  double* red = smem + PBE * T::STRIDE;   // [PB][3] block reduction scratch
  double* stg = red + 3 * PBE;            // [RB][SD] RAMBO staging
  const int sg = threadIdx.x / SUB, gl = threadIdx.x % SUB;
  const unsigned long long lo_all = m.first_index, hi_all = m.first_index + m.n_points;
  const unsigned long long c_begin = lo_all / m.chunk, c_end = (hi_all + m.chunk - 1) / m.chunk;
  const double vol = rambo_volume<K>(m.sqrt_s * m.sqrt_s);
  for (unsigned long long c = c_begin + blockIdx.x; c < c_end; c += gridDim.x) {
    const unsigned long long lo = max(lo_all, c * (unsigned long long)m.chunk);
    const unsigned long long hi = min(hi_all, (c + 1) * (unsigned long long)m.chunk);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;  // thread 0 only: fixed summation order over the chunk
    for (unsigned long long r0 = lo; r0 < hi; r0 += RB) {
      // RAMBO round: subgroup sg generates point r0 + sg (step 1 one lane per particle, steps 2-4 across the
      // subgroup: rambo_group; every sum in particle order, as in the oracle)
      if (sg < RB) {
        const unsigned long long idx = r0 + sg;
        double* st = stg + sg * SD;
        if (gl < K) rambo_massless(idx < hi ? idx : hi - 1, gl, m, st + 8 + 4 * gl);
        __syncwarp();
        const double w = rambo_group<K, SUB>(st + 8, m, vol, st, gl);
        __syncwarp();
        if (gl == 0) {
          bool pass = true;
          for (int i = 1; i < K; ++i) pass = pass && (st[8 + 4 * i] >= m.omega_min);
          st[SD - 2] = w;
          st[SD - 1] = pass ? 1.0 : 0.0;
        }
      }
      __syncthreads();
      for (int q0 = 0; q0 < RB; q0 += PBE) {
        const int q = q0 + (PB > 0 ? pb : 0);
        const unsigned long long idx = r0 + q;
        const bool valid = idx < hi;
        const double* st = stg + q * SD;
        for (int t = g; t < 4 * (T::N + 2); t += G) base[T::MOM + t] = st[t];
        group_sync<T>(pb);
        double msq;
        if constexpr (mma_of<T>::value) {
          msq = mma_eval<T, V, 2>(smem, base, g, pb, a, 0);
        } else {
          double amp[2 * T::NAMP];
          eval_point<T, V::AS, V::SB, dp_of<V>::value>(base, g, pb, a, amp);
          msq = group_msq<T>(amp, g, pb, base, a);
        }
        if (g == 0) {
          const bool pass = valid && st[SD - 1] != 0.0;
          const double v = pass ? st[SD - 2] * msq : 0.0;
          red[3 * pb] = v;
          red[3 * pb + 1] = v * v;
          red[3 * pb + 2] = pass ? 1.0 : 0.0;
        }
        __syncthreads();
        if (threadIdx.x == 0)
          for (int qq = 0; qq < PBE; ++qq) { s0 += red[3 * qq]; s1 += red[3 * qq + 1]; s2 += red[3 * qq + 2]; }
        __syncthreads();
      }
    }
    if (threadIdx.x == 0) {
      m.partials[3 * c] += s0;
      m.partials[3 * c + 1] += s1;
      m.partials[3 * c + 2] += s2;
    }
  }
}

}  // namespace qed
