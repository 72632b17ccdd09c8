// qed_eval_regs.cuh -- register-resident |M|^2 kernel for small processes (N = 2, 3 photons).
//
// The generated body (csrc/generated/qed_regs_N{N}.cu, gen/emit_regs.py) evaluates the
// node-reduced diagram DAG (App. C) of one phase-space point for one
// outgoing-electron spin s' as straight-line code: two threads per point, amplitudes of the
// 2^(N+1) configurations (s, lam_1..lam_N) accumulated in registers, the in-side leaves phi
// exchanged between the two threads through a small shared-memory slot.  Used for n = 1, 2
// where the group kernel (qed_eval_kernel.cuh) is bound by shared-memory traffic.
#pragma once
#include "qed_device.cuh"
#include "qed_sparse.cuh"
#include "qed_kernel_args.h"

namespace qed {


// momentum element: global (read-only path) or the cp.async staging buffer in shared memory
__device__ __forceinline__ double ld_mom(const double* p) { return *p; }

// eps(k, 1), eps(k, 2) as in external_eps, into registers
__device__ __forceinline__ void eps_regs(const double* k, double (&e)[2][3]) {
  const double kperp = sqrt(k[1] * k[1] + k[2] * k[2]);
  const double kn = sqrt(kperp * kperp + k[3] * k[3]);
  const double ct = k[3] / kn, st = kperp / kn;
  double cf = 1.0, sf = 0.0;
  if (kperp > 0.0) {
    cf = k[1] / kperp;
    sf = k[2] / kperp;
  }
  e[0][0] = ct * cf; e[0][1] = ct * sf; e[0][2] = -st;
  e[1][0] = -sf; e[1][1] = cf; e[1][2] = 0.0;
}

// u(p, s) = (n chi_s, sigma.p chi_s / n), n = sqrt(E + m)
__device__ __forceinline__ spinor u_spinor(const double* p, int s) {
  const double r = rsqrt(p[0] + 1.0), n = (p[0] + 1.0) * r;
  spinor u;
  if (s == 0) {
    u.v[0] = {n, 0}; u.v[1] = {0, 0}; u.v[2] = {p[3] * r, 0}; u.v[3] = {p[1] * r, p[2] * r};
  } else {
    u.v[0] = {0, 0}; u.v[1] = {n, 0}; u.v[2] = {p[1] * r, -p[2] * r}; u.v[3] = {-p[3] * r, 0};
  }
  return u;
}

// ubar(p', s') = u(p', s')^dagger gamma^0
__device__ __forceinline__ spinor ubar_spinor(const double* p, int s) {
  const double r = rsqrt(p[0] + 1.0), n = (p[0] + 1.0) * r;
  spinor u;
  if (s == 0) {
    u.v[0] = {n, 0}; u.v[1] = {0, 0}; u.v[2] = {-p[3] * r, 0}; u.v[3] = {-p[1] * r, p[2] * r};
  } else {
    u.v[0] = {0, 0}; u.v[1] = {n, 0}; u.v[2] = {-p[1] * r, -p[2] * r}; u.v[3] = {p[3] * r, 0};
  }
  return u;
}

// propagator constants of S(Q_S) for photon subset `mask`: (Qp, Qm, qx, qy, qz, 0) -> out[6]
template <int N>
__device__ __forceinline__ void mask_store(const double* p, const double (&q)[N][4], int mask, double* out) {
  double Q0 = p[0], Q1 = p[1], Q2 = p[2], Q3 = p[3];
#pragma unroll
  for (int i = 0; i < N; ++i)
    if ((mask >> i) & 1) {
      Q0 += q[i][0]; Q1 += q[i][1]; Q2 += q[i][2]; Q3 += q[i][3];
    }
  const double D = Q0 * Q0 - Q1 * Q1 - Q2 * Q2 - Q3 * Q3 - 1.0;
  const double inv = 1.0 / D;
  reinterpret_cast<double2*>(out)[0] = make_double2((Q0 + 1.0) * inv, (1.0 - Q0) * inv);
  reinterpret_cast<double2*>(out)[1] = make_double2(Q1 * inv, Q2 * inv);
  reinterpret_cast<double2*>(out)[2] = make_double2(Q3 * inv, 0.0);
}

// propagator constants of S(Q) for the one-photon subset {i}: Q = p + sg k_i  -> out[5] in registers
__device__ __forceinline__ void mask_regs(const double* p, const double* k, double sg, double (&out)[5]) {
  const double Q0 = fma(sg, k[0], p[0]), Q1 = fma(sg, k[1], p[1]), Q2 = fma(sg, k[2], p[2]), Q3 = fma(sg, k[3], p[3]);
  const double D = Q0 * Q0 - Q1 * Q1 - Q2 * Q2 - Q3 * Q3 - 1.0;
  const double inv = 1.0 / D;
  out[0] = (Q0 + 1.0) * inv; out[1] = (1.0 - Q0) * inv; out[2] = Q1 * inv; out[3] = Q2 * inv; out[4] = Q3 * inv;
}

// Shared-memory spinor load that the compiler may not hoist, merge or cache in registers:
// the phi leaves are re-read per out-side block so that only one phi spinor is live at a time.
__device__ __forceinline__ spinor ld_spinor_stream(const double* p) {
  const unsigned addr = (unsigned)__cvta_generic_to_shared(p);
  spinor s;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(s.v[c].r), "=d"(s.v[c].i) : "r"(addr + 16 * c));
  return s;
}

// streamed loads of eps (3 doubles, 16-byte aligned) and propagator constants (5 doubles)
__device__ __forceinline__ void ld_stream_eps(const double* p, double (&e)[3]) {
  const unsigned addr = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(e[0]), "=d"(e[1]) : "r"(addr));
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(e[2]) : "r"(addr + 16));
}
// transverse eps(k, 2): only (e1, e2) are loaded (e3 = 0 is structural)
__device__ __forceinline__ void ld_stream_eps_t(const double* p, double (&e)[3]) {
  const unsigned addr = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(e[0]), "=d"(e[1]) : "r"(addr));
  e[2] = 0.0;
}
__device__ __forceinline__ void ld_stream_mask(const double* p, double (&m)[5]) {
  const unsigned addr = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(m[0]), "=d"(m[1]) : "r"(addr));
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(m[2]), "=d"(m[3]) : "r"(addr + 16));
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(m[4]) : "r"(addr + 32));
}

// a += b (Berends-Giele current sums)
__device__ __forceinline__ void add_to(spinor& a, const spinor& b) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    a.v[c].r += b.v[c].r;
    a.v[c].i += b.v[c].i;
  }
}

// acc += sum_c a[c] b[c]  (S2 join: 4 complex multiply-accumulates, 16 DFMA)
__device__ __forceinline__ void cdot_acc(const spinor& a, const spinor& b, double& re, double& im) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    re = fma(a.v[c].r, b.v[c].r, fma(-a.v[c].i, b.v[c].i, re));
    im = fma(a.v[c].r, b.v[c].i, fma(a.v[c].i, b.v[c].r, im));
  }
}

// V: launch variant (WPB warps per block, MIN_BLOCKS resident blocks, PF L2 prefetch).
// T: generated body; T::TPP threads per point (2: thread = (point, s'); 4: (point, s', lam_0)),
// T::NACC amplitudes per thread, T::config_of(idx, sub) = internal configuration index.
// cp.async staging of one warp's batch of momenta: rows 4(N+2) x PPW points, 8-byte copies
template <int ROWS, int PPW>
__device__ __forceinline__ void stage_batch(double* dst, const double* __restrict__ mom, long long n, long long p0, int lane) {
#pragma unroll
  for (int e = lane; e < ROWS * PPW; e += 32) {
    const int r = e / PPW, q = e % PPW;
    long long pt = p0 + q;
    pt = pt < n ? pt : n - 1;
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst + e);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(mom + (long long)r * n + pt) : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// 8 joins of one out-side block, DFMAs interleaved across the pairs: pairs (l0, ph[k]) -> acc[ix[k]],
// (l1, ph[k]) -> acc[ix[4 + k]]
template <int NA>
__device__ __forceinline__ void cdot8_acc(const spinor& l0, const spinor& l1, const spinor (&ph)[4], const int (&ix)[8],
                                          double (&acc)[NA]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const spinor& L = q < 4 ? l0 : l1;
      const c2 b = ph[q & 3].v[c];
      acc[2 * ix[q]] = fma(-L.v[c].i, b.i, acc[2 * ix[q]]);
      acc[2 * ix[q] + 1] = fma(L.v[c].i, b.r, acc[2 * ix[q] + 1]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const spinor& L = q < 4 ? l0 : l1;
      const c2 b = ph[q & 3].v[c];
      acc[2 * ix[q]] = fma(L.v[c].r, b.r, acc[2 * ix[q]]);
      acc[2 * ix[q] + 1] = fma(L.v[c].r, b.i, acc[2 * ix[q] + 1]);
    }
  }
}

// T::PASSES (bodies that hand their amplitudes over pass by pass); 1 when absent
template <class T, class = void>
struct passes_of {
  static constexpr int value = 1;
};
template <class T>
struct passes_of<T, decltype(void(T::PASSES))> {
  static constexpr int value = T::PASSES;
};

template <class T, class V, bool PER_CONFIG>
__global__ void __launch_bounds__(V::WPB * 32, V::MIN_BLOCKS) qed_regs_kernel(QedEvalArgs a) {
  extern __shared__ __align__(16) double smem[];
  constexpr int N = T::N;
  constexpr int TPP = T::TPP;
  constexpr int PPW = 32 / TPP;            // points per warp
  constexpr int NACC = T::NACC;
  constexpr int ROWS = 4 * (N + 2);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int sub = lane % TPP;
  double* sl = smem + (warp * PPW + lane / TPP) * T::STRIDE;
  // PF == 2: double-buffered cp.async staging of the momenta (after the point slots)
  double* stage = smem + V::WPB * PPW * T::STRIDE + warp * 2 * ROWS * PPW;
  const long long n = a.n_points;
  const long long warps_total = (long long)gridDim.x * V::WPB;
  const long long first = ((long long)blockIdx.x * V::WPB + warp) * PPW;
  if (V::PF == 2 && first < n) stage_batch<ROWS, PPW>(stage, a.mom, n, first, lane);
  int buf = 0;
#pragma unroll 1
  for (long long p0 = first; p0 < n; p0 += warps_total * PPW) {
    const long long pt = p0 + lane / TPP;
    const bool valid = pt < n;
    const long long ptc = valid ? pt : n - 1;
    const double* msrc = a.mom;
    long long mstride = n, mpt = ptc;
    if (V::PF == 2) {
      const long long nx = p0 + warps_total * PPW;
      if (nx < n) {
        stage_batch<ROWS, PPW>(stage + (buf ^ 1) * ROWS * PPW, a.mom, n, nx, lane);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      __syncwarp();
      msrc = stage + buf * ROWS * PPW;
      mstride = PPW;
      mpt = lane / TPP;
      buf ^= 1;
    } else if (V::PF == 1) {
      // L2 prefetch of this warp's next batch of momenta: every 128-byte line of every row (one per lane)
      const long long nx = p0 + warps_total * PPW;
      constexpr int SEG = (PPW * 8 + 127) / 128;   // 128-byte lines per row of the batch
#pragma unroll
      for (int e = lane; e < ROWS * SEG; e += 32) {
        const long long q = nx + (e % SEG) * 16;
        if (q < n) {
          const double* r = a.mom + (long long)(e / SEG) * n + q;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(r));
        }
      }
    }
    // amplitudes of NACC configurations -> per-configuration |M|^2 stores, or this thread's part of the sum
    double sum = 0.0;
    auto fin = [&](const double (&acc)[2 * NACC], int sub_) {
      if (PER_CONFIG) {
        if (valid) {
#pragma unroll
          for (int idx = 0; idx < NACC; ++idx) {
            const unsigned h = T::config_of(idx, sub_);
            if (h == 0xffffffffu) continue;   // duplicate holder of this amplitude (split bodies)
            unsigned hx = 0;
#pragma unroll
            for (int b = 0; b < N + 2; ++b) hx |= ((h >> b) & 1u) << ((a.ext_bit >> (4 * b)) & 15);
            a.out[pt * (1LL << (N + 2)) + hx] = a.coupling * fma(acc[2 * idx], acc[2 * idx], acc[2 * idx + 1] * acc[2 * idx + 1]);
          }
        }
      } else if (a.fixed_mask == 0) {
        // four interleaved partial sums: one chain of 2 NACC dependent DFMAs held the pass's tail
        // (3.2 % of the n = 2 stall samples, profiles/r02/lines_n2.txt)
        double part[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int idx = 0; idx < NACC; ++idx)
          part[idx & 3] = fma(acc[2 * idx], acc[2 * idx], fma(acc[2 * idx + 1], acc[2 * idx + 1], part[idx & 3]));
        if (T::config_of(0, sub_) != 0xffffffffu) sum += (part[0] + part[1]) + (part[2] + part[3]);
      } else {
#pragma unroll
        for (int idx = 0; idx < NACC; ++idx) {
          const unsigned h = T::config_of(idx, sub_);
          const double t = fma(acc[2 * idx], acc[2 * idx], acc[2 * idx + 1] * acc[2 * idx + 1]);
          sum += (h != 0xffffffffu && (h & a.fixed_mask) == a.fixed_val) ? t : 0.0;
        }
      }
    };
    if constexpr (passes_of<T>::value > 1) {
      T::body_passes(msrc, mstride, mpt, sl, a, fin);   // calls fin once per pass
    } else {
      double acc[2 * NACC];
#pragma unroll
      for (int i = 0; i < 2 * NACC; ++i) acc[i] = 0.0;
      T::body(msrc, mstride, mpt, sub, sl, a, acc);
      fin(acc, sub);
    }
    if (!PER_CONFIG) {
#pragma unroll
      for (int o = 1; o < TPP; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (valid && sub == 0) a.out[pt] = a.norm * sum;
    }
    __syncwarp();  // the slot is reused by the next point
  }
}

}  // namespace qed
