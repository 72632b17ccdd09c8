// qed_eval_kernel.cuh -- lane-group |M|^2 kernel for one process size (sm_100a, FP64 CUDA cores).
//
// Instantiated once per photon count N = n+1 by the generated translation units
// csrc/generated/qed_eval_N{N}.cu, which carry the lowered node-reduction fixpoint of the
// paper's CDAG (App. C; gen/lower.py) as task tables and a traits struct T.
//
// Mapping: a group of T::G = 2^N lanes evaluates one phase-space point (a quarter, half, one or
// two warps).  Lane g owns the 4 configurations (s, s') x (lam_i = bit i of g) and accumulates
// their amplitudes in registers over all (n+1)! diagrams.  Shared memory holds the point's
// external states, propagator constants, interior trie nodes and the leaves of the current
// photon subset (layouts: gen/lower.py).  Groups of 64 lanes synchronise with a named barrier.
//
// Algorithmic work per point: gen/lower.py Plan.flops.
#pragma once
#include <utility>

#include "qed_device.cuh"
#include "qed_kernel_args.h"

namespace qed {

// ---- shared-memory spinor layouts (gen/lower.py aos_slot / swz): interior spinors have a pitch of SP
// doubles; SP = 10: components contiguous; SP = 8: component c at 16-byte slot c ^ ((off >> 4) & 3)
template <int SP>
__device__ __forceinline__ int aos_slot(int off, int c) {
  if constexpr (SP == 8) return off + 2 * (c ^ ((off >> 4) & 3));
  else return off + 2 * c;
}
__device__ __forceinline__ int swz(int h) { return (h & ~7) | ((h + (h >> 3)) & 7); }

template <int SP>
__device__ __forceinline__ spinor ld_aos(const double* base, int off) {
  spinor s;
#pragma unroll
  for (int c = 0; c < 4; ++c) s.v[c] = ld2(base + aos_slot<SP>(off, c));
  return s;
}
template <int SP>
__device__ __forceinline__ void st_aos(double* base, int off, const spinor& s) {
#pragma unroll
  for (int c = 0; c < 4; ++c) st2(base + aos_slot<SP>(off, c), s.v[c]);
}
// leaf spinor store: p = component 0 (gen/lower.py leaf_off), components NH (helicity columns) apart
template <int NH>
__device__ __forceinline__ void st_leaf(double* p, const spinor& s) {
#pragma unroll
  for (int c = 0; c < 4; ++c) st2(p + c * NH * 2, s.v[c]);
}
__device__ __forceinline__ void ld_eps(const double* p, double (&e)[3]) {
  const double2 e01 = *reinterpret_cast<const double2*>(p);
  e[0] = e01.x; e[1] = e01.y; e[2] = p[2];
}
__device__ __forceinline__ void ld_mask(const double* p, double (&m)[5]) {
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  m[0] = a.x; m[1] = a.y; m[2] = b.x; m[3] = b.y; m[4] = p[4];
}

// plans with tensor-core joins define MMA = true (gen/emit.py); every other traits struct reads false
template <class T, class = void>
struct mma_of {
  static constexpr bool value = false;
};
template <class T>
struct mma_of<T, decltype(void(T::MMA))> {
  static constexpr bool value = T::MMA;
};

// tensor-core CDAG plans with the u-bar leaves built and joined in T::TCH chunks of tau orderings (less shared
// memory per point); every other plan reads 1
template <class T, class = void>
struct tch_of {
  static constexpr int value = 1;
};
template <class T>
struct tch_of<T, decltype(void(T::TCH))> {
  static constexpr int value = T::TCH;
};

// ---- task kinds (one trie node x one helicity state); descriptor = (parent, eps, mask, out)
template <class T>
struct Tasks {
  // in-side V+S1 (interior): out = S(Q) epsslash parent
  static __device__ __forceinline__ void vs_col(double* b, ushort4 t) {
    double e[3], m[5];
    ld_eps(b + t.y, e);
    ld_mask(b + t.z, m);
    st_aos<T::SP>(b, t.w, prop_col(m, eslash_col(e, ld_aos<T::SP>(b, t.x))));
  }
  // out-side V+S1 (interior): out = (parent epsslash) S(Q)
  static __device__ __forceinline__ void vs_row(double* b, ushort4 t) {
    double e[3], m[5];
    ld_eps(b + t.y, e);
    ld_mask(b + t.z, m);
    st_aos<T::SP>(b, t.w, prop_row(m, eslash_row(e, ld_aos<T::SP>(b, t.x))));
  }
  // in-side leaf: phi = S(Q_A) epsslash parent  (V + the propagation half of S2)
  static __device__ __forceinline__ void phi(double* b, ushort4 t) {
    double e[3], m[5];
    ld_eps(b + t.y, e);
    ld_mask(b + t.z, m);
    const spinor v = prop_col(m, eslash_col(e, ld_aos<T::SP>(b, t.x)));
    if constexpr (mma_of<T>::value) st_aos<8>(b, t.w, v);   // tensor-core joins: AoS leaves (64-byte pitch, XOR swizzle)
    else st_leaf<T::NHI>(b + t.w, v);
  }
  // out-side leaf: ubar = parent epsslash
  static __device__ __forceinline__ void ub(double* b, ushort4 t) {
    double e[3];
    ld_eps(b + t.y, e);
    const spinor v = eslash_row(e, ld_aos<T::SP>(b, t.x));
    if constexpr (mma_of<T>::value) st_aos<8>(b, t.w, v);
    else st_leaf<T::NHO>(b + t.w, v);
  }
};

// ---- Berends-Giele current tasks (gen/lower_bg.py): descriptor = T::DW ushort (8 or 16)
// [mask, out, parent_1, eps_1, ..., parent_K, eps_K, pad...]; node = sum_q V(eps_q, parent_q), then S(Q)
template <int DW>
struct Desc {
  uint4 v[DW / 8];
};
template <class T>
struct BGTasks {
  using D = Desc<T::DW>;
  template <int K, bool ROW>
  static __device__ __forceinline__ spinor vsum(const double* b, const D& raw) {
    const unsigned short* d = reinterpret_cast<const unsigned short*>(&raw);
    double e[3];
    ld_eps(b + d[3], e);
    spinor acc = ROW ? eslash_row(e, ld_aos<T::SP>(b, d[2])) : eslash_col(e, ld_aos<T::SP>(b, d[2]));
#pragma unroll
    for (int q = 1; q < K; ++q) {
      ld_eps(b + d[3 + 2 * q], e);
      if (ROW) eslash_row_acc(e, ld_aos<T::SP>(b, d[2 + 2 * q]), acc);
      else eslash_col_acc(e, ld_aos<T::SP>(b, d[2 + 2 * q]), acc);
    }
    return acc;
  }
  template <int K>
  static __device__ __forceinline__ void in_node(double* b, const D& raw) {
    const unsigned short* d = reinterpret_cast<const unsigned short*>(&raw);
    double m[5];
    ld_mask(b + d[0], m);
    st_aos<T::SP>(b, d[1], prop_col(m, vsum<K, false>(b, raw)));
  }
  template <int K>
  static __device__ __forceinline__ void out_node(double* b, const D& raw) {
    const unsigned short* d = reinterpret_cast<const unsigned short*>(&raw);
    double m[5];
    ld_mask(b + d[0], m);
    st_aos<T::SP>(b, d[1], prop_row(m, vsum<K, true>(b, raw)));
  }
  // leaf descriptor field out = offset of the leaf spinor (its subset's leaf buffer, swizzled column)
  template <int K>
  static __device__ __forceinline__ void in_leaf(double* b, const D& raw) {
    const unsigned short* d = reinterpret_cast<const unsigned short*>(&raw);
    double m[5];
    ld_mask(b + d[0], m);
    const spinor v = prop_col(m, vsum<K, false>(b, raw));
    if constexpr (mma_of<T>::value) st_aos<8>(b, d[1], v);   // tensor-core joins: AoS leaves
    else st_leaf<T::NHI>(b + d[1], v);
  }
  template <int K>
  static __device__ __forceinline__ void out_leaf(double* b, const D& raw) {
    const unsigned short* d = reinterpret_cast<const unsigned short*>(&raw);
    const spinor v = vsum<K, true>(b, raw);
    if constexpr (mma_of<T>::value) st_aos<8>(b, d[1], v);
    else st_leaf<T::NHO>(b + d[1], v);
  }
};

// task functors (always inlined; passed as template arguments by the generated schedules)
template <class T, int KIND>
struct TaskFn {  // KIND: 0 vs_col, 1 vs_row, 2 phi, 3 ub
  __device__ __forceinline__ void operator()(double* b, ushort4 d) const {
    if (KIND == 0) Tasks<T>::vs_col(b, d);
    else if (KIND == 1) Tasks<T>::vs_row(b, d);
    else if (KIND == 2) Tasks<T>::phi(b, d);
    else Tasks<T>::ub(b, d);
  }
};
template <class T, int K, int KIND>
struct BGFn {  // KIND: 0 in_node, 1 out_node, 2 in_leaf, 3 out_leaf
  __device__ __forceinline__ void operator()(double* b, const Desc<T::DW>& d) const {
    if (KIND == 0) BGTasks<T>::template in_node<K>(b, d);
    else if (KIND == 1) BGTasks<T>::template out_node<K>(b, d);
    else if (KIND == 2) BGTasks<T>::template in_leaf<K>(b, d);
    else BGTasks<T>::template out_leaf<K>(b, d);
  }
};

// ---- grouped Berends-Giele tasks (profiles/r03; gen/lower_bg.py gtask): one descriptor computes the 2^F nodes
// (S, spin, lam_fixed, mu) of one photon set S, mu = the polarisations of the LAST F photons of S (helicity
// bits K-F+1..K).  Descriptor [mask, out_0, (parent_0, eps_0) per photon p of S, (leaf tasks:) h0] for node
// mu = 0.  Interior levels are stored helicity-major, so node mu's output and parents sit at fixed strides
// (doubles, gen/lower_bg.py group_strides): output SO mu; parent through a fixed photon SF mu; through a free
// photon q SR (mu without bit q) -- loaded once for both of its polarisations (eps(lam = 1) 4 doubles after
// eps(lam = 0), transverse: eps^3 = 0).  Leaf outputs: column swz(h0 + mu 2^(K-F+1)) of the rows at out_0.
template <class T, int K, int F, int KIND, int SO, int SF, int SR>
struct BGGroupFn {  // KIND: 0 in_node, 1 out_node, 2 in_leaf, 3 out_leaf
  __device__ __forceinline__ void operator()(double* b, const Desc<T::DW>& raw) const {
    if constexpr (F == 0) {
      BGFn<T, K, KIND>{}(b, raw);
    } else {
      static_assert(F <= K, "free photons are photons of the node set");
      constexpr bool ROW = KIND & 1;
      constexpr int M = 1 << F, FX = K - F;
      const unsigned short* d = reinterpret_cast<const unsigned short*>(&raw);
      spinor acc[M];
#pragma unroll
      for (int q = 0; q < F; ++q) {   // free photons first: their first vertex initialises every node
        const int p = FX + q;
        double e0[3], e1[2];
        ld_eps(b + d[3 + 2 * p], e0);
        const double2 t = *reinterpret_cast<const double2*>(b + d[3 + 2 * p] + 4);
        e1[0] = t.x;
        e1[1] = t.y;
#pragma unroll
        for (int mr = 0; mr < M / 2; ++mr) {
          const spinor P = ld_aos<T::SP>(b, d[2 + 2 * p] + mr * SR);
          const int mu0 = (mr & ((1 << q) - 1)) | ((mr >> q) << (q + 1)), mu1 = mu0 | (1 << q);
          if (q == 0) {
            acc[mu0] = ROW ? eslash_row(e0, P) : eslash_col(e0, P);
            acc[mu1] = ROW ? eslash_row_t(e1, P) : eslash_col_t(e1, P);
          } else {
            if (ROW) { eslash_row_acc(e0, P, acc[mu0]); eslash_row_t_acc(e1, P, acc[mu1]); }
            else { eslash_col_acc(e0, P, acc[mu0]); eslash_col_t_acc(e1, P, acc[mu1]); }
          }
        }
      }
#pragma unroll
      for (int p = 0; p < FX; ++p) {
        double e[3];
        ld_eps(b + d[3 + 2 * p], e);
#pragma unroll
        for (int mu = 0; mu < M; ++mu) {
          const spinor P = ld_aos<T::SP>(b, d[2 + 2 * p] + mu * SF);
          if (ROW) eslash_row_acc(e, P, acc[mu]);
          else eslash_col_acc(e, P, acc[mu]);
        }
      }
      if constexpr (KIND != 3) {
        double m[5];
        ld_mask(b + d[0], m);
#pragma unroll
        for (int mu = 0; mu < M; ++mu) acc[mu] = ROW ? prop_row(m, acc[mu]) : prop_col(m, acc[mu]);
      }
      if constexpr (KIND >= 2) {
        const int h0 = d[2 + 2 * K];
#pragma unroll
        for (int mu = 0; mu < M; ++mu) {
          const int h = h0 + (mu << (FX + 1));
          st_leaf<KIND == 2 ? T::NHI : T::NHO>(b + d[1] + 2 * swz(h), acc[mu]);
        }
      } else {
#pragma unroll
        for (int mu = 0; mu < M; ++mu) st_aos<T::SP>(b, d[1] + mu * SO, acc[mu]);
      }
    }
  }
};

// run_tasks8 split in two (BG T::SD / load_set / run_set_d): descriptors into registers ...
template <class T, int COUNT, int OFF>
__device__ __forceinline__ void load_tasks8(Desc<T::DW> (&d)[(COUNT + T::G - 1) / T::G], int g, const Desc<T::DW>* __restrict__ tbl) {
  constexpr int TRIPS = (COUNT + T::G - 1) / T::G;
  const int gl = (g + T::G - OFF) % T::G;
#pragma unroll
  for (int k = 0; k < TRIPS; ++k) {
    const int t = gl + k * T::G;
#pragma unroll
    for (int w = 0; w < T::DW / 8; ++w) {
      d[k].v[w] = make_uint4(0, 0, 0, 0);
      if (t < COUNT) d[k].v[w] = tbl[t].v[w];
    }
  }
}
// ... and the tasks
template <class T, int COUNT, class F, int OFF>
__device__ __forceinline__ void exec_tasks8(double* base, int g, const Desc<T::DW> (&d)[(COUNT + T::G - 1) / T::G], F f) {
  constexpr int TRIPS = (COUNT + T::G - 1) / T::G;
  const int gl = (g + T::G - OFF) % T::G;
#pragma unroll
  for (int k = 0; k < TRIPS; ++k)
    if (COUNT % T::G == 0 || gl + k * T::G < COUNT) f(base, d[k]);
}

// OFF: lane offset, so that two task kinds of one stage occupy different lanes / warps
template <class T, int COUNT, class F, int OFF = 0>
__device__ __forceinline__ void run_tasks8(double* base, int g, const Desc<T::DW>* __restrict__ tbl, F f) {
  constexpr int TRIPS = (COUNT + T::G - 1) / T::G;
  const int gl = (g + T::G - OFF) % T::G;
  Desc<T::DW> d[TRIPS];
#pragma unroll
  for (int k = 0; k < TRIPS; ++k) {
    const int t = gl + k * T::G;
#pragma unroll
    for (int w = 0; w < T::DW / 8; ++w) d[k].v[w] = (t < COUNT) ? tbl[t].v[w] : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < TRIPS; ++k)
    if (COUNT % T::G == 0 || gl + k * T::G < COUNT) f(base, d[k]);
}

// run COUNT tasks of one kind over the G lanes of the group (compile-time trip count, descriptors
// loaded up front so the table latency overlaps)
template <class T, int COUNT, class F, int OFF = 0>
__device__ __forceinline__ void run_tasks(double* base, int g, const ushort4* __restrict__ tbl, F f) {
  constexpr int TRIPS = (COUNT + T::G - 1) / T::G;
  const int gl = (g + T::G - OFF) % T::G;
  ushort4 d[TRIPS];
#pragma unroll
  for (int k = 0; k < TRIPS; ++k) {
    const int t = gl + k * T::G;
    d[k] = (t < COUNT) ? tbl[t] : make_ushort4(0, 0, 0, 0);
  }
#pragma unroll
  for (int k = 0; k < TRIPS; ++k)
    if (COUNT % T::G == 0 || gl + k * T::G < COUNT) f(base, d[k]);
}

// run_tasks split in two (T::SD / load_set / run_set_d): descriptors of one task list into registers ...
// (kept as raw 64-bit words: unpacking them into ushort4 right after the load would wait for it)
template <class T, int COUNT, int OFF>
__device__ __forceinline__ void load_tasks(uint2 (&d)[(COUNT + T::G - 1) / T::G], int g, const ushort4* __restrict__ tbl) {
  constexpr int TRIPS = (COUNT + T::G - 1) / T::G;
  const int gl = (g + T::G - OFF) % T::G;
  const uint2* __restrict__ raw = reinterpret_cast<const uint2*>(tbl);
#pragma unroll
  for (int k = 0; k < TRIPS; ++k) {
    const int t = gl + k * T::G;
    d[k] = make_uint2(0u, 0u);
    if (t < COUNT) d[k] = raw[t];
  }
}
// ... and the tasks themselves
template <class T, int COUNT, class F, int OFF>
__device__ __forceinline__ void exec_tasks(double* base, int g, const uint2 (&d)[(COUNT + T::G - 1) / T::G], F f) {
  constexpr int TRIPS = (COUNT + T::G - 1) / T::G;
  const int gl = (g + T::G - OFF) % T::G;
#pragma unroll
  for (int k = 0; k < TRIPS; ++k)
    if (COUNT % T::G == 0 || gl + k * T::G < COUNT)
      f(base, make_ushort4(d[k].x & 0xffffu, d[k].x >> 16, d[k].y & 0xffffu, d[k].y >> 16));
}

template <class T>
__device__ __forceinline__ void group_sync(int pb) {
  if constexpr (T::G <= 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + pb), "r"(T::G) : "memory");
  }
}

template <class T>
__device__ __forceinline__ void stage_externals(double* base, int g, const QedEvalArgs& a) {
  constexpr int N = T::N;
  constexpr int NM = (1 << N) - 2;
  // propagator constants of S(Q_S) for every proper photon subset S = m (uniform loop, no divergence):
  // Q_S = p + sum_{i in S} q_i, q = +k (in) / -k (out)
  for (int t = g; t < NM; t += T::G) {
    const int m = t + 1;
    double Q0 = base[T::MOM + 0], Q1 = base[T::MOM + 1], Q2 = base[T::MOM + 2], Q3 = base[T::MOM + 3];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      const double* k = base + T::MOM + 4 * ((a.photon_particle >> (4 * i)) & 15);
      const double w = ((m >> i) & 1) ? (i < a.n_in_ph ? 1.0 : -1.0) : 0.0;
      Q0 = fma(w, k[0], Q0); Q1 = fma(w, k[1], Q1); Q2 = fma(w, k[2], Q2); Q3 = fma(w, k[3], Q3);
    }
    const double D = Q0 * Q0 - Q1 * Q1 - Q2 * Q2 - Q3 * Q3 - 1.0;
    const double inv = 1.0 / D;
    double* mk = base + T::MASK + 6 * m;
    reinterpret_cast<double2*>(mk)[0] = make_double2((Q0 + 1.0) * inv, (1.0 - Q0) * inv);
    reinterpret_cast<double2*>(mk)[1] = make_double2(Q1 * inv, Q2 * inv);
    reinterpret_cast<double2*>(mk)[2] = make_double2(Q3 * inv, 0.0);
  }
  // polarisation vectors
  for (int t = g; t < N; t += T::G)
    external_eps(base + T::MOM + 4 * ((a.photon_particle >> (4 * t)) & 15), base + T::EPS + 8 * t);
  // electron spinors: lane 0 u(p, s), lane 1 ubar(p', s')
  if (g < 2) {
    const double* p = base + T::MOM + (g == 0 ? 0 : 4 * a.e_out_particle);
    const double r = rsqrt(p[0] + 1.0), nn = (p[0] + 1.0) * r, sg = g == 0 ? 1.0 : -1.0;
    // u(p, s) = (n chi_s, sigma.p chi_s / n);  ubar(p', s') = u^dagger gamma^0 (conjugated lower half negated)
    spinor u0, u1;
    u0.v[0] = {nn, 0}; u0.v[1] = {0, 0}; u0.v[2] = {sg * p[3] * r, 0}; u0.v[3] = {sg * p[1] * r, p[2] * r};
    u1.v[0] = {0, 0}; u1.v[1] = {nn, 0}; u1.v[2] = {sg * p[1] * r, -p[2] * r}; u1.v[3] = {-sg * p[3] * r, 0};
    st_aos<T::SP>(base, g == 0 ? T::U : T::UB, u0);
    st_aos<T::SP>(base, (g == 0 ? T::U : T::UB) + T::SP, u1);
  }
}

// Joins of one photon subset A (S2 contraction + Sum), tile (s, s') per lane:
// acc[c & 1][s | s' << 1] += sum_{sigma, tau} ubar_tau[ho + s'] . phi_sigma[hi + s]
// phi of one sigma stays in registers across the tau loop; loops are rolled so that ptxas
// cannot hoist every leaf load of the subset (which spills).
// hh: packed (2 swz(hi), 2 swz(hi + 1), 2 swz(ho), 2 swz(ho + 1)) of this lane and subset (gen tables)
// SB > 1: SB sigma rows of phi stay in registers across the tau loop (1/SB of the ubar reloads)
template <class T, int AS, int SB>
__device__ __forceinline__ void join_set_sb(const double* __restrict__ base, int h0, int h1, int o0, int o1,
                                            double (&acc)[AS][8]) {
  static_assert(T::NSIG % SB == 0, "sigma blocking must divide NSIG");
#pragma unroll 1
  for (int sg = 0; sg < T::NSIG; sg += SB) {
    c2 p0[SB][4], p1[SB][4];
#pragma unroll
    for (int b = 0; b < SB; ++b) {
      const double* prow = base + T::PHI + (sg + b) * 4 * T::NHI * 2;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        p0[b][c] = ld2(prow + c * T::NHI * 2 + h0);
        p1[b][c] = ld2(prow + c * T::NHI * 2 + h1);
      }
    }
#pragma unroll 1
    for (int tu = 0; tu < T::NTAU; ++tu) {
      const double* urow = base + T::UBL + tu * 4 * T::NHO * 2;
      c2 u0[4], u1[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        u0[c] = ld2(urow + c * T::NHO * 2 + o0);
        u1[c] = ld2(urow + c * T::NHO * 2 + o1);
      }
#pragma unroll
      for (int b = 0; b < SB; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          double* A = acc[(c + b * (AS > 2 ? 2 : 1)) % AS];
          A[0] = fma(u0[c].r, p0[b][c].r, fma(-u0[c].i, p0[b][c].i, A[0]));
          A[1] = fma(u0[c].r, p0[b][c].i, fma(u0[c].i, p0[b][c].r, A[1]));
          A[2] = fma(u0[c].r, p1[b][c].r, fma(-u0[c].i, p1[b][c].i, A[2]));
          A[3] = fma(u0[c].r, p1[b][c].i, fma(u0[c].i, p1[b][c].r, A[3]));
          A[4] = fma(u1[c].r, p0[b][c].r, fma(-u1[c].i, p0[b][c].i, A[4]));
          A[5] = fma(u1[c].r, p0[b][c].i, fma(u1[c].i, p0[b][c].r, A[5]));
          A[6] = fma(u1[c].r, p1[b][c].r, fma(-u1[c].i, p1[b][c].i, A[6]));
          A[7] = fma(u1[c].r, p1[b][c].i, fma(u1[c].i, p1[b][c].r, A[7]));
        }
    }
  }
}

template <class T, int AS, int SB = 1>
__device__ __forceinline__ void join_set(const double* __restrict__ base, unsigned hh, double (&acc)[AS][8], int lb = 0) {
  const int h0 = hh & 255, h1 = (hh >> 8) & 255, o0 = (hh >> 16) & 255, o1 = hh >> 24;
  base += lb * T::LEAFB;   // leaf buffer of the lb-th subset of a batch (T::SETB subsets per stage)
  if constexpr (SB > 1) {
    join_set_sb<T, AS, SB>(base, h0, h1, o0, o1, acc);
    return;
  }
#pragma unroll 1
  for (int sg = 0; sg < T::NSIG; ++sg) {
    c2 p0[4], p1[4];
    const double* prow = base + T::PHI + sg * 4 * T::NHI * 2;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      p0[c] = ld2(prow + c * T::NHI * 2 + h0);
      p1[c] = ld2(prow + c * T::NHI * 2 + h1);
    }
#pragma unroll(T::NTAU >= 4 ? 2 : 1)   // two tau per iteration: next tau's leaf loads overlap this tau's MACs
    for (int tu = 0; tu < T::NTAU; ++tu) {
      const double* urow = base + T::UBL + tu * 4 * T::NHO * 2;
      c2 u0[4], u1[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        u0[c] = ld2(urow + c * T::NHO * 2 + o0);
        u1[c] = ld2(urow + c * T::NHO * 2 + o1);
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double* A = acc[c % AS];
        // (s, s') = (0,0) (1,0) (0,1) (1,1)
        A[0] = fma(u0[c].r, p0[c].r, fma(-u0[c].i, p0[c].i, A[0]));
        A[1] = fma(u0[c].r, p0[c].i, fma(u0[c].i, p0[c].r, A[1]));
        A[2] = fma(u0[c].r, p1[c].r, fma(-u0[c].i, p1[c].i, A[2]));
        A[3] = fma(u0[c].r, p1[c].i, fma(u0[c].i, p1[c].r, A[3]));
        A[4] = fma(u1[c].r, p0[c].r, fma(-u1[c].i, p0[c].i, A[4]));
        A[5] = fma(u1[c].r, p0[c].i, fma(u1[c].i, p0[c].r, A[5]));
        A[6] = fma(u1[c].r, p1[c].r, fma(-u1[c].i, p1[c].i, A[6]));
        A[7] = fma(u1[c].r, p1[c].i, fma(u1[c].i, p1[c].r, A[7]));
      }
    }
  }
}

// Two-half joins (T::HS == 2, gen/lower.py hs_table; Berends-Giele plans, NSIG = NTAU = 1): lane g' of
// either half owns the 8 configurations (s, s', lam_x), x = N - 1, in acc[2 k], k = s | s' << 1 |
// lam_x << 2.  XIN (x in A): 4 phi (lam_x, s) x 2 ubar (s'); else 2 phi (s) x 4 ubar (lam_x, s').
// 6 spinor loads per 8 joins instead of 4 per 4: the join's shared-memory traffic drops by a quarter.
template <class T, bool XIN>
__device__ __forceinline__ void join_set_hs(const double* __restrict__ base, uint2 w, double (&acc)[16], int lb) {
  static_assert(T::NSIG == 1 && T::NTAU == 1, "two-half joins: one phi and one ubar row per subset");
  constexpr int NP = XIN ? 4 : 2, NU = XIN ? 2 : 4;
  base += lb * T::LEAFB;
  int po[NP], uo[NU];
#pragma unroll
  for (int i = 0; i < NP; ++i) po[i] = (w.x >> (8 * i)) & 255;
#pragma unroll
  for (int i = 0; i < NU; ++i) uo[i] = (w.y >> (8 * i)) & 255;
  const double* prow = base + T::PHI;
  const double* urow = base + T::UBL;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    c2 p[NP], u[NU];
#pragma unroll
    for (int i = 0; i < NP; ++i) p[i] = ld2(prow + c * T::NHI * 2 + po[i]);
#pragma unroll
    for (int i = 0; i < NU; ++i) u[i] = ld2(urow + c * T::NHO * 2 + uo[i]);
#pragma unroll
    for (int ip = 0; ip < NP; ++ip)
#pragma unroll
      for (int iu = 0; iu < NU; ++iu) {
        const int k = XIN ? ((ip & 1) | (iu << 1) | ((ip >> 1) << 2)) : (ip | ((iu & 1) << 1) | ((iu >> 1) << 2));
        acc[2 * k] = fma(u[iu].r, p[ip].r, fma(-u[iu].i, p[ip].i, acc[2 * k]));
        acc[2 * k + 1] = fma(u[iu].r, p[ip].i, fma(u[iu].i, p[ip].r, acc[2 * k + 1]));
      }
  }
}

// ---- tensor-core joins (T::MMA; gen/lower.py make_plan(mma=True)).  For one photon subset A the joins of
// all (sigma, tau) diagrams over every configuration are complex matrix products
//   C[row][col] += sum_c ubar_tau[row][c] phi_sigma[col][c],
// rows = (s', lam of the complement's photons), cols = (s, lam of A's photons), run on the FP64 tensor core
// as DMMA m8n8k4 (4 per 8 x 8 tile: C_re += U_re P_re - U_im P_im, C_im += U_re P_im + U_im P_re).  DMMA and
// DFMA share one FP64 datapath on B200 (tools/micro/dmma_peak.cu: 37.1 TF/s alone, the serial sum
// together), but a DMMA carries 512 flop per warp instruction from 2 register operands per lane, so the
// join needs 1/8 of the issue slots and half the shared-memory wavefronts of the CUDA-core join.
// Fragment layout (tools/micro/dmma_layout.cu): lane t holds A[t >> 2][t & 3], B[t & 3][t >> 2] and
// C[t >> 2][2 (t & 3) + r].  Accumulator bits: row = lane bits 2..4 (+ tile TR), col = r, lane bits 0..1
// (+ tile TC); which photon's polarisation sits on which bit depends on the subset and changes by one
// exchange of two bits between consecutive subsets (Johnson order, T::mma_swap).
struct MmaAcc {
  double re[2], im[2];
};
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
template <class T>
struct Mma {
  static constexpr int TR = T::NHO / 8 > 0 ? T::NHO / 8 : 1, TC = T::NHI / 8 > 0 ? T::NHI / 8 : 1;
  static constexpr int P = T::G < 32 ? 32 / T::G : 1;   // points per warp
};
// joins of sigma rows [sg0, sg1) of the point whose slot is pbase into acc
template <class T>
__device__ __forceinline__ void join_mma(const double* __restrict__ pbase, int lane, int sg0, int sg1,
                                         MmaAcc (&acc)[Mma<T>::TR][Mma<T>::TC]) {
  constexpr int TR = Mma<T>::TR, TC = Mma<T>::TC;
  const int ri = lane >> 2, c = lane & 3;
#pragma unroll 1
  for (int sg = sg0; sg < sg1; ++sg) {
    double bre[TC], bim[TC];
#pragma unroll
    for (int tc = 0; tc < TC; ++tc) {
      const c2 v = ld2(pbase + aos_slot<8>(T::PHI + (sg * T::NHI + tc * 8 + ri) * 8, c));
      bre[tc] = v.r;
      bim[tc] = v.i;
    }
#pragma unroll 2
    for (int tu = 0; tu < T::NTAU / tch_of<T>::value; ++tu) {   // the tau orderings of the resident chunk
#pragma unroll
      for (int tr = 0; tr < TR; ++tr) {
        const c2 u = ld2(pbase + aos_slot<8>(T::UBL + (tu * T::NHO + tr * 8 + ri) * 8, c));
        const double nui = -u.i;
#pragma unroll
        for (int tc = 0; tc < TC; ++tc) {
          dmma(acc[tr][tc].re[0], acc[tr][tc].re[1], u.r, bre[tc]);
          dmma(acc[tr][tc].im[0], acc[tr][tc].im[1], u.r, bim[tc]);
          dmma(acc[tr][tc].re[0], acc[tr][tc].re[1], nui, bim[tc]);
          dmma(acc[tr][tc].im[0], acc[tr][tc].im[1], u.i, bre[tc]);
        }
      }
    }
  }
}
// exchanges of two accumulator bits (T::mma_swap, generated): lane bit A <-> lane bit B
template <int A, int B, int TR, int TC>
__device__ __forceinline__ void mma_swap_ll(MmaAcc (&acc)[TR][TC], int lane) {
  const int src = (lane & ~((1 << A) | (1 << B))) | (((lane >> A) & 1) << B) | (((lane >> B) & 1) << A);
#pragma unroll
  for (int tr = 0; tr < TR; ++tr)
#pragma unroll
    for (int tc = 0; tc < TC; ++tc)
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        acc[tr][tc].re[r] = __shfl_sync(0xffffffffu, acc[tr][tc].re[r], src);
        acc[tr][tc].im[r] = __shfl_sync(0xffffffffu, acc[tr][tc].im[r], src);
      }
}
// lane bit A <-> tile index bit (ROW: the row tile TR, else the column tile TC).  Element (lane L, tile t) takes
// the element of tile bit(L, A) from the lane whose bit A is t: a lane keeps tile bit(L, A) and swaps the other
// tile with its partner L ^ (1 << A) -- one shuffle per pair of tiles
template <int A, bool ROW, int TR, int TC>
__device__ __forceinline__ void mma_swap_lt(MmaAcc (&acc)[TR][TC], int lane) {
  const bool la = (lane >> A) & 1;
#pragma unroll
  for (int o = 0; o < (ROW ? TC : TR); ++o) {
    MmaAcc& t0 = ROW ? acc[0][o] : acc[o][0];
    MmaAcc& t1 = ROW ? acc[TR - 1][o] : acc[o][TC - 1];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const double sre = la ? t0.re[r] : t1.re[r], sim = la ? t0.im[r] : t1.im[r];   // the tile the partner needs
      const double zre = __shfl_xor_sync(0xffffffffu, sre, 1 << A), zim = __shfl_xor_sync(0xffffffffu, sim, 1 << A);
      if (la) { t0.re[r] = zre; t0.im[r] = zim; }
      else { t1.re[r] = zre; t1.im[r] = zim; }
    }
  }
}
// column tile <-> row tile
template <int TR, int TC>
__device__ __forceinline__ void mma_swap_tt(MmaAcc (&acc)[TR][TC]) {
  static_assert(TR == 2 && TC == 2, "tile exchange needs both tile bits");
  const MmaAcc t = acc[0][1];
  acc[0][1] = acc[1][0];
  acc[1][0] = t;
}

// Stages 1-3 for the point whose momenta are in base[T::MOM..].  On return lane g holds the
// amplitudes (without e^N) of its configurations in amp[s | s' << 1] (re, im).
// launch-variant field DP (descriptor prefetch; plans that emit T::SD); variants without the field read 0
template <class V, class = void>
struct dp_of {
  static constexpr int value = 0;
};
template <class V>
struct dp_of<V, decltype(void(V::DP))> {
  static constexpr int value = V::DP;
};

// launch-variant field UR (tensor-core plans): the subset loop fully unrolled, so every accumulator exchange
// is straight-line code (no switch on the subset index); variants without the field read 0
template <class V, class = void>
struct ur_of {
  static constexpr int value = 0;
};
template <class V>
struct ur_of<V, decltype(void(V::UR))> {
  static constexpr int value = V::UR;
};

struct NoSD {};
template <class T, bool HAS>
struct sd_of {
  using type = NoSD;
};
template <class T>
struct sd_of<T, true> {
  using type = typename T::SD;
};

// DP: leaf-stage descriptors loaded one subset (batch) ahead (T::SD / load_set / run_set_d)
template <class T, int AS = 2, int SB = 1, int DP = 0>
__device__ __forceinline__ void eval_point(double* base, int g, int pb, const QedEvalArgs& a, double (&amp)[2 * T::NAMP]) {
  static_assert(!mma_of<T>::value, "tensor-core-join plans run mma_eval");
  stage_externals<T>(base, g, a);
  group_sync<T>(pb);
  T::run_interiors(base, g, pb);
  if constexpr (T::HS == 2) {
    // half q joins subsets s0 + q, s0 + q + 2, ... of every batch; the halves' partial amplitudes are
    // summed into half 0 at the end through shared memory (the dead U.. region of the point's slot)
    constexpr int GH = T::G / 2;
    const int q = g / GH, gh = g % GH;
    double acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0.0;
    typename sd_of<T, DP != 0>::type sd;
    if constexpr (DP) T::load_set(sd, g, 0);
#pragma unroll 1
    for (int s0 = 0; s0 < T::NSETS; s0 += T::SETB) {
      uint2 ww[T::SETB / 2];   // join offsets: loaded before the leaf stage so their latency overlaps it
#pragma unroll
      for (int lb = 0; lb < T::SETB; lb += 2) ww[lb / 2] = T::hs_offsets(s0 + lb + q, gh);
      if constexpr (DP) {
        T::run_set_d(base, g, pb, sd);
        group_sync<T>(pb);
        if (s0 + T::SETB < T::NSETS) T::load_set(sd, g, s0 + T::SETB);
      } else {
        T::run_set(base, g, pb, s0);
        group_sync<T>(pb);
      }
#pragma unroll
      for (int lb = 0; lb < T::SETB; lb += 2) {
        const int si = s0 + lb + q;
        if (T::NSETS_REAL % T::SETB == 0 || si < T::NSETS_REAL) {
          const uint2 w = ww[lb / 2];
          if ((T::set_mask(si) >> (T::N - 1)) & 1) join_set_hs<T, true>(base, w, acc, lb + q);
          else join_set_hs<T, false>(base, w, acc, lb + q);
        }
      }
      group_sync<T>(pb);
    }
    double* red = base + T::U;
    if (q == 1) {
#pragma unroll
      for (int i = 0; i < 16; ++i) red[i * GH + gh] = acc[i];
    }
    group_sync<T>(pb);
#pragma unroll
    for (int i = 0; i < 16; ++i) amp[i] = q == 0 ? acc[i] + red[i * GH + gh] : 0.0;
    return;
  } else {
  double acc[AS][8];   // AS independent partial sums per amplitude (ILP across the c loop)
#pragma unroll
  for (int q = 0; q < AS; ++q)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[q][i] = 0.0;
  if constexpr (DP) {
    // leaf-stage descriptors one batch ahead: batch s0 + SETB's are loaded before batch s0's joins
    typename T::SD sd;
    T::load_set(sd, g, 0);
#pragma unroll 1
    for (int s0 = 0; s0 < T::NSETS; s0 += T::SETB) {
      unsigned hh[T::SETB];
#pragma unroll
      for (int lb = 0; lb < T::SETB; ++lb) hh[lb] = T::hiho(s0 + lb, g);
      T::run_set_d(base, g, pb, sd);
      group_sync<T>(pb);
      if (s0 + T::SETB < T::NSETS) T::load_set(sd, g, s0 + T::SETB);
#pragma unroll
      for (int lb = 0; lb < T::SETB; ++lb)
        if (T::NSETS_REAL % T::SETB == 0 || s0 + lb < T::NSETS_REAL) join_set<T, AS, SB>(base, hh[lb], acc, lb);
      group_sync<T>(pb);
    }
  } else {
#pragma unroll 1
  for (int s0 = 0; s0 < T::NSETS; s0 += T::SETB) {
    unsigned hh[T::SETB];   // join offsets: loaded before the leaf stage so their latency overlaps it
#pragma unroll
    for (int lb = 0; lb < T::SETB; ++lb) hh[lb] = T::hiho(s0 + lb, g);
    T::run_set(base, g, pb, s0);      // leaves of subsets s0 .. s0 + SETB - 1
    group_sync<T>(pb);
#pragma unroll
    for (int lb = 0; lb < T::SETB; ++lb)   // padding subsets of a ragged last batch: leaves only, no join
      if (T::NSETS_REAL % T::SETB == 0 || s0 + lb < T::NSETS_REAL) join_set<T, AS, SB>(base, hh[lb], acc, lb);
    group_sync<T>(pb);
  }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double s = acc[0][i];
#pragma unroll
    for (int q = 1; q < AS; ++q) s += acc[q][i];
    amp[i] = s;
  }
  }
}

// internal configuration of amplitude k of lane g: s | lam << 1 | s' << (N+1); with two-half joins
// lane g' = g mod G/2 holds lam_0..lam_{N-2} and k = s | s' << 1 | lam_{N-1} << 2 (half 0 only)
template <class T>
__device__ __forceinline__ unsigned config_of(int k, int g) {
  if constexpr (T::HS == 2) {
    const unsigned gh = g % (T::G / 2);
    return (k & 1) | (gh << 1) | ((unsigned)((k >> 2) & 1) << T::N) | ((unsigned)((k >> 1) & 1) << (T::N + 1));
  }
  return (k & 1) | ((unsigned)g << 1) | ((unsigned)(k >> 1) << (T::N + 1));
}
template <class T>
__device__ __forceinline__ bool holds_amps(int g) { return T::HS == 1 || g < T::G / 2; }

// sum over the group's configurations allowed by the spec of |amp|^2, times norm (valid in every
// lane of groups of <= 32 lanes, and in every lane of 64-lane groups after the barrier exchange)
template <class T>
__device__ __forceinline__ double group_msq(const double (&amp)[2 * T::NAMP], int g, int pb, double* base, const QedEvalArgs& a) {
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < T::NAMP; ++k) {
    const double t = fma(amp[2 * k], amp[2 * k], amp[2 * k + 1] * amp[2 * k + 1]);
    sum += ((config_of<T>(k, g) & a.fixed_mask) == a.fixed_val) ? t : 0.0;
  }
  constexpr int W = T::G < 32 ? T::G : 32;
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if constexpr (T::G > 32) {
    if ((g & 31) == 0) base[T::RED + (g >> 5)] = sum;
    group_sync<T>(pb);
    sum = 0.0;
#pragma unroll
    for (int w = 0; w < T::G / 32; ++w) sum += base[T::RED + w];
  }
  return a.norm * sum;
}

// joins of subset si (leaf buffer lb) for the warp's points, chunk by chunk of tau orderings (T::TCH; chunks
// after the first are built here, between two group barriers), then the subset's accumulator bit exchange
template <class T, int P>
__device__ __forceinline__ void mma_subset_joins(double* smem, double* base, int g, int pb, int w, int lane, int half,
                                                 int sg0, int sg1, int si, int lb,
                                                 MmaAcc (&acc)[P][Mma<T>::TR][Mma<T>::TC]) {
  constexpr bool SPLIT_SET = T::G > 32 && T::NSIG == 1;
#pragma unroll
  for (int ch = 0; ch < tch_of<T>::value; ++ch) {
    if constexpr (tch_of<T>::value > 1) {
      if (ch > 0) {
        group_sync<T>(pb);                 // the previous chunk's u-bar leaves are joined
        T::run_leaf_chunk(base, g, pb, si, ch);
        group_sync<T>(pb);
      }
    }
#pragma unroll
    for (int p = 0; p < P; ++p) {
      const double* pbase = (T::G > 32 ? base : smem + (w * P + p) * T::STRIDE) + lb * T::LEAFB;
      if (!SPLIT_SET || (si & 1) == half) join_mma<T>(pbase, lane, sg0, sg1, acc[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < P; ++p)
    if (si + 1 < T::NSETS_REAL) T::mma_swap(acc[p], lane, si);
}

// the subset loop of mma_eval unrolled (launch field UR): batch B is a compile-time constant, so
// T::mma_swap(acc, lane, si) folds to the one exchange of that subset
template <class T, int DP, int P, int B, class SD>
__device__ __forceinline__ void mma_batch(double* smem, double* base, int g, int pb, int w, int lane, int half, int sg0, int sg1,
                                          SD& sd, MmaAcc (&acc)[P][Mma<T>::TR][Mma<T>::TC]) {
  constexpr int s0 = B * T::SETB;
  if constexpr (DP) {
    T::run_set_d(base, g, pb, sd);
    group_sync<T>(pb);
    if constexpr (s0 + T::SETB < T::NSETS) T::load_set(sd, g, s0 + T::SETB);
  } else {
    T::run_set(base, g, pb, s0);
    group_sync<T>(pb);
  }
#pragma unroll
  for (int lb = 0; lb < T::SETB; ++lb) {
    const int si = s0 + lb;
    if (si < T::NSETS_REAL)
      mma_subset_joins<T, P>(smem, base, g, pb, w, lane, half, sg0, sg1, si, lb, acc);
  }
  group_sync<T>(pb);
}
template <class T, int DP, int P, class SD, int... Bs>
__device__ __forceinline__ void mma_subsets(double* smem, double* base, int g, int pb, int w, int lane, int half, int sg0,
                                            int sg1, SD& sd, MmaAcc (&acc)[P][Mma<T>::TR][Mma<T>::TC],
                                            std::integer_sequence<int, Bs...>) {
  (mma_batch<T, DP, P, Bs>(smem, base, g, pb, w, lane, half, sg0, sg1, sd, acc), ...);
}

// Stages 1-4 of a tensor-core-join plan for the points of this warp (after stage 0).  Groups of G <= 32 lanes
// run their own point's tasks; the joins are warp-wide, one point after the other (P per warp).  A 64-lane
// group splits the sigma rows between its two warps and sums the halves through shared memory.
// MODE 0: the averaged |M|^2 to a.out; 1: per configuration to a.out; 2: no store, returns the group's
// averaged |M|^2 (every lane; the fused MC kernel)
template <class T, class V, int MODE>
__device__ __forceinline__ double mma_eval(double* smem, double* base, int g, int pb, const QedEvalArgs& a, long long p0) {
  constexpr bool PER_CONFIG = MODE == 1;
  static_assert(tch_of<T>::value == 1 || dp_of<V>::value == 0, "descriptor prefetch covers whole subsets only");
  constexpr int TR = Mma<T>::TR, TC = Mma<T>::TC, P = Mma<T>::P;
  constexpr int DP = dp_of<V>::value;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  stage_externals<T>(base, g, a);
  group_sync<T>(pb);
  T::run_interiors(base, g, pb);
  MmaAcc acc[P][TR][TC];
#pragma unroll
  for (int p = 0; p < P; ++p)
#pragma unroll
    for (int tr = 0; tr < TR; ++tr)
#pragma unroll
      for (int tc = 0; tc < TC; ++tc) acc[p][tr][tc] = MmaAcc{{0.0, 0.0}, {0.0, 0.0}};
  // a 64-lane group: its two warps take half of the sigma rows (CDAG) or every other subset (Berends-Giele,
  // one sigma row); both apply every accumulator exchange
  const int half = T::G > 32 ? (threadIdx.x >> 5) & 1 : 0;
  constexpr bool SPLIT_SIG = T::G > 32 && T::NSIG > 1;
  const int sg0 = SPLIT_SIG ? half * (T::NSIG / 2) : 0, sg1 = SPLIT_SIG ? sg0 + T::NSIG / 2 + (half ? T::NSIG % 2 : 0) : T::NSIG;
  typename sd_of<T, DP != 0>::type sd;
  if constexpr (DP) T::load_set(sd, g, 0);
  if constexpr (ur_of<V>::value) {
    mma_subsets<T, DP, P>(smem, base, g, pb, w, lane, half, sg0, sg1, sd, acc, std::make_integer_sequence<int, T::NSETS / T::SETB>{});
  } else {
#pragma unroll 1
  for (int s0 = 0; s0 < T::NSETS; s0 += T::SETB) {   // leaf stage of SETB subsets (CDAG: one)
    if constexpr (DP) {
      T::run_set_d(base, g, pb, sd);
      group_sync<T>(pb);
      if (s0 + T::SETB < T::NSETS) T::load_set(sd, g, s0 + T::SETB);
    } else {
      T::run_set(base, g, pb, s0);
      group_sync<T>(pb);
    }
#pragma unroll
    for (int lb = 0; lb < T::SETB; ++lb) {
      const int si = s0 + lb;
      if (T::NSETS_REAL % T::SETB == 0 || si < T::NSETS_REAL)   // padding subsets: leaves only
        mma_subset_joins<T, P>(smem, base, g, pb, w, lane, half, sg0, sg1, si, lb, acc);
    }
    group_sync<T>(pb);
  }
  }
  if constexpr (T::G > 32) {   // second warp's partial tiles -> the (dead) leaf rows of the point, summed by the first
    double* red = base + T::PHI;
    if (half == 1) {
#pragma unroll
      for (int tr = 0; tr < TR; ++tr)
#pragma unroll
        for (int tc = 0; tc < TC; ++tc)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            red[((tr * TC + tc) * 4 + r) * 32 + lane] = acc[0][tr][tc].re[r];
            red[((tr * TC + tc) * 4 + 2 + r) * 32 + lane] = acc[0][tr][tc].im[r];
          }
    }
    group_sync<T>(pb);
    if (half == 0) {
#pragma unroll
      for (int tr = 0; tr < TR; ++tr)
#pragma unroll
        for (int tc = 0; tc < TC; ++tc)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            acc[0][tr][tc].re[r] += red[((tr * TC + tc) * 4 + r) * 32 + lane];
            acc[0][tr][tc].im[r] += red[((tr * TC + tc) * 4 + 2 + r) * 32 + lane];
          }
    }
  }
  // stage 4: |amp|^2 per configuration (config of each accumulator element: T::mma_config)
  const long long n = a.n_points;
  double mine = 0.0;
#pragma unroll
  for (int p = 0; p < P; ++p) {
    const long long ptp = T::G > 32 ? p0 + pb : p0 + w * P + p;
    if (PER_CONFIG) {
      if (ptp < n && half == 0) {
#pragma unroll
        for (int tr = 0; tr < TR; ++tr)
#pragma unroll
          for (int tc = 0; tc < TC; ++tc)
#pragma unroll
            for (int r = 0; r < 2; ++r) {
              const unsigned h = T::mma_config(lane, r, tr, tc);
              unsigned hx = 0;
#pragma unroll
              for (int b = 0; b < T::N + 2; ++b) hx |= ((h >> b) & 1u) << ((a.ext_bit >> (4 * b)) & 15);
              const double re = acc[p][tr][tc].re[r], im = acc[p][tr][tc].im[r];
              a.out[ptp * (1LL << (T::N + 2)) + hx] = a.coupling * fma(re, re, im * im);
            }
      }
    } else {
      double sum = 0.0;
#pragma unroll
      for (int tr = 0; tr < TR; ++tr)
#pragma unroll
        for (int tc = 0; tc < TC; ++tc)
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const unsigned h = T::mma_config(lane, r, tr, tc);
            const double re = acc[p][tr][tc].re[r], im = acc[p][tr][tc].im[r];
            sum += ((h & a.fixed_mask) == a.fixed_val) ? fma(re, re, im * im) : 0.0;
          }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      if (MODE == 2) {
        if (T::G > 32 || p == (pb % P)) mine = a.norm * sum;
      } else if (ptp < n && half == 0 && (T::G > 32 ? lane == 0 : lane == p * T::G)) {
        a.out[ptp] = a.norm * sum;
      }
    }
  }
  if constexpr (MODE == 2 && T::G > 32) {   // the second warp's sum is partial (its acc was added into the first's)
    group_sync<T>(pb);
    if (half == 0 && lane == 0) base[T::RED] = mine;
    group_sync<T>(pb);
    mine = base[T::RED];
  }
  return mine;
}

// V: launch variant (WPB warps per block, MIN_BLOCKS resident blocks, AS accumulator split, PF prefetch)
template <class T, class V, bool PER_CONFIG>
__global__ void __launch_bounds__(V::WPB * 32, V::MIN_BLOCKS) qed_eval_kernel(QedEvalArgs a) {
  extern __shared__ __align__(16) double smem[];
  constexpr int G = T::G;
  constexpr int PB = V::WPB * 32 / G;   // points per block
  const int g = threadIdx.x % G;
  const int pb = threadIdx.x / G;
  double* base = smem + pb * T::STRIDE;
  const long long n = a.n_points;
  const long long stride_pts = (long long)gridDim.x * PB;
  // PF == 2: the next point's momenta are loaded into registers (MR per lane) while this point is evaluated
  constexpr int MR = (4 * (T::N + 2) + G - 1) / G;
  double mnext[MR];
  if (V::PF == 2) {
    const long long pt = (long long)blockIdx.x * PB + pb;
    const long long ptc = pt < n ? pt : n - 1;
#pragma unroll
    for (int k = 0; k < MR; ++k) {
      const int t = g + k * G;
      mnext[k] = t < 4 * (T::N + 2) ? __ldg(a.mom + (long long)t * n + ptc) : 0.0;
    }
  }
#pragma unroll 1
  for (long long p0 = (long long)blockIdx.x * PB; p0 < n; p0 += stride_pts) {
    const long long pt = p0 + pb;
    const bool valid = pt < n;
    const long long ptc = valid ? pt : n - 1;
    // stage 0: momenta, SoA layout mom[(4 j + mu) n + i]; L2 prefetch of the next batch
    if (V::PF == 2) {
#pragma unroll
      for (int k = 0; k < MR; ++k)
        if (g + k * G < 4 * (T::N + 2)) base[T::MOM + g + k * G] = mnext[k];
      const long long nx = pt + stride_pts < n ? pt + stride_pts : n - 1;
#pragma unroll
      for (int k = 0; k < MR; ++k) {
        const int t = g + k * G;
        if (t < 4 * (T::N + 2)) mnext[k] = __ldg(a.mom + (long long)t * n + nx);
      }
    } else {
      for (int t = g; t < 4 * (T::N + 2); t += G) {
        base[T::MOM + t] = __ldg(a.mom + (long long)t * n + ptc);
        if (V::PF && pt + stride_pts < n) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.mom + (long long)t * n + pt + stride_pts));
      }
    }
    group_sync<T>(pb);
    if constexpr (mma_of<T>::value) {
      mma_eval<T, V, PER_CONFIG ? 1 : 0>(smem, base, g, pb, a, p0);
    } else {
    double amp[2 * T::NAMP];
    eval_point<T, V::AS, V::SB, dp_of<V>::value>(base, g, pb, a, amp);
    // stage 4: |amp|^2 and the spin/polarisation sum or average
    if (PER_CONFIG) {
      if (valid && holds_amps<T>(g)) {
#pragma unroll
        for (int k = 0; k < T::NAMP; ++k) {
          const unsigned h = config_of<T>(k, g);
          unsigned hx = 0;
#pragma unroll
          for (int b = 0; b < T::N + 2; ++b) hx |= ((h >> b) & 1u) << ((a.ext_bit >> (4 * b)) & 15);
          a.out[pt * (1LL << (T::N + 2)) + hx] = a.coupling * fma(amp[2 * k], amp[2 * k], amp[2 * k + 1] * amp[2 * k + 1]);
        }
      }
    } else {
      const double msq = group_msq<T>(amp, g, pb, base, a);
      if (valid && g == 0) a.out[pt] = msq;
    }
    }
    group_sync<T>(pb);   // the slot is reused by the next point
  }
}

}  // namespace qed
