// qed_device.cuh -- per-node device arithmetic of the QED CDAG kernels (sm_100a, FP64).
//
// Kernels of the paper's QED CDAG (§2.2, App. D 465-472):
//   U  base_state  : eps(k, lam), u(p, s), ubar(p', s')             -> external_*()
//   V  vertex      : epsslash psi (column) / psibar epsslash (row)   -> vs_col / v_row / vs_row
//   S1 propagator  : (Qslash + m) psi / (Q^2 - m^2)                  -> fused into vs_col / vs_row
//   S2 join        : propagate one side, contract with the other     -> leaf vs_col + join MACs
//   Sum            : sum of diagram values                           -> register accumulation
//
// Conventions: metric (+,-,-,-), m_e = 1, Dirac representation
//   gamma^0 = diag(1,1,-1,-1), gamma^i = [[0, sigma^i], [-sigma^i, 0]];
// with eps^0 = 0:  epsslash = [[0, -E], [E, 0]],  E = eps.sigma = [[e3, e1 - i e2], [e1 + i e2, -e3]];
// (Qslash + m)/D = [[Qp, -K], [K, Qm]],  Qp = (Q0+m)/D, Qm = (m-Q0)/D, K = (Q/D).sigma.
// Every real output is one DMUL + FMAs (flop model in gen/lower.py FLOPS).
//
// This file is independent of oracle/ (no shared code); its math is checked
// against the oracle by tests/test_gpu_parity.py.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qed {

struct c2 {
  double r, i;
};

__device__ __forceinline__ c2 ld2(const double* p) {
  double2 v = *reinterpret_cast<const double2*>(p);
  return {v.x, v.y};
}
__device__ __forceinline__ void st2(double* p, c2 v) {
  *reinterpret_cast<double2*>(p) = make_double2(v.r, v.i);
}

struct spinor {
  c2 v[4];
};

__device__ __forceinline__ spinor ld_spinor(const double* p) {
  spinor s;
#pragma unroll
  for (int c = 0; c < 4; ++c) s.v[c] = ld2(p + 2 * c);
  return s;
}
__device__ __forceinline__ void st_spinor(double* p, const spinor& s) {
#pragma unroll
  for (int c = 0; c < 4; ++c) st2(p + 2 * c, s.v[c]);
}

// ---- E (x, y)^T  with E = [[e3, e1 - i e2], [e1 + i e2, -e3]], optionally negated
// out0 = e3 x + (e1 - i e2) y ; out1 = (e1 + i e2) x - e3 y
__device__ __forceinline__ void emul_col(double e1, double e2, double e3, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  // re(o0) = e3 xr + e1 yr + e2 yi ; im(o0) = e3 xi + e1 yi - e2 yr
  double se1 = sgn * e1, se2 = sgn * e2, se3 = sgn * e3;
  o0.r = fma(se2, y.i, fma(se1, y.r, se3 * x.r));
  o0.i = fma(-se2, y.r, fma(se1, y.i, se3 * x.i));
  // re(o1) = e1 xr - e2 xi - e3 yr ; im(o1) = e1 xi + e2 xr - e3 yi
  o1.r = fma(-se3, y.r, fma(-se2, x.i, se1 * x.r));
  o1.i = fma(-se3, y.i, fma(se2, x.r, se1 * x.i));
}

// ---- (x, y) E  (row vector times E):  out0 = x e3 + y (e1 + i e2) ; out1 = x (e1 - i e2) - y e3
__device__ __forceinline__ void emul_row(double e1, double e2, double e3, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  double se1 = sgn * e1, se2 = sgn * e2, se3 = sgn * e3;
  // re(o0) = e3 xr + e1 yr - e2 yi ; im(o0) = e3 xi + e1 yi + e2 yr
  o0.r = fma(-se2, y.i, fma(se1, y.r, se3 * x.r));
  o0.i = fma(se2, y.r, fma(se1, y.i, se3 * x.i));
  // re(o1) = e1 xr + e2 xi - e3 yr ; im(o1) = e1 xi - e2 xr - e3 yi
  o1.r = fma(-se3, y.r, fma(se2, x.i, se1 * x.r));
  o1.i = fma(-se3, y.i, fma(-se2, x.r, se1 * x.i));
}

// epsslash psi = (-E psi_bot, E psi_top)                                       [V, 40 flop]
__device__ __forceinline__ spinor eslash_col(const double* e, const spinor& p) {
  spinor o;
  emul_col(e[0], e[1], e[2], p.v[2], p.v[3], -1.0, o.v[0], o.v[1]);
  emul_col(e[0], e[1], e[2], p.v[0], p.v[1], 1.0, o.v[2], o.v[3]);
  return o;
}
// psibar epsslash = (psibar_bot E, -psibar_top E)                              [V, 40 flop]
__device__ __forceinline__ spinor eslash_row(const double* e, const spinor& p) {
  spinor o;
  emul_row(e[0], e[1], e[2], p.v[2], p.v[3], 1.0, o.v[0], o.v[1]);
  emul_row(e[0], e[1], e[2], p.v[0], p.v[1], -1.0, o.v[2], o.v[3]);
  return o;
}

// transverse polarisation eps(k, 2) = (-sin phi, cos phi, 0): e3 = 0 is structural (SURVEY.md §8(c)
// item 4), so its vertex drops the e3 terms: 8 real outputs x 2 ops            [V_T, 24 flop]
__device__ __forceinline__ void emul_col_t(double e1, double e2, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  double se1 = sgn * e1, se2 = sgn * e2;
  o0.r = fma(se2, y.i, se1 * y.r);
  o0.i = fma(-se2, y.r, se1 * y.i);
  o1.r = fma(-se2, x.i, se1 * x.r);
  o1.i = fma(se2, x.r, se1 * x.i);
}
__device__ __forceinline__ void emul_row_t(double e1, double e2, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  double se1 = sgn * e1, se2 = sgn * e2;
  o0.r = fma(-se2, y.i, se1 * y.r);
  o0.i = fma(se2, y.r, se1 * y.i);
  o1.r = fma(se2, x.i, se1 * x.r);
  o1.i = fma(-se2, x.r, se1 * x.i);
}
__device__ __forceinline__ spinor eslash_col_t(const double* e, const spinor& p) {
  spinor o;
  emul_col_t(e[0], e[1], p.v[2], p.v[3], -1.0, o.v[0], o.v[1]);
  emul_col_t(e[0], e[1], p.v[0], p.v[1], 1.0, o.v[2], o.v[3]);
  return o;
}
__device__ __forceinline__ spinor eslash_row_t(const double* e, const spinor& p) {
  spinor o;
  emul_row_t(e[0], e[1], p.v[2], p.v[3], 1.0, o.v[0], o.v[1]);
  emul_row_t(e[0], e[1], p.v[0], p.v[1], -1.0, o.v[2], o.v[3]);
  return o;
}

// accumulating vertices (Berends-Giele currents): acc += epsslash psi / acc += psibar epsslash
// (8 real outputs x 3 FMA = 48 flop)
__device__ __forceinline__ void emul_col_acc(double e1, double e2, double e3, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  double se1 = sgn * e1, se2 = sgn * e2, se3 = sgn * e3;
  o0.r = fma(se2, y.i, fma(se1, y.r, fma(se3, x.r, o0.r)));
  o0.i = fma(-se2, y.r, fma(se1, y.i, fma(se3, x.i, o0.i)));
  o1.r = fma(-se3, y.r, fma(-se2, x.i, fma(se1, x.r, o1.r)));
  o1.i = fma(-se3, y.i, fma(se2, x.r, fma(se1, x.i, o1.i)));
}
__device__ __forceinline__ void emul_row_acc(double e1, double e2, double e3, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  double se1 = sgn * e1, se2 = sgn * e2, se3 = sgn * e3;
  o0.r = fma(-se2, y.i, fma(se1, y.r, fma(se3, x.r, o0.r)));
  o0.i = fma(se2, y.r, fma(se1, y.i, fma(se3, x.i, o0.i)));
  o1.r = fma(-se3, y.r, fma(se2, x.i, fma(se1, x.r, o1.r)));
  o1.i = fma(-se3, y.i, fma(-se2, x.r, fma(se1, x.i, o1.i)));
}
__device__ __forceinline__ void eslash_col_acc(const double* e, const spinor& p, spinor& o) {
  emul_col_acc(e[0], e[1], e[2], p.v[2], p.v[3], -1.0, o.v[0], o.v[1]);
  emul_col_acc(e[0], e[1], e[2], p.v[0], p.v[1], 1.0, o.v[2], o.v[3]);
}
__device__ __forceinline__ void eslash_row_acc(const double* e, const spinor& p, spinor& o) {
  emul_row_acc(e[0], e[1], e[2], p.v[2], p.v[3], 1.0, o.v[0], o.v[1]);
  emul_row_acc(e[0], e[1], e[2], p.v[0], p.v[1], -1.0, o.v[2], o.v[3]);
}

// transverse accumulating vertices (eps^3 = 0; grouped Berends-Giele tasks, where lam = 1 is known at
// build time): 8 real outputs x 2 FMA = 32 flop
__device__ __forceinline__ void emul_col_t_acc(double e1, double e2, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  double se1 = sgn * e1, se2 = sgn * e2;
  o0.r = fma(se2, y.i, fma(se1, y.r, o0.r));
  o0.i = fma(-se2, y.r, fma(se1, y.i, o0.i));
  o1.r = fma(-se2, x.i, fma(se1, x.r, o1.r));
  o1.i = fma(se2, x.r, fma(se1, x.i, o1.i));
}
__device__ __forceinline__ void emul_row_t_acc(double e1, double e2, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  double se1 = sgn * e1, se2 = sgn * e2;
  o0.r = fma(-se2, y.i, fma(se1, y.r, o0.r));
  o0.i = fma(se2, y.r, fma(se1, y.i, o0.i));
  o1.r = fma(se2, x.i, fma(se1, x.r, o1.r));
  o1.i = fma(-se2, x.r, fma(se1, x.i, o1.i));
}
__device__ __forceinline__ void eslash_col_t_acc(const double* e, const spinor& p, spinor& o) {
  emul_col_t_acc(e[0], e[1], p.v[2], p.v[3], -1.0, o.v[0], o.v[1]);
  emul_col_t_acc(e[0], e[1], p.v[0], p.v[1], 1.0, o.v[2], o.v[3]);
}
__device__ __forceinline__ void eslash_row_t_acc(const double* e, const spinor& p, spinor& o) {
  emul_row_t_acc(e[0], e[1], p.v[2], p.v[3], 1.0, o.v[0], o.v[1]);
  emul_row_t_acc(e[0], e[1], p.v[0], p.v[1], -1.0, o.v[2], o.v[3]);
}

// (Qslash + m)/D psi = (Qp t - K b, K t + Qm b), K = q.sigma (q = Q/D)        [S1, 56 flop]
__device__ __forceinline__ spinor prop_col(const double* mk, const spinor& p) {
  const double qp = mk[0], qm = mk[1], qx = mk[2], qy = mk[3], qz = mk[4];
  spinor o;
  c2 a = p.v[0], b = p.v[1], c = p.v[2], d = p.v[3];
  // K (c, d): k0 = qz c + (qx - i qy) d ; k1 = (qx + i qy) c - qz d ; top = Qp (a, b) - K (c, d)
  o.v[0].r = fma(qp, a.r, -fma(qy, d.i, fma(qx, d.r, qz * c.r)));
  o.v[0].i = fma(qp, a.i, -fma(-qy, d.r, fma(qx, d.i, qz * c.i)));
  o.v[1].r = fma(qp, b.r, -fma(-qz, d.r, fma(-qy, c.i, qx * c.r)));
  o.v[1].i = fma(qp, b.i, -fma(-qz, d.i, fma(qy, c.r, qx * c.i)));
  // bottom = K (a, b) + Qm (c, d)
  o.v[2].r = fma(qm, c.r, fma(qy, b.i, fma(qx, b.r, qz * a.r)));
  o.v[2].i = fma(qm, c.i, fma(-qy, b.r, fma(qx, b.i, qz * a.i)));
  o.v[3].r = fma(qm, d.r, fma(-qz, b.r, fma(-qy, a.i, qx * a.r)));
  o.v[3].i = fma(qm, d.i, fma(-qz, b.i, fma(qy, a.r, qx * a.i)));
  return o;
}

// psibar (Qslash + m)/D = (Qp t + b K, -t K + Qm b); (x, y) K = (x qz + y (qx + i qy), x (qx - i qy) - y qz)
__device__ __forceinline__ spinor prop_row(const double* mk, const spinor& p) {
  const double qp = mk[0], qm = mk[1], qx = mk[2], qy = mk[3], qz = mk[4];
  spinor o;
  c2 a = p.v[0], b = p.v[1], c = p.v[2], d = p.v[3];
  // (c, d) K : r0 = c qz + d (qx + i qy) ; r1 = c (qx - i qy) - d qz
  o.v[0].r = fma(qp, a.r, fma(-qy, d.i, fma(qx, d.r, qz * c.r)));
  o.v[0].i = fma(qp, a.i, fma(qy, d.r, fma(qx, d.i, qz * c.i)));
  o.v[1].r = fma(qp, b.r, fma(-qz, d.r, fma(qy, c.i, qx * c.r)));
  o.v[1].i = fma(qp, b.i, fma(-qz, d.i, fma(-qy, c.r, qx * c.i)));
  // -(a, b) K + Qm (c, d)
  o.v[2].r = fma(qm, c.r, -fma(-qy, b.i, fma(qx, b.r, qz * a.r)));
  o.v[2].i = fma(qm, c.i, -fma(qy, b.r, fma(qx, b.i, qz * a.i)));
  o.v[3].r = fma(qm, d.r, -fma(-qz, b.r, fma(qy, a.i, qx * a.r)));
  o.v[3].i = fma(qm, d.i, -fma(-qz, b.i, fma(-qy, a.r, qx * a.i)));
  return o;
}

// ---- external states (U): written to shared memory
// eps(k, 1) = (cos t cos f, cos t sin f, -sin t), eps(k, 2) = (-sin f, cos f, 0),
// t = atan2(k_perp, k_z), f = atan2(k_y, k_x) (f := 0 for k_perp = 0)      [SURVEY.md §8(c) item 4]
// cos t = k_z / |k|, sin t = k_perp / |k|, cos f = k_x / k_perp, sin f = k_y / k_perp, evaluated with two
// reciprocal square roots (MUFU + Newton, <= 1 ulp) instead of two sqrt and four IEEE divisions.
__device__ __forceinline__ void eps_consts(const double* k, double& ct, double& st, double& cf, double& sf) {
  const double kp2 = k[1] * k[1] + k[2] * k[2];
  const double rkn = rsqrt(fma(k[3], k[3], kp2));
  double rkp = 0.0;
  cf = 1.0;
  sf = 0.0;
  if (kp2 > 0.0) {
    rkp = rsqrt(kp2);
    cf = k[1] * rkp;
    sf = k[2] * rkp;
  }
  ct = k[3] * rkn;
  st = (kp2 * rkp) * rkn;
}
__device__ __forceinline__ void external_eps(const double* k, double* out /* [2][4] */) {
  double ct, st, cf, sf;
  eps_consts(k, ct, st, cf, sf);
  reinterpret_cast<double2*>(out)[0] = make_double2(ct * cf, ct * sf);
  reinterpret_cast<double2*>(out)[1] = make_double2(-st, 0.0);
  reinterpret_cast<double2*>(out)[2] = make_double2(-sf, cf);
  reinterpret_cast<double2*>(out)[3] = make_double2(0.0, 0.0);
}
// u(p, s) = (n chi_s, sigma.p chi_s / n), n = sqrt(E + m)      [SURVEY.md §8(c) item 3]
__device__ __forceinline__ void external_u(const double* p, double* out /* [2][8] */) {
  const double r = rsqrt(p[0] + 1.0), n = (p[0] + 1.0) * r;
  double* o = out;
  st2(o + 0, {n, 0}); st2(o + 2, {0, 0}); st2(o + 4, {p[3] * r, 0}); st2(o + 6, {p[1] * r, p[2] * r});
  o += 8;
  st2(o + 0, {0, 0}); st2(o + 2, {n, 0}); st2(o + 4, {p[1] * r, -p[2] * r}); st2(o + 6, {-p[3] * r, 0});
}
// ubar(p', s') = u(p', s')^dagger gamma^0
__device__ __forceinline__ void external_ubar(const double* p, double* out /* [2][8] */) {
  const double r = rsqrt(p[0] + 1.0), n = (p[0] + 1.0) * r;
  double* o = out;
  st2(o + 0, {n, 0}); st2(o + 2, {0, 0}); st2(o + 4, {-p[3] * r, 0}); st2(o + 6, {-p[1] * r, p[2] * r});
  o += 8;
  st2(o + 0, {0, 0}); st2(o + 2, {n, 0}); st2(o + 4, {-p[1] * r, -p[2] * r}); st2(o + 6, {p[3] * r, 0});
}

}  // namespace qed
