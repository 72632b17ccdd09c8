// qed_sparse.cuh -- vertex and propagator kernels on spinors with structural zeros (register kernels, n <= 2).
//
// The external spinors have four structural zeros each (Dirac representation):
//   u(p, 0) = (n, 0, pz/n, (px + i py)/n),  u(p, 1) = (0, n, (px - i py)/n, -pz/n),  n = sqrt(E + m),
// and ubar(p', s') = u^dagger gamma^0 has the same pattern.  nvcc may not drop a product with a literal 0.0
// operand (IEEE: 0 x NaN = NaN), so the generic vertex V (qed_device.cuh eslash_*) and propagator S (prop_*)
// spend pipe slots on them.  The templates below take the zero pattern Z as a compile-time mask
// (bit 2c + j: component c, j = 0 real / 1 imaginary) and issue only the non-zero products, in the SAME
// association order as the generic functions: for finite inputs the results are bitwise those of
// qed_device.cuh (a skipped product is an exact +-0 addend).  Each output with k non-zero products costs
// 2k - 1 flops (one DMUL + k - 1 DFMA); gen/emit_regs.py sparse_* mirrors these counts for the flop model.
//
// Independent of oracle/ (no shared code); checked against the oracle by tests/test_gpu_parity.py.
#pragma once
#include <utility>

#include "qed_device.cuh"

namespace qed {

__host__ __device__ constexpr bool zb(unsigned Z, int k) { return (Z >> k) & 1u; }

// structural zero patterns of the external spinors (qed_eval_regs.cuh u_spinor / ubar_spinor)
constexpr unsigned ZU0 = (1u << 1) | (1u << 2) | (1u << 3) | (1u << 5);   // v0.i, v1, v2.i
constexpr unsigned ZU1 = (1u << 0) | (1u << 1) | (1u << 3) | (1u << 7);   // v0, v1.i, v3.i
constexpr unsigned ZUX = ZU0 & ZU1;                                       // s chosen at run time: v0.i, v1.i

// a1 x1 + a2 x2 + a3 x3 with the structurally zero terms skipped; association of the generic code:
// fma(a3, x3, fma(a2, x2, a1 * x1))
template <bool Z1, bool Z2, bool Z3>
__device__ __forceinline__ double sp3(double a1, double x1, double a2, double x2, double a3, double x3) {
  if constexpr (!Z1) {
    double t = a1 * x1;
    if constexpr (!Z2) t = fma(a2, x2, t);
    if constexpr (!Z3) t = fma(a3, x3, t);
    return t;
  } else if constexpr (!Z2) {
    double t = a2 * x2;
    if constexpr (!Z3) t = fma(a3, x3, t);
    return t;
  } else if constexpr (!Z3) {
    return a3 * x3;
  } else {
    return 0.0;
  }
}
// q x +- inner (the propagator's diagonal term added last, as fma(q, x, +-inner) in the generic code)
template <bool ZX, bool ZI, bool NEG>
__device__ __forceinline__ double sfin(double q, double x, double inner) {
  if constexpr (!ZX && !ZI) return fma(q, x, NEG ? -inner : inner);
  else if constexpr (!ZX) return q * x;
  else if constexpr (!ZI) return NEG ? -inner : inner;
  else return 0.0;
}

// ---- V: epsslash psi (column) and psibar epsslash (row); T: transverse eps (e3 = 0, e[2] not read)
// emul_col terms (x, y = the two input components, s = +-1):
//   o0.r = s (e3 x.r + e1 y.r + e2 y.i)   o0.i = s (e3 x.i + e1 y.i - e2 y.r)
//   o1.r = s (e1 x.r - e2 x.i - e3 y.r)   o1.i = s (e1 x.i + e2 x.r - e3 y.i)
template <unsigned Z, int XC, int YC, bool T>
__device__ __forceinline__ void emul_col_z(const double* e, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  constexpr bool xr = zb(Z, 2 * XC), xi = zb(Z, 2 * XC + 1), yr = zb(Z, 2 * YC), yi = zb(Z, 2 * YC + 1);
  const double se1 = sgn * e[0], se2 = sgn * e[1], se3 = T ? 0.0 : sgn * e[2];
  o0.r = sp3<T || xr, yr, yi>(se3, x.r, se1, y.r, se2, y.i);
  o0.i = sp3<T || xi, yi, yr>(se3, x.i, se1, y.i, -se2, y.r);
  o1.r = sp3<xr, xi, T || yr>(se1, x.r, -se2, x.i, -se3, y.r);
  o1.i = sp3<xi, xr, T || yi>(se1, x.i, se2, x.r, -se3, y.i);
}
__host__ __device__ constexpr unsigned zemul_col(unsigned Z, int XC, int YC, bool T, int OC) {
  const bool xr = zb(Z, 2 * XC), xi = zb(Z, 2 * XC + 1), yr = zb(Z, 2 * YC), yi = zb(Z, 2 * YC + 1);
  const bool o0r = (T || xr) && yr && yi, o0i = (T || xi) && yi && yr;
  const bool o1r = xr && xi && (T || yr), o1i = xi && xr && (T || yi);
  return ((unsigned)o0r << (2 * OC)) | ((unsigned)o0i << (2 * OC + 1)) | ((unsigned)o1r << (2 * OC + 2)) |
         ((unsigned)o1i << (2 * OC + 3));
}
// emul_row terms: o0.r = e3 x.r + e1 y.r - e2 y.i   o0.i = e3 x.i + e1 y.i + e2 y.r
//                 o1.r = e1 x.r + e2 x.i - e3 y.r   o1.i = e1 x.i - e2 x.r - e3 y.i   (times s)
template <unsigned Z, int XC, int YC, bool T>
__device__ __forceinline__ void emul_row_z(const double* e, c2 x, c2 y, double sgn, c2& o0, c2& o1) {
  constexpr bool xr = zb(Z, 2 * XC), xi = zb(Z, 2 * XC + 1), yr = zb(Z, 2 * YC), yi = zb(Z, 2 * YC + 1);
  const double se1 = sgn * e[0], se2 = sgn * e[1], se3 = T ? 0.0 : sgn * e[2];
  o0.r = sp3<T || xr, yr, yi>(se3, x.r, se1, y.r, -se2, y.i);
  o0.i = sp3<T || xi, yi, yr>(se3, x.i, se1, y.i, se2, y.r);
  o1.r = sp3<xr, xi, T || yr>(se1, x.r, se2, x.i, -se3, y.r);
  o1.i = sp3<xi, xr, T || yi>(se1, x.i, -se2, x.r, -se3, y.i);
}
// (the row terms have the same zero structure as the column terms)
__host__ __device__ constexpr unsigned zemul_row(unsigned Z, int XC, int YC, bool T, int OC) { return zemul_col(Z, XC, YC, T, OC); }

// zero pattern of epsslash psi / psibar epsslash for input pattern Z
__host__ __device__ constexpr unsigned z_eslash(unsigned Z, bool T) { return zemul_col(Z, 2, 3, T, 0) | zemul_col(Z, 0, 1, T, 2); }

template <unsigned Z, bool T>
__device__ __forceinline__ spinor eslash_col_z(const double* e, const spinor& p) {
  spinor o;
  emul_col_z<Z, 2, 3, T>(e, p.v[2], p.v[3], -1.0, o.v[0], o.v[1]);
  emul_col_z<Z, 0, 1, T>(e, p.v[0], p.v[1], 1.0, o.v[2], o.v[3]);
  return o;
}
template <unsigned Z, bool T>
__device__ __forceinline__ spinor eslash_row_z(const double* e, const spinor& p) {
  spinor o;
  emul_row_z<Z, 2, 3, T>(e, p.v[2], p.v[3], 1.0, o.v[0], o.v[1]);
  emul_row_z<Z, 0, 1, T>(e, p.v[0], p.v[1], -1.0, o.v[2], o.v[3]);
  return o;
}

// ---- S: (Qslash + m)/D psi (column) and psibar (Qslash + m)/D (row); a, b, c, d = components 0..3
// bits of the four components: a 0/1, b 2/3, c 4/5, d 6/7
template <unsigned Z>
__device__ __forceinline__ spinor prop_col_z(const double* mk, const spinor& p) {
  const double qp = mk[0], qm = mk[1], qx = mk[2], qy = mk[3], qz = mk[4];
  const c2 a = p.v[0], b = p.v[1], c = p.v[2], d = p.v[3];
  spinor o;
  o.v[0].r = sfin<zb(Z, 0), zb(Z, 4) && zb(Z, 6) && zb(Z, 7), true>(qp, a.r, sp3<zb(Z, 4), zb(Z, 6), zb(Z, 7)>(qz, c.r, qx, d.r, qy, d.i));
  o.v[0].i = sfin<zb(Z, 1), zb(Z, 5) && zb(Z, 7) && zb(Z, 6), true>(qp, a.i, sp3<zb(Z, 5), zb(Z, 7), zb(Z, 6)>(qz, c.i, qx, d.i, -qy, d.r));
  o.v[1].r = sfin<zb(Z, 2), zb(Z, 4) && zb(Z, 5) && zb(Z, 6), true>(qp, b.r, sp3<zb(Z, 4), zb(Z, 5), zb(Z, 6)>(qx, c.r, -qy, c.i, -qz, d.r));
  o.v[1].i = sfin<zb(Z, 3), zb(Z, 5) && zb(Z, 4) && zb(Z, 7), true>(qp, b.i, sp3<zb(Z, 5), zb(Z, 4), zb(Z, 7)>(qx, c.i, qy, c.r, -qz, d.i));
  o.v[2].r = sfin<zb(Z, 4), zb(Z, 0) && zb(Z, 2) && zb(Z, 3), false>(qm, c.r, sp3<zb(Z, 0), zb(Z, 2), zb(Z, 3)>(qz, a.r, qx, b.r, qy, b.i));
  o.v[2].i = sfin<zb(Z, 5), zb(Z, 1) && zb(Z, 3) && zb(Z, 2), false>(qm, c.i, sp3<zb(Z, 1), zb(Z, 3), zb(Z, 2)>(qz, a.i, qx, b.i, -qy, b.r));
  o.v[3].r = sfin<zb(Z, 6), zb(Z, 0) && zb(Z, 1) && zb(Z, 2), false>(qm, d.r, sp3<zb(Z, 0), zb(Z, 1), zb(Z, 2)>(qx, a.r, -qy, a.i, -qz, b.r));
  o.v[3].i = sfin<zb(Z, 7), zb(Z, 1) && zb(Z, 0) && zb(Z, 3), false>(qm, d.i, sp3<zb(Z, 1), zb(Z, 0), zb(Z, 3)>(qx, a.i, qy, a.r, -qz, b.i));
  return o;
}
template <unsigned Z>
__device__ __forceinline__ spinor prop_row_z(const double* mk, const spinor& p) {
  const double qp = mk[0], qm = mk[1], qx = mk[2], qy = mk[3], qz = mk[4];
  const c2 a = p.v[0], b = p.v[1], c = p.v[2], d = p.v[3];
  spinor o;
  o.v[0].r = sfin<zb(Z, 0), zb(Z, 4) && zb(Z, 6) && zb(Z, 7), false>(qp, a.r, sp3<zb(Z, 4), zb(Z, 6), zb(Z, 7)>(qz, c.r, qx, d.r, -qy, d.i));
  o.v[0].i = sfin<zb(Z, 1), zb(Z, 5) && zb(Z, 7) && zb(Z, 6), false>(qp, a.i, sp3<zb(Z, 5), zb(Z, 7), zb(Z, 6)>(qz, c.i, qx, d.i, qy, d.r));
  o.v[1].r = sfin<zb(Z, 2), zb(Z, 4) && zb(Z, 5) && zb(Z, 6), false>(qp, b.r, sp3<zb(Z, 4), zb(Z, 5), zb(Z, 6)>(qx, c.r, qy, c.i, -qz, d.r));
  o.v[1].i = sfin<zb(Z, 3), zb(Z, 5) && zb(Z, 4) && zb(Z, 7), false>(qp, b.i, sp3<zb(Z, 5), zb(Z, 4), zb(Z, 7)>(qx, c.i, -qy, c.r, -qz, d.i));
  o.v[2].r = sfin<zb(Z, 4), zb(Z, 0) && zb(Z, 2) && zb(Z, 3), true>(qm, c.r, sp3<zb(Z, 0), zb(Z, 2), zb(Z, 3)>(qz, a.r, qx, b.r, -qy, b.i));
  o.v[2].i = sfin<zb(Z, 5), zb(Z, 1) && zb(Z, 3) && zb(Z, 2), true>(qm, c.i, sp3<zb(Z, 1), zb(Z, 3), zb(Z, 2)>(qz, a.i, qx, b.i, qy, b.r));
  o.v[3].r = sfin<zb(Z, 6), zb(Z, 0) && zb(Z, 1) && zb(Z, 2), true>(qm, d.r, sp3<zb(Z, 0), zb(Z, 1), zb(Z, 2)>(qx, a.r, qy, a.i, -qz, b.r));
  o.v[3].i = sfin<zb(Z, 7), zb(Z, 1) && zb(Z, 0) && zb(Z, 3), true>(qm, d.i, sp3<zb(Z, 1), zb(Z, 0), zb(Z, 3)>(qx, a.i, -qy, a.r, -qz, b.i));
  return o;
}

// V then S on an external spinor with zero pattern Z: the in-side leaf phi = S(Q) epsslash u (column) and
// the out-side node ubar epsslash S(Q) (row)
template <unsigned Z, bool T>
__device__ __forceinline__ spinor vs_col_z(const double* mk, const double* e, const spinor& u) {
  return prop_col_z<z_eslash(Z, T)>(mk, eslash_col_z<Z, T>(e, u));
}
template <unsigned Z, bool T>
__device__ __forceinline__ spinor vs_row_z(const double* mk, const double* e, const spinor& ub) {
  return prop_row_z<z_eslash(Z, T)>(mk, eslash_row_z<Z, T>(e, ub));
}

// ubar(p', s') epsslash S(Q) with s' a warp-uniform run-time value (the register kernels' pass index): one
// specialisation per spin behind a uniform branch, so each pass skips all four zeros of its ubar
template <bool T>
__device__ __forceinline__ spinor vs_row_ub(const double* mk, const double* e, const spinor& ub, int sp) {
  spinor o;
  if (sp == 0) {
    o = vs_row_z<ZU0, T>(mk, e, ub);
  } else {
    o = vs_row_z<ZU1, T>(mk, e, ub);
  }
  return o;
}

}  // namespace qed
