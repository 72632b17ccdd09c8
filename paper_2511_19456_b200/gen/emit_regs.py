"""Emit the register-resident straight-line kernel body for small processes (N = 2, 3 photons).

Build-time only.  Same node-reduced DAG as gen/lower.py with tie position j = 1
(App. C), but lowered to explicit
per-thread statements instead of task tables:

  thread = (phase-space point, s')      -- two threads per point
  in-side leaves   phi_a[s][lam_a] = S(Q_{a}) epsslash_a(lam_a) u(p, s)
                   thread s' computes the s = s' half; both halves are exchanged
                   through a 768-byte shared-memory slot per point (no recomputation)
  out-side trie    ubar(p', s') epsslash_b(lam_b) [S(Q_{all \\ b}) epsslash_c(lam_c)]
                   walked depth-first: every interior (S1) and leaf (V) computed once
  joins (S2+Sum)   acc[s, lam] += leaf . phi_a   for every diagram and configuration

Everything else (external states, propagator constants) is computed in registers;
the only shared memory is the phi exchange.  The emitted code is straight-line: no
task tables, no loops over nodes (fully inlined code lets the
compiler deduplicate at instruction level).
"""
from __future__ import annotations

import itertools
import os

from .lower import FLOPS


def _flops(N: int) -> dict:
    """Flops per point of the emitted body.  Half of every vertex count has lam = 1, whose
    polarisation eps(k, 2) is transverse (eps^3 = 0): V_T = 24 instead of V = 40; vertices and propagators
    applied to the external spinors skip those spinors' structural zeros (sparse_v / sparse_s)."""
    H = 1 << (N + 2)
    n_phi = N * 4                                   # leaves phi_a[s][lam]
    if N == 2:
        n_int, n_leaf = 0, N * 2 * 2                # leaves ubar eps_b, both s'
    else:
        n_int = N * 2 * 2                           # ubar eps_b S, both s'
        n_leaf = N * (N - 1) * 4 * 2                # (b, c) x lam_b lam_c x s'
    import math
    V2 = FLOPS["V"] + FLOPS["V_T"]                  # one vertex of each polarisation
    # vertices on the external spinors skip their structural zeros (qed_sparse.cuh): the phi leaves on
    # u(p, s) and the out-side first level on ubar(p', s'), s and s' known at build time (n = 1) or selected per
    # pass by a uniform branch (n = 2, vs_row_ub)
    vs_u = sum(sparse_vs(ZU[s_], lam == 1) for s_ in range(2) for lam in range(2))          # one photon
    if N == 2:
        v_ub = sum(sparse_v(ZU[s_], lam == 1)[0] for s_ in range(2) for lam in range(2))   # one photon
        trie_out = N * v_ub
    else:
        vs_ub = sum(sparse_vs(ZU[s_], lam == 1) for s_ in range(2) for lam in range(2))   # one photon, both s'
        trie_out = N * vs_ub + n_leaf // 2 * V2
    return {
        "external": N * FLOPS["EPS"] + 2 * FLOPS["SPINOR"],
        "propagator_constants": (N + (N if N > 2 else 0)) * FLOPS["MASK"],
        "trie_in": N * vs_u,
        "trie_out": trie_out,
        "join": math.factorial(N) * H * FLOPS["JOIN"],
        "msq": H * FLOPS["ABS2"],
    }


def slot_layout(N: int) -> dict:
    """Per-point shared-memory slot (doubles): phi[a][s][lam] spinors, eps[i][lam][4], masks[m][6]."""
    lay = {"PHI": 0}
    off = N * 4 * 8
    lay["EPS"] = off
    off += N * 2 * 4
    lay["MASK"] = off                 # slot k: k < N -> {k}; k >= N -> all \ {k - N}
    n_masks = N if N == 2 else 2 * N
    off += n_masks * 6
    if (off // 2) % 2 == 0:
        off += 2                      # odd number of 16-byte slots per point (bank spread)
    lay["STRIDE"] = off
    return lay


T_ = ("", "_t")   # vertex of polarisation lam: eps(k, 2) (lam = 1) is transverse, eps^3 = 0

# Structural zeros of the external spinors (csrc/qed_sparse.cuh ZU0 / ZU1 / ZUX; bit 2c + j = component c,
# j = 0 real / 1 imaginary): u(p, 0) = ubar-pattern(p', 0) = (n, 0, ., 0 + ...), u(p, 1) likewise; ZUX = both
# (spin chosen at run time).  The register bodies skip the products with them (qed_sparse.cuh).
ZU = (0b00101110, 0b10001011)
ZUX = ZU[0] & ZU[1]


def _zb(Z: int, k: int) -> bool:
    return bool((Z >> k) & 1)


def _cnt(zero_flags) -> int:
    """flops of one real output that sums the non-zero products among its terms: 1 DMUL + (k - 1) DFMA."""
    k = sum(1 for z in zero_flags if not z)
    return 2 * k - 1 if k else 0


def sparse_v(Z: int, T: bool) -> tuple[int, int]:
    """(flops, output zero pattern) of the vertex epsslash psi / psibar epsslash on input pattern Z, mirroring
    qed_sparse.cuh emul_col_z / emul_row_z; T: transverse eps (e3 = 0).  Z = 0 gives the generic 40 / 24."""
    fl, zout = 0, 0
    for oc, (xc, yc) in ((0, (2, 3)), (2, (0, 1))):
        xr, xi, yr, yi = _zb(Z, 2 * xc), _zb(Z, 2 * xc + 1), _zb(Z, 2 * yc), _zb(Z, 2 * yc + 1)
        outs = [[T or xr, yr, yi], [T or xi, yi, yr], [xr, xi, T or yr], [xi, xr, T or yi]]
        for k, terms in enumerate(outs):
            fl += _cnt(terms)
            if all(terms):
                zout |= 1 << (2 * oc + k)
    return fl, zout


def sparse_s(Z: int) -> int:
    """flops of the propagator (Qslash + m)/D on input pattern Z (qed_sparse.cuh prop_col_z / prop_row_z, same
    term structure); Z = 0 gives the generic 56."""
    z = [_zb(Z, k) for k in range(8)]
    outs = [[z[0], z[4], z[6], z[7]], [z[1], z[5], z[7], z[6]], [z[2], z[4], z[5], z[6]], [z[3], z[5], z[4], z[7]],
            [z[4], z[0], z[2], z[3]], [z[5], z[1], z[3], z[2]], [z[6], z[0], z[1], z[2]], [z[7], z[1], z[0], z[3]]]
    return sum(_cnt(t) for t in outs)


def sparse_vs(Z: int, T: bool) -> int:
    """V then S on an external spinor with zero pattern Z (qed_sparse.cuh vs_col_z / vs_row_z)."""
    fv, zv = sparse_v(Z, T)
    return fv + sparse_s(zv)


def emit_regs_body(N: int) -> str:
    assert N in (2, 3)
    lay = slot_layout(N)
    full = (1 << N) - 1
    L = []
    w = L.append
    w(f"// ---- generated straight-line body, N = {N} (thread = point x s'), j = 1")
    w(f"// slot layout (doubles): PHI {lay['PHI']}, EPS {lay['EPS']}, MASK {lay['MASK']}, stride {lay['STRIDE']}")
    w("template <class ARGS>")
    w(f"__device__ __forceinline__ void regs_body_N{N}(const double* __restrict__ mom, long long n, long long pt, int sp,")
    w("                                              double* __restrict__ sl, const ARGS& a, double (&acc)[%d]) {" % (2 << (N + 1)))
    w("  // U: external states (PAPER.md App. D ComputeTaskQED_U), split over the two threads of the point")
    w("  const int e_out = a.e_out_particle;")
    w("  double pe[4], pp[4];")
    w("  for (int mu = 0; mu < 4; ++mu) {")
    w("    pe[mu] = qed::ld_mom(mom + (long long)mu * n + pt);")
    w("    pp[mu] = qed::ld_mom(mom + (long long)(4 * e_out + mu) * n + pt);")
    w("  }")
    w("  // external polarisations and propagator constants, split evenly over the two threads of the")
    w("  // point without divergence: thread s' takes photons i = s', s'+2, ... and subsets k = s', s'+2, ...")
    w(f"  for (int i = sp; i < {N}; i += 2) {{")
    w("    const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("    double k[4];")
    w("    for (int mu = 0; mu < 4; ++mu) k[mu] = qed::ld_mom(mom + (long long)(4 * pj + mu) * n + pt);")
    w(f"    qed::external_eps(k, sl + {lay['EPS']} + 8 * i);")
    w("  }")
    w("  {")
    w(f"    double q[{N}][4];")
    w(f"    for (int i = 0; i < {N}; ++i) {{")
    w("      const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("      const double sg = i < a.n_in_ph ? 1.0 : -1.0;")
    w("      for (int mu = 0; mu < 4; ++mu) q[i][mu] = sg * qed::ld_mom(mom + (long long)(4 * pj + mu) * n + pt);")
    w("    }")
    masks = [1 << i for i in range(N)] + ([full & ~(1 << b) for b in range(N)] if N == 3 else [])
    w(f"    for (int k = sp; k < {len(masks)}; k += 2)   // subsets: k < N -> {{k}}, k >= N -> all \\ {{k - N}}")
    w(f"      qed::mask_store(pe, q, k < {N} ? (1 << k) : ({full} & ~(1 << (k - {N}))), sl + {lay['MASK']} + 6 * k);")
    w("  }")
    w("  const qed::spinor u = qed::u_spinor(pe, sp);      // u(p, s = s'): this thread's half of phi")
    w("  const qed::spinor ub = qed::ubar_spinor(pp, sp);  // ubar(p', s')")
    w("  __syncwarp();")
    w("  // in-side leaves phi_a[s = s'][lam] = S(Q_a) epsslash_a(lam) u   (V + S2 propagation)")
    for i in range(N):
        for lam in range(2):
            w(f"  qed::st_spinor(sl + (({i} * 2 + sp) * 2 + {lam}) * 8, qed::prop_col(sl + {lay['MASK'] + 6 * i}, "
              f"qed::eslash_col{T_[lam]}(sl + {lay['EPS'] + 8 * i + 4 * lam}, u)));")
    w("  __syncwarp();")
    w("  // out-side trie, depth first; joins against phi of the remaining photon")
    for b in range(N):
        for lb in range(2):
            e_b = lay["EPS"] + 8 * b + 4 * lb
            if N == 2:
                a_ = 1 - b
                w(f"  {{  // tau = ({b}), lam_{b} = {lb}, remaining photon {a_}")
                w(f"    double eb[3]; qed::ld_stream_eps{T_[lb]}(sl + {e_b}, eb);")
                w(f"    const qed::spinor leaf = qed::eslash_row{T_[lb]}(eb, ub);")
                w("    #pragma unroll")
                w("    for (int k = 0; k < 4; ++k) {")
                w(f"      const qed::spinor ph = qed::ld_spinor_stream(sl + ({a_} * 4 + k) * 8);")
                w(f"      const int idx = (k >> 1) | ((k & 1) << {1 + a_}) | ({lb} << {1 + b});")
                w("      qed::cdot_acc(leaf, ph, acc[2 * idx], acc[2 * idx + 1]);")
                w("    }")
                w("  }")
            else:
                w(f"  {{  // tau_1 = photon {b}, lam_{b} = {lb}")
                w("    __syncwarp();")
                w(f"    double eb[3], mb[5]; qed::ld_stream_eps{T_[lb]}(sl + {e_b}, eb); qed::ld_stream_mask(sl + {lay['MASK'] + 6 * (N + b)}, mb);")
                w(f"    const qed::spinor I = qed::prop_row(mb, qed::eslash_row{T_[lb]}(eb, ub));")
                for c in range(N):
                    if c == b:
                        continue
                    a_ = 3 - b - c
                    w(f"    {{  // tau_2 = photon {c}, remaining photon {a_}")
                    w("      __syncwarp();  // scheduling fence: ptxas would otherwise hoist every phi load and spill")
                    w(f"      double ec0[3], ec1[3]; qed::ld_stream_eps(sl + {lay['EPS'] + 8 * c}, ec0); qed::ld_stream_eps_t(sl + {lay['EPS'] + 8 * c + 4}, ec1);")
                    w(f"      const qed::spinor l0 = qed::eslash_row(ec0, I);")
                    w(f"      const qed::spinor l1 = qed::eslash_row_t(ec1, I);")
                    w("      #pragma unroll")
                    w("      for (int k = 0; k < 4; ++k) {")
                    w(f"        const qed::spinor ph = qed::ld_spinor_stream(sl + ({a_} * 4 + k) * 8);")
                    w(f"        const int i0 = (k >> 1) | ((k & 1) << {1 + a_}) | ({lb} << {1 + b});")
                    w(f"        qed::cdot_acc(l0, ph, acc[2 * i0], acc[2 * i0 + 1]);")
                    w(f"        qed::cdot_acc(l1, ph, acc[2 * (i0 | {1 << (1 + c)})], acc[2 * (i0 | {1 << (1 + c)}) + 1]);")
                    w("      }")
                    w("    }")
                w("  }")
    w("  __syncwarp();")
    w("}")
    return "\n".join(L) + "\n"


def emit_regs_body1(N: int) -> str:
    """N = 2 body with ONE thread per point: the thread holds all 16 amplitudes and the four phi leaves
    of the current in-side photon in registers, so no shared-memory exchange and no warp fences.
    Same DAG, same flops as emit_regs_body(2) (nothing is recomputed)."""
    assert N == 2
    L = []
    w = L.append
    w("// ---- generated straight-line body, N = 2 (thread = point), j = 1, everything in registers")
    w("template <class ARGS>")
    w("__device__ __forceinline__ void regs_body1_N2(const double* __restrict__ mom, long long n, long long pt, int,")
    w("                                               double* __restrict__, const ARGS& a, double (&acc)[32]) {")
    w("  const int e_out = a.e_out_particle;")
    w("  double pe[4], pp[4], q[2][4];")
    w("  for (int mu = 0; mu < 4; ++mu) {")
    w("    pe[mu] = qed::ld_mom(mom + (long long)mu * n + pt);")
    w("    pp[mu] = qed::ld_mom(mom + (long long)(4 * e_out + mu) * n + pt);")
    w("  }")
    w("  for (int i = 0; i < 2; ++i) {")
    w("    const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("    for (int mu = 0; mu < 4; ++mu) q[i][mu] = qed::ld_mom(mom + (long long)(4 * pj + mu) * n + pt);")
    w("  }")
    w("  // U: eps(k_i, lam) (lam = 1 transverse, eps^3 = 0), propagator constants of S(Q_{i}), u, ubar")
    w("  double e[2][2][3], m[2][5];")
    w("  for (int i = 0; i < 2; ++i) {")
    w("    double ct, st, cf, sf;")
    w("    qed::eps_consts(q[i], ct, st, cf, sf);")
    w("    e[i][0][0] = ct * cf; e[i][0][1] = ct * sf; e[i][0][2] = -st;")
    w("    e[i][1][0] = -sf; e[i][1][1] = cf; e[i][1][2] = 0.0;")
    w("  }")
    w("  for (int i = 0; i < 2; ++i) {")
    w("    const double sg = i < a.n_in_ph ? 1.0 : -1.0;")
    w("    qed::mask_regs(pe, q[i], sg, m[i]);")
    w("  }")
    w("  const qed::spinor u0 = qed::u_spinor(pe, 0), u1 = qed::u_spinor(pe, 1);")
    w("  const qed::spinor ub0 = qed::ubar_spinor(pp, 0), ub1 = qed::ubar_spinor(pp, 1);")
    for a_ in range(2):
        b = 1 - a_
        w(f"  {{  // in-side photon {a_}: phi[s][lam_{a_}] = S(Q_{a_}) epsslash u(p, s); out-side leaves ubar(s') epsslash_{b}")
        w("    qed::spinor ph[2][2];")
        for s, us in ((0, "u0"), (1, "u1")):
            w(f"    ph[{s}][0] = qed::vs_col_z<qed::ZU{s}, false>(m[{a_}], e[{a_}][0], {us});")
            w(f"    ph[{s}][1] = qed::vs_col_z<qed::ZU{s}, true>(m[{a_}], e[{a_}][1], {us});")
        for lb in range(2):
            for sp, ubs in ((0, "ub0"), (1, "ub1")):
                w(f"    {{ const qed::spinor leaf = qed::eslash_row_z<qed::ZU{sp}, {'true' if lb else 'false'}>(e[{b}][{lb}], {ubs});")
                for s in range(2):
                    for la in range(2):
                        idx = s | (la << (1 + a_)) | (lb << (1 + b)) | (sp << 3)
                        w(f"      qed::cdot_acc(leaf, ph[{s}][{la}], acc[{2 * idx}], acc[{2 * idx + 1}]);")
                w("    }")
        w("  }")
    w("}")
    return "\n".join(L) + "\n"


def emit_regs_body1p(N: int, fence: bool = True, inter: bool = False) -> str:
    """N = 3 body with ONE thread per point, in two passes over the outgoing-electron spin s'.
    The thread's 12 phi leaves go to a private shared-memory slot (no exchange, no sharing); each pass
    walks the out-side trie of u-bar(p', s') depth first with the 32 amplitudes of that s' in registers
    and hands them to `fin` (|amp|^2 or per-configuration store) before the next pass reuses them.
    Same DAG, same flops as emit_regs_body(3) (nothing is recomputed)."""
    assert N == 3
    L = []
    w = L.append
    fn = "regs_body1p_N3" if fence else "regs_body1q_N3"
    if inter:
        fn = "regs_body1pi_N3"
    w(f"// ---- generated straight-line body, N = 3 (thread = point, two passes over s'), j = 1")
    w("template <class ARGS, class FIN>")
    w(f"__device__ __forceinline__ void {fn}(const double* __restrict__ mom, long long n, long long pt,")
    w("                                               double* __restrict__ sl, const ARGS& a, FIN&& fin) {")
    w("  const int e_out = a.e_out_particle;")
    w("  double pe[4], pp[4], q[3][4], sg[3];")
    w("  for (int mu = 0; mu < 4; ++mu) {")
    w("    pe[mu] = qed::ld_mom(mom + (long long)mu * n + pt);")
    w("    pp[mu] = qed::ld_mom(mom + (long long)(4 * e_out + mu) * n + pt);")
    w("  }")
    w("  for (int i = 0; i < 3; ++i) {")
    w("    const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("    sg[i] = i < a.n_in_ph ? 1.0 : -1.0;")
    w("    for (int mu = 0; mu < 4; ++mu) q[i][mu] = qed::ld_mom(mom + (long long)(4 * pj + mu) * n + pt);")
    w("  }")
    w("  double e[3][2][3];")
    w("  for (int i = 0; i < 3; ++i) {")
    w("    double ct, st, cf, sf;")
    w("    qed::eps_consts(q[i], ct, st, cf, sf);")
    w("    e[i][0][0] = ct * cf; e[i][0][1] = ct * sf; e[i][0][2] = -st;")
    w("    e[i][1][0] = -sf; e[i][1][1] = cf; e[i][1][2] = 0.0;")
    w("  }")
    w("  // in-side leaves phi_a[s][lam] = S(Q_{a}) epsslash_a(lam) u(p, s) -> private slot, spinor a * 4 + s * 2 + lam")
    w("  {")
    w("    const qed::spinor u0 = qed::u_spinor(pe, 0), u1 = qed::u_spinor(pe, 1);")
    for a_ in range(3):
        w(f"    {{ double m[5]; qed::mask_regs(pe, q[{a_}], sg[{a_}], m);")
        for s_, us in ((0, "u0"), (1, "u1")):
            for lam in range(2):
                w(f"      qed::st_spinor(sl + {(a_ * 4 + s_ * 2 + lam) * 8}, qed::vs_col_z<qed::ZU{s_}, {'true' if lam else 'false'}>(m, e[{a_}][{lam}], {us}));")
        w("    }")
    w("  }")
    w("  // propagator constants of S(Q_{all \\ b}): Q = p + sum_{i != b} sg_i k_i")
    w("  double mc[3][5];")
    w("  for (int b = 0; b < 3; ++b) {")
    w("    double Q0 = pe[0], Q1 = pe[1], Q2 = pe[2], Q3 = pe[3];")
    w("    for (int i = 0; i < 3; ++i)")
    w("      if (i != b) { Q0 = fma(sg[i], q[i][0], Q0); Q1 = fma(sg[i], q[i][1], Q1); Q2 = fma(sg[i], q[i][2], Q2); Q3 = fma(sg[i], q[i][3], Q3); }")
    w("    const double D = Q0 * Q0 - Q1 * Q1 - Q2 * Q2 - Q3 * Q3 - 1.0;")
    w("    const double inv = 1.0 / D;")
    w("    mc[b][0] = (Q0 + 1.0) * inv; mc[b][1] = (1.0 - Q0) * inv; mc[b][2] = Q1 * inv; mc[b][3] = Q2 * inv; mc[b][4] = Q3 * inv;")
    w("  }")
    w("  #pragma unroll 1")
    w("  for (int sp = 0; sp < 2; ++sp) {")
    w("    double acc[32];")
    w("    #pragma unroll")
    w("    for (int i = 0; i < 32; ++i) acc[i] = 0.0;")
    w("    const qed::spinor ub = qed::ubar_spinor(pp, sp);")
    # s' is the run-time pass index: the out-side first level branches (warp-uniformly) to the specialisation of
    # ubar(p', s') for that spin (vs_row_ub, all four zeros skipped; +2.3 %, profiles/ab_s3_ub.jsonl); instantiating
    # the whole pass per spin instead measured 5-10 % slower (code size, sweep_s3_unroll_rejected)
    for b in range(3):
        for lb in range(2):
            w(f"    {{  // tau_1 = photon {b}, lam_{b} = {lb}")
            w(f"      const qed::spinor I = qed::vs_row_ub<{'true' if lb else 'false'}>(mc[{b}], e[{b}][{lb}], ub, sp);")
            for c in range(3):
                if c == b:
                    continue
                a_ = 3 - b - c
                w(f"      {{  // tau_2 = photon {c}, remaining photon {a_}")
                if fence:
                    w("        __syncwarp();  // scheduling fence: keeps ptxas from hoisting every phi load")
                w(f"        const qed::spinor l0 = qed::eslash_row(e[{c}][0], I);")
                w(f"        const qed::spinor l1 = qed::eslash_row_t(e[{c}][1], I);")
                if inter:
                    w("        qed::spinor ph[4];")
                    w("        #pragma unroll")
                    w(f"        for (int k = 0; k < 4; ++k) ph[k] = qed::ld_spinor_stream(sl + ({a_} * 4 + k) * 8);")
                    w("        int ix[8];")
                    w("        #pragma unroll")
                    w(f"        for (int k = 0; k < 4; ++k) {{ ix[k] = (k >> 1) | ((k & 1) << {1 + a_}) | ({lb} << {1 + b}); ix[4 + k] = ix[k] | {1 << (1 + c)}; }}")
                    w("        qed::cdot8_acc(l0, l1, ph, ix, acc);")
                    w("      }")
                    continue
                w("        #pragma unroll")
                w("        for (int k = 0; k < 4; ++k) {")
                w(f"          const qed::spinor ph = qed::ld_spinor_stream(sl + ({a_} * 4 + k) * 8);")
                w(f"          const int i0 = (k >> 1) | ((k & 1) << {1 + a_}) | ({lb} << {1 + b});")
                w("          qed::cdot_acc(l0, ph, acc[2 * i0], acc[2 * i0 + 1]);")
                w(f"          qed::cdot_acc(l1, ph, acc[2 * (i0 | {1 << (1 + c)})], acc[2 * (i0 | {1 << (1 + c)}) + 1]);")
                w("        }")
                w("      }")
            w("    }")
    w("    fin(acc, sp);")
    w("  }")
    w("}")
    return "\n".join(L) + "\n"


def bg_flops(N: int = 3) -> dict:
    """Algorithmic flops per point of the Berends-Giele register body (emit_regs_body_bg): every current
    once.  K_out({b, c}) = P_out({b}) epsslash_c + P_out({c}) epsslash_b costs two vertices and 8 adds."""
    assert N == 3
    V2 = FLOPS["V"] + FLOPS["V_T"]
    H = 1 << (N + 2)
    return {
        "external": N * FLOPS["EPS"] + 2 * FLOPS["SPINOR"],
        "propagator_constants": 2 * N * FLOPS["MASK"],
        "currents_in": N * sum(sparse_vs(ZU[s_], lam == 1) for s_ in range(2) for lam in range(2)),  # J_in({a})[s][lam]
        "currents_out": N * 2 * sum(sparse_vs(ZUX, lam == 1) for lam in range(2)),   # P_out({b})[s'][lam], s' per pass
        "k_sums": 2 * 3 * (2 * 2 * V2 + 4 * 8),             # K_out(A^c)[s'][lam_b][lam_c]
        "join": 2 * 3 * 4 * 4 * FLOPS["JOIN"],              # one join per subset {a} and configuration
        "msq": H * FLOPS["ABS2"],
    }


def emit_regs_body_bg(N: int = 3) -> str:
    """Berends-Giele rewrite (DESIGN.md kernel 2b) of the N = 3 body, one thread per point,
    two passes over s'.  j = 1: M = sum_a K_out({b, c}) . J_in({a}), J_in({a}) = S(Q_a) epsslash_a u (the phi
    leaves, private shared-memory slot as in T1P), P_out({x}) = ubar epsslash_x S(Q_{all \\ x}) and
    K_out({b, c}) = P_out({b}) epsslash_c + P_out({c}) epsslash_b: one join per subset instead of two.
    P_out(1) is recomputed once per pass (two of the three P_out pairs are held in registers at a time)."""
    assert N == 3
    L = []
    w = L.append
    w("// ---- generated straight-line body, N = 3, Berends-Giele currents (thread = point, two passes over s'), j = 1")
    w("template <class ARGS, class FIN>")
    w("__device__ __forceinline__ void regs_body_bg_N3(const double* __restrict__ mom, long long n, long long pt,")
    w("                                                double* __restrict__ sl, const ARGS& a, FIN&& fin) {")
    w("  const int e_out = a.e_out_particle;")
    w("  double pe[4], pp[4], q[3][4], sg[3];")
    w("  for (int mu = 0; mu < 4; ++mu) {")
    w("    pe[mu] = qed::ld_mom(mom + (long long)mu * n + pt);")
    w("    pp[mu] = qed::ld_mom(mom + (long long)(4 * e_out + mu) * n + pt);")
    w("  }")
    w("  for (int i = 0; i < 3; ++i) {")
    w("    const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("    sg[i] = i < a.n_in_ph ? 1.0 : -1.0;")
    w("    for (int mu = 0; mu < 4; ++mu) q[i][mu] = qed::ld_mom(mom + (long long)(4 * pj + mu) * n + pt);")
    w("  }")
    w("  double e[3][2][3];")
    w("  for (int i = 0; i < 3; ++i) {")
    w("    double ct, st, cf, sf;")
    w("    qed::eps_consts(q[i], ct, st, cf, sf);")
    w("    e[i][0][0] = ct * cf; e[i][0][1] = ct * sf; e[i][0][2] = -st;")
    w("    e[i][1][0] = -sf; e[i][1][1] = cf; e[i][1][2] = 0.0;")
    w("  }")
    w("  // J_in({a})[s][lam] = S(Q_a) epsslash_a(lam) u(p, s) -> private slot, spinor a * 4 + s * 2 + lam")
    w("  {")
    w("    const qed::spinor u0 = qed::u_spinor(pe, 0), u1 = qed::u_spinor(pe, 1);")
    for a_ in range(3):
        w(f"    {{ double m[5]; qed::mask_regs(pe, q[{a_}], sg[{a_}], m);")
        for s_, us in ((0, "u0"), (1, "u1")):
            for lam in range(2):
                w(f"      qed::st_spinor(sl + {(a_ * 4 + s_ * 2 + lam) * 8}, qed::vs_col_z<qed::ZU{s_}, {'true' if lam else 'false'}>(m, e[{a_}][{lam}], {us}));")
        w("    }")
    w("  }")
    w("  double mc[3][5];   // S(Q_{all \\ x})")
    w("  for (int x = 0; x < 3; ++x) {")
    w("    double Q0 = pe[0], Q1 = pe[1], Q2 = pe[2], Q3 = pe[3];")
    w("    for (int i = 0; i < 3; ++i)")
    w("      if (i != x) { Q0 = fma(sg[i], q[i][0], Q0); Q1 = fma(sg[i], q[i][1], Q1); Q2 = fma(sg[i], q[i][2], Q2); Q3 = fma(sg[i], q[i][3], Q3); }")
    w("    const double D = Q0 * Q0 - Q1 * Q1 - Q2 * Q2 - Q3 * Q3 - 1.0;")
    w("    const double inv = 1.0 / D;")
    w("    mc[x][0] = (Q0 + 1.0) * inv; mc[x][1] = (1.0 - Q0) * inv; mc[x][2] = Q1 * inv; mc[x][3] = Q2 * inv; mc[x][4] = Q3 * inv;")
    w("  }")
    w("  #pragma unroll 1")
    w("  for (int sp = 0; sp < 2; ++sp) {")
    w("    double acc[32];")
    w("    #pragma unroll")
    w("    for (int i = 0; i < 32; ++i) acc[i] = 0.0;")
    w("    const qed::spinor ub = qed::ubar_spinor(pp, sp);")
    w("    qed::spinor P[3][2];   // P_out({x})[lam_x] (two of the three held at a time)")

    def pout(x):
        for lam in range(2):
            # (the per-spin specialisation of vs_row_ub spills 436 bytes in this body and measured -5.6 %)
            w(f"    P[{x}][{lam}] = qed::vs_row_z<qed::ZUX, {'true' if lam else 'false'}>(mc[{x}], e[{x}][{lam}], ub);")

    def block(a_, b, c):
        w(f"    {{  // subset {{{a_}}}: K_out({{{b}, {c}}}) . J_in({{{a_}}})")
        for lb in range(2):
            w(f"      {{ __syncwarp();  // scheduling fence: keeps ptxas from hoisting every J_in load")
            w(f"        qed::spinor K0 = qed::eslash_row(e[{c}][0], P[{b}][{lb}]), K1 = qed::eslash_row_t(e[{c}][1], P[{b}][{lb}]);")
            # accumulating vertex (3 DFMA per output, no DMUL + DADD): same 48-flop model, 8 fewer pipe slots
            w(f"        qed::eslash_row{T_[lb]}_acc(e[{b}][{lb}], P[{c}][0], K0);")
            w(f"        qed::eslash_row{T_[lb]}_acc(e[{b}][{lb}], P[{c}][1], K1);")
            w("        #pragma unroll")
            w("        for (int k = 0; k < 4; ++k) {")
            w(f"          const qed::spinor ph = qed::ld_spinor_stream(sl + ({a_} * 4 + k) * 8);")
            w(f"          const int i0 = (k >> 1) | ((k & 1) << {1 + a_}) | ({lb} << {1 + b});")
            w("          qed::cdot_acc(K0, ph, acc[2 * i0], acc[2 * i0 + 1]);")
            w(f"          qed::cdot_acc(K1, ph, acc[2 * (i0 | {1 << (1 + c)})], acc[2 * (i0 | {1 << (1 + c)}) + 1]);")
            w("        }")
            w("      }")
        w("    }")

    pout(1)
    pout(2)
    block(0, 1, 2)
    pout(0)
    block(1, 0, 2)
    pout(1)   # recomputed (P_out({1}) was dropped for P_out({0}))
    block(2, 0, 1)
    w("    fin(acc, sp);")
    w("  }")
    w("}")
    return "\n".join(L) + "\n"


def emit_regs_body4(N: int) -> str:
    """N = 3 body with four threads per point: thread = (point, s', lam_0).  Photon 0's polarisation
    is fixed per thread, so out-side nodes that do not involve photon 0 are computed by both lam_0
    threads (+14 % executed flops) in exchange for half the accumulators (more resident warps)."""
    assert N == 3
    lay = slot_layout(N)
    full = (1 << N) - 1
    L = []
    w = L.append
    w(f"// ---- generated straight-line body, N = {N} (thread = point x s' x lam_0), j = 1")
    w("template <class ARGS>")
    w(f"__device__ __forceinline__ void regs_body4_N{N}(const double* __restrict__ mom, long long n, long long pt, int sub,")
    w("                                               double* __restrict__ sl, const ARGS& a, double (&acc)[16]) {")
    w("  const int sp = sub & 1, l0 = sub >> 1;")
    w("  const int e_out = a.e_out_particle;")
    w("  double pe[4], pp[4];")
    w("  for (int mu = 0; mu < 4; ++mu) {")
    w("    pe[mu] = qed::ld_mom(mom + (long long)mu * n + pt);")
    w("    pp[mu] = qed::ld_mom(mom + (long long)(4 * e_out + mu) * n + pt);")
    w("  }")
    w("  if (sub == 0) {")
    w(f"    for (int i = 0; i < {N}; ++i) {{")
    w("      const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("      double k[4];")
    w("      for (int mu = 0; mu < 4; ++mu) k[mu] = qed::ld_mom(mom + (long long)(4 * pj + mu) * n + pt);")
    w(f"      qed::external_eps(k, sl + {lay['EPS']} + 8 * i);")
    w("    }")
    w("  } else if (sub == 1 || sub == 2) {")
    w(f"    double q[{N}][4];")
    w(f"    for (int i = 0; i < {N}; ++i) {{")
    w("      const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("      const double sg = i < a.n_in_ph ? 1.0 : -1.0;")
    w("      for (int mu = 0; mu < 4; ++mu) q[i][mu] = sg * qed::ld_mom(mom + (long long)(4 * pj + mu) * n + pt);")
    w("    }")
    masks = [1 << i for i in range(N)] + [full & ~(1 << b) for b in range(N)]
    w("    if (sub == 1) {")
    for k, msk in enumerate(masks[:3]):
        w(f"      qed::mask_store(pe, q, {msk}, sl + {lay['MASK']} + {6 * k});")
    w("    } else {")
    for k, msk in enumerate(masks[3:]):
        w(f"      qed::mask_store(pe, q, {msk}, sl + {lay['MASK']} + {6 * (k + 3)});")
    w("    }")
    w("  }")
    w("  __syncwarp();")
    w("  // in-side leaves phi_a[s][lam]: 12 spinors, 3 per thread (entry e = 4 k + sub)")
    w("  #pragma unroll")
    w("  for (int k = 0; k < 3; ++k) {")
    w("    const int e = 4 * k + sub, ai = e >> 2, s = (e >> 1) & 1, lam = e & 1;")
    w("    const qed::spinor u = qed::u_spinor(pe, s);")
    w(f"    qed::st_spinor(sl + e * 8, qed::prop_col(sl + {lay['MASK']} + 6 * ai, qed::eslash_col(sl + {lay['EPS']} + 8 * ai + 4 * lam, u)));")
    w("  }")
    w("  const qed::spinor ub = qed::ubar_spinor(pp, sp);  // ubar(p', s')")
    w("  __syncwarp();")
    for b in range(N):
        lbs = ["l0"] if b == 0 else ["0", "1"]
        for lb in lbs:
            lb_bit = "" if b == 0 else f" | ({lb} << {b})"   # acc idx: s | lam1 << 1 | lam2 << 2
            w(f"  {{  // tau_1 = photon {b}, lam_{b} = {lb}")
            w("    __syncwarp();")
            w(f"    double eb[3], mb[5]; qed::ld_stream_eps(sl + {lay['EPS']} + 8 * {b} + 4 * ({lb}), eb); "
              f"qed::ld_stream_mask(sl + {lay['MASK'] + 6 * (N + b)}, mb);")
            w("    const qed::spinor I = qed::prop_row(mb, qed::eslash_row(eb, ub));")
            for c in range(N):
                if c == b:
                    continue
                a_ = 3 - b - c
                lcs = ["l0"] if c == 0 else ["0", "1"]
                w(f"    {{  // tau_2 = photon {c}, remaining photon {a_}")
                w("      __syncwarp();")
                for li, lc in enumerate(lcs):
                    w(f"      double ec{li}[3]; qed::ld_stream_eps(sl + {lay['EPS']} + 8 * {c} + 4 * ({lc}), ec{li});")
                    w(f"      const qed::spinor lf{li} = qed::eslash_row(ec{li}, I);")
                # phi_a[s][lam_a]: lam_a = l0 if a == 0 else both
                las = ["l0"] if a_ == 0 else ["0", "1"]
                w("      #pragma unroll")
                w("      for (int s = 0; s < 2; ++s) {")
                for la in las:
                    w(f"        {{ const qed::spinor ph = qed::ld_spinor_stream(sl + (({a_} * 2 + s) * 2 + ({la})) * 8);")
                    for li, lc in enumerate(lcs):
                        bits = []
                        for (ph_, lam) in ((b, lb), (c, lc), (a_, la)):
                            if ph_ != 0:
                                bits.append(f"(({lam}) << {ph_})")
                        idx = "s | " + " | ".join(bits) if bits else "s"
                        w(f"          {{ const int idx = {idx}; qed::cdot_acc(lf{li}, ph, acc[2 * idx], acc[2 * idx + 1]); }}")
                    w("        }")
                w("      }")
                w("    }")
            w("  }")
    w("  __syncwarp();")
    w("}")
    return "\n".join(L) + "\n"


def emit_regs_body_interleaved(N: int) -> str:
    """Same DAG and thread mapping as emit_regs_body(3), but each (b, lam_b, c) block loads its four
    phi spinors first and issues the 8 joins' DFMAs interleaved (8 independent chains in a row)."""
    assert N == 3
    src = emit_regs_body(N)
    src = src.replace(f"regs_body_N{N}(", f"regs_bodyi_N{N}(")
    lines = src.split("\n")
    out = []
    i = 0
    while i < len(lines):
        ln = lines[i]
        if ln.strip() == "#pragma unroll" and i + 1 < len(lines) and "for (int k = 0; k < 4; ++k) {" in lines[i + 1] \
                and "ld_spinor_stream" in lines[i + 2] and "i0 =" in lines[i + 3]:
            # lines: pragma, for, ph load, i0, cdot l0, cdot l1, close
            load = lines[i + 2].strip()
            i0 = lines[i + 3].strip()
            bit = lines[i + 5].split("(i0 | ")[1].split(")")[0]
            ind = ln[: len(ln) - len(ln.lstrip())]
            base_expr = load.split("ld_spinor_stream(")[1].rsplit(");", 1)[0]
            i0_expr = i0.split("=", 1)[1].strip().rstrip(";")
            out.append(f"{ind}qed::spinor ph[4];")
            out.append(f"{ind}#pragma unroll")
            out.append(f"{ind}for (int k = 0; k < 4; ++k) ph[k] = qed::ld_spinor_stream({base_expr});")
            out.append(f"{ind}int ix[8];")
            out.append(f"{ind}#pragma unroll")
            out.append(f"{ind}for (int k = 0; k < 4; ++k) {{ ix[k] = {i0_expr}; ix[4 + k] = ix[k] | {bit}; }}")
            out.append(f"{ind}qed::cdot8_acc(l0, l1, ph, ix, acc);")
            i += 7
            continue
        out.append(ln)
        i += 1
    return "\n".join(out)


def emit_regs_source(N: int) -> str:
    fl = _flops(N)
    total = sum(fl.values())
    flops_comment = "\n".join(f"//   {k:22s} {v:>10d}" for k, v in fl.items())
    vs = regs_variants(N)
    ns = f"qedregs_N{N}"
    lay = slot_layout(N)
    variant_structs = "".join(
        f"struct V{i} {{ static constexpr int WPB = {w}, MIN_BLOCKS = {m}, PF = {p}; }};\n"
        for i, (d, w, m, p) in enumerate(vs))
    kernel_cases = "\n".join(
        f"    {'default' if i == 0 else f'case {i}'}: return per_config ? (const void*)qed::qed_regs_kernel<{ns}::{d}, {ns}::V{i}, true>\n"
        f"                                      : (const void*)qed::qed_regs_kernel<{ns}::{d}, {ns}::V{i}, false>;"
        for i, (d, w, m, p) in enumerate(vs))
    tpp = "{" + ", ".join("4" if d in ("T4", "TH") else "1" if d.startswith("T1") else "2" for d, *_ in vs) + "}"
    body4 = emit_regs_body4(N) + "\n" + emit_regs_body_interleaved(N) + "\n" + emit_regs_body1p(N) + "\n" + \
        emit_regs_body1p(N, inter=True) + "\n" + emit_regs_body_bg(N) if N == 3 else ""
    t4 = f"""
// four threads per point: (point, s', lam_0); accumulators s | lam_1 << 1 | lam_2 << 2
struct T4 {{
  static constexpr int N = {N}, TPP = 4, NACC = 8, STRIDE = {lay['STRIDE']};
  template <class ARGS2>
  static __device__ __forceinline__ void body(const double* mom, long long n, long long pt, int sub, double* sl,
                                              const ARGS2& a, double (&acc)[16]) {{
    regs_body4_N{N}(mom, n, pt, sub, sl, a, acc);
  }}
  static __device__ __forceinline__ unsigned config_of(int idx, int sub) {{
    return (idx & 1) | ((unsigned)(sub >> 1) << 1) | ((unsigned)(idx >> 1) << 2) | ((unsigned)(sub & 1) << (N + 1));
  }}
}};
// two threads per point, joins issued interleaved across the 8 (leaf, phi) pairs of a block
struct TI : T {{
  template <class ARGS2>
  static __device__ __forceinline__ void body(const double* mom, long long n, long long pt, int sub, double* sl,
                                              const ARGS2& a, double (&acc)[{2 << (N + 1)}]) {{
    regs_bodyi_N{N}(mom, n, pt, sub, sl, a, acc);
  }}
}};
// one thread per point, two passes over s' (32 amplitudes live per pass), phi in a private slot
struct T1P {{
  static constexpr int N = {N}, TPP = 1, NACC = {1 << (N + 1)}, STRIDE = 98, PASSES = 2;
  template <class ARGS2, class FIN>
  static __device__ __forceinline__ void body_passes(const double* mom, long long n, long long pt, double* sl,
                                                     const ARGS2& a, FIN&& fin) {{
    regs_body1p_N{N}(mom, n, pt, sl, a, fin);
  }}
  static __device__ __forceinline__ unsigned config_of(int idx, int sub) {{ return idx | ((unsigned)sub << (N + 1)); }}
}};
// Berends-Giele currents, one thread per point, two passes over s' (QED_ALGO_BERENDS_GIELE at n = 2)
struct T1B : T1P {{
  static constexpr long long FLOPS_PER_POINT = {sum(bg_flops(N).values()) if N == 3 else 0}LL;
  template <class ARGS2, class FIN>
  static __device__ __forceinline__ void body_passes(const double* mom, long long n, long long pt, double* sl,
                                                     const ARGS2& a, FIN&& fin) {{
    regs_body_bg_N{N}(mom, n, pt, sl, a, fin);
  }}
}};
// T1P with each out-side block's 8 joins issued interleaved (T1PI)
struct T1PI : T1P {{
  template <class ARGS2, class FIN>
  static __device__ __forceinline__ void body_passes(const double* mom, long long n, long long pt, double* sl,
                                                     const ARGS2& a, FIN&& fin) {{
    regs_body1pi_N{N}(mom, n, pt, sl, a, fin);
  }}
}};""" if N == 3 else ""
    if N == 2:
        body4 = emit_regs_body1(N)
        t4 = f"""
// one thread per point: all 16 amplitudes and the phi leaves in registers, no shared-memory slot
struct T1 {{
  static constexpr int N = {N}, TPP = 1, NACC = {1 << (N + 2)}, STRIDE = 0;
  template <class ARGS2>
  static __device__ __forceinline__ void body(const double* mom, long long n, long long pt, int sub, double* sl,
                                              const ARGS2& a, double (&acc)[{2 << (N + 2)}]) {{
    regs_body1_N{N}(mom, n, pt, sub, sl, a, acc);
  }}
  static __device__ __forceinline__ unsigned config_of(int idx, int) {{ return idx; }}
}};"""
    bg_c = ""
    if N == 3:
        # Berends-Giele variants; r32 sweep: 2.91e9 pts/s without the L2 prefetch, 2.81e9 with it
        # (r44: moving the complement propagator constants to the private slot, at 7 warps/SM, measured -12 %).
        # Session-3 A/B (profiles/ab_s3_t1b.jsonl): with the accumulating K_out vertices the L2 prefetch
        # variant is 1.9 % ahead (3.11e9 vs 3.06e9) -> first
        bvs = [("T1B", 8, 1, 1), ("T1B", 8, 1, 0), ("T1B", 4, 2, 1)]
        variant_structs += "".join(
            f"struct B{i} {{ static constexpr int WPB = {w_}, MIN_BLOCKS = {m}, PF = {p_}; }};\n" for i, (d, w_, m, p_) in enumerate(bvs))
        bcases = "\n".join(
            f"    {'default' if i == 0 else f'case {i}'}: return per_config ? (const void*)qed::qed_regs_kernel<{ns}::{d}, {ns}::B{i}, true>\n"
            f"                                      : (const void*)qed::qed_regs_kernel<{ns}::{d}, {ns}::B{i}, false>;"
            for i, (d, *_) in enumerate(bvs))
        bg_c = f"""// Berends-Giele rewrite in registers (one thread per point)
int qedregsbg_num_variants_N{N}(void) {{ return {len(bvs)}; }}
const void* qedregsbg_kernel_N{N}(int per_config, int variant) {{
  switch (variant) {{
{bcases}
  }}
}}
void qedregsbg_config_N{N}(int variant, int* warps_per_block, int* points_per_warp, long long* smem_per_block,
                           long long* flops_per_point) {{
  static const int wpb[{len(bvs)}] = {{{", ".join(str(v[1]) for v in bvs)}}};
  *warps_per_block = wpb[variant];
  *points_per_warp = 32;
  *smem_per_block = (long long)wpb[variant] * 32 * {ns}::T1B::STRIDE * 8;
  *flops_per_point = {ns}::T1B::FLOPS_PER_POINT;
}}
"""
    return f"""// GENERATED by paper_2511_19456_b200/gen/emit_regs.py -- do not edit.
// Register-resident kernel for N = {N} photons (n = {N - 1}); thread = (point, s') [T] or (point, s', lam_0) [T4].
// Algorithmic FP64 flops per point:
{flops_comment}
//   {'total':22s} {total:>10d}
#include "../qed_eval_regs.cuh"

namespace {ns} {{
{emit_regs_body(N)}
{body4}
// two threads per point: (point, s'); accumulators s | lam_i << (1 + i)
struct T {{
  static constexpr int N = {N}, TPP = 2, NACC = {1 << (N + 1)}, STRIDE = {lay['STRIDE']};
  static constexpr long long FLOPS_PER_POINT = {total}LL;
  template <class ARGS2>
  static __device__ __forceinline__ void body(const double* mom, long long n, long long pt, int sub, double* sl,
                                              const ARGS2& a, double (&acc)[{2 << (N + 1)}]) {{
    regs_body_N{N}(mom, n, pt, sub, sl, a, acc);
  }}
  static __device__ __forceinline__ unsigned config_of(int idx, int sub) {{ return idx | ((unsigned)sub << (N + 1)); }}
}};{t4}
{variant_structs}}}  // namespace {ns}

extern "C" {{
int qedregs_num_variants_N{N}(void) {{ return {len(vs)}; }}
const void* qedregs_kernel_N{N}(int per_config, int variant) {{
  switch (variant) {{
{kernel_cases}
  }}
}}
void qedregs_config_N{N}(int variant, int* warps_per_block, int* points_per_warp, long long* smem_per_block,
                         long long* flops_per_point) {{
  static const int wpb[{len(vs)}] = {{{", ".join(str(v[1]) for v in vs)}}};
  static const int tpp[{len(vs)}] = {tpp};
  *warps_per_block = wpb[variant];
  *points_per_warp = 32 / tpp[variant];
  static const int pf[{len(vs)}] = {{{", ".join(str(v[3]) for v in vs)}}};
  static const int stride[{len(vs)}] = {{{", ".join(f"{ns}::{v[0]}::STRIDE" if v[0].startswith("T1") else f"{ns}::T::STRIDE" for v in vs)}}};
  *smem_per_block = (long long)wpb[variant] * (32 / tpp[variant]) * stride[variant] * 8 +
                    (pf[variant] == 2 ? (long long)wpb[variant] * 2 * {4 * (N + 2)} * (32 / tpp[variant]) * 8 : 0);
  *flops_per_point = {ns}::T::FLOPS_PER_POINT;
}}
{bg_c}}}
"""


def regs_variants(N: int) -> list[tuple[str, int, int, int]]:
    """Launch variants (body, warps per block, min resident blocks, L2 prefetch); QED_VARIANT selects.
    Variant 0 = best of the latest sweep (profiles/sweep_*.jsonl)."""
    if N == 3:
        # r20 sweep: the interleaved join body TI >= T at n = 2 once the transverse vertices shortened T
        # r28 sweep: one thread per point in two s' passes (T1P) 2.31e9 pts/s (62.5 %) vs 2.01e9 for TI;
        # r30: interleaved joins (T1PI) +1.1 %, one fence per tau_1 block (T1PJ) +0.3 % (dropped)
        # r41: the L2 prefetch now covers both 128-byte lines of each 32-point row: +4 % (2.44e9, 66 %);
        #      an L1 prefetch instead measured the same (+0.3 %, dropped)
        return [("T1PI", 8, 1, 1), ("T1P", 8, 1, 1), ("T1P", 8, 1, 0), ("T1P", 4, 2, 1), ("TI", 4, 1, 2), ("T", 4, 1, 2),
                ("T", 4, 1, 1), ("T", 4, 1, 0), ("T", 2, 5, 2), ("T4", 4, 4, 1), ("T4", 4, 3, 2), ("TI", 4, 1, 1)]
    # t1 sweep: one thread per point (T1) 1.19e10 pts/s (68 % of FP64 peak) vs 8.18e9 for T
    return [("T1", 8, 1, 2), ("T1", 4, 2, 2), ("T1", 2, 4, 2), ("T1", 4, 2, 1), ("T", 2, 6, 2), ("T", 4, 1, 0),
            ("T", 4, 1, 1), ("T", 2, 6, 1), ("T", 4, 1, 2)]


def generate_regs(out_dir: str, Ns=(2, 3)) -> list[str]:
    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for N in Ns:
        path = os.path.join(out_dir, f"qed_regs_N{N}.cu")
        src = emit_regs_source(N)
        if not os.path.exists(path) or open(path).read() != src:
            with open(path, "w") as f:
                f.write(src)
        paths.append(path)
    return paths
