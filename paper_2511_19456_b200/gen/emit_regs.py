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
    H = 1 << (N + 2)
    n_phi = N * 4                                   # leaves phi_a[s][lam]
    if N == 2:
        n_int, n_leaf = 0, N * 2 * 2                # leaves ubar eps_b, both s'
    else:
        n_int = N * 2 * 2                           # ubar eps_b S, both s'
        n_leaf = N * (N - 1) * 4 * 2                # (b, c) x lam_b lam_c x s'
    import math
    return {
        "external": N * FLOPS["EPS"] + 2 * FLOPS["SPINOR"],
        "propagator_constants": (N + (N if N > 2 else 0)) * FLOPS["MASK"],
        "trie_in": n_phi * (FLOPS["V"] + FLOPS["S"]),
        "trie_out": n_int * (FLOPS["V"] + FLOPS["S"]) + n_leaf * FLOPS["V"],
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
    w("    pe[mu] = __ldg(mom + (long long)mu * n + pt);")
    w("    pp[mu] = __ldg(mom + (long long)(4 * e_out + mu) * n + pt);")
    w("  }")
    w("  if (sp == 0) {")
    w("    // polarisation vectors of every photon -> slot EPS")
    w(f"    for (int i = 0; i < {N}; ++i) {{")
    w("      const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("      double k[4];")
    w("      for (int mu = 0; mu < 4; ++mu) k[mu] = __ldg(mom + (long long)(4 * pj + mu) * n + pt);")
    w(f"      qed::external_eps(k, sl + {lay['EPS']} + 8 * i);")
    w("    }")
    w("  } else {")
    w("    // propagator constants: in-side leaves S(Q_{a}), out-side interiors S(Q_{all \\ b})")
    w(f"    double q[{N}][4];")
    w(f"    for (int i = 0; i < {N}; ++i) {{")
    w("      const int pj = (a.photon_particle >> (4 * i)) & 15;")
    w("      const double sg = i < a.n_in_ph ? 1.0 : -1.0;")
    w("      for (int mu = 0; mu < 4; ++mu) q[i][mu] = sg * __ldg(mom + (long long)(4 * pj + mu) * n + pt);")
    w("    }")
    masks = [1 << i for i in range(N)] + ([full & ~(1 << b) for b in range(N)] if N == 3 else [])
    for k, msk in enumerate(masks):
        w(f"    qed::mask_store(pe, q, {msk}, sl + {lay['MASK']} + {6 * k});")
    w("  }")
    w("  const qed::spinor u = qed::u_spinor(pe, sp);      // u(p, s = s'): this thread's half of phi")
    w("  const qed::spinor ub = qed::ubar_spinor(pp, sp);  // ubar(p', s')")
    w("  __syncwarp();")
    w("  // in-side leaves phi_a[s = s'][lam] = S(Q_a) epsslash_a(lam) u   (V + S2 propagation)")
    for i in range(N):
        for lam in range(2):
            w(f"  qed::st_spinor(sl + (({i} * 2 + sp) * 2 + {lam}) * 8, qed::prop_col(sl + {lay['MASK'] + 6 * i}, "
              f"qed::eslash_col(sl + {lay['EPS'] + 8 * i + 4 * lam}, u)));")
    w("  __syncwarp();")
    w("  // out-side trie, depth first; joins against phi of the remaining photon")
    for b in range(N):
        for lb in range(2):
            e_b = lay["EPS"] + 8 * b + 4 * lb
            if N == 2:
                a_ = 1 - b
                w(f"  {{  // tau = ({b}), lam_{b} = {lb}, remaining photon {a_}")
                w(f"    double eb[3]; qed::ld_stream_eps(sl + {e_b}, eb);")
                w(f"    const qed::spinor leaf = qed::eslash_row(eb, ub);")
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
                w(f"    double eb[3], mb[5]; qed::ld_stream_eps(sl + {e_b}, eb); qed::ld_stream_mask(sl + {lay['MASK'] + 6 * (N + b)}, mb);")
                w(f"    const qed::spinor I = qed::prop_row(mb, qed::eslash_row(eb, ub));")
                for c in range(N):
                    if c == b:
                        continue
                    a_ = 3 - b - c
                    w(f"    {{  // tau_2 = photon {c}, remaining photon {a_}")
                    w("      __syncwarp();  // scheduling fence: ptxas would otherwise hoist every phi load and spill")
                    w(f"      double ec0[3], ec1[3]; qed::ld_stream_eps(sl + {lay['EPS'] + 8 * c}, ec0); qed::ld_stream_eps(sl + {lay['EPS'] + 8 * c + 4}, ec1);")
                    w(f"      const qed::spinor l0 = qed::eslash_row(ec0, I);")
                    w(f"      const qed::spinor l1 = qed::eslash_row(ec1, I);")
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


def emit_regs_source(N: int) -> str:
    fl = _flops(N)
    total = sum(fl.values())
    flops_comment = "\n".join(f"//   {k:22s} {v:>10d}" for k, v in fl.items())
    vs = regs_variants(N)
    ns = f"qedregs_N{N}"
    variant_structs = "namespace " + ns + " {\n" + "".join(
        f"struct V{i} {{ static constexpr int WPB = {w}, MIN_BLOCKS = {m}, PF = {p}; }};\n"
        for i, (w, m, p) in enumerate(vs)) + "}\n"
    kernel_cases = "\n".join(
        f"    {'default' if i == 0 else f'case {i}'}: return per_config ? (const void*)qed::qed_regs_kernel<{ns}::T, {ns}::V{i}, true>\n"
        f"                                      : (const void*)qed::qed_regs_kernel<{ns}::T, {ns}::V{i}, false>;"
        for i in range(len(vs)))
    return f"""// GENERATED by paper_2511_19456_b200/gen/emit_regs.py -- do not edit.
// Register-resident kernel for N = {N} photons (n = {N - 1}); thread = (point, s').
// Algorithmic FP64 flops per point:
{flops_comment}
//   {'total':22s} {total:>10d}
#include "../qed_eval_regs.cuh"

namespace qedregs_N{N} {{
{emit_regs_body(N)}
struct T {{
  static constexpr int N = {N};
  static constexpr long long FLOPS_PER_POINT = {total}LL;
  static constexpr int STRIDE = {slot_layout(N)['STRIDE']};
  template <class ARGS2>
  static __device__ __forceinline__ void body(const double* mom, long long n, long long pt, int sp, double* sl,
                                              const ARGS2& a, double (&acc)[{2 << (N + 1)}]) {{
    regs_body_N{N}(mom, n, pt, sp, sl, a, acc);
  }}
}};
}}  // namespace qedregs_N{N}

{variant_structs}
extern "C" {{
int qedregs_num_variants_N{N}(void) {{ return {len(vs)}; }}
const void* qedregs_kernel_N{N}(int per_config, int variant) {{
  switch (variant) {{
{kernel_cases}
  }}
}}
void qedregs_config_N{N}(int variant, int* warps_per_block, int* points_per_warp, long long* smem_per_block,
                         long long* flops_per_point) {{
  static const int wpb[{len(vs)}] = {{{", ".join(str(v[0]) for v in vs)}}};
  *warps_per_block = wpb[variant];
  *points_per_warp = 16;
  *smem_per_block = (long long)wpb[variant] * 16 * qedregs_N{N}::T::STRIDE * 8;
  *flops_per_point = qedregs_N{N}::T::FLOPS_PER_POINT;
}}
}}
"""


def regs_variants(N: int) -> list[tuple[int, int, int]]:
    """Launch variants (warps per block, min resident blocks, L2 prefetch), QED_VARIANT selects."""
    # variant 0 = best of the r01 sweep (profiles/sweep_r01.jsonl)
    if N == 3:
        return [(4, 1, 1), (4, 1, 0), (2, 6, 1), (2, 6, 0), (2, 5, 1)]
    return [(2, 6, 1), (4, 1, 0), (4, 1, 1), (2, 8, 0), (2, 8, 1)]


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
