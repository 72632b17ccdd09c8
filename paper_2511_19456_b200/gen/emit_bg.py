"""Emit the CUDA translation unit of the Berends-Giele variant of one process size (NEXT #1).

Build-time only.  Writes csrc/generated/qed_bg_N{N}.cu from gen/lower_bg.py: 8-ushort task tables
for the current levels and the per-subset leaves, a traits struct T (NSIG = NTAU = 1: one join per
photon subset), and entry points used by the runtime when a process is created with
QED_ALGO_BERENDS_GIELE.  The kernels are the templates of qed_eval_kernel.cuh / qed_mc_kernel.cuh.
"""
from __future__ import annotations

import os

from .emit import _mma_members, choose_launch, lane_offset
from .lower import hiho_table, hs_table
import math

from .lower_bg import BGPlan, group_strides, make_bg_plan


def _tbl(name, tasks, dw):
    rows = []
    for d in tasks:
        assert len(d) <= dw and max(d) < 65536
        rows.append(list(d) + [0] * (dw - len(d)))
    if not rows:
        return f"__device__ const qed::Desc<{dw}> {name}[1] = {{}};\n"
    packed = []
    for r in rows:
        w = [r[i] | (r[i + 1] << 16) for i in range(0, dw, 2)]
        quads = ["{" + ", ".join(f"0x{x:08x}u" for x in w[q:q + 4]) + "}" for q in range(0, len(w), 4)]
        packed.append("{{" + ", ".join(quads) + "}}")
    body = ",\n  ".join(", ".join(packed[i:i + 2]) for i in range(0, len(packed), 2))
    return f"__device__ const qed::Desc<{dw}> {name}[{len(rows)}] = {{\n  {body}}};\n"


def _fn(plan: BGPlan, K: int, F: int, kind: int) -> str:
    """Task functor of one stage: BGGroupFn with the plan's strides (doubles) for K, F."""
    so, sf, sr = group_strides(K, F, math.comb(plan.N, K), math.comb(plan.N, K - 1) if K > 1 else 0) if F else (0, 0, 0)
    return f"qed::BGGroupFn<T, {K}, {F}, {kind}, {so * plan.sp}, {sf * plan.sp}, {sr * plan.sp}>"


def emit_bg_ns(plan: BGPlan, ns: str, extra: bool = False) -> tuple[str, list]:
    """Namespace `ns` of one plan: tables, traits T, launch variants V*.  extra: a candidate plan beside the
    default one (two variants: PF = 2 with and without the descriptor prefetch)."""
    N, L = plan.N, plan.layout
    wpb, mb = choose_launch(plan)
    mb4 = max(1, min(mb, 65536 // (152 * wpb * 32)))
    # r06/r10 sweeps: AS = 4 first unless its register budget costs resident blocks (n >= 7)
    vs = [(wpb, mb4, 4, 1), (wpb, mb, 2, 1)] if mb4 == mb else [(wpb, mb, 2, 1), (wpb, mb4, 4, 1)]
    # PF = 2: the next point's momenta prefetched into registers (round 2)
    vs += [v[:3] + (2,) for v in vs]
    # r35 sweep: the prefetching copy of the old default is as fast or faster for n = 4..7 (+0.2..2 %);
    # at n = 3 the AS = 4 variant with it wins by 10 %
    d = {4: 3}.get(N, 2 if N <= 8 else 0)
    vs = [vs[d]] + vs[:d] + vs[d + 1:]
    lev_flat, lines = [], []
    prev_count, prev_k = 0, None
    for i, (kind, K, tasks, F) in enumerate(plan.levels):
        off = lane_offset(prev_count, plan.G) if (kind == "out" and prev_k == K) else 0
        kid = 0 if kind == "in" else 1
        fn = _fn(plan, K, F, kid)
        lines.append(f"    qed::run_tasks8<T, {len(tasks)}, {fn}, {off}>(base, g, k_levels + {len(lev_flat)}, {fn}{{}});")
        prev_count, prev_k = len(tasks), K
        lev_flat += tasks
        # a level depends on the previous level of the same side only: sync after each in/out pair
        nxt = plan.levels[i + 1] if i + 1 < len(plan.levels) else None
        if nxt is None or nxt[1] != K:
            lines.append("    qed::group_sync<T>(pb);")
    interiors = "\n".join(lines) if lines else "    (void)base; (void)g; (void)pb;"
    B = plan.setb
    n_in, n_out = B * len(plan.set_in[0]), B * len(plan.set_out[0])
    stage_struct = [[(kind, K, len(t), F) for kind, K, t, F in st] for st in plan.set_stages[0]]
    n_rec = sum(c for st in stage_struct for _, _, c, _ in st)
    set_flat = []
    for s0 in range(0, len(plan.sets), B):       # one batch: recomputed levels, all in-leaves, all out-leaves
        for lvl in range(len(stage_struct)):      # level by level, every subset of the batch
            for kk in range(len(stage_struct[lvl])):
                for q in range(B):
                    set_flat += plan.set_stages[s0 + q][lvl][kk][2]
        for q in range(B):
            set_flat += plan.set_in[s0 + q]
        for q in range(B):
            set_flat += plan.set_out[s0 + q]
    n_rec *= B
    per_set = n_rec + n_in + n_out
    rec_lines, off = [], 0
    sd_fields, ld_lines, ex_lines = [], [], []     # the same leaf stage split for descriptor prefetch (DP)

    def _sd(cnt, lo, off_, K, kid, F):
        f = f"d{len(sd_fields)}"
        fn = _fn(plan, K, F, kid)
        sd_fields.append(f"qed::Desc<DW> {f}[{(cnt + plan.G - 1) // plan.G}];")
        ld_lines.append(f"    qed::load_tasks8<T, {cnt}, {lo}>(d.{f}, g, k_sets + (si / {B}) * {per_set} + {off_});")
        ex_lines.append(f"    qed::exec_tasks8<T, {cnt}, {fn}, {lo}>(base, g, d.{f}, {fn}{{}});")

    for st in stage_struct:
        prev = 0
        st = [(kind, K, cnt * B, F) for kind, K, cnt, F in st]
        for q, (kind, K, cnt, F) in enumerate(st):
            lo = lane_offset(prev, plan.G) if q > 0 else 0
            kid = 0 if kind == "in" else 1
            fn = _fn(plan, K, F, kid)
            rec_lines.append(f"    qed::run_tasks8<T, {cnt}, {fn}, {lo}>(base, g, "
                             f"k_sets + (si / {B}) * {per_set} + {off}, {fn}{{}});")
            _sd(cnt, lo, off, K, kid, F)
            off += cnt
            prev = cnt
        rec_lines.append("    qed::group_sync<T>(pb);")
        ex_lines.append("    qed::group_sync<T>(pb);")
    rec_code = "\n".join(rec_lines) + ("\n" if rec_lines else "")
    lo = lane_offset(n_in, plan.G)
    _sd(n_in, 0, n_rec, plan.j, 2, plan.f_in)
    _sd(n_out, lo, n_rec + n_in, N - plan.j, 3, plan.f_out)
    trips = sum(((c + plan.G - 1) // plan.G) for c in [n_in, n_out] + [cnt * B for st in stage_struct for _, _, cnt, _ in st])
    if trips * plan.dw // 2 <= 24:   # descriptor prefetch variants where the prefetched words fit in a few registers
        vs += [vs[0][:4] + (1,), vs[1][:4] + (1,)]
    vs = [v if len(v) == 5 else v + (0,) for v in vs]
    # r39 sweep: the descriptor prefetch +4.5 % at n = 3 and +4.3 % at n = 6, -1 % at n = 4, 5
    if N in (4, 7):
        vs = [vs[4]] + vs[:4] + vs[5:]
    if extra:   # candidate plan: PF = 2, AS = 2, at the shared-memory occupancy and at <= 12 blocks (170
        # registers: the grouped tasks' 2^F accumulators are live beside the join's), + the descriptor prefetch
        w0, m0 = vs[0][0], max(v[1] for v in vs)
        m12 = max(1, min(m0, (12 * 32) // (w0 * 32) if w0 * 32 <= 384 else 1))
        vs = [(w0, m0, 2, 2, 0), (w0, m12, 2, 2, 0)] + ([(w0, m12, 2, 2, 1)] if any(v[4] for v in vs) else [])
    sd_struct = " ".join(sd_fields)
    load_set = "\n".join(ld_lines)
    run_set_d = "\n".join(ex_lines)
    fin = _fn(plan, plan.j, plan.f_in, 2)
    fout = _fn(plan, N - plan.j, plan.f_out, 3)
    run_set = rec_code + (f"    qed::run_tasks8<T, {n_in}, {fin}, 0>(base, g, k_sets + (si / {B}) * {per_set} + {n_rec}, {fin}{{}});\n"
                          f"    qed::run_tasks8<T, {n_out}, {fout}, {lo}>(base, g, k_sets + (si / {B}) * {per_set} + {n_rec + n_in}, "
                          f"{fout}{{}});")
    set_pos = [p for ps in plan.set_pos for p in ps]
    set_mask = [sum(1 << x for x in A) for A in plan.sets]
    hiho = hiho_table(plan)
    hst = hs_table(plan) if plan.hs == 2 else [0, 0]
    flops_comment = "\n".join(f"//   {k:22s} {v:>10d}" for k, v in plan.flops.items())
    lay = ", ".join(f"{k} = {L[k]}" for k in ("MOM", "RED", "EPS", "MASK", "U", "UB", "PHI", "UBL"))
    variant_structs = "".join(f"struct V{i} {{ static constexpr int WPB = {w}, MIN_BLOCKS = {m}, AS = {a}, PF = {p}, SB = 1, DP = {dp}; }};\n"
                              for i, (w, m, a, p, dp) in enumerate(vs))
    grp_note = f"node groups F = {plan.grp} (level 1, levels >= 2, in-leaf, out-leaf, recomputed)" if any(plan.grp) else "one node per task"
    code = f"""// ---- plan {ns}: G = {plan.G} lanes per point, {B} subsets per leaf stage, {plan.stride * 8} B shared memory per point,
// {grp_note}; current levels <= {plan.store} stored (deeper ones recomputed per subset: +{plan.recompute_flops} executed flops);
// variants {vs}.  FP64 flops per point:
{flops_comment}
//   {'total':22s} {plan.flops_per_point:>10d}
namespace {ns} {{

{_tbl("k_levels", lev_flat, plan.dw)}{_tbl("k_sets", set_flat, plan.dw)}
__device__ const unsigned char k_set_pos[{len(set_pos)}] = {{{", ".join(map(str, set_pos))}}};
__device__ const unsigned k_set_mask[{len(set_mask)}] = {{{", ".join(map(str, set_mask))}}};
// per (subset, lane): packed 2 swz(hi), 2 swz(hi + 1), 2 swz(ho), 2 swz(ho + 1) (leaf-row offsets of the lane's tile)
__device__ const unsigned k_hiho[{len(hiho)}] = {{{", ".join(f"0x{x:08x}u" for x in hiho)}}};
// two-half joins (hs = {plan.hs}): per (subset, lane of a half) phi / ubar offsets of the (s, s', lam_x) tile
__device__ const uint2 k_hs[{max(1, len(hst) // 2)}] = {{{", ".join(f"{{0x{hst[i]:08x}u, 0x{hst[i + 1]:08x}u}}" for i in range(0, len(hst), 2))}}};

struct T {{
  static constexpr int N = {N}, J = {plan.j}, G = {plan.G}, DW = {plan.dw};
  static constexpr int STRIDE = {plan.stride}, SP = {plan.sp};
  static constexpr int {lay};
  static constexpr int NSIG = 1, NTAU = 1, NHI = {plan.n_hi}, NHO = {plan.n_ho};
  static constexpr int NSETS = {len(plan.sets)}, NSETS_REAL = {plan.n_sets_real}, SETB = {B}, LEAFB = {L['LEAFB']};
  static constexpr int HS = {plan.hs}, NAMP = 4 * HS;   // join halves, amplitudes per lane
  static constexpr long long FLOPS_PER_POINT = {plan.flops_per_point}LL;
{_mma_members(plan) if getattr(plan, "mma", False) else ""}  static __device__ __forceinline__ unsigned set_mask(int si) {{ return k_set_mask[si]; }}
  static __device__ __forceinline__ int set_pos(int si, int i) {{ return k_set_pos[si * N + i]; }}
  static __device__ __forceinline__ unsigned hiho(int si, int g) {{ return __ldg(k_hiho + si * G + g); }}
  static __device__ __forceinline__ uint2 hs_offsets(int si, int gh) {{ return __ldg(k_hs + si * (G / 2) + gh); }}
  static __device__ __forceinline__ void run_interiors(double* base, int g, int pb) {{
{interiors}
  }}
  static __device__ __forceinline__ void run_set(double* base, int g, int pb, int si) {{
{run_set}
  }}
  // the same leaf stage split in two for DP = 1: descriptors of batch si into registers (issued one batch ahead,
  // during the previous batch's joins), then the tasks
  struct SD {{ {sd_struct} }};
  static __device__ __forceinline__ void load_set(SD& d, int g, int si) {{
{load_set}
  }}
  static __device__ __forceinline__ void run_set_d(double* base, int g, int pb, const SD& d) {{
{run_set_d}
  }}
}};
{variant_structs}
}}  // namespace {ns}
"""
    return code, [(ns, i, v, plan) for i, v in enumerate(vs)]


def emit_bg_source(plan: BGPlan, extras: tuple = ()) -> str:
    """The translation unit of one size: the default plan (variants 0..) and candidate plans `extras`
    (node-grouped, profiles/r03) appended as further launch variants."""
    N = plan.N
    code, allv = emit_bg_ns(plan, f"qedbg_N{N}")
    for i, p in enumerate(extras):
        c, v = emit_bg_ns(p, f"qedbg_N{N}_x{i + 1}", extra=True)
        code += c
        allv += v
    if N in PROMOTE and extras:      # a candidate variant measured faster than the default plan becomes variant 0
        ci, vi = PROMOTE[N]
        k = len(allv) - sum(len(emit_bg_ns(p, "x", extra=True)[1]) for p in extras[ci:]) + vi
        allv = [allv[k]] + allv[:k] + allv[k + 1:]
    kcases = "\n".join(
        f"    {'default' if i == 0 else f'case {i}'}: return per_config ? (const void*)qed::qed_eval_kernel<{ns}::T, {ns}::V{k}, true>\n"
        f"                                      : (const void*)qed::qed_eval_kernel<{ns}::T, {ns}::V{k}, false>;"
        for i, (ns, k, _, _) in enumerate(allv))
    n = len(allv)
    # the fused MC kernel runs the eval default too: with RAMBO batched per block (qed_mc_kernel.cuh) the promoted
    # n = 4 tensor-core plan is the fastest MC plan as well (profiles/mc_sweep_r63.jsonl: 1.54e8 vs 1.47e8 points/s)
    mcv = 0
    mcases = "\n".join(f"    {'default' if i == 0 else f'case {i}'}: return (const void*)qed::qed_mc_kernel<{ns}::T, {ns}::V{k}>;"
                       for i, (ns, k, _, p) in enumerate(allv))
    return f"""// GENERATED by paper_2511_19456_b200/gen/emit_bg.py -- do not edit.
// Berends-Giele (distributive rewrite of the node-reduced CDAG, NEXT #1) for N = {N} photons (n = {N - 1}):
// {plan.n_sets_real} photon subsets A (|A| = j = {plan.j}), one join each, {plan.H} configurations per point.
// {n} launch variants over {1 + len(extras)} plan(s); variant 0 is the default.
#include "../qed_mc_kernel.cuh"

{code}
extern "C" {{
int qedbg_num_variants_N{N}(void) {{ return {n}; }}
int qedbg_mc_variant_N{N}(void) {{ return {mcv}; }}
const void* qedbg_kernel_N{N}(int per_config, int variant) {{
  switch (variant) {{
{kcases}
  }}
}}
const void* qedbg_mc_kernel_N{N}(int variant) {{
  switch (variant) {{
{mcases}
  }}
}}
void qedbg_config_N{N}(int variant, int* warps_per_block, int* points_per_warp, long long* smem_per_block,
                       long long* flops_per_point) {{
  static const int wpb[{n}] = {{{", ".join(str(v[0]) for _, _, v, _ in allv)}}};
  static const int ppw[{n}] = {{{", ".join(str(32 // p.G if p.G <= 32 else 0) for _, _, _, p in allv)}}};
  static const long long stride[{n}] = {{{", ".join(str(p.stride) for _, _, _, p in allv)}}};
  static const long long flops[{n}] = {{{", ".join(str(p.flops_per_point) + "LL" for _, _, _, p in allv)}}};
  static const int G[{n}] = {{{", ".join(str(p.G) for _, _, _, p in allv)}}};
  const int w = wpb[variant];
  *warps_per_block = w;
  *points_per_warp = ppw[variant];
  *smem_per_block = (long long)(w * 32 / G[variant]) * stride[variant] * 8;
  *flops_per_point = flops[variant];
}}
}}
"""


# node-grouped candidate plans (profiles/r03), compiled beside the default as further launch variants and
# measured with QED_VARIANT (tools/sweep.sh): grp = F per stage kind (level 1, levels >= 2, in-leaf,
# out-leaf, recomputed), setb = subsets per leaf stage
# (profiles/sweep_r50, r51: every grouped candidate but the n = 5 one measured 20-45 % slower at n = 3, 4 --
# the wider tasks leave more lanes idle in each divergent in-/out-leaf phase, lower_bg.simt_utilisation);
# ungrouped candidates with the subset batch the SIMT model prefers (sweep r52)
CANDIDATES = {
    4: [dict(mma=True)],
    5: [dict(setb=4), dict(setb=3), dict(mma=True, setb=4)],
    6: [dict(grp=(1, 2, 1, 1, 1), setb=4), dict(setb=4), dict(setb=6)],
    7: [dict(setb=5, hs=1)],
}


# (candidate, its variant) promoted to variant 0 where the sweep measured it faster than the default plan
# (B200 at 1965 MHz): n = 5 SETB 4 at 12 blocks/SM +8.7 %, n = 6 SETB 5 with one-tile joins +7.2 %
# (profiles/sweep_r52_setb.jsonl); tensor-core joins (make_bg_plan(mma=True), profiles/sweep_r58_bg_mma.jsonl)
# n = 3 +4.9 %, n = 4 +3.8 % over the previous defaults -- at n = 5 the accumulator exchanges (one per subset,
# against only one (sigma, tau) join each) cost more than the joins save: -16 %, -9 % with the one-shuffle
# lane-tile exchange (r62), not kept; n = 7, 8 candidates
# (SETB 3, 4, one-tile joins) measured 2-26 % slower (profiles/sweep_r53_setb_n7n8.jsonl).
PROMOTE = {4: (0, 2), 5: (2, 2), 6: (1, 1), 7: (0, 0)}


def candidate_plans(N: int) -> list[dict]:
    return CANDIDATES.get(N, [])


def generate_bg(out_dir: str, Ns=(2, 3, 4, 5, 6, 7, 8, 9)) -> list[str]:
    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for N in Ns:
        path = os.path.join(out_dir, f"qed_bg_N{N}.cu")
        src = emit_bg_source(make_bg_plan(N), tuple(make_bg_plan(N, **kw) for kw in candidate_plans(N)))
        if not os.path.exists(path) or open(path).read() != src:
            with open(path, "w") as f:
                f.write(src)
        paths.append(path)
    return paths
