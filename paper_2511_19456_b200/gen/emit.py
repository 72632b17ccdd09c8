"""Emit the CUDA translation unit of one process size from its lowered Plan.

Build-time only.  Writes csrc/generated/qed_eval_N{N}.cu: the task tables of the
node-reduced trie (gen/lower.py), a traits struct T with the shared-memory layout
and the straight-line stage schedule (stored interior levels, then per photon
subset: recomputed deep levels, leaves), and the C entry points that the runtime
(csrc/qed_runtime.cu) uses to size and launch the kernel templates of
csrc/qed_eval_kernel.cuh and csrc/qed_mc_kernel.cuh.
"""
from __future__ import annotations

import os

from .lower import MMA_COL_POS, MMA_ROW_POS, Plan, hiho_table, lane_offset, make_plan

_LANE_BIT = {"L0": 0, "L1": 1, "L3": 3, "L4": 4}


def _mma_members(plan: Plan) -> str:
    """Traits members of a tensor-core-join plan: MMA, the accumulator bit exchange after each subset
    (lower.mma_assignments) and the configuration of each accumulator element in the final layout."""
    cases = []
    for si, (pa, pc) in enumerate(plan.mma_swaps):
        if pa in _LANE_BIT and pc in _LANE_BIT:
            call = f"qed::mma_swap_ll<{_LANE_BIT[pa]}, {_LANE_BIT[pc]}>(acc, lane)"
        elif pa in _LANE_BIT and pc == "TR":
            call = f"qed::mma_swap_lt<{_LANE_BIT[pa]}, true>(acc, lane)"
        elif pa == "TC" and pc in _LANE_BIT:
            call = f"qed::mma_swap_lt<{_LANE_BIT[pc]}, false>(acc, lane)"
        else:
            assert (pa, pc) == ("TC", "TR"), (pa, pc)
            call = "qed::mma_swap_tt(acc)"
        cases.append(f"      case {si}: {call}; break;")
    bit = {"L0": "(lane & 1)", "L1": "((lane >> 1) & 1)", "L3": "((lane >> 3) & 1)", "L4": "((lane >> 4) & 1)",
           "TR": "tr", "TC": "tc"}
    terms = [f"((unsigned){bit[pos]} << {1 + x})" for x, pos in sorted(plan.mma_assign[-1].items())]
    cfg = " | ".join(["(unsigned)r", f"((unsigned)((lane >> 2) & 1) << {plan.N + 1})"] + terms)
    return f"""  // tensor-core joins (gen/lower.py make_plan(mma=True)): subsets in Johnson order; after subset si the two
  // accumulator bits whose photons changed sides are exchanged; mma_config = the configuration of element
  // (lane, r, row tile, column tile) in the final layout
  static constexpr bool MMA = true;
  template <class ACC>
  static __device__ __forceinline__ void mma_swap(ACC& acc, int lane, int si) {{
    switch (si) {{
{chr(10).join(cases)}
      default: break;
    }}
  }}
  static __device__ __forceinline__ unsigned mma_config(int lane, int r, int tr, int tc) {{
    (void)tr; (void)tc;
    return {cfg};
  }}
"""

SMEM_PER_SM = 228 * 1024
SMEM_RESERVED_PER_BLOCK = 1024
SMEM_MAX_PER_BLOCK = 227 * 1024
MIN_REGS = 96


def choose_launch(plan: Plan) -> tuple[int, int]:
    """(warps per block, resident blocks per SM) maximising resident warps under the
    shared-memory limit, keeping >= MIN_REGS registers per thread."""
    best = (0, 1, 1)
    for wpb in (1, 2, 4, 8, 16):
        if wpb * 32 < plan.G or (wpb * 32) % plan.G:
            continue
        pb = wpb * 32 // plan.G
        blk = pb * plan.stride * 8 + 8 * 3 * wpb     # + MC block-reduction scratch
        if blk > SMEM_MAX_PER_BLOCK:
            break
        blocks = min(32, SMEM_PER_SM // (blk + SMEM_RESERVED_PER_BLOCK), 64 // wpb)
        blocks = min(blocks, 65536 // (MIN_REGS * wpb * 32))
        if blocks < 1:
            continue
        if blocks * wpb > best[0]:
            best = (blocks * wpb, wpb, blocks)
    return best[1], best[2]


def variants(plan: Plan) -> list[tuple[int, int, int, int]]:
    """Launch variants compiled into the library, selected at run time with QED_VARIANT:
    (warps per block, min resident blocks, accumulator split AS, L2 prefetch, sigma block SB).  Variant 0 is
    the default (chosen from measurements)."""
    wpb, mb = choose_launch(plan)
    mb4 = max(1, min(mb, 65536 // (152 * wpb * 32)))
    if plan.N >= 5:   # r01 sweep: 4 partial accumulators win for n >= 4
        vs = [(wpb, mb4, 4, 1), (wpb, mb, 2, 1), (wpb, mb, 2, 0)]
    else:
        vs = [(wpb, mb, 2, 1), (wpb, mb4, 4, 1), (wpb, mb, 2, 0)]
    vs = [v + (1,) for v in vs]
    if plan.n_sigma % 2 == 0:   # sigma blocked in the join (SB phi rows held across the tau loop)
        mb6 = max(1, min(mb, 65536 // (184 * wpb * 32)))
        sb = [(wpb, mb6, 4, 1, 2), (wpb, mb4, 2, 1, 2)]
        if plan.n_sigma % 3 == 0:
            sb.append((wpb, max(1, min(mb, 65536 // (216 * wpb * 32))), 4, 1, 3))
        # r22 sweep: SB = 2 wins at n = 4 (+6 %) and n = 5 (+5 %), loses at n = 3
        vs = sb + vs if plan.N >= 5 else vs + sb
    # DP = 1: leaf-stage descriptors one subset ahead; PF = 2: next point's momenta prefetched into registers
    vs = [v + (0,) for v in vs]
    vs += [vs[0][:3] + (2, vs[0][4], 1), vs[1][:3] + (2, vs[1][4], 1), vs[0][:3] + (1, vs[0][4], 1), vs[0][:3] + (2, vs[0][4], 0)]
    # (r29: holding the point-independent interior descriptors in registers for the whole kernel measured
    # 1-5 % slower at n = 3..5 and was dropped)
    # r28 sweep: register prefetch of the momenta +1.6 % at n = 3; with the descriptor prefetch +2 % at n = 4
    # r40: register prefetch of the momenta +0.7 % at n = 5
    promote = {4: len(vs) - 1, 5: len(vs) - 4, 6: len(vs) - 1}.get(plan.N)
    if promote is not None:
        vs = [vs[promote]] + vs[:promote] + vs[promote + 1:]
    if plan.N == 4:   # n = 3: sigma blocking at 16 warps/SM (128 registers); r37 sweep: +7 % -> the default
        # r40: + the descriptor prefetch (raw words) +1.4 % -> the default
        # (r43: AS = 4 at 12 warps measured -0.8 %)
        vs = [(wpb, min(mb, 4), 2, 2, 2, 1), (wpb, min(mb, 4), 2, 2, 2, 0)] + vs + [(wpb, min(mb, 4), 2, 2, 1, 0)]
    # (r33: prefetching the next tau's u-bar rows in the sigma-blocked join measured 5 % slower at n = 4: dropped)
    return vs


def _tasks(name, tasks):
    if not tasks:
        return f"__device__ const ushort4 {name}[1] = {{{{0, 0, 0, 0}}}};\n"
    body = ",\n  ".join(", ".join(f"{{{a}, {b}, {c}, {d}}}" for a, b, c, d in tasks[i:i + 6])
                        for i in range(0, len(tasks), 6))
    return f"__device__ const ushort4 {name}[{len(tasks)}] = {{\n  {body}}};\n"


KIND_FN = {"vs_col": "vs_col", "vs_row": "vs_row", "phi": "phi", "ub": "ub"}


def _chunk_members(tch: int, chunk_lines: list[str]) -> str:
    """Traits members of a tau-chunked tensor-core plan: TCH and the leaf chunks after the first."""
    if tch == 1:
        return ""
    body = "\n".join(chunk_lines)
    return f"""  // u-bar leaves built and joined in TCH chunks of tau orderings (make_plan(tau_chunks=...))
  static constexpr int TCH = {tch};
  static __device__ __forceinline__ void run_leaf_chunk(double* base, int g, int pb, int si, int ch) {{
    (void)pb;
    switch (ch) {{
{body}
      default: break;
    }}
  }}
"""


def emit_plan_namespace(plan: Plan, ns: str) -> str:
    """Task tables + traits struct T of one lowered plan, in namespace `ns`."""
    N, L = plan.N, plan.layout
    in_flat, out_flat, lines = [], [], []
    for lv in range(max(len(plan.in_levels), len(plan.out_levels))):
        if lv < len(plan.in_levels):
            t = plan.in_levels[lv]
            lines.append(f"    qed::run_tasks<T, {len(t)}>(base, g, k_in_tasks + {len(in_flat)}, qed::TaskFn<T, 0>{{}});")
            in_flat += t
        if lv < len(plan.out_levels):
            t = plan.out_levels[lv]
            off = lane_offset(len(plan.in_levels[lv]), plan.G) if lv < len(plan.in_levels) else 0
            lines.append(f"    qed::run_tasks<T, {len(t)}, qed::TaskFn<T, 1>, {off}>(base, g, k_out_tasks + {len(out_flat)}, "
                         "qed::TaskFn<T, 1>{});")
            out_flat += t
        lines.append("    qed::group_sync<T>(pb);")
    interiors = "\n".join(lines) if lines else "    (void)base; (void)g; (void)pb;"
    struct = [[(k, len(t)) for k, t in st] for st in plan.set_stages[0]]
    per_set = sum(c for st in struct for _, c in st)
    set_flat = []
    for stages in plan.set_stages:
        assert [[(k, len(t)) for k, t in st] for st in stages] == struct
        for st in stages:
            for _, t in st:
                set_flat += t
    lines, off = [], 0
    sd_fields, ld_lines, ex_lines = [], [], []
    tch = getattr(plan, "tau_chunks", 1)
    chunk_lines = []                 # tau-chunked tensor-core plans: the leaf chunks after the first
    n_main = len(struct) - (tch - 1)
    for i, st in enumerate(struct):
        if i >= n_main:
            c_lines = []
            for q, (kind, cnt) in enumerate(st):
                kid = {"vs_col": 0, "vs_row": 1, "phi": 2, "ub": 3}[kind]
                c_lines.append(f"qed::run_tasks<T, {cnt}, qed::TaskFn<T, {kid}>, 0>(base, g, "
                               f"k_set_tasks + si * {per_set} + {off}, qed::TaskFn<T, {kid}>{{}});")
                off += cnt
            chunk_lines.append(f"      case {i - n_main + 1}: " + " ".join(c_lines) + " break;")
            continue
        if i > 0:
            lines.append("    qed::group_sync<T>(pb);")
            ex_lines.append("    qed::group_sync<T>(pb);")
        prev = 0
        for q, (kind, cnt) in enumerate(st):
            lo = lane_offset(prev, plan.G) if q > 0 else 0
            kid = {"vs_col": 0, "vs_row": 1, "phi": 2, "ub": 3}[kind]
            lines.append(f"    qed::run_tasks<T, {cnt}, qed::TaskFn<T, {kid}>, {lo}>(base, g, "
                         f"k_set_tasks + si * {per_set} + {off}, qed::TaskFn<T, {kid}>{{}});")
            f = f"d{len(sd_fields)}"
            sd_fields.append(f"uint2 {f}[{(cnt + plan.G - 1) // plan.G}];")
            ld_lines.append(f"    qed::load_tasks<T, {cnt}, {lo}>(d.{f}, g, k_set_tasks + si * {per_set} + {off});")
            ex_lines.append(f"    qed::exec_tasks<T, {cnt}, qed::TaskFn<T, {kid}>, {lo}>(base, g, d.{f}, qed::TaskFn<T, {kid}>{{}});")
            off += cnt
            prev = cnt
    run_set = "\n".join(lines)
    sd_struct = " ".join(sd_fields)
    load_set = "\n".join(ld_lines)
    run_set_d = "\n".join(ex_lines)
    set_pos = [p for ps in plan.set_pos for p in ps]
    set_mask = [sum(1 << x for x in A) for A in plan.sets]
    hiho = hiho_table(plan)
    for tbl in (in_flat, out_flat, set_flat):
        for t in tbl:
            assert max(t) < 65536
    lay = ", ".join(f"{k} = {L[k]}" for k in ("MOM", "RED", "EPS", "MASK", "U", "UB", "PHI", "UBL"))
    return f"""namespace {ns} {{

{_tasks("k_in_tasks", in_flat)}{_tasks("k_out_tasks", out_flat)}{_tasks("k_set_tasks", set_flat)}
__device__ const unsigned char k_set_pos[{len(set_pos)}] = {{{", ".join(map(str, set_pos))}}};
__device__ const unsigned k_set_mask[{len(set_mask)}] = {{{", ".join(map(str, set_mask))}}};
// per (subset, lane): packed 2 swz(hi), 2 swz(hi + 1), 2 swz(ho), 2 swz(ho + 1) (leaf-row offsets of the lane's tile)
__device__ const unsigned k_hiho[{len(hiho)}] = {{{", ".join(f"0x{x:08x}u" for x in hiho)}}};

// interior levels <= {plan.store} stored per point, {plan.stride * 8} B shared memory per point
struct T {{
  static constexpr int N = {N}, J = {plan.j}, G = {plan.G};
  static constexpr int STRIDE = {plan.stride}, SP = {plan.sp};
  static constexpr int {lay};
  static constexpr int NSIG = {plan.n_sigma}, NTAU = {plan.n_tau}, NHI = {plan.n_hi}, NHO = {plan.n_ho};
  static constexpr int NSETS = {len(plan.sets)}, NSETS_REAL = NSETS, SETB = 1, LEAFB = 0;
  static constexpr int HS = 1, NAMP = 4;
  static constexpr long long FLOPS_PER_POINT = {plan.flops_per_point}LL;
{_mma_members(plan) if getattr(plan, "mma", False) else ""}{_chunk_members(tch, chunk_lines)}
  static __device__ __forceinline__ unsigned set_mask(int si) {{ return k_set_mask[si]; }}
  static __device__ __forceinline__ int set_pos(int si, int i) {{ return k_set_pos[si * N + i]; }}
  static __device__ __forceinline__ unsigned hiho(int si, int g) {{ return __ldg(k_hiho + si * G + g); }}
  static __device__ __forceinline__ void run_interiors(double* base, int g, int pb) {{
{interiors}
  }}
  static __device__ __forceinline__ void run_set(double* base, int g, int pb, int si) {{
{run_set}
  }}
  // the same leaf stage split in two: descriptors of subset si into registers (issued one subset ahead,
  // so their latency overlaps the previous subset's joins), then the tasks
  struct SD {{ {sd_struct} }};
  static __device__ __forceinline__ void load_set(SD& d, int g, int si) {{
{load_set}
  }}
  static __device__ __forceinline__ void run_set_d(double* base, int g, int pb, const SD& d) {{
{run_set_d}
  }}
}};

}}  // namespace {ns}
"""


# tensor-core-join variant promoted to variant 0 (index among the mma variants), where measured faster
# (profiles/sweep_r55_mma.jsonl: n = 3 +17 %, n = 4 +19 %, n = 5 +24 % over the CUDA-core join, with the
# descriptor prefetch)
# + (r60) the unrolled subset loop at n = 3
MMA_PROMOTE: dict[int, int] = {4: 3, 5: 0, 6: 0}


def plan_variants(N: int) -> list[Plan]:
    """Lowered plans compiled for one process size: the default, plus (n = 4) one that recomputes the
    second out-side trie level per subset (22 KB -> 15 KB of shared memory per point), plus (n = 3..5) the
    tensor-core-join plan (make_plan(mma=True))."""
    plans = [make_plan(N)]
    if N in (4, 5, 6):
        plans.append(make_plan(N, mma=True))
    # (r68: u-bar leaves built and joined in 2 or 3 chunks of tau orderings -- 12-16 % less shared memory per
    # point, 1-2 more resident points per SM -- measured 4-28 % slower at n = 4, 5: the extra leaf phases and
    # barriers cost more than the occupancy gains; make_plan(tau_chunks=...) is kept, not compiled)
    if N == 5:
        plans.append(make_plan(N, store=1))
        # (r56: tensor-core joins with less shared memory per point -- level 2 recomputed per subset, or the
        # 64-byte interior pitch at 2 warps per block -- measured 15-24 % slower than the default tensor-core plan)
        # (r65: the 64-byte pitch again at one warp per block, 9 resident points: -23 %, dropped)
        # (r38: the 64-byte spinor pitch, 22 KB per point and 10 resident points per SM, measured 11-16 % slower)
    return plans


def emit_source(plan: Plan, extra: list[Plan] | None = None) -> str:
    N = plan.N
    plans = [plan] + list(extra or [])
    nss = [f"qedgen_N{N}"] + [f"qedgen_N{N}_p{i}" for i in range(1, len(plans))]
    vs = []   # (plan index, wpb, min blocks, AS, PF)
    for pi, p in enumerate(plans):
        if getattr(p, "mma", False):   # tensor-core joins: no accumulator split / sigma blocking; +- descriptor prefetch
            wpb, mb = choose_launch(p)
            if p.G == 32 and wpb > 1:   # one point per block: the same residency in finer blocks
                mb, wpb = mb * wpb, 1
            if getattr(p, "tau_chunks", 1) > 1:   # leaf chunks between joins: no descriptor prefetch (whole subsets)
                vs += [(pi, wpb, mb, 2, 2, 1, 0), (pi, wpb, mb, 2, 2, 1, 0, 1)]
                continue
            vs += [(pi, wpb, mb, 2, 2, 1, 1), (pi, wpb, mb, 2, 2, 1, 0)]
            if N <= 5:   # unrolled subset loop (UR); r60: n = 3 +5.6 %, n = 4 +0.8 %, n = 5 -28 % (20 subsets: code size)
                vs += [(pi, wpb, mb, 2, 2, 1, 1, 1), (pi, wpb, mb, 2, 2, 1, 0, 1)]
        else:
            vs += [(pi,) + v for v in variants(p)]
    mma_v = [i for i, v in enumerate(vs) if getattr(plans[v[0]], "mma", False)]
    if N in MMA_PROMOTE and mma_v:
        k = mma_v[MMA_PROMOTE[N]]
        vs = [vs[k]] + vs[:k] + vs[k + 1:]
    mc_v = 0   # the fused MC kernel runs the eval default (tensor-core joins included; profiles/mc_sweep_r63.jsonl)
    fl = plan.flops
    flops_comment = "\n".join(f"//   {k:22s} {v:>10d}   (executed {plan.executed_flops[k]})" for k, v in fl.items())
    bodies = "\n".join(emit_plan_namespace(p, ns) for p, ns in zip(plans, nss))
    variant_structs = "".join(
        f"namespace {nss[v[0]]} {{ struct V{i} {{ static constexpr int WPB = {v[1]}, MIN_BLOCKS = {v[2]}, AS = {v[3]}, PF = {v[4]}, "
        f"SB = {v[5]}, DP = {v[6]}{f', UR = {v[7]}' if len(v) > 7 else ''}; }}; }}\n"
        for i, v in enumerate(vs))
    kernel_cases = "\n".join(
        f"    {'default' if i == 0 else f'case {i}'}: return per_config ? (const void*)qed::qed_eval_kernel<{nss[pi]}::T, {nss[pi]}::V{i}, true>\n"
        f"                                      : (const void*)qed::qed_eval_kernel<{nss[pi]}::T, {nss[pi]}::V{i}, false>;"
        for i, (pi, *_) in enumerate(vs))
    mc_cases = "\n".join(
        f"    {'default' if i == 0 else f'case {i}'}: return (const void*)qed::qed_mc_kernel<{nss[pi]}::T, {nss[pi]}::V{i}>;"
        for i, (pi, *_) in enumerate(vs))
    strides = ", ".join(str(plans[pi].stride) for pi, *_ in vs)
    flops = ", ".join(f"{plans[pi].flops_per_point}LL" for pi, *_ in vs)
    return f"""// GENERATED by paper_2511_19456_b200/gen/emit.py -- do not edit.
// Process size N = {N} photons (n = {N - 1}): {len(plan.sets)} photon subsets A (|A| = j = {plan.j}),
// {plan.n_sigma} x {plan.n_tau} diagrams per subset, {plan.H} spin/polarisation configurations,
// G = {plan.G} lanes per point; launch variants (plan, warps/block, min blocks/SM, acc split, prefetch):
// {vs}
// Algorithmic FP64 flops per point (node-reduced, helicity-shared DAG):
{flops_comment}
//   {'total':22s} {plan.flops_per_point:>10d}   (executed {sum(plan.executed_flops.values())})
#include "../qed_mc_kernel.cuh"

{bodies}
{variant_structs}
extern "C" {{
int qedgen_num_variants_N{N}(void) {{ return {len(vs)}; }}
int qedgen_mc_variant_N{N}(void) {{ return {mc_v}; }}
const void* qedgen_kernel_N{N}(int per_config, int variant) {{
  switch (variant) {{
{kernel_cases}
  }}
}}
const void* qedgen_mc_kernel_N{N}(int variant) {{
  switch (variant) {{
{mc_cases}
  }}
}}
void qedgen_config_N{N}(int variant, int* warps_per_block, int* points_per_warp, long long* smem_per_block,
                        long long* flops_per_point) {{
  static const int wpb[{len(vs)}] = {{{", ".join(str(v[1]) for v in vs)}}};
  static const int stride[{len(vs)}] = {{{strides}}};
  static const long long flops[{len(vs)}] = {{{flops}}};
  const int w = wpb[variant];
  *warps_per_block = w;
  *points_per_warp = 32 / {plan.G};   // 0 when a point spans several warps
  *smem_per_block = (long long)(w * 32 / {plan.G}) * stride[variant] * 8;
  *flops_per_point = flops[variant];  // algorithmic (identical for every plan of this size)
}}
}}
"""


def generate_all(out_dir: str, Ns=(2, 3, 4, 5, 6)) -> list[str]:
    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for N in Ns:
        plans = plan_variants(N)
        path = os.path.join(out_dir, f"qed_eval_N{N}.cu")
        src = emit_source(plans[0], plans[1:])
        if not os.path.exists(path) or open(path).read() != src:
            with open(path, "w") as f:
                f.write(src)
        paths.append(path)
    return paths


if __name__ == "__main__":
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in generate_all(os.path.join(here, "csrc", "generated")):
        print(p)
