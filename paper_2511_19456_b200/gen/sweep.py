"""Node-reduction sweep: the B200 analogue of the paper's Fig. 9.

PAPER.md §3.4 lines 190-201 (Fig. 9): speedup of e- gamma^4 -> e- gamma (fixed spins and
polarisations) as node reductions (App. C) are applied one at a time, against the speedup
predicted from the FLOPs of the CDAG, on CPU and GPU; and line 200: with full inlining the compiler
"removes any duplicated instructions (i.e., essentially performs node reduction on instruction
level), which leads to the same device code produced, regardless of the optimization state".

This module emits, for one CDAG state (any partially reduced graph from gen/dag.py), a straight-line
device function with ONE statement per compute node -- the paper's code generation scheme
(App. D) -- wrapped in a thread-per-point kernel.  Every S1/S2 node computes its own
propagator (its denominator included), so an unreduced graph really recomputes shared subexpressions
unless the compiler deduplicates them.  tools/reduction_sweep.py builds several states, times them on
the GPU and compares with the FLOP prediction.  Build-time / experiment code, not the product path.
"""
from __future__ import annotations

import random

from .dag import CDAG, Process, build_unreduced

# flop model per node (FMA = 2): used for the Fig. 9 "theoretical speedup" curve
NODE_FLOPS = {"U_e": 10, "U_ph": 12, "V": 40, "S1": 20 + 56, "S2": 20 + 56 + 32}


def reduction_states(proc: Process, checkpoints: list[float], seed: int = 0) -> list[tuple[int, CDAG]]:
    """Apply node reductions one at a time in random order (the fixpoint does not
    depend on the order); return (number of reductions applied, graph copy) at the given fractions of
    the total number of reductions."""
    import copy
    g = build_unreduced(proc)
    # count the total number of single reductions first
    tmp = copy.deepcopy(g)
    rng = random.Random(seed)
    total = 0
    while True:
        groups = tmp.reducible_groups()
        if not groups:
            break
        grp = rng.choice(groups)
        for d in grp[1:]:
            tmp._merge(grp[0], d)
        total += 1
    marks = sorted({int(round(f * total)) for f in checkpoints})
    out = []
    rng = random.Random(seed)
    done = 0
    for m in marks:
        while done < m:
            groups = g.reducible_groups()
            grp = rng.choice(groups)
            for d in grp[1:]:
                g._merge(grp[0], d)
            done += 1
        out.append((done, copy.deepcopy(g)))
    return out


def _topo(g: CDAG) -> list[int]:
    indeg = {i: len(set(n.parents)) for i, n in g.nodes.items()}
    ready = sorted(i for i, d in indeg.items() if d == 0)
    order = []
    while ready:
        i = ready.pop(0)
        order.append(i)
        for c in sorted(g.nodes[i].children):
            indeg[c] -= 1
            if indeg[c] == 0:
                ready.append(c)
    return order


def emit_state(g: CDAG, proc: Process, name: str) -> tuple[str, int]:
    """Device function `name`(mom, n, pt, out_msq) for one CDAG state; returns (source, predicted flops)."""
    N = proc.N
    nodes = g.nodes
    info: dict[int, tuple] = {}     # data node -> (kind, side, absorbed set)
    L = [f"__device__ __forceinline__ double {name}(const double* __restrict__ mom, long long n, long long pt) {{"]
    w = L.append
    flops = 0
    var = {}
    for nid in _topo(g):
        nd = nodes[nid]
        if nd.kind == "data":
            if not nd.parents:                       # entry node: a particle momentum
                info[nid] = ("entry", nd.label)
                continue
            src = nd.parents[0]
            var[nid] = var[src]
            info[nid] = info[src]
            continue
        pars = nd.parents
        v = f"v{nid}"
        if nd.kind == "U":
            lab = info[pars[0]][1]
            if lab[0] == "e_in":
                w(f"  const qed::spinor {v} = qed::sweep_u(mom, n, pt);")
                info[nid] = ("spinor", "in", frozenset())
                flops += NODE_FLOPS["U_e"]
            elif lab[0] == "e_out":
                w(f"  const qed::spinor {v} = qed::sweep_ubar(mom, n, pt, {proc.n_in_ph + 1});")
                info[nid] = ("spinor", "out", frozenset())
                flops += NODE_FLOPS["U_e"]
            else:
                i = lab[1]
                part = 1 + i if i < proc.n_in_ph else proc.n_in_ph + 2 + (i - proc.n_in_ph)
                w(f"  double {v}[3]; qed::sweep_eps(mom, n, pt, {part}, {v});")
                info[nid] = ("photon", i)
                flops += NODE_FLOPS["U_ph"]
        elif nd.kind == "V":
            ph, fe = pars
            i = info[ph][1]
            _, side, ab = info[fe]
            fn = "eslash_col" if side == "in" else "eslash_row"
            w(f"  const qed::spinor {v} = qed::{fn}({var[ph]}, {var[fe]});")
            info[nid] = ("spinor", side, ab | {i})
            flops += NODE_FLOPS["V"]
        elif nd.kind == "S1":
            _, side, ab = info[pars[0]]
            mask = sum(1 << x for x in ab) if side == "in" else ((1 << N) - 1) & ~sum(1 << x for x in ab)
            fn = "prop_col" if side == "in" else "prop_row"
            w(f"  const qed::spinor {v} = qed::{fn}_m(mom, n, pt, {mask}, {var[pars[0]]});")
            info[nid] = ("spinor", side, ab)
            flops += NODE_FLOPS["S1"]
        elif nd.kind == "S2":
            a, b = pars
            ia, ib = info[a], info[b]
            if ia[1] != "in":
                a, b, ia, ib = b, a, ib, ia
            mask = sum(1 << x for x in ia[2])
            w(f"  const qed::c2 {v} = qed::sweep_join(mom, n, pt, {mask}, {var[a]}, {var[b]});")
            info[nid] = ("scalar",)
            flops += NODE_FLOPS["S2"]
        elif nd.kind == "Sum":
            terms = [var[p] for p in pars]
            w(f"  qed::c2 {v} = {terms[0]};")
            for t in terms[1:]:
                w(f"  {v}.r += {t}.r; {v}.i += {t}.i;")
            info[nid] = ("scalar",)
            flops += 2 * (len(terms) - 1)
        var[nid] = v
        var_out = v
    w(f"  return {var_out}.r * {var_out}.r + {var_out}.i * {var_out}.i;")
    w("}")
    return "\n".join(L) + "\n", flops


def emit_sweep_files(proc: Process, states: list[tuple[int, CDAG]], stem: str) -> tuple[dict[str, str], list[dict]]:
    """One translation unit per CDAG state (kernel k_state<k> + getter) and one with the timing entry
    point, so that the states compile in parallel; and per-state metadata.  Returns ({file: source}, meta)."""
    N, nin = proc.N, proc.n_in_ph
    files, meta = {}, []
    pre = _prelude(proc, len(states))
    for k, (done, g) in enumerate(states):
        src, fl = emit_state(g, proc, f"state{k}")
        meta.append({"state": k, "reductions": done, "nodes": len(g), "predicted_flops": fl})
        files[f"{stem}_s{k}.cu"] = (pre + src + f"""
__global__ void __launch_bounds__(128) k_state{k}(const double* __restrict__ mom, long long n, double* out, double norm) {{
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = norm * state{k}(mom, n, i);
}}
}}  // namespace qed

extern "C" const void* sweep_kernel_{k}(void) {{ return (const void*)qed::k_state{k}; }}
""")
    decl = "".join(f'extern "C" const void* sweep_kernel_{k}(void);\n' for k in range(len(states)))
    table = ", ".join(f"sweep_kernel_{k}()" for k in range(len(states)))
    files[f"{stem}_main.cu"] = f"""// GENERATED by paper_2511_19456_b200/gen/sweep.py -- timing entry point of the node-reduction sweep.
#include <cuda_runtime.h>
{decl}
extern "C" int sweep_num_states(void) {{ return {len(states)}; }}
// run state k over n points (momenta SoA on the device), reps timed launches; returns ms per launch
extern "C" int sweep_run(int k, const double* mom, long long n, double* out, double norm, int reps, float* ms) {{
  const void* kern[] = {{ {table} }};
  if (k < 0 || k >= {len(states)}) return 1;
  const int threads = 128;
  const unsigned blocks = (unsigned)((n + threads - 1) / threads);
  void* args[] = {{(void*)&mom, (void*)&n, (void*)&out, (void*)&norm}};
  cudaLaunchKernel(kern[k], dim3(blocks), dim3(threads), args, 0, 0);   // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cudaLaunchKernel(kern[k], dim3(blocks), dim3(threads), args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float t = 0; cudaEventElapsedTime(&t, e0, e1);
  *ms = t / reps;
  cudaEventDestroy(e0); cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}}
"""
    return files, meta


def _prelude(proc: Process, n_states: int) -> str:
    N, nin = proc.N, proc.n_in_ph
    return f"""// GENERATED by paper_2511_19456_b200/gen/sweep.py -- node-reduction sweep (PAPER.md Fig. 9 analogue).
// Process e- + {nin} gamma -> e- + {proc.n_out_ph} gamma, fixed spins/polarisations (all 0), one thread per
// point, one statement per CDAG compute node; {n_states} reduction states, one per translation unit.
#include <cuda_runtime.h>
#include "../qed_device.cuh"

namespace qed {{
constexpr int SW_N = {N}, SW_NIN = {nin};
// SWEEP_NOCSE: every momentum read is a volatile load, so the compiler cannot deduplicate identical node
// computations (the paper's "without always_inline" case, PAPER.md line 200); otherwise plain loads and
// full instruction-level CSE across nodes.
__device__ __forceinline__ double swm(const double* mom, long long n, long long pt, int j, int mu) {{
#ifdef SWEEP_NOCSE
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(mom + (long long)(4 * j + mu) * n + pt));
  return v;
#else
  return __ldg(mom + (long long)(4 * j + mu) * n + pt);
#endif
}}
__device__ __forceinline__ int sw_part(int i) {{ return i < SW_NIN ? 1 + i : SW_NIN + 2 + (i - SW_NIN); }}
__device__ __forceinline__ spinor sweep_u(const double* mom, long long n, long long pt) {{
  const double E = swm(mom, n, pt, 0, 0), r = rsqrt(E + 1.0), nn = (E + 1.0) * r;
  spinor u;
  u.v[0] = {{nn, 0}}; u.v[1] = {{0, 0}}; u.v[2] = {{swm(mom, n, pt, 0, 3) * r, 0}};
  u.v[3] = {{swm(mom, n, pt, 0, 1) * r, swm(mom, n, pt, 0, 2) * r}};
  return u;
}}
__device__ __forceinline__ spinor sweep_ubar(const double* mom, long long n, long long pt, int j) {{
  const double E = swm(mom, n, pt, j, 0), r = rsqrt(E + 1.0), nn = (E + 1.0) * r;
  spinor u;
  u.v[0] = {{nn, 0}}; u.v[1] = {{0, 0}}; u.v[2] = {{-swm(mom, n, pt, j, 3) * r, 0}};
  u.v[3] = {{-swm(mom, n, pt, j, 1) * r, swm(mom, n, pt, j, 2) * r}};
  return u;
}}
__device__ __forceinline__ void sweep_eps(const double* mom, long long n, long long pt, int j, double* e) {{
  double k[4] = {{swm(mom, n, pt, j, 0), swm(mom, n, pt, j, 1), swm(mom, n, pt, j, 2), swm(mom, n, pt, j, 3)}};
  double ct, st, cf, sf;
  eps_consts(k, ct, st, cf, sf);
  e[0] = ct * cf; e[1] = ct * sf; e[2] = -st;
}}
// propagator constants of subset `mask` computed inside the node (an unreduced graph recomputes them)
__device__ __forceinline__ void sweep_mask(const double* mom, long long n, long long pt, int mask, double* mk) {{
  double Q0 = swm(mom, n, pt, 0, 0), Q1 = swm(mom, n, pt, 0, 1), Q2 = swm(mom, n, pt, 0, 2), Q3 = swm(mom, n, pt, 0, 3);
#pragma unroll
  for (int i = 0; i < SW_N; ++i)
    if ((mask >> i) & 1) {{
      const double sg = i < SW_NIN ? 1.0 : -1.0;
      const int j = sw_part(i);
      Q0 += sg * swm(mom, n, pt, j, 0); Q1 += sg * swm(mom, n, pt, j, 1);
      Q2 += sg * swm(mom, n, pt, j, 2); Q3 += sg * swm(mom, n, pt, j, 3);
    }}
  const double inv = 1.0 / (Q0 * Q0 - Q1 * Q1 - Q2 * Q2 - Q3 * Q3 - 1.0);
  mk[0] = (Q0 + 1.0) * inv; mk[1] = (1.0 - Q0) * inv; mk[2] = Q1 * inv; mk[3] = Q2 * inv; mk[4] = Q3 * inv;
}}
__device__ __forceinline__ spinor prop_col_m(const double* mom, long long n, long long pt, int mask, const spinor& s) {{
  double mk[5]; sweep_mask(mom, n, pt, mask, mk); return prop_col(mk, s);
}}
__device__ __forceinline__ spinor prop_row_m(const double* mom, long long n, long long pt, int mask, const spinor& s) {{
  double mk[5]; sweep_mask(mom, n, pt, mask, mk); return prop_row(mk, s);
}}
// S2: propagate the in-side half with S(Q_A) and contract with the out-side half
__device__ __forceinline__ c2 sweep_join(const double* mom, long long n, long long pt, int mask, const spinor& in,
                                         const spinor& out) {{
  const spinor ph = prop_col_m(mom, n, pt, mask, in);
  c2 r = {{0, 0}};
#pragma unroll
  for (int c = 0; c < 4; ++c) {{
    r.r = fma(out.v[c].r, ph.v[c].r, fma(-out.v[c].i, ph.v[c].i, r.r));
    r.i = fma(out.v[c].r, ph.v[c].i, fma(out.v[c].i, ph.v[c].r, r.i));
  }}
  return r;
}}
"""
