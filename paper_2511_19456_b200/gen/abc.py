"""ABC-model code generation (second half; §1.3 line 56, App. F 521-531).

The ABC model has the diagram structure of QED Compton scattering (one A/C line, the N = n + 1 B-ons
attached in every order: N! diagrams) with scalar kernels: a vertex is the coupling g and a propagator
is 1/(Q^2 - m^2), the line species alternating C, A, C, ... along the line (App. F).  The paper
uses it to compare kernel weight between QED and a model with the same graph structure (line 530).

Two per-point straight-line bodies are emitted, as for QED:

* CDAG (the paper's method): the node-reduced two-sided trie of gen/lower.py with split j = N/2.
  In-side prefix nodes in(s_1..s_i) = in(s_1..s_{i-1}) r(S_i), out-side nodes from the outgoing A
  out(t_1..t_i) = out(t_1..t_{i-1}) r(all \\ {t_1..t_{i-1}}), one FMA per diagram at the joins
  M += in(sigma) out(tau) over every ordering sigma of A and tau of A^c, |A| = j.
* BG (the distributive rewrite): J(S) = r(S) sum_{i in S} J(S \\ i),
  M = sum_i J(all \\ i).

r(S) = 1 / (Q_S^2 - m_{X(|S|)}^2), Q_S = p_A + sum_{i in S} q_i, q = +k (incoming) / -k (outgoing),
X = C for odd |S|, A for even |S|.  Algorithmic flops count FMA = 2, add / mul / div = 1.
"""
from __future__ import annotations

import itertools
import math
import os

MASS_A, MASS_B, MASS_C = 1.0, 0.5, 1.2       # DESIGN.md reading A2 (include/abc.h)
SIZES_CDAG = (2, 4, 6)                         # N = n + 1 B-ons (even: tree diagrams exist only for odd n)
SIZES_BG = (2, 4, 6)                           # N = 8 would keep ~C(8,4) currents live: spills


def _name(S) -> str:
    return "".join(str(i) for i in S)


BATCH_INV_MIN_N = 6   # r54: N = 6 +43 % (CDAG) / +108 % (BG); N = 4 (HBM-bound) -5 % with it


def _subset_prelude(N, L):
    """Q_S and r(S) for every proper non-empty subset, by increasing size (Q_S = Q_{S minus max} + q_max).
    For N >= BATCH_INV_MIN_N the reciprocals of one size are taken together (Montgomery's batch inversion:
    prefix products, one division, two multiplications back per subset), so a subset costs 3
    multiplications and a Newton step (2 FMA) instead of an FP64 division (a reciprocal-estimate + Newton sequence, ~8 FP64 pipe
    operations); the chains of the N - 1 sizes are independent."""
    if N < BATCH_INV_MIN_N:
        return _subset_prelude_div(N, L)
    flops = 0
    for size in range(1, N):
        subs = list(itertools.combinations(range(N), size))
        for S in subs:
            prev = "pA" if size == 1 else f"Q{_name(S[:-1])}"
            b = S[-1]
            L.append(f"  double Q{_name(S)}[4];")
            L.append(f"  for (int mu = 0; mu < 4; ++mu) Q{_name(S)}[mu] = fma(sg[{b}], k[{b}][mu], {prev}[mu]);")
            m2 = "kMC2" if size % 2 else "kMA2"
            q = f"Q{_name(S)}"
            L.append(f"  const double d{_name(S)} = fma({q}[0], {q}[0], -fma({q}[1], {q}[1], "
                     f"fma({q}[2], {q}[2], fma({q}[3], {q}[3], {m2}))));")
            flops += 8 + 8          # 4 fma for Q, 4 fma for D
        # batch inversion of this size's denominators
        names = [_name(S) for S in subs]
        L.append(f"  const double pp{size}_0 = d{names[0]};")
        for i in range(1, len(names)):
            L.append(f"  const double pp{size}_{i} = pp{size}_{i - 1} * d{names[i]};")
        L.append(f"  double iv{size} = 1.0 / pp{size}_{len(names) - 1};")
        for i in range(len(names) - 1, 0, -1):
            L.append(f"  const double q{names[i]} = iv{size} * pp{size}_{i - 1};")
            L.append(f"  iv{size} *= d{names[i]};")
        L.append(f"  const double q{names[0]} = iv{size};")
        # one Newton step per reciprocal: the chain's error grows with its length (and the diagram sum can
        # cancel by 1e5, tests/test_abc_gpu.py full-size case); r = q + q (1 - d q) is back to ~1 ulp
        for nm in names:
            L.append(f"  const double r{nm} = fma(q{nm}, fma(-d{nm}, q{nm}, 1.0), q{nm});")
        flops += 3 * (len(names) - 1) + 1 + 4 * len(names)
    return flops


def _subset_prelude_div(N, L):
    """The same with one division per subset (HBM-bound sizes: the serial product chains cost more there)."""
    flops = 0
    for size in range(1, N):
        for S in itertools.combinations(range(N), size):
            prev = "pA" if size == 1 else f"Q{_name(S[:-1])}"
            b = S[-1]
            L.append(f"  double Q{_name(S)}[4];")
            L.append(f"  for (int mu = 0; mu < 4; ++mu) Q{_name(S)}[mu] = fma(sg[{b}], k[{b}][mu], {prev}[mu]);")
            m2 = "kMC2" if size % 2 else "kMA2"
            q = f"Q{_name(S)}"
            L.append(f"  const double r{_name(S)} = 1.0 / fma({q}[0], {q}[0], -fma({q}[1], {q}[1], "
                     f"fma({q}[2], {q}[2], fma({q}[3], {q}[3], {m2}))));")
            flops += 8 + 9          # 4 fma for Q, D: 3 fma + 1 fma-with-mass (8), division (1)
    return flops


def emit_cdag(N: int) -> tuple[str, int]:
    j = N // 2
    L = [f"__device__ __forceinline__ double abc_cdag_N{N}(const double (&pA)[4], const double (&k)[{N}][4], "
         f"const double (&sg)[{N}]) {{"]
    flops = _subset_prelude(N, L)
    full = tuple(range(N))
    # in-side trie: prefixes of length 1..j (leaves include r(A), the propagation half of S2)
    for i in range(1, j + 1):
        for sig in itertools.permutations(range(N), i):
            S = tuple(sorted(sig))
            if i == 1:
                L.append(f"  const double in{_name(sig)} = r{_name(S)};")
            else:
                L.append(f"  const double in{_name(sig)} = in{_name(sig[:-1])} * r{_name(S)};")
                flops += 1
    # out-side trie: prefixes from the outgoing A, length 1..N-j (leaf = product of N-j-1 propagators)
    for i in range(2, N - j + 1):
        for tau in itertools.permutations(range(N), i):
            rest = tuple(x for x in full if x not in tau[:-1])
            prev = f"ou{_name(tau[:-1])}" if i > 2 else None
            if prev is None:
                L.append(f"  const double ou{_name(tau)} = r{_name(rest)};")
            else:
                L.append(f"  const double ou{_name(tau)} = {prev} * r{_name(rest)};")
                flops += 1
    # joins: one per diagram, into NACC independent partial sums (a single accumulator makes the N! FMAs one
    # dependent chain: latency-bound at N = 6), summed pairwise at the end
    NACC = 4 if N >= 4 else 1
    L.append("  double " + ", ".join(f"M{a} = 0.0" for a in range(NACC)) + ";")
    d = 0
    for A in itertools.combinations(range(N), j):
        Ac = tuple(x for x in full if x not in A)
        for sig in itertools.permutations(A):
            for tau in itertools.permutations(Ac):
                a = d % NACC
                if N - j == 1:
                    L.append(f"  M{a} += in{_name(sig)};")
                    flops += 1
                else:
                    L.append(f"  M{a} = fma(in{_name(sig)}, ou{_name(tau)}, M{a});")
                    flops += 2
                d += 1
    if NACC == 4:
        L.append("  return (M0 + M1) + (M2 + M3);")
        flops += 3
    else:
        L.append("  return M0;")
    L.append("}")
    return "\n".join(L) + "\n", flops


def emit_bg(N: int) -> tuple[str, int]:
    L = [f"__device__ __forceinline__ double abc_bg_N{N}(const double (&pA)[4], const double (&k)[{N}][4], "
         f"const double (&sg)[{N}]) {{"]
    flops = _subset_prelude(N, L)
    for size in range(1, N):
        for S in itertools.combinations(range(N), size):
            if size == 1:
                L.append(f"  const double J{_name(S)} = r{_name(S)};")
                continue
            terms = [f"J{_name(tuple(x for x in S if x != i))}" for i in S]
            L.append(f"  const double J{_name(S)} = r{_name(S)} * ({' + '.join(terms)});")
            flops += size          # size - 1 adds + 1 mul
    full = tuple(range(N))
    terms = [f"J{_name(tuple(x for x in full if x != i))}" for i in full]
    L.append(f"  return {' + '.join(terms)};")
    flops += N - 1
    L.append("}")
    return "\n".join(L) + "\n", flops


def generate_abc(out_dir: str) -> list[str]:
    """csrc/generated/abc_N{N}.cu: the bodies, their kernels and their flop counts."""
    os.makedirs(out_dir, exist_ok=True)
    paths = []
    for N in SIZES_BG:
        parts, entries = [], []
        for alg, sizes, emit in (("cdag", SIZES_CDAG, emit_cdag), ("bg", SIZES_BG, emit_bg)):
            if N not in sizes:
                entries.append((alg, None, 0))
                continue
            src, fl = emit(N)
            parts.append(src)
            entries.append((alg, f"abc_{alg}_N{N}", fl))
        body = "".join(parts)
        getters = []
        for alg, fn, fl in entries:
            if fn is None:
                getters.append(f'extern "C" const void* abcgen_kernel_{alg}_N{N}(void) {{ return nullptr; }}\n'
                               f'extern "C" long long abcgen_flops_{alg}_N{N}(void) {{ return 0; }}\n')
            else:
                getters.append(
                    f"struct Body_{alg} {{\n"
                    f"  static __device__ __forceinline__ double amp(const double (&pA)[4], const double (&k)[{N}][4], "
                    f"const double (&sg)[{N}]) {{ return {fn}(pA, k, sg); }}\n}};\n"
                    f'extern "C" const void* abcgen_kernel_{alg}_N{N}(void) {{ '
                    f"return (const void*)qed::abc_kernel<{N}, Body_{alg}>; }}\n"
                    f'extern "C" long long abcgen_flops_{alg}_N{N}(void) {{ return {fl}; }}\n')
        src = (f"// GENERATED by paper_2511_19456_b200/gen/abc.py -- do not edit.\n"
               f"// ABC model (PAPER.md App. F), N = {N} B-ons ({math.factorial(N)} diagrams): straight-line per-point\n"
               f"// bodies (CDAG: node-reduced two-sided trie; BG: Berends-Giele currents).\n"
               f'#include "../abc_kernel.cuh"\n\nnamespace abcgen_N{N} {{\n'
               f"using qed::kMA2;\nusing qed::kMC2;\n{body}\n" + "".join(getters) + f"}}  // namespace abcgen_N{N}\n")
        # extern "C" inside a namespace keeps C linkage
        path = os.path.join(out_dir, f"abc_N{N}.cu")
        if not os.path.exists(path) or open(path).read() != src:
            with open(path, "w") as f:
                f.write(src)
        paths.append(path)
    return paths
