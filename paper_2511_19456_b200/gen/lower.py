"""Lower the node-reduced CDAG (two-sided prefix trie) of one process size to the
tables the sm_100a kernel executes.  Build-time only.

The fixpoint of node reduction (gen/dag.py, App. C) keeps one
V node per ordered photon prefix grown from each electron end, one S1 node per
interior prefix, one S2 (join) per diagram and one Sum.
The kernel evaluates exactly that DAG, with every node expanded over the spin /
polarisation states its subtree depends on (reuse "where the
same Feynman diagram must be evaluated repeatedly for many combinations of
inputs"):

  in-side  node  psi(sigma_1..sigma_i; s, lam_sigma)        2^(i+1) states
  out-side node  ubar(tau_1..tau_i; s', lam_tau)            2^(i+1) states
  leaf (i = j)   phi_sigma = S(Q_A) psi_sigma              (S2's "propagate one side")
  join           amp[h] += ubar_tau(h_out) . phi_sigma(h_in)  for every diagram
                 (sigma, tau), set(sigma) = A, set(tau) = complement of A.

Schedule (the static schedule of PAPER.md line 113, one device):
  stage 0  load momenta of one phase-space point into shared memory
  stage 1  external states (U): eps(k_i, lam), u(p, s), ubar(p', s'); and for
           every proper photon subset S the propagator constants of
           S(Q_S) = (Qslash_S + m)/(Q_S^2 - m^2), Q_S = p + sum_{i in S} q_i
  stage 2  interior trie levels (fused V+S1 tasks), in-side and out-side
  stage 3  for each subset A with |A| = j: its leaves (fused V+S tasks for phi,
           V tasks for ubar) then the joins of all j!(N-j)! diagrams of A for
           all 2^(N+2) configurations, accumulated in registers
  stage 4  |amp|^2, sum / average over configurations, one store per point.

A group of G lanes evaluates one point; lane l owns the 8 configurations with
free bits (s, lam_0, s') and fixed lam_i = bit (i-1) of l for photons i >= 1.
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

from .dag import balanced_split, perm_count

# flop model of the emitted device code (FMA = 2, add/mul = 1; gen/../csrc/qed_device.cuh)
FLOPS = {
    "V": 40,          # epsslash psi: 8 real outputs x (1 mul + 2 fma)
    "S": 56,          # (Qslash+m)/D psi with pre-scaled constants: 8 x (1 mul + 3 fma)
    "JOIN": 32,       # 4 complex multiply-accumulates
    "ABS2": 4,        # |amp|^2 accumulated: fma + fma
    "MASK": 20,       # Q_S (4 add), D (1 mul + 3 fma + 1 add), 1/D (1), 5 scaled constants (1 add + 5 mul ... )
    "EPS": 12,        # per photon: 2 sqrt, 3 div, products (counted as 1 each)
    "SPINOR": 10,     # per electron: sqrt, div, 4 products, both spins
}


@dataclass
class Plan:
    N: int
    j: int
    G: int
    tile: int
    sets: list[tuple[int, ...]]
    sigmas: list[list[tuple[int, ...]]]
    taus: list[list[tuple[int, ...]]]
    layout: dict[str, int]
    stride: int
    in_levels: list[list[tuple[int, int, int, int]]] = field(default_factory=list)
    out_levels: list[list[tuple[int, int, int, int]]] = field(default_factory=list)
    set_phi_tasks: list[list[tuple[int, int, int, int]]] = field(default_factory=list)
    set_ub_tasks: list[list[tuple[int, int, int, int]]] = field(default_factory=list)
    set_pos: list[list[int]] = field(default_factory=list)
    set_x_in: list[int] = field(default_factory=list)
    flops: dict[str, int] = field(default_factory=dict)

    @property
    def H(self) -> int:
        return 1 << (self.N + 2)

    @property
    def n_sigma(self) -> int:
        return math.factorial(self.j)

    @property
    def n_tau(self) -> int:
        return math.factorial(self.N - self.j)

    @property
    def n_hi(self) -> int:
        return 1 << (self.j + 1)

    @property
    def n_ho(self) -> int:
        return 1 << (self.N - self.j + 1)

    @property
    def flops_per_point(self) -> int:
        return sum(self.flops.values())


def _prefixes(N: int, i: int):
    return list(itertools.permutations(range(N), i))


def make_plan(N: int, j: int | None = None) -> Plan:
    if N < 2:
        raise ValueError("need at least two photons (n >= 1)")
    if j is None:
        j = balanced_split(N)
    assert 1 <= j <= N - 1
    G = 1 << (N - 1)
    tile = 8
    assert G * tile == 1 << (N + 2)

    # ---------------------------------------------------------------- shared-memory layout (doubles)
    lay: dict[str, int] = {}
    off = 0

    def alloc(name, size):
        nonlocal off
        lay[name] = off
        off += size
        off += off & 1          # keep 16-byte alignment

    alloc("MOM", 4 * (N + 2))
    alloc("EPS", N * 2 * 4)          # [photon][lam][e1,e2,e3,pad]
    alloc("U", 2 * 8)                # [s][4 complex]
    alloc("UB", 2 * 8)               # [s'][4 complex]
    alloc("MASK", (1 << N) * 6)      # [subset][Qp, Qm, qx, qy, qz, pad]
    in_nodes: list[dict[tuple, int]] = []
    for i in range(1, j):
        pre = _prefixes(N, i)
        alloc(f"IN{i}", len(pre) * (1 << (i + 1)) * 8)
        in_nodes.append({p: k for k, p in enumerate(pre)})
    out_nodes: list[dict[tuple, int]] = []
    for i in range(1, N - j):
        pre = _prefixes(N, i)
        alloc(f"OUT{i}", len(pre) * (1 << (i + 1)) * 8)
        out_nodes.append({p: k for k, p in enumerate(pre)})
    n_sigma, n_tau = math.factorial(j), math.factorial(N - j)
    n_hi, n_ho = 1 << (j + 1), 1 << (N - j + 1)
    alloc("PHI", n_sigma * n_hi * 8)
    alloc("UBL", n_tau * n_ho * 8)
    stride = off
    # spread consecutive points of a warp over the 32 banks (LDS.128 phases of 8 lanes)
    if stride % 16 == 0:
        stride += 4
    elif stride % 16 == 8:
        stride += 2
    lay["STRIDE"] = stride

    def eps_off(i, lam):
        return lay["EPS"] + (i * 2 + lam) * 4

    def mask_off(m):
        return lay["MASK"] + m * 6

    full = (1 << N) - 1

    def in_node_off(prefix, hidx):
        i = len(prefix)
        k = in_nodes[i - 1][prefix]
        return lay[f"IN{i}"] + (k * (1 << (i + 1)) + hidx) * 8

    def out_node_off(prefix, hidx):
        i = len(prefix)
        k = out_nodes[i - 1][prefix]
        return lay[f"OUT{i}"] + (k * (1 << (i + 1)) + hidx) * 8

    def mask_of(ph):
        m = 0
        for x in ph:
            m |= 1 << x
        return m

    plan = Plan(N=N, j=j, G=G, tile=tile, sets=[], sigmas=[], taus=[], layout=lay, stride=stride)

    # ---------------------------------------------------------------- interior trie levels (V+S1 fused)
    # in-side node (sigma_1..sigma_i), helicity index s | lam_{sigma_1} << 1 | ... (by position)
    for i in range(1, j):
        tasks = []
        for pre in _prefixes(N, i):
            for h in range(1 << (i + 1)):
                parent = lay["U"] + (h & 1) * 8 if i == 1 else in_node_off(pre[:-1], h & ((1 << i) - 1))
                lam = (h >> i) & 1
                tasks.append((parent, eps_off(pre[-1], lam), mask_off(mask_of(pre)), in_node_off(pre, h)))
        plan.in_levels.append(tasks)
    # out-side node (tau_1..tau_i) counted from the outgoing electron; propagator momentum
    # Q_{all \ set(tau)} (momentum of the line = p + photons still on the in-side)
    for i in range(1, N - j):
        tasks = []
        for pre in _prefixes(N, i):
            for h in range(1 << (i + 1)):
                parent = lay["UB"] + (h & 1) * 8 if i == 1 else out_node_off(pre[:-1], h & ((1 << i) - 1))
                lam = (h >> i) & 1
                tasks.append((parent, eps_off(pre[-1], lam), mask_off(full & ~mask_of(pre)), out_node_off(pre, h)))
        plan.out_levels.append(tasks)

    # ---------------------------------------------------------------- per-set leaves
    for A in itertools.combinations(range(N), j):
        Ac = tuple(x for x in range(N) if x not in A)
        sig = list(itertools.permutations(A))
        tau = list(itertools.permutations(Ac))
        plan.sets.append(A)
        plan.sigmas.append(sig)
        plan.taus.append(tau)
        pos = [0] * N
        for k, x in enumerate(A):
            pos[x] = 1 + k
        for k, x in enumerate(Ac):
            pos[x] = 1 + k
        plan.set_pos.append(pos)
        plan.set_x_in.append(1 if 0 in A else 0)
        # phi_sigma[hi], hi = s | lam_{A sorted} (bit 1 + sorted position)
        phi = []
        for si, sg in enumerate(sig):
            for hi in range(n_hi):
                lam = {x: (hi >> pos[x]) & 1 for x in A}
                hpar = (hi & 1) | sum(lam[sg[l]] << (l + 1) for l in range(j - 1))
                parent = lay["U"] + (hi & 1) * 8 if j == 1 else in_node_off(sg[:-1], hpar)
                phi.append((parent, eps_off(sg[-1], lam[sg[-1]]), mask_off(mask_of(A)),
                            lay["PHI"] + (si * n_hi + hi) * 8))
        ub = []
        for ti, tu in enumerate(tau):
            for ho in range(n_ho):
                lam = {x: (ho >> pos[x]) & 1 for x in Ac}
                L = N - j
                hpar = (ho & 1) | sum(lam[tu[l]] << (l + 1) for l in range(L - 1))
                parent = lay["UB"] + (ho & 1) * 8 if L == 1 else out_node_off(tu[:-1], hpar)
                ub.append((parent, eps_off(tu[-1], lam[tu[-1]]), 0, lay["UBL"] + (ti * n_ho + ho) * 8))
        plan.set_phi_tasks.append(phi)
        plan.set_ub_tasks.append(ub)

    # ---------------------------------------------------------------- algorithmic flops per point
    n_in_int = sum(len(t) for t in plan.in_levels)
    n_out_int = sum(len(t) for t in plan.out_levels)
    n_phi = sum(len(t) for t in plan.set_phi_tasks)
    n_ub = sum(len(t) for t in plan.set_ub_tasks)
    H = 1 << (N + 2)
    plan.flops = {
        "external": N * FLOPS["EPS"] + 2 * FLOPS["SPINOR"],
        "propagator_constants": ((1 << N) - 2) * FLOPS["MASK"],
        "trie_in": (n_in_int + n_phi) * (FLOPS["V"] + FLOPS["S"]),
        "trie_out": n_out_int * (FLOPS["V"] + FLOPS["S"]) + n_ub * FLOPS["V"],
        "join": math.factorial(N) * H * FLOPS["JOIN"],
        "msq": H * FLOPS["ABS2"],
    }
    return plan


def trie_node_counts(plan: Plan) -> dict[str, int]:
    """V / S1 / S2 node counts of the lowered trie before helicity expansion (must equal the
    node-reduction fixpoint of gen/dag.py)."""
    N, j = plan.N, plan.j
    V = sum(perm_count(N, i) for i in range(1, j + 1)) + sum(perm_count(N, i) for i in range(1, N - j + 1))
    S1 = sum(len(t) >> (i + 2) for i, t in enumerate(plan.in_levels)) + \
        sum(len(t) >> (i + 2) for i, t in enumerate(plan.out_levels))
    S2 = sum(len(s) * len(t) for s, t in zip(plan.sigmas, plan.taus))
    return {"V": V, "S1": S1, "S2": S2}
