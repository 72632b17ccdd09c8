"""Lower the node-reduced CDAG (two-sided prefix trie) of one process size to the
tables the sm_100a lane-group kernel executes.  Build-time only.

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

Static schedule (one device), one group of G = 2^N lanes per point:
  stage 0  momenta of the point -> shared memory
  stage 1  external states (U) and, for every proper photon subset S, the constants of
           S(Q_S) = (Qslash_S + m)/(Q_S^2 - m^2), Q_S = p + sum_{i in S} q_i
  stage 2  stored interior trie levels (fused V+S1 tasks), in-side and out-side
  stage 3  for each subset A with |A| = j: the interior levels deeper than `store`
           restricted to the prefixes inside A / its complement (recomputed per subset to
           keep shared memory small), the leaves (V+S tasks for phi, V tasks for ubar),
           then the joins of its j!(N-j)! diagrams, accumulated in registers
  stage 4  |amp|^2, sum / average over configurations, one store per point.

Lane g owns the 4 configurations (s, s') x fixed (lam_0..lam_{N-1}) = bits of g.

Shared-memory spinor layouts (bank-conflict free for the access patterns):
  interior / external spinors: 4 complex components contiguous, pitch SP = 10 doubles (80 B: consecutive
      spinors written by consecutive lanes fall in distinct bank slots, no address arithmetic);
  leaves: component-major rows  [sigma][c][hi'] / [tau][c][ho'], hi' = swz(hi) (see swz()).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

from .dag import balanced_split, perm_count

# flop model of the emitted device code (FMA = 2, add/mul = 1; csrc/qed_device.cuh)
FLOPS = {
    "V": 40,          # epsslash psi: 8 real outputs x (1 mul + 2 fma)
    "V_T": 24,        # the same for the transverse eps(k, 2) (eps^3 = 0): 8 x (1 mul + 1 fma); regs kernels
    "S": 56,          # (Qslash+m)/D psi with pre-scaled constants: 8 x (1 mul + 3 fma)
    "JOIN": 32,       # 4 complex multiply-accumulates
    "ABS2": 4,        # |amp|^2 accumulated: fma + fma
    "MASK": 20,       # Q_S (4 add), D (1 mul + 3 fma + 1 add), 1/D (1), 5 scaled constants
    "EPS": 12,        # per photon: 2 sqrt, 3 div, products (counted as 1 each)
    "SPINOR": 10,     # per electron: sqrt, div, 4 products, both spins
}


def swz(h: int) -> int:
    """Leaf-row position of helicity index h: rotate each aligned group of 8 by h >> 3."""
    return (h & ~7) | ((h + (h >> 3)) & 7)


SP = 10   # default spinor pitch (doubles) for plans that do not choose one


def aos_slot(off: int, c: int, sp: int = SP) -> int:
    """Double offset of component c of the interior spinor starting at `off`.
    sp = 10: components contiguous, 80-byte pitch (8 consecutive spinors hit 8 distinct 16-byte bank slots,
    no address arithmetic); sp = 8: 64-byte pitch, component c at slot c ^ ((off >> 4) & 3) (same bank
    property, 20 % less shared memory, 4 integer ops per component)."""
    if sp == 8:
        assert off % 8 == 0
        return off + 2 * (c ^ ((off >> 4) & 3))
    assert off % 2 == 0
    return off + 2 * c


# measured per process size (profiles/sweep_r12.jsonl vs r10/r11): the 80-byte pitch wins where the kernel
# is issue-bound, the 64-byte pitch where shared memory limits occupancy
PITCH_CDAG = {2: 8, 3: 8, 4: 8, 5: 10, 6: 8}
PITCH_BG = {2: 8, 3: 8, 4: 10, 5: 8, 6: 8, 7: 8, 8: 10, 9: 10}


@dataclass
class Plan:
    N: int
    j: int
    G: int
    store: int                      # interior levels <= store are stored once per point
    sets: list[tuple[int, ...]]
    sigmas: list[list[tuple[int, ...]]]
    taus: list[list[tuple[int, ...]]]
    layout: dict[str, int]
    stride: int
    in_levels: list[list[tuple[int, int, int, int]]] = field(default_factory=list)
    out_levels: list[list[tuple[int, int, int, int]]] = field(default_factory=list)
    # per set: list of stages; each stage = (kind, tasks); kinds: "vs_col", "vs_row", "phi", "ub"
    set_stages: list[list[list[tuple[str, list]]]] = field(default_factory=list)
    set_pos: list[list[int]] = field(default_factory=list)
    flops: dict[str, int] = field(default_factory=dict)
    executed_flops: dict[str, int] = field(default_factory=dict)

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


def _prefixes_in(elems, i: int):
    return list(itertools.permutations(elems, i))


def default_store(N: int, j: int) -> int:
    """Interior levels stored per point; deeper ones are recomputed per subset when storing them
    would exceed ~26 KB of shared memory per point (n = 5: level 2, 30 KB -> 2 x 3 KB per subset)."""
    return 1 if N >= 6 else max(j, N - j)


def johnson_order(N: int, j: int) -> list[tuple[int, ...]]:
    """The j-subsets of range(N) in an order where consecutive subsets differ by exchanging one element
    (a Hamiltonian path of the Johnson graph, found by depth-first search; it exists for every N, j)."""
    subs = list(itertools.combinations(range(N), j))
    n = len(subs)
    adj = {a: [b for b in subs if len(set(a) & set(b)) == j - 1] for a in subs}
    path, seen = [subs[0]], {subs[0]}

    def dfs():
        if len(path) == n:
            return True
        for b in adj[path[-1]]:
            if b not in seen:
                seen.add(b)
                path.append(b)
                if dfs():
                    return True
                path.pop()
                seen.discard(b)
        return False
    assert dfs()
    return path


# tensor-core join (DMMA m8n8k4 f64) physical positions of the photons' polarisation bits in the accumulator
# layout: the in-set A's photons take the column positions, the complement's the row positions
MMA_COL_POS = ("L0", "L1", "TC")      # lane bit 0, lane bit 1, column-tile index
MMA_ROW_POS = ("L3", "L4", "TR")      # lane bit 3, lane bit 4, row-tile index


def mma_assignments(N: int, j: int, order: list[tuple[int, ...]]):
    """Photon -> physical position for every subset of `order`, and the position pair exchanged at each
    transition.  The first subset assigns sorted photons to positions in order; at a transition the photon
    entering A takes the position of the photon leaving it and vice versa, so the accumulators of every
    configuration move by one exchange of two physical bits (qed_eval_kernel.cuh mma_swap)."""
    assert j <= len(MMA_COL_POS) and N - j <= len(MMA_ROW_POS)
    A0 = order[0]
    Ac0 = tuple(x for x in range(N) if x not in A0)
    cur = {x: MMA_COL_POS[k] for k, x in enumerate(A0)}
    cur.update({x: MMA_ROW_POS[k] for k, x in enumerate(Ac0)})
    assigns, swaps = [dict(cur)], []
    for a, b in zip(order, order[1:]):
        (out_,), (in_,) = set(a) - set(b), set(b) - set(a)
        pa, pc = cur[out_], cur[in_]
        cur[out_], cur[in_] = pc, pa
        assigns.append(dict(cur))
        swaps.append((pa, pc))
    return assigns, swaps


def make_plan(N: int, j: int | None = None, store: int | None = None, sp: int | None = None,
              mma: bool = False, tau_chunks: int = 1) -> Plan:
    if N < 2:
        raise ValueError("need at least two photons (n >= 1)")
    if j is None:
        j = balanced_split(N)
    assert 1 <= j <= N - 1
    if store is None:
        store = default_store(N, j)
    G = 1 << N
    full = (1 << N) - 1
    SP = sp if sp is not None else PITCH_CDAG.get(N, 10)

    lay: dict[str, int] = {}
    off = 0

    def alloc(name, size, align=2):
        nonlocal off
        off = (off + align - 1) // align * align
        lay[name] = off
        off += size

    alloc("MOM", 4 * (N + 2))
    alloc("RED", max(2, G // 32))    # cross-warp reduction scratch (groups of > 32 lanes)
    alloc("EPS", N * 2 * 4)          # [photon][lam][e1, e2, e3, pad]
    alloc("MASK", (1 << N) * 6)      # [subset][Qp, Qm, qx, qy, qz, pad]
    alloc("U", 2 * SP, 8)             # [s] spinor (AoS, swizzled)
    alloc("UB", 2 * SP, 8)            # [s'] spinor
    in_nodes: dict[int, dict[tuple, int]] = {}
    out_nodes: dict[int, dict[tuple, int]] = {}
    for i in range(1, min(j, store + 1)):
        pre = _prefixes_in(range(N), i)
        alloc(f"IN{i}", len(pre) * (1 << (i + 1)) * SP, 8)
        in_nodes[i] = {p: k for k, p in enumerate(pre)}
    for i in range(1, min(N - j, store + 1)):
        pre = _prefixes_in(range(N), i)
        alloc(f"OUT{i}", len(pre) * (1 << (i + 1)) * SP, 8)
        out_nodes[i] = {p: k for k, p in enumerate(pre)}
    # per-set recomputed interior levels: prefixes of length i inside a set of size j / N-j
    set_in_nodes: dict[int, dict[tuple, int]] = {}
    set_out_nodes: dict[int, dict[tuple, int]] = {}
    for i in range(store + 1, j):
        alloc(f"SIN{i}", perm_count(j, i) * (1 << (i + 1)) * SP, 8)
    for i in range(store + 1, N - j):
        alloc(f"SOUT{i}", perm_count(N - j, i) * (1 << (i + 1)) * SP, 8)
    n_sigma, n_tau = math.factorial(j), math.factorial(N - j)
    n_hi, n_ho = 1 << (j + 1), 1 << (N - j + 1)
    assert tau_chunks == 1 or (mma and n_tau % tau_chunks == 0)
    assert not mma or (n_hi >= 8 and n_ho >= 8), "tensor-core tiles are 8 x 8: both sides need >= 2 photons"
    if mma:   # AoS leaves (64-byte pitch, XOR component swizzle): spinor (row, slot) at row * NH + slot; with
        # tau_chunks > 1 the u-bar leaves of one chunk of tau orderings at a time (joined chunk by chunk)
        alloc("PHI", n_sigma * n_hi * 8, 8)
        alloc("UBL", n_tau // tau_chunks * n_ho * 8, 8)
    else:
        alloc("PHI", n_sigma * 4 * n_hi * 2, 8)
        alloc("UBL", n_tau * 4 * n_ho * 2, 8)
    stride = off
    # odd number of 16-byte slots per point: consecutive points of a warp start in different banks
    stride = (stride + 1) // 2 * 2
    if (stride // 2) % 2 == 0:
        stride += 2
    lay["STRIDE"] = stride

    def eps_off(i, lam):
        return lay["EPS"] + (i * 2 + lam) * 4

    def mask_off(m):
        return lay["MASK"] + m * 6

    def mask_of(ph):
        m = 0
        for x in ph:
            m |= 1 << x
        return m

    plan = Plan(N=N, j=j, G=G, store=store, sets=[], sigmas=[], taus=[], layout=lay, stride=stride)
    plan.sp = SP
    plan.mma = mma
    plan.tau_chunks = tau_chunks
    order = johnson_order(N, j) if mma else list(itertools.combinations(range(N), j))
    if mma:
        plan.mma_assign, plan.mma_swaps = mma_assignments(N, j, order)

    def mma_slot(assign, side_photons, h, prim):
        """Accumulator-layout index of leaf helicity h (bit 0 = s / s', bit 1 + k = lam of the k-th sorted
        photon of the side): bit 0 <- the spin, bit 1 <- the photon at L0 / L3, bit 2 <- L1 / L4, bit 3 <- the
        tile index TC / TR."""
        slot = h & 1
        for k, x in enumerate(side_photons):
            lam = (h >> (1 + k)) & 1
            p_ = assign[x]
            bit = {prim[0]: 1, prim[1]: 2, prim[2]: 3}[p_]
            slot |= lam << bit
        return slot

    # ---------------------------------------------------------------- stored interior levels (V+S1 fused)
    def in_off(prefix, h, set_local=None):
        i = len(prefix)
        if i in in_nodes:
            return lay[f"IN{i}"] + (in_nodes[i][prefix] * (1 << (i + 1)) + h) * SP
        return lay[f"SIN{i}"] + (set_local[prefix] * (1 << (i + 1)) + h) * SP

    def out_off(prefix, h, set_local=None):
        i = len(prefix)
        if i in out_nodes:
            return lay[f"OUT{i}"] + (out_nodes[i][prefix] * (1 << (i + 1)) + h) * SP
        return lay[f"SOUT{i}"] + (set_local[prefix] * (1 << (i + 1)) + h) * SP

    def in_task(pre, h, local=None):
        i = len(pre)
        parent = lay["U"] + (h & 1) * SP if i == 1 else in_off(pre[:-1], h & ((1 << i) - 1), local)
        return (parent, eps_off(pre[-1], (h >> i) & 1), mask_off(mask_of(pre)), in_off(pre, h, local))

    def out_task(pre, h, local=None):
        i = len(pre)
        parent = lay["UB"] + (h & 1) * SP if i == 1 else out_off(pre[:-1], h & ((1 << i) - 1), local)
        return (parent, eps_off(pre[-1], (h >> i) & 1), mask_off(full & ~mask_of(pre)), out_off(pre, h, local))

    for i in sorted(in_nodes):
        plan.in_levels.append([in_task(pre, h) for pre in _prefixes_in(range(N), i) for h in range(1 << (i + 1))])
    for i in sorted(out_nodes):
        plan.out_levels.append([out_task(pre, h) for pre in _prefixes_in(range(N), i) for h in range(1 << (i + 1))])

    # ---------------------------------------------------------------- per-set stages
    n_set_in_int = n_set_out_int = 0
    for si_, A in enumerate(order):
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
        stages: list[list[tuple[str, list]]] = []
        local_in: dict[tuple, int] = {}
        local_out: dict[tuple, int] = {}
        for i in range(store + 1, max(j, N - j)):
            st = []
            if i < j:
                pres = _prefixes_in(A, i)
                for k, p in enumerate(pres):
                    local_in[p] = k
                st.append(("vs_col", [in_task(p, h, local_in) for p in pres for h in range(1 << (i + 1))]))
                n_set_in_int += len(st[-1][1])
            if i < N - j:
                pres = _prefixes_in(Ac, i)
                for k, p in enumerate(pres):
                    local_out[p] = k
                st.append(("vs_row", [out_task(p, h, local_out) for p in pres for h in range(1 << (i + 1))]))
                n_set_out_int += len(st[-1][1])
            stages.append(st)
        # leaves: phi_sigma[hi], hi = s | lam_{A sorted} << (1 + position); write index = sigma * n_hi + hi
        phi = []
        for si, sg in enumerate(sig):
            for hi in range(n_hi):
                lam = {x: (hi >> pos[x]) & 1 for x in A}
                hpar = (hi & 1) | sum(lam[sg[l]] << (l + 1) for l in range(j - 1))
                parent = lay["U"] + (hi & 1) * SP if j == 1 else in_off(sg[:-1], hpar, local_in)
                if mma:
                    sl = mma_slot(plan.mma_assign[si_], A, hi, MMA_COL_POS)
                    dst = lay["PHI"] + (si * n_hi + sl) * 8
                else:
                    dst = leaf_off(lay["PHI"], n_hi, si, hi)
                phi.append((parent, eps_off(sg[-1], lam[sg[-1]]), mask_off(mask_of(A)), dst))
        ub = []
        L = N - j
        for ti, tu in enumerate(tau):
            for ho in range(n_ho):
                lam = {x: (ho >> pos[x]) & 1 for x in Ac}
                hpar = (ho & 1) | sum(lam[tu[l]] << (l + 1) for l in range(L - 1))
                parent = lay["UB"] + (ho & 1) * SP if L == 1 else out_off(tu[:-1], hpar, local_out)
                if mma:
                    sl = mma_slot(plan.mma_assign[si_], Ac, ho, MMA_ROW_POS)
                    dst = lay["UBL"] + ((ti % (n_tau // tau_chunks)) * n_ho + sl) * 8
                else:
                    dst = leaf_off(lay["UBL"], n_ho, ti, ho)
                ub.append((parent, eps_off(tu[-1], lam[tu[-1]]), 0, dst))
        if mma:   # consecutive lanes store consecutive AoS spinors (conflict-free with the XOR swizzle)
            phi.sort(key=lambda t: t[3])
            per = len(ub) // tau_chunks          # ub was built tau-major: chunk c = taus c * per / n_ho ..
            chunks = [sorted(ub[c * per:(c + 1) * per], key=lambda t: t[3]) for c in range(tau_chunks)]
            stages.append([("phi", phi), ("ub", chunks[0])])
            for c in range(1, tau_chunks):       # leaf chunk stages: each follows the joins of the previous chunk
                stages.append([("ub", chunks[c])])
        else:
            stages.append([("phi", phi), ("ub", ub)])
        plan.set_stages.append(stages)

    # ---------------------------------------------------------------- algorithmic flops per point
    # (the node-reduced DAG: every distinct trie node once, whether stored or recomputed)
    def trie_count(levels):
        return sum(perm_count(N, i) * (1 << (i + 1)) for i in levels)

    n_in_int = trie_count(range(1, j))
    n_out_int = trie_count(range(1, N - j))
    n_phi = perm_count(N, j) * n_hi
    n_ub = perm_count(N, N - j) * n_ho
    H = 1 << (N + 2)
    plan.flops = {
        "external": N * FLOPS["EPS"] + 2 * FLOPS["SPINOR"],
        "propagator_constants": ((1 << N) - 2) * FLOPS["MASK"],
        "trie_in": (n_in_int + n_phi) * (FLOPS["V"] + FLOPS["S"]),
        "trie_out": n_out_int * (FLOPS["V"] + FLOPS["S"]) + n_ub * FLOPS["V"],
        "join": math.factorial(N) * H * FLOPS["JOIN"],
        "msq": H * FLOPS["ABS2"],
    }
    # executed (includes the per-set recomputation of deep interior levels)
    n_in_exec = sum(len(t) for t in plan.in_levels) + n_set_in_int
    n_out_exec = sum(len(t) for t in plan.out_levels) + n_set_out_int
    plan.executed_flops = dict(plan.flops)
    plan.executed_flops["trie_in"] = (n_in_exec + n_phi) * (FLOPS["V"] + FLOPS["S"])
    plan.executed_flops["trie_out"] = n_out_exec * (FLOPS["V"] + FLOPS["S"]) + n_ub * FLOPS["V"]
    return plan


def trie_node_counts(plan: Plan) -> dict[str, int]:
    """V / S1 / S2 node counts of the lowered trie before helicity expansion (must equal the
    node-reduction fixpoint of gen/dag.py)."""
    N, j = plan.N, plan.j
    V = sum(perm_count(N, i) for i in range(1, j + 1)) + sum(perm_count(N, i) for i in range(1, N - j + 1))
    S1 = sum(perm_count(N, i) for i in range(1, j)) + sum(perm_count(N, i) for i in range(1, N - j))
    S2 = sum(len(s) * len(t) for s, t in zip(plan.sigmas, plan.taus))
    return {"V": V, "S1": S1, "S2": S2}


def lane_offset(count_first: int, G: int) -> int:
    """Start lane of the second task kind of a stage: right after the first kind's last lane,
    rounded up to a warp boundary when the group spans several warps (no intra-warp divergence)."""
    off = count_first % G
    if G > 32 and off:
        off = ((off + 31) // 32 * 32) % G
    return off


def leaf_off(region: int, nh: int, row: int, h: int) -> int:
    """Offset (doubles) of component 0 of leaf spinor (row, h) in a component-major leaf region of nh
    helicity columns; component c sits c * 2 nh further.  Leaf descriptors carry this directly."""
    off = region + row * 4 * nh * 2 + 2 * swz(h)
    assert off < 65536
    return off


def hiho_table(plan) -> list[int]:
    """Per (subset si, lane g): the lane's leaf-row offsets for the join, packed in one word:
    2 swz(hi) | 2 swz(hi + 1) << 8 | 2 swz(ho) << 16 | 2 swz(ho + 1) << 24, with hi = s=0 | lam_A bits at
    their positions in A, ho likewise on the complement (lam_i = bit i of g)."""
    out = []
    for si, A in enumerate(plan.sets):
        pos = plan.set_pos[si]
        for g in range(plan.G):
            hi = ho = 0
            for i in range(plan.N):
                lam = (g >> i) & 1
                if i in A:
                    hi |= lam << pos[i]
                else:
                    ho |= lam << pos[i]
            w = [2 * swz(hi), 2 * swz(hi + 1), 2 * swz(ho), 2 * swz(ho + 1)]
            assert max(w) < 256
            out.append(w[0] | w[1] << 8 | w[2] << 16 | w[3] << 24)
    return out


def hs_table(plan) -> list[int]:
    """Two-half join tables (plan.hs == 2).  The last photon x = N - 1 leaves the lane index: lane
    g' < G/2 of either half owns the 8 configurations (s, s', lam_x) x (lam_i = bit i of g', i < x).
    Per (subset si, g') two words of four byte offsets (2 swz(h), leaf rows as in hiho_table):
      x in A:  phi for (lam_x, s) = (0,0) (0,1) (1,0) (1,1), ubar for s' = 0, 1 (bytes 2, 3 zero)
      x in Ac: phi for s = 0, 1 (bytes 2, 3 zero), ubar for (lam_x, s') = (0,0) (0,1) (1,0) (1,1)
    Flattened as [si][g'][word]."""
    N, x = plan.N, plan.N - 1
    out = []
    for si, A in enumerate(plan.sets):
        pos = plan.set_pos[si]
        for gp in range(plan.G // 2):
            hi = ho = 0
            for i in range(x):
                lam = (gp >> i) & 1
                if i in A:
                    hi |= lam << pos[i]
                else:
                    ho |= lam << pos[i]
            if x in A:
                ph = [2 * swz(s | hi | (lx << pos[x])) for lx in (0, 1) for s in (0, 1)]
                ub = [2 * swz(sp | ho) for sp in (0, 1)] + [0, 0]
            else:
                ph = [2 * swz(s | hi) for s in (0, 1)] + [0, 0]
                ub = [2 * swz(sp | ho | (lx << pos[x])) for lx in (0, 1) for sp in (0, 1)]
            assert max(ph + ub) < 256
            out.append(ph[0] | ph[1] << 8 | ph[2] << 16 | ph[3] << 24)
            out.append(ub[0] | ub[1] << 8 | ub[2] << 16 | ub[3] << 24)
    return out
