"""Berends-Giele lowering: the distributive rewrite of the node-reduced CDAG.

PAPER.md line 160 (§3.1): node reduction alone "does not lower the computational complexity below
a factorial"; lines 220 and 378 name term rewriting with distributivity as the way to exponential
scaling.  Applied to the two-sided trie of gen/lower.py, distributivity pulls the sum over the
orderings of a photon subset inside the propagators:

  J_in(S)  = S(Q_S) sum_{i in S} epsslash_i J_in(S \\ i),        J_in({}) = u(p, s)
             (= sum over all orderings sigma of S of phi_sigma: the in-side current of subset S)
  P_out(T) = [sum_{i in T} P_out(T \\ i) epsslash_i] S(Q_{all \\ T}),  P_out({}) = ubar(p', s')
  K_out(T) = sum_{i in T} P_out(T \\ i) epsslash_i                 (leaf level |T| = N - j, no propagator)
  M(h)     = sum_{|A| = j} K_out(A^c)[s', lam_{A^c}] . J_in(A)[s, lam_A]

This is exactly the same sum of (n+1)! diagrams (the oracle is unchanged); the work per point drops
from factorial to exponential: 232 k instead of 6.2 M flops at n = 5.  Each node is expanded over the
spin/polarisation states of its subset (2^(|S|+1)), as in gen/lower.py.

Task descriptors (ushort): [mask, out, parent_1, eps_1, ..., parent_K, eps_K] with K = |S|.
Layouts and swizzles are those of gen/lower.py (interiors: AoS spinors with XOR component
swizzle; leaves: component-major rows with swz()).
"""
from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

from .dag import balanced_split
from .lower import FLOPS, MMA_COL_POS, MMA_ROW_POS, PITCH_BG, johnson_order, lane_offset, leaf_off, mma_assignments

FLOPS_BG = dict(FLOPS)
FLOPS_BG["VACC"] = 48    # accumulating vertex: 8 real outputs x 3 fma
FLOPS_BG["VACC_T"] = 32  # accumulating transverse vertex (eps^3 = 0, lam = 1 known at build time): 8 x 2 fma


@dataclass
class BGPlan:
    N: int
    j: int
    G: int
    sets: list[tuple[int, ...]]
    layout: dict[str, int]
    stride: int
    # interior levels: list of (kind, K, tasks) in execution order; kind "in" (col, with S) / "out" (row, with S)
    levels: list[tuple[str, int, list[list[int]]]] = field(default_factory=list)
    # per set: (J_in leaf tasks [K = j], K_out leaf tasks [K = N - j])
    set_in: list[list[list[int]]] = field(default_factory=list)
    set_out: list[list[list[int]]] = field(default_factory=list)
    set_pos: list[list[int]] = field(default_factory=list)
    flops: dict[str, int] = field(default_factory=dict)
    n_sets_real: int = 0     # C(N, j); sets[n_sets_real:] pad the last batch to SETB subsets
    hs: int = 1              # join halves (lower.hs_table): 1 = lane tile (s, s'); 2 = (s, s', lam_{N-1})
    # node groups (profiles/r03): F free polarisation bits per task of each stage kind; a task computes the 2^F
    # nodes (S, spin, lam_fixed, mu) of one subset S, mu = the polarisations of the first F photons of S
    grp: tuple = (0, 0, 0, 0, 0)   # (level 1, levels >= 2, in-leaf, out-leaf, recomputed levels)

    @property
    def H(self) -> int:
        return 1 << (self.N + 2)

    @property
    def n_hi(self) -> int:
        return 1 << (self.j + 1)

    @property
    def n_ho(self) -> int:
        return 1 << (self.N - self.j + 1)

    @property
    def flops_per_point(self) -> int:
        return sum(self.flops.values())


def _subsets(N, k):
    return list(itertools.combinations(range(N), k))


def lane_utilisation(plan) -> tuple[float, dict]:
    """Lane-utilisation model of one point's schedule on the G lanes of its group: every barrier-
    separated phase (interior level pair, per-batch recompute stage, leaf stage, join) lasts as long as
    its busiest lane (task costs from FLOPS_BG; lane placement as in qed_eval_kernel.cuh run_tasks8).
    Returns (executed flops / (G x sum of phase maxima), per-phase-kind [span, work]).  Latency is
    ignored, so this bounds what the schedule shape allows; tools/bg_util.py prints it."""
    F = FLOPS_BG
    G, B, N = plan.G, plan.setb, plan.N

    def cost(kind, K, F=0, leaf=False):
        return task_flops(K, F, kind == "in" or not leaf)

    def phase(groups):
        lane = [0.0] * G
        for cnt, c, off in groups:
            for t in range(cnt):
                lane[(t + off) % G] += c
        return max(lane), sum(cnt * c for cnt, c, _ in groups)

    phases = []
    i = 0
    while i < len(plan.levels):
        kind, K, t, F0 = plan.levels[i]
        grp = [(len(t), cost(kind, K, F0), 0)]
        if i + 1 < len(plan.levels) and plan.levels[i + 1][1] == K:
            k2, _, t2, F2 = plan.levels[i + 1]
            grp.append((len(t2), cost(k2, K, F2), lane_offset(len(t), G)))
            i += 1
        phases.append(("int", phase(grp)))
        i += 1
    for _ in range(len(plan.sets) // B):
        for st in plan.set_stages[0]:
            grp, prev = [], 0
            for q, (kind, K, t, F0) in enumerate(st):
                grp.append((len(t) * B, cost(kind, K, F0), lane_offset(prev, G) if q > 0 else 0))
                prev = len(t) * B
            phases.append(("rec", phase(grp)))
        n_in, n_out = B * len(plan.set_in[0]), B * len(plan.set_out[0])
        phases.append(("leaf", phase([(n_in, cost("in", plan.j, plan.f_in, True), 0),
                                      (n_out, cost("out", N - plan.j, plan.f_out, True), lane_offset(n_in, G))])))
    n_join = plan.n_sets_real * 4 * F["JOIN"]      # padding subsets skip their join
    phases.append(("join", (float(n_join), float(n_join * G))))
    by: dict[str, list[float]] = {}
    for k, (m, w) in phases:
        a = by.setdefault(k, [0.0, 0.0])
        a[0] += m
        a[1] += w
    span = sum(a[0] for a in by.values())
    return sum(a[1] for a in by.values()) / (G * span), by


def simt_utilisation(plan) -> tuple[float, dict]:
    """SIMT-aware variant of lane_utilisation: the task kinds of one phase are different code paths, so a
    warp runs them one after the other, each for as many trips as its busiest lane needs (idle lanes of a
    path are lost, not filled by the other kind).  Phase cost = max over the group's warps of the sum over
    kinds of (trips x task cost).  It explains the round-3 grouped-task measurements (profiles/sweep_r51:
    n = 4 (1,2,2,2,2)/5 modelled 0.66 of the default's utilisation, measured 0.80 of its rate)."""
    G, B, N = plan.G, plan.setb, plan.N
    W = max(1, G // 32)

    def cost(kind, K, F=0, leaf=False):
        return task_flops(K, F, kind == "in" or not leaf)

    def phase(groups):
        worst = 0.0
        for w in range(W):
            lanes = range(w * 32, min(G, (w + 1) * 32))
            tot = 0.0
            for cnt, c, off in groups:
                trips = max(sum(1 for t in range(cnt) if (t + off) % G == g) for g in lanes)
                tot += trips * c
            worst = max(worst, tot)
        return worst, sum(cnt * c for cnt, c, _ in groups) / W

    phases = []
    i = 0
    while i < len(plan.levels):
        kind, K, t, F0 = plan.levels[i]
        grp = [(len(t), cost(kind, K, F0), 0)]
        if i + 1 < len(plan.levels) and plan.levels[i + 1][1] == K:
            k2, _, t2, F2 = plan.levels[i + 1]
            grp.append((len(t2), cost(k2, K, F2), lane_offset(len(t), G)))
            i += 1
        phases.append(("int", phase(grp)))
        i += 1
    for _ in range(len(plan.sets) // B):
        for st in plan.set_stages[0]:
            grp, prev = [], 0
            for q, (kind, K, t, F0) in enumerate(st):
                grp.append((len(t) * B, cost(kind, K, F0), lane_offset(prev, G) if q > 0 else 0))
                prev = len(t) * B
            phases.append(("rec", phase(grp)))
        n_in, n_out = B * len(plan.set_in[0]), B * len(plan.set_out[0])
        phases.append(("leaf", phase([(n_in, cost("in", plan.j, plan.f_in, True), 0),
                                      (n_out, cost("out", N - plan.j, plan.f_out, True), lane_offset(n_in, G))])))
    n_join = plan.n_sets_real * 4 * FLOPS_BG["JOIN"]
    phases.append(("join", (float(n_join), float(n_join * min(G, 32)))))
    by: dict[str, list[float]] = {}
    for k, (m, w) in phases:
        a = by.setdefault(k, [0.0, 0.0])
        a[0] += m
        a[1] += w
    span = sum(a[0] for a in by.values())
    return sum(a[1] for a in by.values()) / (min(G, 32) * span), by


# sizes where the GPU sweep overrules the model (profiles/sweep_r18.jsonl: the modelled batch of 2 at
# n = 2 and of 4 at n = 7 measured 3 % and 6 % slower than 1 and 2)
SETB_MEASURED = {(3, 1): 1, (8, 4): 2}


def default_setb(N: int, j: int, store: int, sp: int) -> int:
    """Subsets per leaf stage (1, 2, 4 or 8, at most 4 when deep levels are recomputed per subset):
    the batch that maximises lane utilisation x occupancy (resident warps per SM, saturating at 16).
    It need not divide the number of subsets: the list is padded with copies of the last subset,
    whose leaves are computed and whose joins are skipped."""
    from .emit import choose_launch
    if (N, j) in SETB_MEASURED:
        return SETB_MEASURED[(N, j)]
    n_sets = math.comb(N, j)
    recompute = store + 1 < max(j, N - j)
    best = (-1.0, 1)
    for b in (1, 2, 4, 8):
        if b > n_sets or (recompute and b > 4):
            break
        p = make_bg_plan(N, j, setb=b, store=store, sp=sp)
        wpb, blocks = choose_launch(p)
        if wpb * 32 < p.G:
            continue
        util, _ = lane_utilisation(p)
        score = util * min(16, wpb * blocks) / 16
        if score > best[0] * 1.01:
            best = (score, b)
    return best[1]


def default_bg_store(N: int, j: int) -> int:
    """Current levels stored per point; deeper interior levels are recomputed per subset when storing
    them would push shared memory past ~110 KB per point (n >= 7)."""
    def spinors(store):
        return sum(math.comb(N, k) << (k + 1) for k in range(1, min(j, store + 1))) + \
            sum(math.comb(N, k) << (k + 1) for k in range(1, min(N - j, store + 1)))
    return N if spinors(N) * 64 <= 110 * 1024 else 2


def default_hs(N: int) -> int:
    """Join halves where they measured faster (profiles/sweep_r21.jsonl vs sweep_r18: n = 6 +6 %,
    n = 8 +11 %; n = 4 -5 %, n = 5 flat, n = 7 -1.5 %)."""
    return 2 if N in (7, 9) else 1


def group_strides(K: int, F: int, nS: int, nR: int) -> tuple[int, int, int]:
    """Node strides between node mu and mu + 1 of a grouped task (free photons = the last F of S, helicity-
    major interior layout: node (S, h) at region + h nS + idx(S); nS / nR = subsets of the task's / parent
    level): (output, parent through a fixed photon, parent through a free photon)."""
    return (1 << (K - F + 1)) * nS, (1 << (K - F)) * nR, (1 << (K - F + 1)) * nR


def swz_h(h: int) -> int:
    return (h & ~7) | ((h + (h >> 3)) & 7)


def leaf_mu(region: int, h0: int, mu: int, K: int, F: int) -> int:
    """Leaf offset of node mu of a grouped leaf task (kernel: BGGroupFn leaf store): helicity h0 + mu
    2^(K-F+1), column swz(h) of the leaf rows starting at region."""
    return region + 2 * swz_h(h0 + mu * (1 << (K - F + 1)))


def task_flops(K: int, F: int, prop: bool) -> int:
    """FP64 flops of one grouped task (2^F nodes): per node K vertices, the first one plain (V or V_T),
    the others accumulating (VACC or VACC_T); a vertex is transverse (eps^3 = 0) when its photon is
    free and its polarisation is 1, which the kernel knows at build time; + S per node."""
    F_ = FLOPS_BG
    tot = 0
    for mu in range(1 << F):
        for q in range(K):
            trans = q >= K - F and (mu >> (q - (K - F))) & 1
            if q == 0 if F == 0 else q == K - F:   # the kernel starts each node with its first free photon
                tot += F_["V_T"] if trans else F_["V"]
            else:
                tot += F_["VACC_T"] if trans else F_["VACC"]
        tot += F_["S"] if prop else 0
    return tot


def mma_leaf_slot(assign: dict, side_photons, h: int, prim) -> int:
    """Accumulator-layout slot of leaf helicity h (bit 0 = s / s', bit 1 + k = lam of the k-th sorted photon
    of the side): bit 0 <- the spin, bits 1, 2, 3 <- the photons at prim[0], prim[1], prim[2] (lower.py)."""
    slot = h & 1
    for k, x in enumerate(side_photons):
        slot |= ((h >> (1 + k)) & 1) << (1 + prim.index(assign[x]))
    return slot


def make_bg_plan(N: int, j: int | None = None, setb: int | None = None, store: int | None = None,
                 sp: int | None = None, hs: int | None = None, grp: tuple | None = None, mma: bool = False) -> BGPlan:
    if j is None:
        j = balanced_split(N)
    assert 1 <= j <= N - 1
    G = 1 << N
    full = (1 << N) - 1
    SP = sp if sp is not None else PITCH_BG.get(N, 10)
    grp = tuple(grp) if grp is not None else (0, 0, 0, 0, 0)
    grouped = any(grp)
    if mma:   # tensor-core joins (qed_eval_kernel.cuh mma_eval): one-tile joins, ungrouped tasks; 8 x 8 tiles
        assert not grouped and (hs in (None, 1)) and 2 <= j <= len(MMA_COL_POS) and 2 <= N - j <= len(MMA_ROW_POS)
        hs = 1
    if store is None:
        store = default_bg_store(N, j)
    assert not grouped or store + 1 >= max(j, N - j), "grouped plans store every interior level"
    if hs is None:
        hs = default_hs(N)
    if setb is None:
        setb = default_setb(N, j, store, SP)
    if hs == 2 and setb % 2:
        setb *= 2                                   # one subset per half and batch at least
    lay: dict[str, int] = {}
    off = 0

    def alloc(name, size, align=2):
        nonlocal off
        off = (off + align - 1) // align * align
        lay[name] = off
        off += size

    alloc("MOM", 4 * (N + 2))
    alloc("RED", max(2, G // 32))
    alloc("EPS", N * 2 * 4)
    alloc("MASK", (1 << N) * 6)
    alloc("U", 2 * SP, 8)
    alloc("UB", 2 * SP, 8)
    in_idx: dict[int, dict[tuple, int]] = {}
    out_idx: dict[int, dict[tuple, int]] = {}
    for k in range(1, min(j, store + 1)):
        subs = _subsets(N, k)
        alloc(f"IN{k}", len(subs) * (1 << (k + 1)) * SP, 8)
        in_idx[k] = {s: i for i, s in enumerate(subs)}
    for k in range(1, min(N - j, store + 1)):
        subs = _subsets(N, k)
        alloc(f"OUT{k}", len(subs) * (1 << (k + 1)) * SP, 8)
        out_idx[k] = {s: i for i, s in enumerate(subs)}
    # per-subset recomputed levels: subsets of size k inside A (|A| = j) / inside A^c (|A^c| = N - j)
    for k in range(store + 1, j):
        alloc(f"SIN{k}", setb * math.comb(j, k) * (1 << (k + 1)) * SP, 8)
    for k in range(store + 1, N - j):
        alloc(f"SOUT{k}", setb * math.comb(N - j, k) * (1 << (k + 1)) * SP, 8)
    set_local: dict[tuple, int] = {}
    cur_slot = [0]
    n_hi, n_ho = 1 << (j + 1), 1 << (N - j + 1)
    leafb = (4 * n_hi * 2 + 4 * n_ho * 2 + 7) // 8 * 8      # doubles per leaf buffer (PHI + UBL; AoS if mma)
    if grouped:   # leaf buffers of one batch skewed by the out-leaf tasks per subset (16-byte columns): the
        # quarter warps storing the same columns of several subsets hit distinct bank groups
        leafb += (2 << max(0, N - j - min(grp[3], N - j) + 1)) % 16
    alloc("PHI", 4 * n_hi * 2, 8)
    alloc("UBL", 4 * n_ho * 2, 8)
    alloc("LEAFX", leafb * (setb - 1) - (lay["UBL"] + 4 * n_ho * 2 - lay["PHI"] - leafb) if setb > 1 else 0, 8)
    lay["LEAFB"] = leafb
    stride = (off + 1) // 2 * 2
    if (stride // 2) % 2 == 0:
        stride += 2
    lay["STRIDE"] = stride
    if hs == 2:    # the halves' amplitude reduction reuses the slot from U on (dead after the last join)
        assert lay["U"] + 16 * (G // 2) <= stride, (N, lay["U"], stride)

    def eps_off(i, lam):
        return lay["EPS"] + (i * 2 + lam) * 4

    def mask_off(m):
        return lay["MASK"] + m * 6

    def msk(S):
        return sum(1 << x for x in S)

    def hel(S, h_bits: dict, spin: int) -> int:
        """helicity index of subset S: spin | lam_{S sorted} << (1 + position)"""
        return spin | sum(h_bits[x] << (1 + p) for p, x in enumerate(S))

    def node_off(side, S, h):
        k = len(S)
        if k == 0:
            return (lay["U"] if side == "in" else lay["UB"]) + h * SP
        if k > store:
            idx = set_local[(side, S)]
            slot = cur_slot[0] * math.comb(j if side == "in" else N - j, k)   # this subset's batch slot
            return lay[f"{'SIN' if side == 'in' else 'SOUT'}{k}"] + ((slot + idx) * (1 << (k + 1)) + h) * SP
        idx = (in_idx if side == "in" else out_idx)[k][S]
        if grouped:   # helicity-major: the nodes of one helicity index are consecutive over the subsets
            return lay[f"{'IN' if side == 'in' else 'OUT'}{k}"] + (h * math.comb(N, k) + idx) * SP
        return lay[f"{'IN' if side == 'in' else 'OUT'}{k}"] + (idx * (1 << (k + 1)) + h) * SP

    def gtask(side, S, F, lf, spin, out_of, mask, leafreg=None):
        """Grouped task of node set S (sorted) for fixed polarisations lf (of the first K-F photons) and
        spin: the 2^F nodes mu = polarisations of the LAST F photons of S (helicity bits K-F+1..K).
        Descriptor [mask, out_0, (parent_0, eps_0) per photon of S, (leaves:) h0]; the kernel steps node mu's
        output / parents by group_strides() (leaf outputs: leaf_mu(out_0 = region, h0)); free photons'
        eps(lam = 1) sit 4 doubles after eps(lam = 0).  Every offset the kernel derives is checked here
        against the plain node layout."""
        K = len(S)
        nS = math.comb(N, K)
        nR = math.comb(N, K - 1) if K > 1 else 0
        so, sf, sr = group_strides(K, F, nS, nR)
        lam0 = {x: (lf >> p) & 1 for p, x in enumerate(S[:K - F])}
        lam0.update({x: 0 for x in S[K - F:]})
        h0 = hel(S, lam0, spin)
        d = [mask, out_of(h0) if leafreg is None else leafreg]
        for q, x in enumerate(S):
            R = tuple(y for y in S if y != x)
            d += [node_off(side, R, hel(R, lam0, spin)), eps_off(x, lam0[x])]
        if leafreg is not None:
            d.append(h0)
        for mu in range(1 << F):                 # layout claims of the kernel, node by node
            lam = dict(lam0)
            lam.update({x: (mu >> q) & 1 for q, x in enumerate(S[K - F:])})
            h = hel(S, lam, spin)
            assert h == h0 + (1 << (K - F + 1)) * mu
            if leafreg is None:
                assert out_of(h) == d[1] + so * SP * mu, (S, mu)
            else:
                assert out_of(h) == leaf_mu(leafreg, h0, mu, K, F), (S, mu)
            for p, x in enumerate(S):
                R = tuple(y for y in S if y != x)
                par = node_off(side, R, hel(R, lam, spin))
                if p >= K - F:
                    q = p - (K - F)
                    mr = (mu & ((1 << q) - 1)) | ((mu >> (q + 1)) << q)
                    assert par == d[2 + 2 * p] + sr * SP * mr, (S, mu, p)
                    assert eps_off(x, lam[x]) == d[3 + 2 * p] + 4 * ((mu >> q) & 1)
                else:
                    assert par == d[2 + 2 * p] + sf * SP * mu, (S, mu, p)
                    assert eps_off(x, lam[x]) == d[3 + 2 * p]
        return d

    def level_tasks(side, Ss, kind, leafreg=None, nh=0):
        """Tasks of the node sets Ss: ungrouped (F = 0) in the original (S, h) order; grouped in (h0, S)
        order, so that consecutive lanes take consecutive nodes of the helicity-major layout."""
        res = []
        K = len(Ss[0])
        F = fsel(kind, K)
        if not grouped:
            assert F == 0
        order = [(lf, sp, S) for lf in range(1 << (K - F)) for sp in range(2) for S in Ss] if grouped else \
            [(lf, sp, S) for S in Ss for lf in range(1 << (K - F)) for sp in range(2)]
        for lf, spin, S in order:
            mask = mask_off(msk(S) if side == "in" else full & ~msk(S))
            if leafreg is None:
                res.append(gtask(side, S, F, lf, spin, lambda h, S=S: node_off(side, S, h), mask))
            else:
                res.append(gtask(side, S, F, lf, spin, lambda h: leaf_off(leafreg, nh, 0, h),
                                 mask if side == "in" else 0, leafreg if grouped else None))
        return res

    def fsel(kind: str, k: int) -> int:
        F = {"lvl": grp[0] if k == 1 else grp[1], "in_leaf": grp[2], "out_leaf": grp[3], "rec": grp[4]}[kind]
        return min(F, k)

    plan = BGPlan(N=N, j=j, G=G, sets=[], layout=lay, stride=stride)
    plan.sp = SP
    plan.setb = setb
    plan.store = store
    plan.grp = grp
    plan.set_stages = []
    for k in range(1, min(max(j, N - j), store + 1)):
        if k < j:
            t = level_tasks("in", _subsets(N, k), "lvl")
            plan.levels.append(("in", k, t, fsel("lvl", k)))
        if k < N - j:
            t = level_tasks("out", _subsets(N, k), "lvl")
            plan.levels.append(("out", k, t, fsel("lvl", k)))
    subsets = johnson_order(N, j) if mma else list(itertools.combinations(range(N), j))
    plan.mma = mma
    if mma:
        plan.mma_assign, plan.mma_swaps = mma_assignments(N, j, subsets)
    if hs == 2:
        # two-half joins (lower.hs_table): subsets containing photon N-1 first, so that the two halves
        # of a batch take the same join shape (at most one mixed pair)
        subsets = [A for A in subsets if N - 1 in A] + [A for A in subsets if N - 1 not in A]
    plan.hs = hs
    plan.n_sets_real = len(subsets)
    subsets += [subsets[-1]] * (-len(subsets) % setb)   # ragged last batch: padding, joins skipped
    plan.f_in, plan.f_out = fsel("in_leaf", j), fsel("out_leaf", N - j)
    for A in subsets:
        Ac = tuple(x for x in range(N) if x not in A)
        plan.sets.append(A)
        pos = [0] * N
        for k, x in enumerate(A):
            pos[x] = 1 + k
        for k, x in enumerate(Ac):
            pos[x] = 1 + k
        plan.set_pos.append(pos)
        # recomputed interior levels of this subset (stored levels are shared by all subsets)
        stages = []
        set_local.clear()
        cur_slot[0] = (len(plan.sets) - 1) % setb
        for k in range(store + 1, max(j, N - j)):
            st = []
            if k < j:
                subs = list(itertools.combinations(A, k))
                for i, S in enumerate(subs):
                    set_local[("in", S)] = i
                st.append(("in", k, level_tasks("in", subs, "rec"), fsel("rec", k)))
            if k < N - j:
                subs = list(itertools.combinations(Ac, k))
                for i, T in enumerate(subs):
                    set_local[("out", T)] = i
                st.append(("out", k, level_tasks("out", subs, "rec"), fsel("rec", k)))
            stages.append(st)
        plan.set_stages.append(stages)
        lb = (len(plan.sets) - 1) % setb          # leaf buffer of this subset within its batch
        phi0, ubl0 = lay["PHI"] + lb * lay["LEAFB"], lay["UBL"] + lb * lay["LEAFB"]
        if mma:   # AoS leaves at their accumulator-layout slot (lower.mma_slot), tasks in slot order
            si_ = min(len(plan.sets) - 1, plan.n_sets_real - 1)
            asg = plan.mma_assign[si_]
            ti = [(d, mma_leaf_slot(asg, A, d_h, MMA_COL_POS)) for d, d_h in
                  zip(level_tasks("in", [A], "in_leaf", phi0, n_hi), range(n_hi))]
            plan.set_in.append(sorted(([d[0], phi0 + sl * 8] + d[2:] for d, sl in ti), key=lambda t: t[1]))
            to = [(d, mma_leaf_slot(asg, Ac, d_h, MMA_ROW_POS)) for d, d_h in
                  zip(level_tasks("out", [Ac], "out_leaf", ubl0, n_ho), range(n_ho))]
            plan.set_out.append(sorted(([d[0], ubl0 + sl * 8] + d[2:] for d, sl in to), key=lambda t: t[1]))
        else:
            plan.set_in.append(level_tasks("in", [A], "in_leaf", phi0, n_hi))
            plan.set_out.append(level_tasks("out", [Ac], "out_leaf", ubl0, n_ho))

    F = FLOPS_BG
    H = 1 << (N + 2)

    def vflops(k):
        return F["V"] + (k - 1) * F["VACC"]

    n_in = sum(math.comb(N, k) * (1 << (k + 1)) * (vflops(k) + F["S"]) for k in range(1, j + 1))
    n_out = sum(math.comb(N, k) * (1 << (k + 1)) * (vflops(k) + F["S"]) for k in range(1, N - j)) + \
        math.comb(N, N - j) * (1 << (N - j + 1)) * vflops(N - j)
    plan.max_k = max(j, N - j)
    plan.dw = 8 if plan.max_k <= 3 and not grouped else 16   # descriptor width in ushort (grouped: + h0)
    rec = sum(len(t) * (vflops(k) + F["S"]) << Fk for stages in plan.set_stages for st in stages for _, k, t, Fk in st)
    stored_rec = sum(math.comb(N, k) * (1 << (k + 1)) * (vflops(k) + F["S"])
                     for k in range(store + 1, j)) + \
        sum(math.comb(N, k) * (1 << (k + 1)) * (vflops(k) + F["S"]) for k in range(store + 1, N - j))
    n_pad = len(plan.sets) - plan.n_sets_real
    pad_leaf = n_pad * ((1 << (j + 1)) * (vflops(j) + F["S"]) + (1 << (N - j + 1)) * vflops(N - j))
    plan.recompute_flops = rec - stored_rec + pad_leaf   # executed on top of the algorithmic count
    plan.flops = {
        "external": N * F["EPS"] + 2 * F["SPINOR"],
        "propagator_constants": ((1 << N) - 2) * F["MASK"],
        "currents_in": n_in,
        "currents_out": n_out,
        "join": math.comb(N, j) * H * F["JOIN"],
        "msq": H * F["ABS2"],
    }
    if grouped:
        # the kernel's own count: a free photon's lam = 1 vertex is the transverse form (eps^3 = 0), known
        # at build time in a grouped task; everything else as above (each node still computed once)
        plan.flops["currents_in"] = sum(math.comb(N, k) * (1 << (k + 1 - fsel("lvl" if k < j else "in_leaf", k)))
                                        * task_flops(k, fsel("lvl" if k < j else "in_leaf", k), True)
                                        for k in range(1, j + 1))
        plan.flops["currents_out"] = sum(math.comb(N, k) * (1 << (k + 1 - fsel("lvl", k))) * task_flops(k, fsel("lvl", k), True)
                                         for k in range(1, N - j)) + \
            math.comb(N, N - j) * (1 << (N - j + 1 - plan.f_out)) * task_flops(N - j, plan.f_out, False)
    return plan
