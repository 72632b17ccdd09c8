"""Build-time generator (paper_2511_19456_b200/gen): the CDAG of PAPER.md §2-3 and App. C,
pinned by the paper's printed node counts, and the lowered kernel tables checked against the
oracle through the table interpreter (no GPU)."""
import math
import os

import numpy as np
import pytest

import oracle
import synthetic
from paper_2511_19456_b200.gen.dag import (build_unreduced, north_star, paper_process, reduced_counts_formula,
                                           table1_closed_form)
from paper_2511_19456_b200.gen.interp import eval_point
from paper_2511_19456_b200.gen.lower import make_plan, trie_node_counts

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden(name):
    out = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.split("#")[0].strip()
        if line:
            out.append(line.split())
    return out


@pytest.mark.parametrize("n,count", [(int(a), int(b)) for a, b in _golden("table1_node_counts.txt")])
def test_table1_closed_form(n, count):
    """nodes(n) = 3(n+3) + 2 + 2(2n+1)(n+1)! reproduces every Table 1 row."""
    assert table1_closed_form(n) == count


@pytest.mark.parametrize("n,count", [(int(a), int(b)) for a, b in _golden("table1_node_counts.txt")][:5])
def test_generated_cdag_matches_table1(n, count):
    """The generated (pre-optimisation) CDAG of e- gamma^n -> e- gamma has exactly Table 1's node count."""
    g = build_unreduced(paper_process(n))
    g.validate()
    assert len(g) == count
    # the north-star direction has the same topology
    assert len(build_unreduced(north_star(n))) == count


def test_n1_composition_fig5():
    g = build_unreduced(paper_process(1))
    c = g.counts()
    entry = sum(1 for nd in g.nodes.values() if nd.kind == "data" and not nd.parents)
    for kind, cnt in _golden("fig5_n1_composition.txt"):
        got = entry if kind == "entry" else c.get(kind, 0) - (entry if kind == "data" else 0)
        assert got == int(cnt), (kind, got)


@pytest.mark.parametrize("n,nodes", [(1, 26), (2, 59), (3, 148), (4, 543), (5, 2234)])
def test_node_reduction_fixpoint(n, nodes):
    """Fixpoint of node reduction (App. C) = two-sided prefix trie
    (SURVEY.md App. A.2); (n+1)! S2 joins survive."""
    g = build_unreduced(north_star(n)).reduce_fixpoint()
    g.validate()
    assert len(g) == nodes
    c = g.counts()
    f = reduced_counts_formula(n + 1, (n + 1) // 2)
    for k in ("V", "S1", "S2", "U", "Sum"):
        assert c.get(k, 0) == f[k]
    assert c["S2"] == math.factorial(n + 1)


@pytest.mark.parametrize("n", [2, 3])
def test_fixpoint_is_order_independent(n):
    """the fully reduced CDAG does not depend on the reduction order."""
    ref = build_unreduced(north_star(n)).reduce_fixpoint().canonical()
    for seed in range(4):
        g = build_unreduced(north_star(n)).reduce_random_order(seed)
        assert g.canonical() == ref


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_lowered_trie_equals_fixpoint(n):
    plan = make_plan(n + 1)
    g = build_unreduced(north_star(n)).reduce_fixpoint()
    c = g.counts()
    t = trie_node_counts(plan)
    assert (t["V"], t["S1"], t["S2"]) == (c["V"], c.get("S1", 0), c["S2"])


@pytest.mark.parametrize("n,npts", [(1, 3), (2, 3), (3, 2), (4, 1), (5, 1)])
def test_tables_interpreted_match_oracle(n, npts):
    """The kernel's task tables, executed with the kernel's shared-memory layout, give the
    oracle's helicity amplitudes (catches any wrong offset before a GPU run)."""
    plan = make_plan(n + 1)
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=300 + n).numpy()
    A = oracle.amps(1, n, mom)
    for k in range(npts):
        B = eval_point(plan, mom[k], 1)
        assert np.max(np.abs(A[k] - B)) <= 1e-12 * np.max(np.abs(A[k]))


@pytest.mark.parametrize("n", [1, 2, 3])
def test_tables_paper_direction(n):
    plan = make_plan(n + 1)
    mom = synthetic.rambo_cm(n, 1, sqrt_s=5.0, seed=400 + n).numpy()
    rev = np.concatenate([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], axis=1)
    A = oracle.amps(n, 1, rev)
    B = eval_point(plan, rev[0], n)
    assert np.max(np.abs(A[0] - B)) <= 1e-12 * np.max(np.abs(A[0]))


def test_flop_counts_documented():
    """Algorithmic flops per point (the roofline numerator) for n = 1..5."""
    got = [make_plan(n + 1).flops_per_point for n in range(1, 6)]
    assert got == [2260, 10672, 65884, 565672, 6212404]


# ---------------------------------------------------------------- Berends-Giele (distributive rewrite, NEXT #1)

@pytest.mark.parametrize("n,npts", [(1, 2), (2, 2), (3, 2), (4, 1), (5, 1)])
def test_bg_tables_interpreted_match_oracle(n, npts):
    """Summing over orderings inside the propagators leaves the
    amplitude unchanged: the BG tables, executed with the device layout, give the oracle's amplitudes."""
    from paper_2511_19456_b200.gen.interp import eval_point_bg
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    plan = make_bg_plan(n + 1)
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=500 + n).numpy()
    A = oracle.amps(1, n, mom)
    for k in range(npts):
        B = eval_point_bg(plan, mom[k], 1)
        assert np.max(np.abs(A[k] - B)) <= 1e-12 * np.max(np.abs(A[k]))


def test_bg_flop_counts():
    """Exponential instead of factorial growth of the algorithmic work per point."""
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    got = [make_bg_plan(n + 1).flops_per_point for n in range(1, 6)]
    assert got == [2260, 7792, 27100, 90792, 310324]
    cdag = [make_plan(n + 1).flops_per_point for n in range(1, 6)]
    assert cdag[4] / got[4] > 19


@pytest.mark.parametrize("N,store", [(5, 1), (6, 1), (7, None)])
def test_bg_recompute_and_large_tables_match_oracle(N, store):
    """Per-subset recomputation of deep current levels (n >= 7 default) and the n = 6 tables."""
    from paper_2511_19456_b200.gen.interp import eval_point_bg
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    n = N - 1
    plan = make_bg_plan(N, store=store)
    mom = synthetic.rambo_cm(n, 1, sqrt_s=5.0, seed=600 + n).numpy()
    A = oracle.amps(1, n, mom)
    B = eval_point_bg(plan, mom[0], 1)
    assert np.max(np.abs(A[0] - B)) <= 1e-12 * np.max(np.abs(A[0]))


def test_bg_default_plans_n7_n8():
    """n = 7, 8: levels above 2 recomputed per subset, several subsets per stage, fits one block's
    shared memory; the subset list is padded to whole batches (C(8,4) = 70, C(9,4) = 126)."""
    import math
    from paper_2511_19456_b200.gen.lower_bg import lane_utilisation, make_bg_plan
    for N in (8, 9):
        p = make_bg_plan(N)
        assert p.store == 2 and p.dw == 16 and p.setb >= 2
        assert p.stride * 8 < 227 * 1024
        assert p.n_sets_real == math.comb(N, p.j) and len(p.sets) % p.setb == 0
        assert len(p.sets) - p.n_sets_real < p.setb
        assert all(A == p.sets[p.n_sets_real - 1] for A in p.sets[p.n_sets_real:])
        assert lane_utilisation(p)[0] > 0.8


def test_bg_lane_utilisation_model():
    """The schedule model: one subset per stage leaves most lanes idle at n = 6 (16 + 32 leaf tasks on
    128 lanes); the default batch recovers it; a perfectly packed stage has utilisation 1."""
    from paper_2511_19456_b200.gen.lower_bg import lane_utilisation, make_bg_plan
    u1, by1 = lane_utilisation(make_bg_plan(7, setb=1, hs=1))
    ud, _ = lane_utilisation(make_bg_plan(7))
    assert by1["leaf"][1] / (128 * by1["leaf"][0]) < 0.4 and ud > u1 + 0.2
    u2, _ = lane_utilisation(make_bg_plan(2))
    assert u2 == 1.0


@pytest.mark.parametrize("N,hs", [(4, 2), (5, 2), (6, 2), (5, 1), (7, 1)])
def test_bg_join_halves_match_oracle(N, hs):
    """Two-half joins (lower.hs_table: lane tile (s, s', lam_{N-1}), subsets split over the halves of
    the group) and the one-tile form, each against the oracle through the interpreter."""
    from paper_2511_19456_b200.gen.interp import eval_point_bg
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    n = N - 1
    plan = make_bg_plan(N, hs=hs)
    assert plan.hs == hs and (hs == 1 or plan.setb % 2 == 0)
    mom = synthetic.rambo_cm(n, 2, sqrt_s=5.0, seed=700 + n).numpy()
    A = oracle.amps(1, n, mom)
    for k in range(2):
        B = eval_point_bg(plan, mom[k], 1)
        assert np.max(np.abs(A[k] - B)) <= 1e-12 * np.max(np.abs(A[k]))


# ---------------------------------------------------------------- register bodies: flop counts from the emitted code
_CALL_FLOPS = {"eslash_col(": 40, "eslash_row(": 40, "eslash_col_t(": 24, "eslash_row_t(": 24, "prop_col(": 56,
               "prop_row(": 56, "cdot_acc(": 32, "cdot8_acc(": 8 * 32, "add_to(": 8,
               "eslash_row_acc(": 48, "eslash_row_t_acc(": 32}


def _sparse_call_flops():
    """qed_sparse.cuh calls on the external spinors, priced by the generator's zero-aware count."""
    from paper_2511_19456_b200.gen.emit_regs import ZU, ZUX, sparse_v, sparse_vs
    out = {}
    for zn, z in (("ZU0", ZU[0]), ("ZU1", ZU[1]), ("ZUX", ZUX)):
        for t in (False, True):
            tn = "true" if t else "false"
            out[f"vs_col_z<qed::{zn}, {tn}>("] = sparse_vs(z, t)
            out[f"vs_row_z<qed::{zn}, {tn}>("] = sparse_vs(z, t)
            out[f"eslash_row_z<qed::{zn}, {tn}>("] = sparse_v(z, t)[0]
            out[f"eslash_col_z<qed::{zn}, {tn}>("] = sparse_v(z, t)[0]
    for t in (False, True):   # vs_row_ub: the spin's own pattern; both spins cost the same
        assert sparse_vs(ZU[0], t) == sparse_vs(ZU[1], t)
        out[f"vs_row_ub<{'true' if t else 'false'}>("] = sparse_vs(ZU[0], t)
    return out


def _count_body_flops(src: str, fn: str) -> int:
    """Flops of the vertex / propagator / join / sum calls in the straight-line body `fn` of generated source,
    each weighted by the trip count of the enclosing `for (...; x < K; ...)` loops (read from the text)."""
    import re
    body = src[src.index(f"void {fn}("):]
    body = body[:body.index("\n}\n")]
    total, stack, pending = 0, [], 1
    for line in body.split("\n"):
        m = re.search(r"for \(int \w+ = 0; \w+ < (\d+); \+\+\w+\)", line)
        mult = 1
        for k in stack:
            mult *= k
        if m:
            pending = int(m.group(1))
        for call, fl in {**_CALL_FLOPS, **_sparse_call_flops()}.items():
            total += mult * (pending if m else 1) * fl * line.count(call)
        for ch in line:
            if ch == "{":
                stack.append(pending if m else 1)
                m, pending = None, 1
            elif ch == "}":
                stack.pop()
    return total


def test_register_body_flops_match_the_flop_model():
    """The roofline numerator of the register kernels (gen/emit_regs.py _flops / bg_flops) equals what their
    emitted straight-line bodies call: n = 1 (T1), n = 2 (T1P, and T1PI: the headline kernel's body) and BG n = 2
    (T1B, whose recomputed P_out({1}) is executed, not algorithmic work)."""
    from paper_2511_19456_b200.gen.emit_regs import _flops, bg_flops, emit_regs_source
    for N, fn, model in ((2, "regs_body1_N2", _flops(2)), (3, "regs_body1p_N3", _flops(3)),
                         (3, "regs_body1pi_N3", _flops(3)), (3, "regs_body_bg_N3", bg_flops(3))):
        src = emit_regs_source(N)
        vertex_part = sum(v for k, v in model.items() if k not in ("external", "propagator_constants", "msq"))
        got = _count_body_flops(src, fn)
        if fn == "regs_body_bg_N3":
            from paper_2511_19456_b200.gen.emit_regs import ZUX, sparse_vs
            got -= 2 * (sparse_vs(ZUX, False) + sparse_vs(ZUX, True))   # P_out({1}) recomputed once per s' pass
        assert got == vertex_part, (fn, got, vertex_part)
    # the generic plan minus the transverse-vertex saving (16 flop per eps(k, 2) vertex, half of all vertices)
    # and minus the structural zeros of u / ubar skipped by the vertices and propagators on them
    from paper_2511_19456_b200.gen.emit_regs import ZU, ZUX, sparse_vs, sparse_v
    gen_vs = {False: 40 + 56, True: 24 + 56}
    save_u = sum(gen_vs[lam == 1] - sparse_vs(ZU[s], lam == 1) for s in range(2) for lam in range(2))
    save_ub1 = sum({False: 40, True: 24}[lam == 1] - sparse_v(ZU[s], lam == 1)[0] for s in range(2) for lam in range(2))
    save_ub = sum(gen_vs[lam == 1] - sparse_vs(ZU[s], lam == 1) for s in range(2) for lam in range(2))
    assert sum(_flops(2).values()) == make_plan(2).flops_per_point - 16 * 8 - 2 * save_u - 2 * save_ub1
    assert sum(_flops(3).values()) == make_plan(3).flops_per_point - 16 * 36 - 3 * save_u - 3 * save_ub


def test_sparse_external_patterns_and_generic_counts():
    """The structural zero patterns the register kernels skip (qed_sparse.cuh ZU0 / ZU1, gen ZU) are exactly the
    zeros of the oracle's u(p, s) and ubar(p, s) at generic momenta, and the zero-aware counts reduce to the
    generic flop model (V 40, V_T 24, S 56) on a spinor without zeros."""
    from paper_2511_19456_b200.gen.emit_regs import ZU, ZUX, sparse_s, sparse_v
    rng = np.random.default_rng(5)
    for _ in range(5):
        pv = rng.normal(size=3)
        p = np.array([np.sqrt(1.0 + pv @ pv), *pv])
        for s in range(2):
            for sp in (oracle.spinor_u(p, s), oracle.spinor_ubar(p, s)):
                re_im = np.stack([sp.real, sp.imag], axis=1).reshape(-1)   # bit 2c + j
                z = sum(1 << k for k in range(8) if re_im[k] == 0.0)
                assert z == ZU[s], (s, bin(z))
    assert ZUX == ZU[0] & ZU[1]
    assert sparse_v(0, False) == (40, 0) and sparse_v(0, True) == (24, 0) and sparse_s(0) == 56
    # a zero input component removes exactly the products it enters (each appears in 3 of the 8 V outputs)
    assert sparse_v(1, False)[0] == 40 - 2 * 3


# ---------------------------------------------------------------- grouped Berends-Giele tasks (round 3)
@pytest.mark.parametrize("N,grp,setb", [(3, (1, 1, 1, 2, 1), 2), (4, (1, 2, 2, 2, 2), 3), (5, (1, 2, 1, 2, 2), 2),
                                        (5, (1, 2, 2, 2, 2), 5), (6, (1, 2, 1, 1, 1), 4), (7, (1, 1, 1, 1, 1), None)])
def test_bg_grouped_tasks_interpreted_match_oracle(N, grp, setb):
    """Grouped tasks (2^F nodes per descriptor, helicity-major interior layout, strided parents, skewed
    leaf buffers; gen/lower_bg.py gtask) executed by the kernel's offset rules give the oracle's amplitudes."""
    from paper_2511_19456_b200.gen.interp import eval_point_bg
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    n = N - 1
    plan = make_bg_plan(N, grp=grp, setb=setb)
    assert plan.grp == grp and plan.dw == 16
    mom = synthetic.rambo_cm(n, 2, sqrt_s=5.0, seed=800 + n).numpy()
    A = oracle.amps(1, n, mom)
    for k in range(2):
        B = eval_point_bg(plan, mom[k], 1)
        assert np.max(np.abs(A[k] - B)) <= 1e-12 * np.max(np.abs(A[k]))


def test_bg_grouped_flops_are_generic_minus_transverse():
    """A grouped task evaluates the same nodes; the only flop difference is the transverse vertex (eps^3 = 0)
    of each free photon with lam = 1: 40 -> 24 as first vertex, 48 -> 32 accumulating."""
    import math
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    for N, grp in [(4, (1, 1, 1, 1, 1)), (5, (1, 2, 2, 2, 2)), (6, (1, 2, 1, 1, 1))]:
        g, u = make_bg_plan(N, grp=grp), make_bg_plan(N)
        j = g.j
        saved = 0

        def level_saving(K, F, count_nodes):
            # per node: half of the nodes have lam = 1 for each free photon; the first free photon's vertex
            # is the plain one (saves 16), the other free photons' vertices accumulate (save 16)
            return count_nodes * F * 16 // 2

        for k in range(1, j):
            saved += level_saving(k, min(grp[0] if k == 1 else grp[1], k), math.comb(N, k) << (k + 1))
        for k in range(1, N - j):
            saved += level_saving(k, min(grp[0] if k == 1 else grp[1], k), math.comb(N, k) << (k + 1))
        saved += level_saving(j, min(grp[2], j), math.comb(N, j) << (j + 1))
        saved += level_saving(N - j, min(grp[3], N - j), math.comb(N, N - j) << (N - j + 1))
        assert u.flops_per_point - g.flops_per_point == saved, N


def test_bg_grouped_layout_claims_fail_on_a_wrong_stride():
    """Self-check of the interpreter: a wrong parent stride (what a kernel / table mismatch looks like)
    breaks the amplitude, so the grouped parity tests above can fail."""
    from paper_2511_19456_b200.gen import interp
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    plan = make_bg_plan(5, grp=(1, 2, 2, 2, 2), setb=5)
    mom = synthetic.rambo_cm(4, 1, sqrt_s=5.0, seed=801).numpy()
    A = oracle.amps(1, 4, mom)
    orig = interp.expand_group

    def wrong(d, K, F, sp, leaf, N):
        e = orig(d, K, F, sp, leaf, N)
        if F and K == 2 and not leaf and len(e) > 1:
            e[1][2] += sp          # node mu = 1 reads the neighbouring parent
        return e
    interp.expand_group = wrong
    try:
        B = interp.eval_point_bg(plan, mom[0], 1)
    finally:
        interp.expand_group = orig
    assert np.max(np.abs(A[0] - B)) > 1e-6 * np.max(np.abs(A[0]))


# ---------------------------------------------------------------- tensor-core joins (DMMA; this round)
def test_johnson_order_exchanges_one_photon_per_step():
    """The subset order of the tensor-core plans visits every j-subset once and consecutive subsets
    exchange exactly one photon, so the accumulator layout changes by one bit exchange (mma_swap)."""
    import itertools
    from paper_2511_19456_b200.gen.lower import johnson_order, mma_assignments
    for N, j in [(4, 2), (5, 2), (6, 3), (7, 3)]:
        order = johnson_order(N, j)
        assert sorted(order) == list(itertools.combinations(range(N), j))
        for a, b in zip(order, order[1:]):
            assert len(set(a) & set(b)) == j - 1
        if N - j <= 3:
            assign, swaps = mma_assignments(N, j, order)
            assert len(swaps) == len(order) - 1
            for A, asg in zip(order, assign):   # A's photons on column positions, the rest on row positions
                assert all(asg[x] in ("L0", "L1", "TC") for x in A)
                assert all(asg[x] in ("L3", "L4", "TR") for x in range(N) if x not in A)
                assert len(set(asg.values())) == N


@pytest.mark.parametrize("N,bg", [(4, False), (5, False), (6, False), (4, True), (5, True), (6, True), (5, "tc2")])
def test_mma_plans_interpreted_match_oracle(N, bg):
    """Tensor-core-join plans (AoS leaves at their accumulator slot, Johnson order, per-subset bit exchanges,
    final configuration map), executed by the interpreter with the kernel's rules, give the oracle's
    amplitudes (CDAG: gen/lower.py make_plan(mma=True); Berends-Giele: make_bg_plan(mma=True))."""
    from paper_2511_19456_b200.gen.interp import eval_point, eval_point_bg
    from paper_2511_19456_b200.gen.lower import make_plan
    from paper_2511_19456_b200.gen.lower_bg import make_bg_plan
    n = N - 1
    if bg == "tc2":   # u-bar leaves in two chunks of tau orderings (make_plan(tau_chunks=2))
        plan, bg = make_plan(N, mma=True, tau_chunks=2), False
    else:
        plan = make_bg_plan(N, mma=True) if bg else make_plan(N, mma=True)
    mom = synthetic.rambo_cm(n, 2, sqrt_s=5.0, seed=1000 + n).numpy()
    A = oracle.amps(1, n, mom)
    for k in range(2):
        B = (eval_point_bg if bg else eval_point)(plan, mom[k], 1)
        assert np.max(np.abs(A[k] - B)) <= 1e-12 * np.max(np.abs(A[k]))


def test_mma_wrong_exchange_is_detected():
    """Self-check: skipping one accumulator bit exchange (or exchanging the wrong pair) scrambles the
    amplitudes, so the interpreter parity above can fail on a generator / kernel mismatch."""
    from paper_2511_19456_b200.gen import interp
    from paper_2511_19456_b200.gen.lower import make_plan
    plan = make_plan(5, mma=True)
    mom = synthetic.rambo_cm(4, 1, sqrt_s=5.0, seed=1001).numpy()
    A = oracle.amps(1, 4, mom)
    plan.mma_swaps = [plan.mma_swaps[0]] * len(plan.mma_swaps)
    B = interp.eval_point(plan, mom[0], 1)
    assert np.max(np.abs(A[0] - B)) > 1e-6 * np.max(np.abs(A[0]))
