"""Shared-memory wavefront model of a Berends-Giele plan (gen/lower_bg.py), offline.

Replays the per-lane task placement of qed_eval_kernel.cuh (run_tasks8: lane g of the group takes tasks
(g - OFF) mod G + k G) and the access sequence of each task functor (BGFn / BGGroupFn), warp instruction by
warp instruction, and counts wavefronts with the bank rule: a warp access costs max over the 32 4-byte
banks of the number of distinct words requested in that bank (same word = broadcast).  Joins replay
join_set (lane tile (s, s'), hiho table).  Prints wavefronts per point by phase; compare with ncu
l1tex__data_pipe_lsu_wavefronts_mem_shared.sum / points.
usage: python tools/bank_model.py N [grp...]"""
import math
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2511_19456_b200.gen.lower import aos_slot, hiho_table  # noqa: E402
from paper_2511_19456_b200.gen.lower_bg import group_strides, leaf_mu, make_bg_plan  # noqa: E402


def wavefronts(acc):
    """acc: per lane (lane index, byte address, size) of one warp instruction.  Accesses wider than 4 bytes
    are served in phases of 128 / size lanes (quarter warps for 16 B, half warps for 8 B); a phase with
    active lanes costs max over banks of the distinct words requested (>= 1)."""
    if not acc:
        return 0
    size = acc[0][2]
    per = 128 // max(4, size)
    phases = defaultdict(list)
    for l, a, n in acc:
        phases[l // per].append((a, n))
    tot = 0
    for ph in phases.values():
        banks = defaultdict(set)
        for a, n in ph:
            for w in range(a // 4, (a + n) // 4):
                banks[w % 32].add(w)
        tot += max(len(s) for s in banks.values())
    return tot


def task_accesses(plan, d, K, F, kind, sp):
    """Ordered list of (bytes offset within the point slot, size) of one task, one entry per instruction."""
    acc = []

    def aos(off):
        return [(8 * aos_slot(off, c, sp), 16) for c in range(4)]

    def eps(off, lam1=False):
        return [(8 * off, 16), (8 * (off + 2), 8)] if not lam1 else [(8 * off, 16)]

    leaf = kind >= 2
    nh = plan.n_hi if kind == 2 else plan.n_ho
    M = 1 << F
    if F == 0:
        for q in range(K):
            acc += eps(d[3 + 2 * q]) + aos(d[2 + 2 * q])
        if kind != 3:
            acc += [(8 * d[0], 16), (8 * (d[0] + 2), 16), (8 * (d[0] + 4), 8)]
        if leaf:
            acc += [(8 * (d[1] + c * nh * 2), 16) for c in range(4)]
        else:
            acc += [(8 * aos_slot(d[1], c, sp), 16) for c in range(4)]
        return acc
    st_out, st_fix, st_free = group_strides(K, F, math.comb(plan.N, K), math.comb(plan.N, K - 1) if K > 1 else 0)
    for p in range(K - F, K):
        acc += eps(d[3 + 2 * p]) + eps(d[3 + 2 * p] + 4, True)
        for mr in range(M // 2):
            acc += aos(d[2 + 2 * p] + mr * st_free * sp)
    for p in range(K - F):
        acc += eps(d[3 + 2 * p])
        for mu in range(M):
            acc += aos(d[2 + 2 * p] + mu * st_fix * sp)
    if kind != 3:
        acc += [(8 * d[0], 16), (8 * (d[0] + 2), 16), (8 * (d[0] + 4), 8)]
    for mu in range(M):
        if leaf:
            o = leaf_mu(d[1], d[2 + 2 * K], mu, K, F)
            acc += [(8 * (o + c * nh * 2), 16) for c in range(4)]
        else:
            acc += [(8 * aos_slot(d[1] + mu * st_out * sp, c, sp), 16) for c in range(4)]
    return acc


def replay_phase(plan, groups, ppw, stride):
    """groups: list of (tasks, K, F, kind, OFF).  Returns wavefronts per warp for this phase (all points of
    the warp run the same tasks at their own slot base)."""
    G = plan.G
    lanes_per_warp = min(32, G)
    nwarps = max(1, G // 32)
    tot = 0
    for tasks, K, F, kind, off in groups:
        trips = (len(tasks) + G - 1) // G
        for w in range(nwarps):
            for k in range(trips):
                per_lane = []
                for l in range(32):
                    pb, g = (l // G, l % G) if G < 32 else (0, w * 32 + l)
                    t = (g + G - off) % G + k * G
                    if t < len(tasks):
                        per_lane.append((l, pb, task_accesses(plan, tasks[t], K, F, kind, plan.sp)))
                if not per_lane:
                    continue
                n_ins = len(per_lane[0][2])
                for i in range(n_ins):
                    tot += wavefronts([(l, pb * stride * 8 + a[i][0], a[i][1]) for l, pb, a in per_lane])
    return tot


def model(plan):
    from paper_2511_19456_b200.gen.emit import lane_offset
    G = plan.G
    ppw = max(1, 32 // G)
    stride = plan.stride
    out = {}
    # interior levels
    prev_count, prev_k, tot = 0, None, 0
    for kind, K, t, F in plan.levels:
        off = lane_offset(prev_count, G) if (kind == "out" and prev_k == K) else 0
        tot += replay_phase(plan, [(t, K, F, 0 if kind == "in" else 1, off)], ppw, stride)
        prev_count, prev_k = len(t), K
    out["interior"] = tot
    B = plan.setb
    tot = 0
    for s0 in range(0, len(plan.sets), B):
        tin = [d for q in range(B) for d in plan.set_in[s0 + q]]
        tout = [d for q in range(B) for d in plan.set_out[s0 + q]]
        tot += replay_phase(plan, [(tin, plan.j, plan.f_in, 2, 0),
                                   (tout, plan.N - plan.j, plan.f_out, 3, lane_offset(len(tin), G))], ppw, stride)
    out["leaves"] = tot
    # joins (join_set, AS/SB = 1 shape: per component 2 phi + 2 ubar loads per lane)
    hh = hiho_table(plan)
    tot = 0
    nwarps = max(1, G // 32)
    for si in range(plan.n_sets_real):
        lb = si % B
        base = lb * plan.layout["LEAFB"]
        for w in range(nwarps):
            for c in range(4):
                for which in range(4):
                    acc = []
                    for l in range(32):
                        pb, g = (l // G, l % G) if G < 32 else (0, w * 32 + l)
                        x = hh[si * G + g]
                        h0, h1, o0, o1 = x & 255, (x >> 8) & 255, (x >> 16) & 255, x >> 24
                        if which < 2:
                            o = plan.layout["PHI"] + base + c * plan.n_hi * 2 + (h0 if which == 0 else h1)
                        else:
                            o = plan.layout["UBL"] + base + c * plan.n_ho * 2 + (o0 if which == 2 else o1)
                        acc.append((l, pb * stride * 8 + 8 * o, 16))
                    tot += wavefronts(acc)
    out["join"] = tot
    return {k: v / ppw for k, v in out.items()}


if __name__ == "__main__":
    N = int(sys.argv[1])
    kw = {}
    if len(sys.argv) > 2:
        kw["grp"] = tuple(int(x) for x in sys.argv[2].split(","))
    if len(sys.argv) > 3:
        kw["setb"] = int(sys.argv[3])
    p = make_bg_plan(N, **kw)
    m = model(p)
    print(N, kw, {k: round(v) for k, v in m.items()}, "total", round(sum(m.values())))
