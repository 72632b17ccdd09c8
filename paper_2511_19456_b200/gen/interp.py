"""Reference interpreter of a lowered Plan (build-time check of the generator).

Executes the generated task tables on a flat per-point "shared memory" array
with exactly the offsets the CUDA kernel uses, so a wrong table entry fails
here (tests/test_generator.py compares it with the oracle) before any GPU
run.  It mirrors the device arithmetic of csrc/qed_device.cuh in numpy; it is
part of the generator's test surface, not of the product path.
"""
from __future__ import annotations

import math

import numpy as np

from .lower import Plan, aos_slot, hiho_table, hs_table

ALPHA = 1 / 137.035999084


def _eslash_col(e, v):
    e1, e2, e3 = e
    a, b, c, d = v
    return np.array([-(e3 * c + (e1 - 1j * e2) * d), -((e1 + 1j * e2) * c - e3 * d),
                     e3 * a + (e1 - 1j * e2) * b, (e1 + 1j * e2) * a - e3 * b])


def _eslash_row(e, v):
    e1, e2, e3 = e
    a, b, c, d = v
    return np.array([c * e3 + d * (e1 + 1j * e2), c * (e1 - 1j * e2) - d * e3,
                     -(a * e3 + b * (e1 + 1j * e2)), -(a * (e1 - 1j * e2) - b * e3)])


def _prop_col(mk, v):
    qp, qm, qx, qy, qz = mk[:5]
    a, b, c, d = v
    Kc = (qz * c + (qx - 1j * qy) * d, (qx + 1j * qy) * c - qz * d)
    Ka = (qz * a + (qx - 1j * qy) * b, (qx + 1j * qy) * a - qz * b)
    return np.array([qp * a - Kc[0], qp * b - Kc[1], Ka[0] + qm * c, Ka[1] + qm * d])


def _prop_row(mk, v):
    qp, qm, qx, qy, qz = mk[:5]
    a, b, c, d = v
    # (t, b) [[Qp, -K], [K, Qm]] = (Qp t + bK, -tK + Qm b); (x, y)K = (x qz + y(qx+iqy), x(qx-iqy) - y qz)
    bK = (c * qz + d * (qx + 1j * qy), c * (qx - 1j * qy) - d * qz)
    tK = (a * qz + b * (qx + 1j * qy), a * (qx - 1j * qy) - b * qz)
    return np.array([qp * a + bK[0], qp * b + bK[1], -tK[0] + qm * c, -tK[1] + qm * d])


def _join_offsets(hiho, si, G, h, N):
    """Leaf-row offsets (in doubles, swizzle applied) of amplitude index h for subset si, from the
    per-(subset, lane) table the kernels read (lane g = the photon-polarisation bits of h)."""
    w = hiho[si * G + ((h >> 1) & (G - 1))]
    s, sp = h & 1, (h >> (N + 1)) & 1
    return (w >> (8 * s)) & 255, (w >> (16 + 8 * sp)) & 255


def _join_offsets_hs(tab, plan, si, h):
    """The same offsets from the two-half table (lower.hs_table): lane g' = lam_0..lam_{N-2}, tile
    (s, s', lam_x), x = N - 1."""
    N, x = plan.N, plan.N - 1
    gp = (h >> 1) & ((1 << x) - 1)
    s, sp, lx = h & 1, (h >> (N + 1)) & 1, (h >> (1 + x)) & 1
    wp, wu = tab[2 * (si * (plan.G // 2) + gp)], tab[2 * (si * (plan.G // 2) + gp) + 1]
    if x in plan.sets[si]:
        return (wp >> (8 * (2 * lx + s))) & 255, (wu >> (8 * sp)) & 255
    return (wp >> (8 * s)) & 255, (wu >> (8 * (2 * lx + sp))) & 255


MMA_BIT = {"L0": ("col", 1), "L1": ("col", 2), "TC": ("col", 3), "L3": ("row", 1), "L4": ("row", 2), "TR": ("row", 3)}


def _mma_swap(acc, swap):
    """Exchange of the two accumulator bits of one subset transition (qed_eval_kernel.cuh mma_swap_*)."""
    pa, pc = swap
    (_, ba), (_, bc) = MMA_BIT[pa], MMA_BIT[pc]
    R, C = acc.shape
    new = np.empty_like(acc)
    for r in range(R):
        for c in range(C):
            r2 = (r & ~(1 << bc)) | (((c >> ba) & 1) << bc)
            c2 = (c & ~(1 << ba)) | (((r >> bc) & 1) << ba)
            new[r][c] = acc[r2][c2]
    return new


def _mma_amp(plan, acc):
    """Accumulator (row, col) -> amplitude of its configuration under the last subset's assignment."""
    N = plan.N
    R, C = acc.shape
    assign = plan.mma_assign[-1] if not hasattr(plan, "n_sets_real") else plan.mma_assign[plan.n_sets_real - 1]
    amp = np.zeros(plan.H, dtype=complex)
    for r in range(R):
        for c in range(C):
            h = (c & 1) | ((r & 1) << (N + 1))
            for x, pos in assign.items():
                side, b = MMA_BIT[pos]
                h |= (((c if side == "col" else r) >> b) & 1) << (1 + x)
            amp[h] = acc[r][c]
    return amp


def _mma_join(plan, sm, run, get_aos_sp8):
    """The tensor-core join of qed_eval_kernel.cuh (join_mma) on one point: per subset (Johnson order),
    C[row][col] += sum_c ubar_tau[row][c] phi_sigma[col][c] over every diagram (sigma, tau), with rows / cols
    the accumulator-layout slots (lower.mma_slot); between subsets the accumulator bits of the exchanged
    positions are swapped (mma_swap); at the end the last subset's assignment maps (row, col) to the
    configuration.  Returns amplitudes in the internal index (s | lam_i << (1+i) | s' << (N+1))."""
    N, L = plan.N, plan.layout
    R, C = plan.n_ho, plan.n_hi
    acc = np.zeros((R, C), dtype=complex)
    TCH = getattr(plan, "tau_chunks", 1)
    NT = plan.n_tau // TCH
    for si, A in enumerate(plan.sets):
        stages = plan.set_stages[si]
        for stage in stages[:len(stages) - TCH + 1]:      # recomputed levels and leaf chunk 0 (phi + ubar)
            for kind, tasks in stage:
                run(kind, tasks)
        for c in range(TCH):
            if c:
                for kind, tasks in stages[len(stages) - TCH + c]:
                    run(kind, tasks)
            U = np.array([[get_aos_sp8(L["UBL"] + (t * R + r) * 8) for r in range(R)] for t in range(NT)])
            P = np.array([[get_aos_sp8(L["PHI"] + (s_ * C + c_) * 8) for c_ in range(C)] for s_ in range(plan.n_sigma)])
            for t in range(NT):
                for s_ in range(plan.n_sigma):
                    acc += U[t] @ P[s_].T
        if si + 1 < len(plan.sets):
            pa, pc = plan.mma_swaps[si]
            (_, ba), (_, bc) = MMA_BIT[pa], MMA_BIT[pc]
            new = np.empty_like(acc)
            for r in range(R):
                for c in range(C):
                    r2 = (r & ~(1 << bc)) | (((c >> ba) & 1) << bc)
                    c2 = (c & ~(1 << ba)) | (((r >> bc) & 1) << ba)
                    new[r][c] = acc[r2][c2]
            acc = new
    assign = plan.mma_assign[-1]
    amp = np.zeros(plan.H, dtype=complex)
    for r in range(R):
        for c in range(C):
            h = (c & 1) | ((r & 1) << (N + 1))
            for x, pos in assign.items():
                side, b = MMA_BIT[pos]
                h |= (((c if side == "col" else r) >> b) & 1) << (1 + x)
            amp[h] = acc[r][c]
    return amp


def eval_point(plan: Plan, mom: np.ndarray, n_in_ph: int) -> np.ndarray:
    """All helicity amplitudes (external bit order, with e^N) at one point, via the tables."""
    N, L = plan.N, plan.layout
    sm = np.zeros(plan.stride + 8)            # real doubles, exactly as the device sees them

    def put_aos(off, v):
        for c in range(4):
            o = aos_slot(off, c, plan.sp)
            sm[o], sm[o + 1] = v[c].real, v[c].imag

    def get_aos(off):
        return np.array([complex(sm[aos_slot(off, c, plan.sp)], sm[aos_slot(off, c, plan.sp) + 1]) for c in range(4)])

    def put_leaf(nh, off, v):     # off: the descriptor's leaf offset (component 0)
        if getattr(plan, "mma", False):   # AoS leaves, 64-byte pitch with the XOR swizzle
            for c in range(4):
                o = aos_slot(off, c, 8)
                sm[o], sm[o + 1] = v[c].real, v[c].imag
            return
        for c in range(4):
            o = off + c * nh * 2
            sm[o], sm[o + 1] = v[c].real, v[c].imag

    hiho = hiho_table(plan)

    def get_leaf_off(base, nh, row, o2):
        o = base + row * 4 * nh * 2 + o2
        return np.array([complex(sm[o + c * nh * 2], sm[o + c * nh * 2 + 1]) for c in range(4)])

    photon_particle = [1 + i if i < n_in_ph else n_in_ph + 2 + (i - n_in_ph) for i in range(N)]
    sign = [1.0 if i < n_in_ph else -1.0 for i in range(N)]
    p, pp = mom[0], mom[n_in_ph + 1]
    for i in range(N):
        k = mom[photon_particle[i]]
        kperp = math.hypot(k[1], k[2])
        kn = math.sqrt(kperp * kperp + k[3] * k[3])
        ct, st = k[3] / kn, kperp / kn
        cf, sf = (k[1] / kperp, k[2] / kperp) if kperp > 0 else (1.0, 0.0)
        sm[L["EPS"] + i * 8: L["EPS"] + i * 8 + 3] = (ct * cf, ct * sf, -st)
        sm[L["EPS"] + i * 8 + 4: L["EPS"] + i * 8 + 7] = (-sf, cf, 0.0)
    n = math.sqrt(p[0] + 1)
    put_aos(L["U"], np.array([n, 0, p[3] / n, (p[1] + 1j * p[2]) / n]))
    put_aos(L["U"] + plan.sp, np.array([0, n, (p[1] - 1j * p[2]) / n, -p[3] / n]))
    n = math.sqrt(pp[0] + 1)
    put_aos(L["UB"], np.array([n, 0, -pp[3] / n, -(pp[1] - 1j * pp[2]) / n]))
    put_aos(L["UB"] + plan.sp, np.array([0, n, -(pp[1] + 1j * pp[2]) / n, pp[3] / n]))
    for m in range(1, (1 << N) - 1):
        Q = p.copy()
        for i in range(N):
            if m >> i & 1:
                Q = Q + sign[i] * mom[photon_particle[i]]
        inv = 1 / (Q[0] ** 2 - Q[1] ** 2 - Q[2] ** 2 - Q[3] ** 2 - 1)
        sm[L["MASK"] + m * 6: L["MASK"] + m * 6 + 5] = ((Q[0] + 1) * inv, (1 - Q[0]) * inv,
                                                        Q[1] * inv, Q[2] * inv, Q[3] * inv)

    def eps(off):
        return sm[off: off + 3]

    def mask(off):
        return sm[off: off + 5]

    def run(kind, tasks):
        for par, e, mk, out in tasks:
            if kind == "vs_col":
                put_aos(out, _prop_col(mask(mk), _eslash_col(eps(e), get_aos(par))))
            elif kind == "vs_row":
                put_aos(out, _prop_row(mask(mk), _eslash_row(eps(e), get_aos(par))))
            elif kind == "phi":
                put_leaf(plan.n_hi, out, _prop_col(mask(mk), _eslash_col(eps(e), get_aos(par))))
            elif kind == "ub":
                put_leaf(plan.n_ho, out, _eslash_row(eps(e), get_aos(par)))

    for tasks in plan.in_levels:
        run("vs_col", tasks)
    for tasks in plan.out_levels:
        run("vs_row", tasks)
    H = plan.H
    amp = np.zeros(H, dtype=complex)      # internal index: s | lam_i << (1+i) | s' << (N+1)
    if getattr(plan, "mma", False):
        amp = _mma_join(plan, sm, run, get_aos_sp8=lambda off: np.array(
            [complex(sm[aos_slot(off, c, 8)], sm[aos_slot(off, c, 8) + 1]) for c in range(4)]))
    for si, A in enumerate(plan.sets if not getattr(plan, "mma", False) else []):
        for stage in plan.set_stages[si]:
            for kind, tasks in stage:
                run(kind, tasks)
        for h in range(H):
            oi, oo = _join_offsets(hiho, si, plan.G, h, N)
            for a in range(plan.n_sigma):
                phi = get_leaf_off(L["PHI"], plan.n_hi, a, oi)
                for b in range(plan.n_tau):
                    amp[h] += get_leaf_off(L["UBL"], plan.n_ho, b, oo) @ phi
    e_n = math.sqrt(4 * math.pi * ALPHA) ** N
    out = np.zeros(H, dtype=complex)
    e_out = n_in_ph + 1
    for h in range(H):
        hx = (h & 1) | (((h >> (N + 1)) & 1) << e_out)
        for i in range(N):
            hx |= ((h >> (1 + i)) & 1) << photon_particle[i]
        out[hx] = e_n * amp[h]
    return out


def expand_group(d, K: int, F: int, sp: int, leaf: bool, N: int) -> list[list[int]]:
    """The 2^F single-node descriptors [mask, out, (parent, eps) x K] of grouped task d, by the kernel's
    offset rules (qed_eval_kernel.cuh BGGroupFn; free photons = the last F of the node set)."""
    from .lower_bg import group_strides, leaf_mu
    if F == 0:
        return [list(d[:2 + 2 * K])]
    so, sf, sr = group_strides(K, F, math.comb(N, K), math.comb(N, K - 1) if K > 1 else 0)
    res = []
    for mu in range(1 << F):
        e = [d[0], leaf_mu(d[1], d[2 + 2 * K], mu, K, F) if leaf else d[1] + so * sp * mu]
        for p in range(K):
            if p >= K - F:
                q = p - (K - F)
                mr = (mu & ((1 << q) - 1)) | ((mu >> (q + 1)) << q)
                e += [d[2 + 2 * p] + sr * sp * mr, d[3 + 2 * p] + 4 * ((mu >> q) & 1)]
            else:
                e += [d[2 + 2 * p] + sf * sp * mu, d[3 + 2 * p]]
        res.append(e)
    return res


def eval_point_bg(plan, mom: np.ndarray, n_in_ph: int) -> np.ndarray:
    """Berends-Giele plan (gen/lower_bg.py) executed with the device layout; returns amplitudes
    in external bit order with e^N (same contract as eval_point)."""
    N, L = plan.N, plan.layout
    sm = np.zeros(plan.stride + 8)

    def put_aos(off, v):
        for c in range(4):
            o = aos_slot(off, c, plan.sp)
            sm[o], sm[o + 1] = v[c].real, v[c].imag

    def get_aos(off):
        return np.array([complex(sm[aos_slot(off, c, plan.sp)], sm[aos_slot(off, c, plan.sp) + 1]) for c in range(4)])

    LB = L["LEAFB"]

    def put_leaf(nh, off, v):     # off: the descriptor's leaf offset (component 0)
        if getattr(plan, "mma", False):   # AoS leaves, 64-byte pitch with the XOR swizzle
            for c in range(4):
                o = aos_slot(off, c, 8)
                sm[o], sm[o + 1] = v[c].real, v[c].imag
            return
        for c in range(4):
            o = off + c * nh * 2
            sm[o], sm[o + 1] = v[c].real, v[c].imag

    hiho = hiho_table(plan)
    hst = hs_table(plan) if getattr(plan, "hs", 1) == 2 else None

    def get_leaf_off(base, nh, o2, lb=0):
        o = base + lb * LB + o2
        return np.array([complex(sm[o + c * nh * 2], sm[o + c * nh * 2 + 1]) for c in range(4)])

    photon_particle = [1 + i if i < n_in_ph else n_in_ph + 2 + (i - n_in_ph) for i in range(N)]
    sign = [1.0 if i < n_in_ph else -1.0 for i in range(N)]
    p, pp = mom[0], mom[n_in_ph + 1]
    for i in range(N):
        k = mom[photon_particle[i]]
        kperp = math.hypot(k[1], k[2])
        kn = math.sqrt(kperp * kperp + k[3] * k[3])
        ct, st = k[3] / kn, kperp / kn
        cf, sf = (k[1] / kperp, k[2] / kperp) if kperp > 0 else (1.0, 0.0)
        sm[L["EPS"] + i * 8: L["EPS"] + i * 8 + 3] = (ct * cf, ct * sf, -st)
        sm[L["EPS"] + i * 8 + 4: L["EPS"] + i * 8 + 7] = (-sf, cf, 0.0)
    n = math.sqrt(p[0] + 1)
    put_aos(L["U"], np.array([n, 0, p[3] / n, (p[1] + 1j * p[2]) / n]))
    put_aos(L["U"] + plan.sp, np.array([0, n, (p[1] - 1j * p[2]) / n, -p[3] / n]))
    n = math.sqrt(pp[0] + 1)
    put_aos(L["UB"], np.array([n, 0, -pp[3] / n, -(pp[1] - 1j * pp[2]) / n]))
    put_aos(L["UB"] + plan.sp, np.array([0, n, -(pp[1] + 1j * pp[2]) / n, pp[3] / n]))
    for m in range(1, (1 << N) - 1):
        Q = p.copy()
        for i in range(N):
            if m >> i & 1:
                Q = Q + sign[i] * mom[photon_particle[i]]
        inv = 1 / (Q[0] ** 2 - Q[1] ** 2 - Q[2] ** 2 - Q[3] ** 2 - 1)
        sm[L["MASK"] + m * 6: L["MASK"] + m * 6 + 5] = ((Q[0] + 1) * inv, (1 - Q[0]) * inv,
                                                        Q[1] * inv, Q[2] * inv, Q[3] * inv)

    def vsum(d, row):
        K = (len(d) - 2) // 2
        acc = np.zeros(4, complex)
        for q in range(K):
            par, e = d[2 + 2 * q], d[3 + 2 * q]
            f = _eslash_row if row else _eslash_col
            acc = acc + f(sm[e: e + 3], get_aos(par))
        return acc

    SPP = plan.sp

    def nodes(tasks, K, F, leaf=False):
        return [e for d in tasks for e in expand_group(d, K, F, SPP, leaf, N)]

    for kind, K, tasks, F in plan.levels:
        for d in nodes(tasks, K, F):
            if kind == "in":
                put_aos(d[1], _prop_col(sm[d[0]: d[0] + 5], vsum(d, False)))
            else:
                put_aos(d[1], _prop_row(sm[d[0]: d[0] + 5], vsum(d, True)))
    H = plan.H
    amp = np.zeros(H, dtype=complex)
    for si, A in enumerate(plan.sets):
        lb = si % plan.setb
        if lb == 0:
            for sj in range(si, si + plan.setb):
                for stage in plan.set_stages[sj]:
                    for kind, K, tasks, F in stage:
                        for d in nodes(tasks, K, F):
                            if kind == "in":
                                put_aos(d[1], _prop_col(sm[d[0]: d[0] + 5], vsum(d, False)))
                            else:
                                put_aos(d[1], _prop_row(sm[d[0]: d[0] + 5], vsum(d, True)))
            for sj in range(si, si + plan.setb):
                for d in nodes(plan.set_in[sj], plan.j, plan.f_in, True):
                    put_leaf(plan.n_hi, d[1], _prop_col(sm[d[0]: d[0] + 5], vsum(d, False)))
                for d in nodes(plan.set_out[sj], N - plan.j, plan.f_out, True):
                    put_leaf(plan.n_ho, d[1], vsum(d, True))
        if si >= plan.n_sets_real:      # padding subset of a ragged last batch
            continue
        if getattr(plan, "mma", False):
            R, C = plan.n_ho, plan.n_hi

            def aos8(off):
                return np.array([complex(sm[aos_slot(off, c, 8)], sm[aos_slot(off, c, 8) + 1]) for c in range(4)])
            U = np.array([aos8(L["UBL"] + lb * LB + r * 8) for r in range(R)])
            P = np.array([aos8(L["PHI"] + lb * LB + c * 8) for c in range(C)])
            mma_acc = (mma_acc if si else np.zeros((R, C), dtype=complex)) + U @ P.T
            if si + 1 < plan.n_sets_real:
                mma_acc = _mma_swap(mma_acc, plan.mma_swaps[si])
            if si + 1 == plan.n_sets_real:
                amp[:] = _mma_amp(plan, mma_acc)
            continue
        for h in range(H):
            if hst is not None:
                oi, oo = _join_offsets_hs(hst, plan, si, h)
            else:
                oi, oo = _join_offsets(hiho, si, plan.G, h, N)
            amp[h] += get_leaf_off(L["UBL"], plan.n_ho, oo, lb) @ get_leaf_off(L["PHI"], plan.n_hi, oi, lb)
    e_n = math.sqrt(4 * math.pi * ALPHA) ** N
    out = np.zeros(H, dtype=complex)
    e_out = n_in_ph + 1
    for h in range(H):
        hx = (h & 1) | (((h >> (N + 1)) & 1) << e_out)
        for i in range(N):
            hx |= ((h >> (1 + i)) & 1) << photon_particle[i]
        out[hx] = e_n * amp[h]
    return out
