"""Pins for the parity oracle (oracle/qed_oracle.c) against what the paper and
the mathematics fix -- never against the oracle itself.

Each test names the passage or identity it follows.  Together they are
chosen so that a plausible slip in the oracle (a dropped propagator, a wrong
sign of an outgoing photon momentum, a transposed gamma matrix, a wrong
spinor, a wrong coupling power, a wrong averaging factor) fails at least one:

* gamma algebra / spinors / polarisations: textbook identities
* n = 1 unpolarised: Peskin & Schroeder eq. (5.87), any frame     (coupling e^4, averaging)
* n = 1 polarised: Klein-Nishina, lab frame                         (photon pol. basis)
* any n, spin-summed: trace identity in the CHIRAL basis           (spinors, basis-independence)
* any n, fully summed: Feynman-gauge polarisation sum               (pol. sum completeness)
* any n: Ward identity eps_i -> k_i                                  (propagators, momentum signs)
* any n: Lorentz invariance, Bose symmetry                           (frame, ordering)
* n = 2 -> 1: soft-photon (eikonal) limit                            (relative normalisation e^2)
* (n+1)! diagram count (§3.1)
* double vs long double (conditioning)
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synthetic

ALPHA = 1 / 137.035999084          # CODATA 2018
E_CHARGE = math.sqrt(4 * math.pi * ALPHA)
G = np.diag([1.0, -1.0, -1.0, -1.0])


def mdot(a, b):
    return a[..., 0] * b[..., 0] - (a[..., 1:] * b[..., 1:]).sum(-1)


# ----------------------------------------------------------------- algebra


def test_gamma_anticommutator():
    g = oracle.gammas()
    for mu in range(4):
        for nu in range(4):
            ac = g[mu] @ g[nu] + g[nu] @ g[mu]
            assert np.abs(ac - 2 * G[mu, nu] * np.eye(4)).max() < 1e-14


def _slash_dirac(a):
    g = oracle.gammas()
    return g[0] * a[0] - g[1] * a[1] - g[2] * a[2] - g[3] * a[3]


def test_spinor_identities():
    rng = np.random.default_rng(11)
    g0 = oracle.gammas()[0]
    for _ in range(20):
        pv = rng.normal(size=3) * rng.choice([0.1, 1, 10])
        p = np.array([math.sqrt(1 + pv @ pv), *pv])
        us = [oracle.spinor_u(p, s) for s in (0, 1)]
        ubs = [oracle.spinor_ubar(p, s) for s in (0, 1)]
        for s in (0, 1):
            assert abs(ubs[s] @ us[s] - 2.0) < 1e-12                      # ubar u = 2m
            assert np.abs(ubs[s] - us[s].conj() @ g0).max() < 1e-14        # ubar = u^dag g0
            assert np.abs((_slash_dirac(p) - np.eye(4)) @ us[s]).max() < 1e-11 * p[0]  # Dirac eq.
        assert abs(ubs[0] @ us[1]) < 1e-12
        comp = sum(np.outer(us[s], ubs[s]) for s in (0, 1))                # sum_s u ubar = pslash + m
        assert np.abs(comp - (_slash_dirac(p) + np.eye(4))).max() < 1e-11 * p[0]


@pytest.mark.parametrize("kdir", ["random", "+z", "-z", "x"])
def test_polarisation_vectors(kdir):
    rng = np.random.default_rng(3)
    for _ in range(10):
        if kdir == "random":
            kv = rng.normal(size=3)
        else:
            kv = {"+z": np.array([0, 0, 1.0]), "-z": np.array([0, 0, -1.0]), "x": np.array([1.0, 0, 0])}[kdir]
            kv = kv * rng.uniform(0.1, 10)
        k = np.array([np.linalg.norm(kv), *kv])
        e1, e2 = oracle.polvec(k, 0), oracle.polvec(k, 1)
        for e in (e1, e2):
            assert e[0] == 0
            assert abs(mdot(e, k)) < 1e-14 * k[0]
            assert abs(mdot(e, e) + 1) < 1e-14
        assert abs(mdot(e1, e2)) < 1e-14


# ----------------------------------------------------------------- Klein-Nishina (n = 1)


def _kn_unpolarised(m):
    """P&S eq. (5.87): 1/4 sum |M|^2 = 2e^4 [p.k'/p.k + p.k/p.k' + 2m^2(1/p.k - 1/p.k') + m^4(1/p.k - 1/p.k')^2]"""
    p, k, kp = m[:, 0], m[:, 1], m[:, 3]
    pk, pkp = mdot(p, k), mdot(p, kp)
    d = 1 / pk - 1 / pkp
    return 2 * E_CHARGE ** 4 * (pkp / pk + pk / pkp + 2 * d + d * d)


def test_klein_nishina_unpolarised_lab_and_boosted():
    mom = synthetic.compton_lab(512, seed=1)
    # lab frame: exact to rounding.  Boosted frame: the boost itself rounds the inputs
    # (conservation/on-shellness broken at ~1e-16 E), amplified by E^2/p.k for soft photons;
    # the long-double oracle shows the same 3e-11, so the bound there is an input bound.
    for m, tol in ((mom, 1e-12), (synthetic.boost_rotate(mom, seed=5), 1e-10)):
        mm = m.numpy()
        got = oracle.msq(1, 1, mm)
        ref = _kn_unpolarised(mm)
        assert np.max(np.abs(got / ref - 1)) < tol


def test_klein_nishina_polarised_lab():
    """1/2 sum_{s,s'} |M|^2 = e^4 [w'/w + w/w' - 2 + 4 (eps.eps')^2]  (electron at rest)."""
    mm = synthetic.compton_lab(256, seed=4).numpy()
    w, wp = mm[:, 1, 0], mm[:, 3, 0]
    for lam in (0, 1):
        for lamp in (0, 1):
            got = oracle.msq(1, 1, mm, spec=[-1, lam, -1, lamp])
            ee = np.array([oracle.polvec(mm[i, 1], lam)[1:] @ oracle.polvec(mm[i, 3], lamp)[1:]
                           for i in range(len(mm))])
            ref = E_CHARGE ** 4 * (wp / w + w / wp - 2 + 4 * ee ** 2)
            assert np.max(np.abs(got / ref - 1)) < 1e-11


# ----------------------------------------------------------------- trace identity (chiral basis)

SIG = [np.array([[0, 1], [1, 0]], complex), np.array([[0, -1j], [1j, 0]]), np.array([[1, 0], [0, -1]], complex)]
Z2, I2 = np.zeros((2, 2)), np.eye(2)
GCH = [np.block([[Z2, I2], [I2, Z2]]).astype(complex)] + [np.block([[Z2, s], [-s, Z2]]) for s in SIG]


def _slash_ch(a):
    return GCH[0] * a[0] - GCH[1] * a[1] - GCH[2] * a[2] - GCH[3] * a[3]


def _gamma_chain_sum(q, p, eps):
    """Gamma = sum_pi epsslash_{pi N} S(Q_{N-1}) ... epsslash_{pi 1} as a 4x4 matrix (chiral basis)."""
    N = len(q)
    tot = np.zeros((4, 4), complex)
    for perm in itertools.permutations(range(N)):
        M = np.eye(4, dtype=complex)
        Q = p.copy()
        for l, i in enumerate(perm):
            M = _slash_ch(eps[i]) @ M
            if l < N - 1:
                Q = Q + q[i]
                M = (_slash_ch(Q) + np.eye(4)) @ M / (mdot(Q, Q) - 1)
        tot += M
    return tot


@pytest.mark.parametrize("n", [1, 2, 3])
def test_trace_identity_spin_sum(n):
    """sum_{s,s'} |ubar' Gamma u|^2 = Tr[(p'slash + m) Gamma (pslash + m) g0 Gamma^dag g0]."""
    mm = synthetic.rambo_cm(n, 6, sqrt_s=5.0, seed=20 + n).numpy()
    N = n + 1
    g0 = GCH[0]
    for pt in mm:
        p, pp = pt[0], pt[2]
        ks = [pt[1]] + [pt[3 + i] for i in range(n)]
        q = [ks[0]] + [-k for k in ks[1:]]
        for lam_bits in range(1 << N):
            lams = [(lam_bits >> i) & 1 for i in range(N)]
            eps = [oracle.polvec(ks[i], lams[i]) for i in range(N)]
            Gm = _gamma_chain_sum(q, p, eps)
            tr = np.trace((_slash_ch(pp) + np.eye(4)) @ Gm @ (_slash_ch(p) + np.eye(4)) @ g0 @ Gm.conj().T @ g0)
            ref = E_CHARGE ** (2 * N) * tr.real
            spec = [-1, lams[0], -1] + lams[1:]
            got = 2 * oracle.msq(1, n, pt[None], spec=spec)[0]   # undo the 1/2 initial-spin average
            assert abs(got / ref - 1) < 1e-11


# ----------------------------------------------------------------- Feynman-gauge polarisation sum


@pytest.mark.parametrize("n", [1, 2])
def test_feynman_gauge_polarisation_sum(n):
    """sum over physical pols = sum_{mu_i} prod(-g_{mu_i mu_i}) |M(eps_i = e_{mu_i})|^2 (valid by
    the Ward identity); independent of how the physical basis is built."""
    mm = synthetic.rambo_cm(n, 4, sqrt_s=5.0, seed=40 + n).numpy()
    N = n + 1
    for pt in mm:
        p, pp = pt[0], pt[2]
        ks = [pt[1]] + [pt[3 + i] for i in range(n)]
        q = np.array([ks[0]] + [-k for k in ks[1:]])
        rhs = 0.0
        for s in (0, 1):
            u = oracle.spinor_u(p, s)
            for sp in (0, 1):
                ub = oracle.spinor_ubar(pp, sp)
                for mus in itertools.product(range(4), repeat=N):
                    eps = np.zeros((N, 4), complex)
                    for i, mu in enumerate(mus):
                        eps[i, mu] = 1.0
                    a, nd = oracle.diagram_sum_explicit(q, p, u, ub, eps)
                    rhs += np.prod([-G[mu, mu] for mu in mus]) * abs(a) ** 2
        rhs *= E_CHARGE ** (2 * N)
        got = 4 * oracle.msq(1, n, pt[None])[0]       # undo the 1/4 initial average
        assert abs(got / rhs - 1) < 1e-11


# ----------------------------------------------------------------- Ward identity


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_ward_identity(n):
    mm = synthetic.rambo_cm(n, 4, sqrt_s=5.0, seed=60 + n).numpy()
    N = n + 1
    for pt in mm:
        p, pp = pt[0], pt[2]
        ks = [pt[1]] + [pt[3 + i] for i in range(n)]
        q = np.array([ks[0]] + [-k for k in ks[1:]])
        u, ub = oracle.spinor_u(p, 0), oracle.spinor_ubar(pp, 1)
        eps_phys = np.array([oracle.polvec(k, 0) for k in ks], dtype=complex)
        for i in range(N):
            eps = eps_phys.copy()
            eps[i] = ks[i] / ks[i][0]
            a, _ = oracle.diagram_sum_explicit(q, p, u, ub, eps)
            # scale: the same diagrams with physical eps_i (O(1) for these kinematics)
            aref, _ = oracle.diagram_sum_explicit(q, p, u, ub, eps_phys)
            scale = max(abs(aref), 1e-3)
            assert abs(a) < 1e-12 * max(1.0, scale), (n, i, a, aref)


def test_ward_identity_detects_wrong_sign():
    """Self-check of the pin: flipping the sign of an outgoing photon's momentum in
    the propagators breaks gauge invariance by O(1)."""
    pt = synthetic.rambo_cm(2, 1, sqrt_s=5.0, seed=3).numpy()[0]
    ks = [pt[1], pt[3], pt[4]]
    q_bad = np.array([ks[0], ks[1], -ks[2]])
    u, ub = oracle.spinor_u(pt[0], 0), oracle.spinor_ubar(pt[2], 0)
    eps = np.array([oracle.polvec(k, 0) for k in ks], dtype=complex)
    eps[0] = ks[0] / ks[0][0]
    a, _ = oracle.diagram_sum_explicit(q_bad, pt[0], u, ub, eps)
    assert abs(a) > 1e-3


# ----------------------------------------------------------------- Lorentz invariance and Bose symmetry


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_lorentz_invariance(n):
    npts = {1: 64, 2: 32, 3: 16, 4: 4}[n]
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=80 + n)
    a = oracle.msq(1, n, mom.numpy())
    b = oracle.msq(1, n, synthetic.boost_rotate(mom, seed=9).numpy())
    assert np.max(np.abs(b / a - 1)) < 1e-10


@pytest.mark.parametrize("n", [2, 3])
def test_bose_symmetry(n):
    mom = synthetic.rambo_cm(n, 8, sqrt_s=5.0, seed=90 + n).numpy()
    perm = np.roll(np.arange(n), 1)
    mom2 = mom.copy()
    mom2[:, 3:] = mom[:, 3 + perm]
    a, b = oracle.msq(1, n, mom), oracle.msq(1, n, mom2)
    assert np.max(np.abs(b / a - 1)) < 1e-12
    # fixed configurations move with the photons: particle 3+i of mom2 is particle 3+perm[i] of mom
    A, B = oracle.amps(1, n, mom), oracle.amps(1, n, mom2)
    H = A.shape[1]
    for h in range(H):
        h2 = h & 0b111
        for i in range(n):
            h2 |= ((h >> (3 + perm[i])) & 1) << (3 + i)
        assert np.max(np.abs(B[:, h2] - A[:, h])) <= 1e-12 * np.max(np.abs(A))


# ----------------------------------------------------------------- soft-photon limit


def _soft_point(sqrt_s, d_hat, lam, n_hat):
    """e- gamma -> e- gamma1 gamma2 with gamma2 = lam (1, n_hat) soft; the hard pair is back to back
    along d_hat in its own rest frame.  lam = 0 gives the n = 1 point."""
    s = sqrt_s ** 2
    kin = (s - 1) / (2 * sqrt_s)
    p = np.array([(s + 1) / (2 * sqrt_s), 0, 0, -kin])
    k = np.array([kin, 0, 0, kin])
    k2 = lam * np.array([1.0, *n_hat])
    P = np.array([sqrt_s, 0, 0, 0]) - k2
    MP = math.sqrt(mdot(P, P))
    ps = (MP * MP - 1) / (2 * MP)
    pe = np.array([math.sqrt(1 + ps * ps), *(ps * d_hat)])
    pg = np.array([ps, *(-ps * d_hat)])
    beta = P[1:] / P[0]
    b2 = beta @ beta
    gam = 1 / math.sqrt(1 - b2)

    def boost(v):
        if b2 == 0:
            return v.copy()
        bp = beta @ v[1:]
        E = gam * (v[0] + bp)
        vec = v[1:] + ((gam - 1) * bp / b2 + gam * v[0]) * beta
        return np.array([E, *vec])

    return p, k, boost(pe), boost(pg), k2


def test_soft_photon_limit():
    """sum|M_{n=2}|^2 -> e^2 [2 p.p'/(p.k p'.k) - m^2/(p.k)^2 - m^2/(p'.k)^2] sum|M_{n=1}|^2 (error O(lam))."""
    d = np.array([0.3, -0.5, 0.81]); d /= np.linalg.norm(d)
    nh = np.array([-0.6, 0.2, 0.3]); nh /= np.linalg.norm(nh)
    p, k, pe, pg, _ = _soft_point(5.0, d, 0.0, nh)
    m1 = oracle.msq(1, 1, np.array([[p, k, pe, pg]]))[0]
    errs = []
    for lam in (1e-3, 1e-4):
        p, k, pe, pg, k2 = _soft_point(5.0, d, lam, nh)
        m2 = oracle.msq(1, 2, np.array([[p, k, pe, pg, k2]]))[0]
        eik = E_CHARGE ** 2 * (2 * mdot(p, pe) / (mdot(p, k2) * mdot(pe, k2)) - 1 / mdot(p, k2) ** 2
                               - 1 / mdot(pe, k2) ** 2)
        errs.append(abs(m2 / (eik * m1) - 1))
    assert errs[0] < 1e-2 and errs[1] < 1e-3 and errs[1] < errs[0] / 5, errs


# ----------------------------------------------------------------- counting and conditioning


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7])
def test_diagram_count_is_factorial(N):
    """(n+1)! orderings of the N = n+1 photons on the electron line (§3.1)."""
    rng = np.random.default_rng(N)
    q = rng.normal(size=(N, 4))
    eps = rng.normal(size=(N, 4)) + 0j
    _, nd = oracle.diagram_sum_explicit(q, np.array([3.0, 0.1, 0.2, 0.3]), np.ones(4, complex),
                                        np.ones(4, complex), eps)
    assert nd == math.factorial(N)


@pytest.mark.parametrize("n,sqrt_s", [(2, 1.5), (2, 1000.0), (3, 5.0), (3, 100.0)])
def test_double_vs_long_double(n, sqrt_s):
    mom = synthetic.rambo_cm(n, 16, sqrt_s=sqrt_s, seed=100 + n).numpy()
    a = oracle.msq(1, n, mom, kind="f64")
    b = oracle.msq(1, n, mom, kind="f80")
    assert np.max(np.abs(a / b - 1)) < 1e-12


def test_modes_consistent_with_amplitudes():
    """fixed / summed / averaged modes are the stated sums of |amp[h]|^2."""
    mom = synthetic.rambo_cm(2, 8, seed=5).numpy()
    A = oracle.amps(1, 2, mom)
    tot = oracle.msq(1, 2, mom)
    assert np.allclose(tot, 0.25 * (np.abs(A) ** 2).sum(1), rtol=1e-14)
    h = 0b10110
    fixed = oracle.msq(1, 2, mom, spec=[(h >> j) & 1 for j in range(5)])
    assert np.allclose(fixed, np.abs(A[:, h]) ** 2, rtol=1e-14)
