"""Pins for the oracle's FIXED-STATE conventions: which state label (0/1) means which
spinor and which polarisation vector.

The identity pins of test_oracle_pins.py hold under any relabelling of the basis
(lambda 0<->1, phi -> -phi, chi_up <-> chi_down).  The pins here do not: each one
fixes the label against a value written out by hand from the definition, or against
a covariant construction that does not go through the oracle's spinor code.

* eps(k, lambda): exact values for k along +x, +y, +z, -z and one generic k,
  evaluated by hand from SURVEY.md §8(c) item 4 (linear basis, PAPER.md:402 `PolX`):
  theta = atan2(k_perp, k_z), phi = atan2(k_y, k_x) (phi := 0 if k_perp = 0),
  eps(k,1) = (0, cos t cos f, cos t sin f, -sin t), eps(k,2) = (0, -sin f, cos f, 0).
  Label 0 is eps(k,1), label 1 is eps(k,2) (include/qed.h, qed_state_spec).
* u(p,s), ubar(p,s): exact values at rest, along +z and for a generic p, from
  SURVEY.md §8(c) item 3: u = sqrt(E+m) (chi_s ; sigma.p chi_s / (E+m)), chi_up = (1,0),
  label 0 = up.
* |M(h)|^2 with every state fixed (n = 1, 2): the covariant spin-projector trace
  u ubar = (pslash + m)(1 + gamma5 Sslash)/2, with S the spin four-vector of a rest-frame
  spin +-z boosted along p (Bjorken-Drell), evaluated in the CHIRAL basis with the
  polarisation vectors built from the literal angles above.  Fixes the electron labels
  (S -> -S under up <-> down) independently of the oracle's Pauli-spinor construction.
* polarised Klein-Nishina with the reference eps.eps' built from the formula.
* mutation self-checks: the same references under each plausible mislabelling
  (lambda swap, phi -> -phi, up <-> down) disagree with the oracle, so the pins above
  can tell them apart.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synthetic

ALPHA = 1 / 137.035999084          # CODATA 2018
E_CHARGE = math.sqrt(4 * math.pi * ALPHA)


def mdot(a, b):
    return a[..., 0] * b[..., 0] - (a[..., 1:] * b[..., 1:]).sum(-1)


# ----------------------------------------------------------------- eps(k, lambda): exact values

R5 = math.sqrt(5.0)
# (k three-vector, eps(k,1) = label 0, eps(k,2) = label 1), each evaluated by hand:
EPS_TABLE = [
    # k || +x: theta = pi/2, phi = 0
    ((2.0, 0.0, 0.0), (0, 0, 0, -1), (0, 0, 1, 0)),
    # k || +y: theta = pi/2, phi = pi/2
    ((0.0, 3.0, 0.0), (0, 0, 0, -1), (0, -1, 0, 0)),
    # k || +z: theta = 0, k_perp = 0 -> phi := 0
    ((0.0, 0.0, 0.5), (0, 1, 0, 0), (0, 0, 1, 0)),
    # k || -z: theta = pi, phi := 0
    ((0.0, 0.0, -4.0), (0, -1, 0, 0), (0, 0, 1, 0)),
    # k = (1, 2, 2): |k| = 3, k_perp = sqrt5, cos t = 2/3, sin t = sqrt5/3, cos f = 1/sqrt5, sin f = 2/sqrt5
    ((1.0, 2.0, 2.0), (0, 2 / (3 * R5), 4 / (3 * R5), -R5 / 3), (0, -2 / R5, 1 / R5, 0)),
    # k = (-1, -2, -2): cos t = -2/3, sin t = sqrt5/3, phi = atan2(-2,-1): cos f = -1/sqrt5, sin f = -2/sqrt5
    ((-1.0, -2.0, -2.0), (0, 2 / (3 * R5), 4 / (3 * R5), -R5 / 3), (0, 2 / R5, -1 / R5, 0)),
]


@pytest.mark.parametrize("kv,e1,e2", EPS_TABLE)
def test_polarisation_vector_exact_values(kv, e1, e2):
    k = np.array([math.sqrt(sum(c * c for c in kv)), *kv])
    assert np.max(np.abs(oracle.polvec(k, 0) - np.array(e1))) < 1e-15
    assert np.max(np.abs(oracle.polvec(k, 1) - np.array(e2))) < 1e-15


def test_polarisation_table_detects_mislabelling():
    """Self-check: the table separates lambda 0<->1 and phi -> -phi at the generic k."""
    kv, e1, e2 = EPS_TABLE[4]
    k = np.array([3.0, *kv])
    assert np.max(np.abs(oracle.polvec(k, 1) - np.array(e1))) > 0.1          # lambda swap
    e2_phi_flipped = np.array([0, 2 / R5, 1 / R5, 0])                         # -sin(-f), cos(-f)
    assert np.max(np.abs(oracle.polvec(k, 1) - e2_phi_flipped)) > 0.1


# ----------------------------------------------------------------- u(p,s), ubar(p,s): exact values


def _u_table():
    """(p, u(p,up), u(p,down)) written out from u = sqrt(E+m)(chi; sigma.p chi/(E+m))."""
    rows = []
    # at rest: u = sqrt(2) (chi; 0)
    r2 = math.sqrt(2.0)
    rows.append(((1.0, 0, 0, 0), (r2, 0, 0, 0), (0, r2, 0, 0)))
    # along +z, |p| = 3/4: E = 5/4, E+m = 9/4, sqrt(E+m) = 3/2; sigma.p chi_up = (pz, 0), chi_dn -> (0, -pz)
    rows.append(((1.25, 0, 0, 0.75), (1.5, 0, 1.5 * 0.75 / 2.25, 0), (0, 1.5, 0, -1.5 * 0.75 / 2.25)))
    # generic p = (1, 2, 2): E = sqrt(10); sigma.p chi_up = (pz, px + i py) = (2, 1 + 2i),
    # sigma.p chi_dn = (px - i py, -pz) = (1 - 2i, -2)
    E = math.sqrt(10.0)
    n = math.sqrt(E + 1)
    rows.append(((E, 1.0, 2.0, 2.0), (n, 0, n * 2 / (E + 1), n * (1 + 2j) / (E + 1)),
                 (0, n, n * (1 - 2j) / (E + 1), n * -2 / (E + 1))))
    return rows


@pytest.mark.parametrize("row", range(3))
def test_spinor_exact_values(row):
    p, uu, ud = _u_table()[row]
    p = np.array(p)
    for s, ref in ((0, uu), (1, ud)):
        ref = np.array(ref, dtype=complex)
        assert np.max(np.abs(oracle.spinor_u(p, s) - ref)) < 1e-15 * max(1, p[0])
        # ubar = u^dagger gamma^0, gamma^0 = diag(1, 1, -1, -1) (Dirac representation)
        ubar_ref = ref.conj() * np.array([1, 1, -1, -1])
        assert np.max(np.abs(oracle.spinor_ubar(p, s) - ubar_ref)) < 1e-15 * max(1, p[0])


def test_spinor_table_detects_mislabelling():
    p, uu, ud = _u_table()[2]
    p = np.array(p)
    assert np.max(np.abs(oracle.spinor_u(p, 0) - np.array(ud))) > 0.1         # up <-> down
    uu_conj = np.array(uu, dtype=complex).conj()                                # py -> -py (phi -> -phi)
    assert np.max(np.abs(oracle.spinor_u(p, 0) - uu_conj)) > 0.1


# ----------------------------------------------------------------- fully fixed |M(h)|^2: spin-projector trace

SIG = [np.array([[0, 1], [1, 0]], complex), np.array([[0, -1j], [1j, 0]]), np.array([[1, 0], [0, -1]], complex)]
Z2, I2 = np.zeros((2, 2)), np.eye(2)
# chiral (Weyl) basis, independent of the oracle's Dirac matrices
GCH = [np.block([[Z2, I2], [I2, Z2]]).astype(complex)] + [np.block([[Z2, s], [-s, Z2]]) for s in SIG]
G5 = 1j * GCH[0] @ GCH[1] @ GCH[2] @ GCH[3]
ONE = np.eye(4, dtype=complex)


def _slash(a):
    return GCH[0] * a[0] - GCH[1] * a[1] - GCH[2] * a[2] - GCH[3] * a[3]


def _eps_formula(k, lam):
    """SURVEY.md §8(c) item 4 written out with the literal angles (not oracle.polvec)."""
    kp = math.hypot(k[1], k[2])
    th = math.atan2(kp, k[3])
    ph = 0.0 if kp == 0 else math.atan2(k[2], k[1])
    if lam == 0:
        return np.array([0, math.cos(th) * math.cos(ph), math.cos(th) * math.sin(ph), -math.sin(th)])
    return np.array([0, -math.sin(ph), math.cos(ph), 0.0])


def _spin_vector(p, s):
    """Rest-frame spin +z (s = 0) or -z (s = 1) boosted along p:
    S = (p.n / m, n + (p.n) p / (m (E + m))), n = +-z, m = 1."""
    nz = 1.0 if s == 0 else -1.0
    pn = p[3] * nz
    return np.array([pn, pn * p[1] / (p[0] + 1), pn * p[2] / (p[0] + 1), nz + pn * p[3] / (p[0] + 1)])


def _projector(p, s):
    """u(p,s) ubar(p,s) = (pslash + m)(1 + gamma5 Sslash) / 2."""
    return (_slash(p) + ONE) @ (ONE + G5 @ _slash(_spin_vector(p, s))) / 2


def _gamma_chain_sum(q, p, eps):
    N = len(q)
    tot = np.zeros((4, 4), complex)
    for perm in itertools.permutations(range(N)):
        M = ONE.copy()
        Q = p.copy()
        for l, i in enumerate(perm):
            M = _slash(eps[i]) @ M
            if l < N - 1:
                Q = Q + q[i]
                M = (_slash(Q) + ONE) @ M / (mdot(Q, Q) - 1)
        tot += M
    return tot


def _fixed_trace(pt, n, s, sp, lams, swap_spin=False, swap_lam=False):
    p, pp = pt[0], pt[2]
    ks = [pt[1]] + [pt[3 + i] for i in range(n)]
    q = [ks[0]] + [-k for k in ks[1:]]
    eps = [_eps_formula(ks[i], (1 - lams[i]) if swap_lam else lams[i]) for i in range(n + 1)]
    Gm = _gamma_chain_sum(q, p, eps)
    g0 = GCH[0]
    ss = (1 - s) if swap_spin else s            # mislabel the incoming electron only (see below)
    ssp = sp
    tr = np.trace(_projector(pp, ssp) @ Gm @ _projector(p, ss) @ g0 @ Gm.conj().T @ g0)
    return E_CHARGE ** (2 * (n + 1)) * tr.real


@pytest.mark.parametrize("n", [1, 2])
def test_fixed_configuration_spin_projector_trace(n):
    """|ubar(p',s') Gamma u(p,s)|^2 = Tr[P(p',s') Gamma P(p,s) g0 Gamma^dag g0] for every
    configuration, in a frame where no momentum lies along z (all labels matter)."""
    mom = synthetic.rambo_cm(n, 3, sqrt_s=5.0, seed=300 + n)
    mm = synthetic.boost_rotate(mom, seed=17).numpy()
    N = n + 1
    for pt in mm:
        for s, sp in itertools.product((0, 1), repeat=2):
            for lams in itertools.product((0, 1), repeat=N):
                spec = [s, lams[0], sp] + list(lams[1:])
                got = oracle.msq(1, n, pt[None], spec=spec)[0]
                ref = _fixed_trace(pt, n, s, sp, lams)
                assert abs(got - ref) <= 1e-11 * abs(ref) + 1e-30, (n, spec, got, ref)


@pytest.mark.parametrize("n", [1, 2])
def test_fixed_configuration_trace_detects_mislabelling(n):
    """Self-check: with the incoming spin label flipped (up<->down) or every photon label flipped
    (lambda 0<->1), the reference no longer matches the oracle.  (Flipping BOTH electron labels at
    once is an exact symmetry of |M(h)| for real polarisation vectors -- see the next test -- so
    that relabelling is unobservable in any output; the exact spinor values above still fix it.)"""
    mom = synthetic.rambo_cm(n, 2, sqrt_s=5.0, seed=310 + n)
    mm = synthetic.boost_rotate(mom, seed=19).numpy()
    N = n + 1
    for kw in ({"swap_spin": True}, {"swap_lam": True}):
        worst = 0.0
        for pt in mm:
            for s, sp in itertools.product((0, 1), repeat=2):
                for lams in itertools.product((0, 1), repeat=N):
                    spec = [s, lams[0], sp] + list(lams[1:])
                    got = oracle.msq(1, n, pt[None], spec=spec)[0]
                    ref = _fixed_trace(pt, n, s, sp, lams, **kw)
                    worst = max(worst, abs(got - ref) / abs(ref))
        assert worst > 1e-2, kw


@pytest.mark.parametrize("n", [1, 2, 3])
def test_both_electron_spins_flipped_is_a_symmetry(n):
    """|M(s, s', lambdas)| = |M(1-s, 1-s', lambdas)| for real eps: evaluated with the independent
    projector trace, so it is a property of the physics, not of the oracle's spinors."""
    mm = synthetic.boost_rotate(synthetic.rambo_cm(n, 1, sqrt_s=5.0, seed=320 + n), seed=21).numpy()
    N = n + 1
    for pt in mm:
        for lams in itertools.product((0, 1), repeat=N):
            a = _fixed_trace(pt, n, 0, 1, lams)
            b = _fixed_trace(pt, n, 1, 0, lams)
            assert abs(a - b) <= 1e-11 * abs(a)


# ----------------------------------------------------------------- polarised Klein-Nishina, eps from the formula


def test_klein_nishina_polarised_lab_formula_basis():
    """1/2 sum_{s,s'} |M|^2 = e^4 [w'/w + w/w' - 2 + 4 (eps.eps')^2]  (electron at rest), with
    eps, eps' from the written-out angles; the lambda-swapped reference must fail."""
    mm = synthetic.compton_lab(256, seed=4).numpy()
    w, wp = mm[:, 1, 0], mm[:, 3, 0]
    for lam in (0, 1):
        for lamp in (0, 1):
            got = oracle.msq(1, 1, mm, spec=[-1, lam, -1, lamp])

            def ref_for(a, b):
                ee = np.array([_eps_formula(mm[i, 1], a)[1:] @ _eps_formula(mm[i, 3], b)[1:]
                               for i in range(len(mm))])
                return E_CHARGE ** 4 * (wp / w + w / wp - 2 + 4 * ee ** 2)

            assert np.max(np.abs(got / ref_for(lam, lamp) - 1)) < 1e-11
            assert np.max(np.abs(got / ref_for(lam, 1 - lamp) - 1)) > 1e-2     # mislabelled eps'
