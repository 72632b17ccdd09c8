"""Pins for the ABC-model oracle (oracle/abc_oracle.c; §1.3 line 56, App. F).

Each pin is fixed by something other than the oracle:
* n = 1 (A B -> A B): the textbook two-diagram amplitude M = g^2 [1/(s - m_C^2) + 1/(u - m_C^2)]
  (s-channel and u-channel C-on exchange);                              (masses, momentum signs)
* the number of diagrams is N! (every ordering of the B-ons on the A/C line, App. F);
* an independent algorithm: the Berends-Giele recursion J(S) = (1/D_S) sum_{i in S} J(S \\ i) over
  B-on subsets, the line species fixed by |S| (C odd, A even), written here in numpy;
* a mutation self-check: with every internal line a C-on the recursion disagrees at n = 3;
* Bose symmetry (outgoing B-ons permuted), time reversal (A B -> A B^n vs A B^n -> A B) and
  Lorentz invariance.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
import synthetic

MA, MB, MC = synthetic.ABC_MASSES


def mdot(a, b):
    return a[..., 0] * b[..., 0] - (a[..., 1:] * b[..., 1:]).sum(-1)


def test_abc_n1_closed_form():
    mom = synthetic.abc_cm(1, 256, sqrt_s=5.0, seed=1).numpy()
    pA, kB, pA2, kB2 = (mom[:, i] for i in range(4))
    s = mdot(pA + kB, pA + kB)
    u = mdot(pA - kB2, pA - kB2)
    for g in (1.0, 0.3):
        ref = (g * g * (1 / (s - MC ** 2) + 1 / (u - MC ** 2))) ** 2
        got = oracle.abc_msq(1, 1, mom, MA, MC, g)
        assert np.max(np.abs(got / ref - 1)) < 1e-13


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8])
def test_abc_diagram_count_is_factorial(N):
    rng = np.random.default_rng(N)
    _, nd = oracle.abc_diagram_sum(rng.normal(size=(N, 4)), np.array([3.0, 0.1, 0.2, 0.3]), MA, MC)
    assert nd == math.factorial(N)


def _bg_recursion(pt, n_in, n_out, m_line):
    """Berends-Giele recursion over B-on subsets (independent of the oracle's enumeration)."""
    N = n_in + n_out
    pA = pt[0]
    ks = [pt[1 + i] for i in range(n_in)] + [pt[n_in + 2 + i] for i in range(n_out)]
    q = [k if i < n_in else -k for i, k in enumerate(ks)]
    J = {(): 1.0}
    for size in range(1, N):
        for S in itertools.combinations(range(N), size):
            Q = pA + sum(q[i] for i in S)
            J[S] = sum(J[tuple(x for x in S if x != i)] for i in S) / (mdot(Q, Q) - m_line(size) ** 2)
    full = tuple(range(N))
    return sum(J[tuple(x for x in full if x != i)] for i in full)


@pytest.mark.parametrize("n", [1, 3, 5])
def test_abc_matches_berends_giele_recursion(n):
    mom = synthetic.abc_cm(n, 6, sqrt_s=5.0, seed=20 + n).numpy()
    got = oracle.abc_msq(1, n, mom, MA, MC)
    for pt, v in zip(mom, got):
        amp = _bg_recursion(pt, 1, n, lambda size: MC if size % 2 else MA)
        assert abs(v / amp ** 2 - 1) < 1e-12


def test_abc_recursion_detects_wrong_line_species():
    """Self-check: with every internal line a C-on (alternation dropped) the reference moves by O(1)."""
    mom = synthetic.abc_cm(3, 4, sqrt_s=5.0, seed=31).numpy()
    got = oracle.abc_msq(1, 3, mom, MA, MC)
    bad = np.array([_bg_recursion(pt, 1, 3, lambda size: MC) ** 2 for pt in mom])
    assert np.min(np.abs(got / bad - 1)) > 1e-2


@pytest.mark.parametrize("n", [3, 5])
def test_abc_bose_symmetry_and_time_reversal(n):
    mom = synthetic.abc_cm(n, 16, sqrt_s=5.0, seed=40 + n).numpy()
    a = oracle.abc_msq(1, n, mom, MA, MC)
    perm = np.roll(np.arange(n), 1)
    mom2 = mom.copy()
    mom2[:, 3:] = mom[:, 3 + perm]
    assert np.max(np.abs(oracle.abc_msq(1, n, mom2, MA, MC) / a - 1)) < 1e-12
    # A B -> A B^n  vs  A B^n -> A B with initial and final states exchanged (PAPER.md:523 direction)
    rev = np.concatenate([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], axis=1)
    assert np.max(np.abs(oracle.abc_msq(n, 1, rev, MA, MC) / a - 1)) < 1e-12


def test_abc_lorentz_invariance():
    mom = synthetic.abc_cm(3, 32, sqrt_s=5.0, seed=50)
    a = oracle.abc_msq(1, 3, mom.numpy(), MA, MC)
    b = oracle.abc_msq(1, 3, synthetic.boost_rotate(mom, seed=4).numpy(), MA, MC)
    assert np.max(np.abs(b / a - 1)) < 1e-10


def test_abc_odd_number_of_b_ons_is_rejected():
    """A B -> A B^n has tree diagrams only for odd n (N = n + 1 even)."""
    mom = synthetic.abc_cm(2, 2, sqrt_s=5.0, seed=1).numpy()
    with pytest.raises(ValueError):
        oracle.abc_msq(1, 2, mom, MA, MC)
