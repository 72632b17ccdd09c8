"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Tolerance (BASELINE.json north_star): relative error <= 1e-10 in FP64 on the
summed/averaged |M|^2 per point; per configuration, |gpu - oracle| <= 1e-10 x the
largest configuration of that point.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu

TOL = 1e-10
# oracle-sized parity batches: several tiles (points per block) and a ragged tail
PARITY_POINTS = {1: 4099, 2: 4099, 3: 2053, 4: 259, 5: 67}


@pytest.fixture(scope="module")
def qed():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_19456_b200 import qed as q
    return q


def _gpu_msq(qed, proc, mom_aos: torch.Tensor) -> np.ndarray:
    soa = synthetic.to_soa(mom_aos).cuda()
    out = torch.full((mom_aos.shape[0],), float("nan"), dtype=torch.float64, device="cuda")
    proc.eval_msq(soa, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _gpu_configs(qed, proc, mom_aos: torch.Tensor) -> np.ndarray:
    n = mom_aos.shape[0]
    soa = synthetic.to_soa(mom_aos).cuda()
    out = torch.full((n * (1 << proc.n_ext),), float("nan"), dtype=torch.float64, device="cuda")
    proc.eval_msq_configs(soa, out, n)
    torch.cuda.synchronize()
    return out.cpu().numpy().reshape(n, -1)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_averaged_msq_matches_oracle(qed, n):
    mom = synthetic.rambo_cm(n, PARITY_POINTS[n], sqrt_s=5.0, seed=1000 + n)
    proc = qed.Process(n)
    got = _gpu_msq(qed, proc, mom)
    ref = oracle.msq(1, n, mom.numpy())
    rel = np.abs(got / ref - 1)
    assert np.all(np.isfinite(got))
    assert rel.max() <= TOL, (rel.max(), int(rel.argmax()))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_per_configuration_matches_oracle(qed, n):
    npts = min(PARITY_POINTS[n], 515)
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=2000 + n)
    proc = qed.Process(n)
    got = _gpu_configs(qed, proc, mom)
    A = oracle.amps(1, n, mom.numpy())
    ref = np.abs(A) ** 2
    err = np.abs(got - ref) / ref.max(axis=1, keepdims=True)
    assert err.max() <= TOL, err.max()


def test_compton_lab_klein_nishina_config(qed):
    """BASELINE.json configs[0]: n = 1, 4096 lab-frame points, averaged and the four
    fixed photon-polarisation pairs (electron spins summed) vs the oracle."""
    mom = synthetic.compton_lab(4096, seed=1)
    ref = oracle.msq(1, 1, mom.numpy())
    got = _gpu_msq(qed, qed.Process(1), mom)
    assert np.max(np.abs(got / ref - 1)) <= TOL
    for lam in (0, 1):
        for lamp in (0, 1):
            proc = qed.Process(1, in_spins=[-1, lam], out_spins=[-1, lamp])
            got = _gpu_msq(qed, proc, mom)
            ref = oracle.msq(1, 1, mom.numpy(), spec=[-1, lam, -1, lamp])
            assert np.max(np.abs(got / ref - 1)) <= TOL


FIXED_POINTS = {1: 301, 2: 301, 3: 301, 4: 67, 5: 13}


@pytest.mark.parametrize("algorithm", ["cdag", "bg"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_fixed_states_match_oracle(qed, n, algorithm):
    """Random partial specs (each particle summed or fixed to 0/1), plus the all-fixed spec, in a
    boosted frame where no momentum lies along z (so every state label matters)."""
    mom = synthetic.boost_rotate(synthetic.rambo_cm(n, FIXED_POINTS[n], seed=3000 + n), seed=31)
    rng = np.random.default_rng(n)
    specs = [[int(x) for x in rng.integers(-1, 2, size=n + 3)] for _ in range(3)]
    specs.append([int(x) for x in rng.integers(0, 2, size=n + 3)])
    scale = oracle.msq(1, n, mom.numpy())
    for spec in specs:
        proc = qed.Process(n, in_spins=spec[:2], out_spins=spec[2:], algorithm=algorithm)
        got = _gpu_msq(qed, proc, mom)
        ref = oracle.msq(1, n, mom.numpy(), spec=spec)
        assert np.max(np.abs(got - ref) / scale) <= TOL, spec


@pytest.mark.parametrize("algorithm", ["cdag", "bg"])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_paper_direction_matches_oracle(qed, n, algorithm):
    """e- gamma^n -> e- gamma: n incoming photons.  Kinematics from
    RAMBO for the north-star process with the photon roles crossed is not physical, so
    build it directly: RAMBO 2 -> (e + gamma) final state from an initial e- + n gamma
    system generated as the 'final' state of a north-star point, reversed."""
    mom = synthetic.rambo_cm(n, {5: 37, 4: 131}.get(n, 257), sqrt_s=5.0, seed=4000 + n).numpy()
    # time-reverse the north-star kinematics: initial <-> final (momenta unchanged)
    # north-star order: e_in, g_in, e_out, g_out*n  ->  paper order: e_in', g_in'*n, e_out', g_out'
    rev = np.concatenate([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], axis=1)
    proc = qed.Process(n, n_in_photons=n, algorithm=algorithm)
    got = _gpu_msq(qed, proc, torch.from_numpy(rev))
    ref = oracle.msq(n, 1, rev)
    assert np.max(np.abs(got / ref - 1)) <= TOL
    # fixed states in the paper direction (the paper evaluates one configuration per call)
    spec = ([0] + [1, 0] * (n + 2))[:n + 3]
    proc = qed.Process(n, n_in_photons=n, in_spins=spec[:n + 1], out_spins=spec[n + 1:], algorithm=algorithm)
    got = _gpu_msq(qed, proc, torch.from_numpy(rev))
    assert np.max(np.abs(got - oracle.msq(n, 1, rev, spec=spec)) / ref) <= TOL


def test_empty_and_single_point(qed):
    proc = qed.Process(2)
    soa = torch.zeros((4 * 5, 0), dtype=torch.float64, device="cuda")
    out = torch.zeros(0, dtype=torch.float64, device="cuda")
    proc.eval_msq(soa, out, n_points=0)
    torch.cuda.synchronize()
    mom = synthetic.rambo_cm(2, 1, seed=5)
    got = _gpu_msq(qed, proc, mom)
    ref = oracle.msq(1, 2, mom.numpy())
    assert abs(got[0] / ref[0] - 1) <= TOL


@pytest.mark.parametrize("npts", [1, 2, 3, 5, 7, 31, 33, 63, 65, 127, 129])
def test_ragged_sizes_n2(qed, npts):
    proc = qed.Process(2)
    mom = synthetic.rambo_cm(2, npts, seed=6000 + npts)
    got = _gpu_msq(qed, proc, mom)
    assert np.max(np.abs(got / oracle.msq(1, 2, mom.numpy()) - 1)) <= TOL


@pytest.mark.parametrize("n,npts,sample", [(2, 1 << 22, 2048), (3, 1 << 21, 512), (4, 1 << 20, 64), (5, 1 << 18, 24)])
def test_full_size_sampled(qed, n, npts, sample):
    """Bench-sized batches (the launch configuration bench.py times): sampled outputs vs the oracle."""
    torch.manual_seed(0)
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=7000 + n, device="cuda")
    soa = synthetic.to_soa(mom)
    out = torch.empty(npts, dtype=torch.float64, device="cuda")
    proc = qed.Process(n)
    proc.eval_msq(soa, out)
    torch.cuda.synchronize()
    idx = torch.cat([torch.tensor([0, npts - 1]), torch.randint(0, npts, (sample,))]).unique()
    got = out[idx.cuda()].cpu().numpy()
    ref = oracle.msq(1, n, mom[idx.cuda()].cpu().numpy())
    assert np.all(np.isfinite(out.cpu().numpy()))
    assert np.max(np.abs(got / ref - 1)) <= TOL


def test_abi_errors(qed):
    with pytest.raises(qed.QedError) as e:
        qed.Process(0)
    assert e.value.status == 2
    with pytest.raises(qed.QedError) as e:
        qed.Process(6)
    assert e.value.status == 2
    proc = qed.Process(1)
    st = qed.library().qed_eval_msq(proc._h, None, 5, None, None)
    assert st == 1
    st = qed.library().qed_eval_msq(proc._h, None, -1, None, None)
    assert st == 1
    # the binding refuses layouts the kernels would misread (row stride = n_points)
    soa = torch.zeros((4 * 4, 10), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        proc.eval_msq(soa, torch.zeros(5, dtype=torch.float64, device="cuda"))   # wider batch than out
    with pytest.raises(ValueError):
        proc.eval_msq(soa.cpu(), torch.zeros(10, dtype=torch.float64, device="cuda"))   # host momenta
    with pytest.raises(ValueError):
        proc.eval_msq_host(soa, torch.zeros(10, dtype=torch.float64), 10)                # device momenta
    with pytest.raises(qed.QedError):
        qed.Process(2, kernel_family="default", variant=10 ** 6)


def test_env_variant_out_of_range_is_an_error(qed, monkeypatch):
    """QED_VARIANT that is not a compiled variant index fails loudly (no silent fallback)."""
    nv = qed.Process(3).info()["n_variants"]
    for bad in (str(nv), "-3", "x"):
        monkeypatch.setenv("QED_VARIANT", bad)
        with pytest.raises(qed.QedError) as e:
            qed.Process(3)
        assert e.value.status == 1
    monkeypatch.setenv("QED_VARIANT", str(nv - 1))
    assert qed.Process(3).info()["variant"] == nv - 1


@pytest.mark.parametrize("n", [1, 2])
def test_lane_group_family_at_small_n(qed, n):
    """kernel_family="lane-group" runs the lane-group kernel at n <= 2 (same results)."""
    mom = synthetic.rambo_cm(n, 1029, seed=3300 + n)
    for algorithm in ("cdag", "bg"):
        proc = qed.Process(n, algorithm=algorithm, kernel_family="lane-group")
        assert proc.info()["lanes_per_point"] == 1 << (n + 1)
        got = _gpu_msq(qed, proc, mom)
        assert np.max(np.abs(got / oracle.msq(1, n, mom.numpy()) - 1)) <= TOL


def test_host_entry_point(qed):
    n = 3
    mom = synthetic.rambo_cm(n, 1001, seed=8000)
    soa = synthetic.to_soa(mom).pin_memory()
    out = torch.empty(1001, dtype=torch.float64).pin_memory()
    proc = qed.Process(n)
    proc.eval_msq_host(soa, out, 1001)
    ref = oracle.msq(1, n, mom.numpy())
    assert np.max(np.abs(out.numpy() / ref - 1)) <= TOL


def test_host_entry_point_pipelined_chunks(qed):
    """qed_eval_msq_host over several pipelined chunks (>= 2^18 points each, two streams, ragged last
    chunk): bitwise equal to the device entry point on the same points, oracle on samples around the
    chunk boundaries; pageable (unpinned) host buffers work too."""
    n, P = 1, 2 * (1 << 18) + 12345
    mom = synthetic.rambo_cm(n, P, seed=8100)
    soa = synthetic.to_soa(mom)
    proc = qed.Process(n)
    dev = torch.empty(P, dtype=torch.float64, device="cuda")
    proc.eval_msq(soa.cuda(), dev)
    torch.cuda.synchronize()
    out = torch.full((P,), float("nan"), dtype=torch.float64).pin_memory()
    proc.eval_msq_host(soa.pin_memory(), out, P)
    assert torch.equal(out, dev.cpu())
    idx = np.unique(np.concatenate([np.arange(0, 50), np.arange((1 << 18) - 50, (1 << 18) + 50),
                                    np.arange(2 * (1 << 18) - 50, 2 * (1 << 18) + 50), np.arange(P - 50, P)]))
    ref = oracle.msq(1, n, mom[idx].numpy())
    assert np.max(np.abs(out.numpy()[idx] / ref - 1)) <= TOL
    out2 = torch.full((P,), float("nan"), dtype=torch.float64)
    proc.eval_msq_host(soa.contiguous(), out2, P)
    assert torch.equal(out2, out)


@pytest.mark.parametrize("conserve", [False, True])
@pytest.mark.parametrize("n,n_in,algorithm", [(2, 1, "cdag"), (3, 3, "bg")])
def test_host_entry_point_onshell(qed, n, n_in, algorithm, conserve):
    """qed_eval_msq_host_ex(QED_HOST_ONSHELL [| QED_HOST_CONSERVE]): only the 3-momenta are uploaded and
    the energies are restored on the device from the mass shell; with CONSERVE the outgoing electron's
    rows are not uploaded either and follow from momentum conservation (include/qed.h).  The rows that
    must not be read are poisoned with NaN on the host; oracle on the original momenta, over pipelined
    chunks with a ragged tail, in the north-star and the paper direction (electron rows 0 and n_in + 1)."""
    P = 2 * (1 << 18) + 777
    mom = synthetic.rambo_cm(n if n_in == 1 else n, P, sqrt_s=5.0, seed=8200 + n).numpy()
    if n_in > 1:   # time-reversed north-star kinematics (test_paper_direction_matches_oracle)
        mom = np.concatenate([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], axis=1)
    soa = synthetic.to_soa(torch.from_numpy(mom))
    dev = torch.empty(P, dtype=torch.float64, device="cuda")
    proc = qed.Process(n, n_in_photons=n_in, algorithm=algorithm)
    proc.eval_msq(soa.cuda(), dev)
    torch.cuda.synchronize()
    poisoned = soa.clone()
    poisoned[0::4] = float("nan")
    if conserve:
        poisoned[4 * (n_in + 1):4 * (n_in + 2)] = float("nan")
    out = torch.full((P,), float("nan"), dtype=torch.float64).pin_memory()
    proc.eval_msq_host(poisoned.pin_memory(), out, P, onshell=True, conserve=conserve)
    got = out.numpy()
    assert np.all(np.isfinite(got))
    # same points as the device path up to the rounding of the given energies, amplified by the
    # conditioning of the propagator denominators (Q^2 - m^2 cancels): ~1e-15 typical, 5.5e-12 worst (r s3b)
    dev_rel = np.abs(got / dev.cpu().numpy() - 1)
    assert np.max(dev_rel) <= TOL
    worst = np.argsort(dev_rel)[-16:]
    idx = np.unique(np.concatenate([np.arange(0, 40), np.arange((1 << 18) - 40, (1 << 18) + 40), np.arange(P - 40, P),
                                    worst]))
    ref = oracle.msq(n_in, n + 1 - n_in, mom[idx])
    assert np.max(np.abs(got[idx] / ref - 1)) <= TOL
    for bad in (2, 4):   # CONSERVE without ONSHELL; an unknown bit
        with pytest.raises(qed.QedError):
            qed._check(qed._lib.qed_eval_msq_host_ex(proc._h, poisoned.data_ptr(), P, out.data_ptr(), bad), "flags")
    # a tiny call (one partial chunk, one block of the completion kernel) and an empty one
    small = synthetic.to_soa(torch.from_numpy(mom[:5]))
    small[0::4] = float("nan")
    if conserve:
        small[4 * (n_in + 1):4 * (n_in + 2)] = float("nan")
    out5 = torch.full((5,), float("nan"), dtype=torch.float64)
    proc.eval_msq_host(small, out5, 5, onshell=True, conserve=conserve)
    assert np.max(np.abs(out5.numpy() / oracle.msq(n_in, n + 1 - n_in, mom[:5]) - 1)) <= TOL
    proc.eval_msq_host(small[:, :0].contiguous(), out5[:0], 0, onshell=True, conserve=conserve)


def test_two_streams_two_handles(qed):
    n = 2
    mom = synthetic.rambo_cm(n, 20000, seed=9000)
    soa = synthetic.to_soa(mom).cuda()
    p1, p2 = qed.Process(n), qed.Process(n, in_spins=[0, -1])
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1 = torch.empty(20000, dtype=torch.float64, device="cuda")
    o2 = torch.empty_like(o1)
    torch.cuda.synchronize()
    p1.eval_msq(soa, o1, stream=s1)
    p2.eval_msq(soa, o2, stream=s2)
    torch.cuda.synchronize()
    ref1 = oracle.msq(1, n, mom[:500].numpy())
    ref2 = oracle.msq(1, n, mom[:500].numpy(), spec=[0, -1, -1, -1, -1])
    assert np.max(np.abs(o1[:500].cpu().numpy() / ref1 - 1)) <= TOL
    assert np.max(np.abs(o2[:500].cpu().numpy() / ref2 - 1)) <= TOL


# ---------------------------------------------------------------- Berends-Giele kernels (QED_ALGO_BERENDS_GIELE)

@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_bg_averaged_msq_matches_oracle(qed, n):
    mom = synthetic.rambo_cm(n, PARITY_POINTS[n], sqrt_s=5.0, seed=1100 + n)
    got = _gpu_msq(qed, qed.Process(n, algorithm="bg"), mom)
    ref = oracle.msq(1, n, mom.numpy())
    assert np.max(np.abs(got / ref - 1)) <= TOL


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_bg_per_configuration_matches_oracle(qed, n):
    npts = min(PARITY_POINTS[n], 257)
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=2100 + n)
    got = _gpu_configs(qed, qed.Process(n, algorithm="bg"), mom)
    ref = np.abs(oracle.amps(1, n, mom.numpy())) ** 2
    assert np.max(np.abs(got - ref) / ref.max(axis=1, keepdims=True)) <= TOL


@pytest.mark.parametrize("n", [2, 4])
def test_bg_paper_direction_and_fixed_states(qed, n):
    mom = synthetic.rambo_cm(n, 129, sqrt_s=5.0, seed=4100 + n).numpy()
    rev = np.concatenate([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], axis=1)
    got = _gpu_msq(qed, qed.Process(n, n_in_photons=n, algorithm="bg"), torch.from_numpy(rev))
    assert np.max(np.abs(got / oracle.msq(n, 1, rev) - 1)) <= TOL
    spec = [0, -1, 1] + [-1] * n
    got = _gpu_msq(qed, qed.Process(n, in_spins=spec[:2], out_spins=spec[2:], algorithm="bg"), torch.from_numpy(mom))
    ref = oracle.msq(1, n, mom, spec=spec)
    assert np.max(np.abs(got - ref) / oracle.msq(1, n, mom)) <= TOL


@pytest.mark.parametrize("n,npts,sample", [(2, 1 << 22, 1024), (3, 1 << 21, 512), (4, 1 << 20, 64),
                                           (5, 1 << 18, 24), (6, 1 << 18, 4)])
def test_bg_full_size_sampled(qed, n, npts, sample):
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=7100 + n, device="cuda")
    out = torch.empty(npts, dtype=torch.float64, device="cuda")
    qed.Process(n, algorithm="bg").eval_msq(synthetic.to_soa(mom), out)
    torch.cuda.synchronize()
    idx = torch.cat([torch.tensor([0, npts - 1]), torch.randint(0, npts, (sample,))]).unique()
    got = out[idx.cuda()].cpu().numpy()
    ref = oracle.msq(1, n, mom[idx.cuda()].cpu().numpy())
    assert np.all(np.isfinite(out.cpu().numpy()))
    assert np.max(np.abs(got / ref - 1)) <= TOL


# ---------------------------------------------------------------- stress kinematics (SURVEY.md §8(d) "Stress")

@pytest.mark.parametrize("algorithm", ["cdag", "bg"])
@pytest.mark.parametrize("n,sqrt_s", [(2, 1.5), (2, 20.0), (2, 100.0), (2, 1000.0), (3, 1.5), (3, 100.0), (4, 20.0)])
def test_extreme_energies(qed, n, sqrt_s, algorithm):
    mom = synthetic.rambo_cm(n, 257, sqrt_s=sqrt_s, seed=int(8000 + 10 * n + sqrt_s))
    got = _gpu_msq(qed, qed.Process(n, algorithm=algorithm), mom)
    ref = oracle.msq(1, n, mom.numpy(), kind="f80")     # long-double oracle: conditioning reference
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got / ref - 1)) <= TOL


@pytest.mark.parametrize("algorithm", ["cdag", "bg"])
def test_photons_along_the_beam_axis(qed, algorithm):
    """k_perp = 0 (phi := 0 reading, R6): n = 1 in the CM frame with the outgoing photon
    exactly along -z (backscatter) and +z (forward), n = 2 with one photon along -z."""
    s5 = 5.0
    kin = (s5 * s5 - 1) / (2 * s5)
    e_in = np.array([(s5 * s5 + 1) / (2 * s5), 0, 0, -kin])
    g_in = np.array([kin, 0, 0, kin])
    pts = []
    for sgn in (-1.0, 1.0):
        g_out = np.array([kin, 0, 0, sgn * kin])
        pts.append([e_in, g_in, e_in + g_in - g_out, g_out])
    mom = torch.tensor(np.array(pts))
    got = _gpu_msq(qed, qed.Process(1, algorithm=algorithm), mom)
    ref = oracle.msq(1, 1, mom.numpy())
    assert np.max(np.abs(got / ref - 1)) <= TOL
    base = synthetic.rambo_cm(2, 16, sqrt_s=s5, seed=77).numpy()
    # rotate each point so that the first outgoing photon lies along -z (exact zeros in k_x, k_y)
    for p in base:
        k = p[3, 1:]
        kn = np.linalg.norm(k)
        ax = np.cross(k / kn, [0, 0, -1.0])
        sa = np.linalg.norm(ax)
        ca = np.dot(k / kn, [0, 0, -1.0])
        ax = ax / sa
        K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
        R = np.eye(3) + sa * K + (1 - ca) * K @ K
        p[:, 1:] = p[:, 1:] @ R.T
        p[3, 1:] = [0.0, 0.0, -kn]
        p[2] = p[0] + p[1] - p[3] - p[4]     # restore exact conservation
    got = _gpu_msq(qed, qed.Process(2, algorithm=algorithm), torch.from_numpy(base))
    ref = oracle.msq(1, 2, base)
    assert np.max(np.abs(got / ref - 1)) <= TOL


# ---------------------------------------------------------------- n = 6..8 (NEXT #2, Berends-Giele only)

def test_bg_n6_matches_oracle(qed):
    n = 6
    mom = synthetic.rambo_cm(n, 16, sqrt_s=5.0, seed=1106)
    got = _gpu_msq(qed, qed.Process(n, algorithm="bg"), mom)
    ref = oracle.msq(1, n, mom.numpy())
    assert np.max(np.abs(got / ref - 1)) <= TOL


@pytest.mark.parametrize("n", [7, 8])
def test_bg_large_n_matches_golden_oracle(qed, n):
    """Oracle values precomputed by tools/make_golden.py (oracle only; ~100 s / 30 min per point)."""
    import json
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", f"oracle_n{n}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    g = json.load(open(path))
    mom = torch.tensor(g["momenta"], dtype=torch.float64)
    got = _gpu_msq(qed, qed.Process(n, algorithm="bg"), mom)
    ref = np.array(g["msq"])
    assert np.max(np.abs(got / ref - 1)) <= TOL


@pytest.mark.parametrize("n", [6, 7, 8])
def test_bg_large_n_invariances(qed, n):
    """Properties that hold at any size: Lorentz invariance of the spin/polarisation-summed |M|^2 and
    Bose symmetry under a permutation of the outgoing photons."""
    mom = synthetic.rambo_cm(n, 1024, sqrt_s=5.0, seed=1200 + n)
    proc = qed.Process(n, algorithm="bg")
    a = _gpu_msq(qed, proc, mom)
    b = _gpu_msq(qed, proc, synthetic.boost_rotate(mom, seed=3, max_rapidity=1.0))
    perm = torch.roll(torch.arange(n), 1)
    mom2 = mom.clone()
    mom2[:, 3:] = mom[:, 3 + perm]
    c = _gpu_msq(qed, proc, mom2)
    assert np.all(np.isfinite(a)) and np.all(a > 0)
    assert np.max(np.abs(b / a - 1)) <= 1e-9
    assert np.max(np.abs(c / a - 1)) <= TOL      # rounding order changes with the permutation


# every compiled launch variant (QED_VARIANT / qed_process_options.variant), averaged and per
# configuration: non-default variants are what the tuning sweeps time, so they are held to parity too
VARIANT_CASES = [("cdag", n) for n in (1, 2, 3, 4, 5)] + [("bg", n) for n in (1, 2, 3, 4, 5, 6)]


@pytest.mark.parametrize("algorithm,n", VARIANT_CASES)
def test_every_launch_variant_matches_oracle(qed, algorithm, n):
    npts = {1: 1029, 2: 1029, 3: 517, 4: 131, 5: 37, 6: 9}[n]
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=3100 + n)
    ref = oracle.msq(1, n, mom.numpy())
    A = oracle.amps(1, n, mom[:5].numpy())
    ref_cfg = np.abs(A) ** 2
    nv = qed.Process(n, algorithm=algorithm).info()["n_variants"]
    assert nv >= 1
    for v in range(nv):
        proc = qed.Process(n, algorithm=algorithm, variant=v)
        assert proc.info()["variant"] == v
        got = _gpu_msq(qed, proc, mom)
        rel = np.abs(got / ref - 1)
        assert rel.max() <= TOL, (v, rel.max())
        cfg = _gpu_configs(qed, proc, mom[:5])
        assert (np.abs(cfg - ref_cfg) / ref_cfg.max(axis=1, keepdims=True)).max() <= TOL, v
    with pytest.raises(qed.QedError):
        qed.Process(n, algorithm=algorithm, variant=nv)
