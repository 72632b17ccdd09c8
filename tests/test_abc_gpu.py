"""GPU parity of the ABC-model kernels (include/abc.h; App. F) against the ABC oracle, through
the C ABI: both algorithms, both directions, oracle-sized batches with a ragged tail, a bench-sized batch
sampled, and the ABI's error codes.  Tolerance 1e-10 relative (north_star)."""
import numpy as np
import pytest
import torch

import oracle
import synthetic

pytestmark = pytest.mark.gpu
TOL = 1e-10
MA, MB, MC = synthetic.ABC_MASSES


@pytest.fixture(scope="module")
def qed():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2511_19456_b200 import qed as q
    assert (q.ABC_MASS_A, q.ABC_MASS_B, q.ABC_MASS_C) == synthetic.ABC_MASSES
    return q


def _run(proc, mom):
    soa = synthetic.to_soa(mom).cuda()
    out = torch.full((mom.shape[0],), float("nan"), dtype=torch.float64, device="cuda")
    proc.eval_msq(soa, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("algorithm", ["cdag", "bg"])
@pytest.mark.parametrize("n", [1, 3, 5])
def test_abc_matches_oracle(qed, n, algorithm):
    mom = synthetic.abc_cm(n, {1: 5003, 3: 5003, 5: 1029}[n], sqrt_s=5.0, seed=100 + n)
    proc = qed.AbcProcess(n, algorithm=algorithm)
    got = _run(proc, mom)
    ref = oracle.abc_msq(1, n, mom.numpy(), MA, MC)
    assert np.all(np.isfinite(got))
    assert np.max(np.abs(got / ref - 1)) <= TOL
    # the paper's direction A B^n -> A B: initial and final states exchanged
    rev = torch.cat([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], dim=1)
    got = _run(qed.AbcProcess(1, n_in=n, algorithm=algorithm), rev)
    assert np.max(np.abs(got / oracle.abc_msq(n, 1, rev.numpy(), MA, MC) - 1)) <= TOL


@pytest.mark.parametrize("algorithm", ["cdag", "bg"])
def test_abc_full_size_sampled(qed, algorithm):
    n, P = 5, 1 << 22
    mom = synthetic.abc_cm(n, P, sqrt_s=5.0, seed=7, device="cuda")
    out = torch.empty(P, dtype=torch.float64, device="cuda")
    qed.AbcProcess(n, algorithm=algorithm).eval_msq(synthetic.to_soa(mom), out)
    torch.cuda.synchronize()
    idx = torch.cat([torch.tensor([0, P - 1]), torch.randint(0, P, (2048,))]).unique().cuda()
    ref = oracle.abc_msq(1, n, mom[idx].cpu().numpy(), MA, MC)
    assert np.all(np.isfinite(out.cpu().numpy()))
    assert np.max(np.abs(out[idx].cpu().numpy() / ref - 1)) <= TOL


def test_abc_abi_errors(qed):
    with pytest.raises(qed.QedError) as e:
        qed.AbcProcess(2)                       # odd number of B-ons
    assert e.value.status == 1
    with pytest.raises(qed.QedError) as e:
        qed.AbcProcess(7)                       # N = 8: not compiled
    assert e.value.status == 2
    proc = qed.AbcProcess(3)
    assert proc.info()["n_diagrams"] == 24 and proc.info()["bytes_per_point"] == 8 * (4 * 5 + 1)
    assert qed.library().abc_eval_msq(proc._h, None, 5, None, None) == 1
