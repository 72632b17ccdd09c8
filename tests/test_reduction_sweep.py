"""Node-reduction sweep (§3.4 Fig. 9): every partially
reduced CDAG state of e- gamma^4 -> e- gamma that build() compiles, in both builds (full CSE / volatile
momentum loads), is the same function: each is compared point by point with the oracle's fixed-
configuration |M|^2 (the states evaluate spins and polarisations all fixed to 0).

CPU part: the libraries exist and export the timing entry point; the metadata follows the reduction
order (node counts fall to the fixpoint 543 of PAPER.md Table 1 / App. C, flops fall with them).
"""
import ctypes
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
import synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2511_19456_b200", "lib")
N_PH = 4
TOL = 1e-10


def _meta():
    return json.load(open(os.path.join(LIB, f"sweep_n{N_PH}_meta.json")))


def _lib(tag):
    lib = ctypes.CDLL(os.path.join(LIB, f"libqed_sweep_n{N_PH}_{tag}.so"))
    lib.sweep_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p, ctypes.c_double,
                              ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    lib.sweep_num_states.restype = ctypes.c_int
    return lib


def test_sweep_libraries_and_metadata():
    meta = _meta()
    assert [m["state"] for m in meta] == list(range(len(meta)))
    assert meta[0]["reductions"] == 0 and meta[0]["nodes"] == 2183          # Table 1, n = 4
    assert meta[-1]["nodes"] == 543                                        # the fixpoint
    nodes = [m["nodes"] for m in meta]
    flops = [m["predicted_flops"] for m in meta]
    assert nodes == sorted(nodes, reverse=True) and flops == sorted(flops, reverse=True)
    for tag in ("cse", "nocse"):
        assert _lib(tag).sweep_num_states() == len(meta)


@pytest.mark.gpu
@pytest.mark.parametrize("tag", ["cse", "nocse"])
def test_every_reduction_state_matches_oracle(tag):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = _lib(tag)
    P = 4099                                          # 33 blocks of 128 threads, ragged tail
    mom = synthetic.rambo_cm(N_PH, P, sqrt_s=5.0, seed=4100)
    rev = torch.cat([mom[:, 2:3], mom[:, 3:], mom[:, 0:1], mom[:, 1:2]], dim=1)   # e- gamma^4 -> e- gamma
    ref = oracle.msq(N_PH, 1, rev.numpy(), spec=[0] * (N_PH + 3))
    soa = synthetic.to_soa(rev).cuda()
    norm = (4 * math.pi / 137.035999084) ** (N_PH + 1)
    for m in _meta():
        out = torch.full((P,), float("nan"), dtype=torch.float64, device="cuda")
        ms = ctypes.c_float()
        rc = lib.sweep_run(m["state"], soa.data_ptr(), P, out.data_ptr(), norm, 1, ctypes.byref(ms))
        torch.cuda.synchronize()
        assert rc == 0, (tag, m)
        got = out.cpu().numpy()
        assert np.max(np.abs(got / ref - 1)) <= TOL, (tag, m["state"])
