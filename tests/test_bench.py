"""bench.py contract: one JSON line with the keys the driver reads, for both arms, one and two ranks.

The two-rank run uses QED_BENCH_DIST_BACKEND=gloo so that both ranks can share the single GPU of
the test box: it exercises sharding, barriers, the max-over-ranks timing and the MC all-reduce
(whose sigma must be bitwise identical to the one-rank run), not multi-GPU performance.
"""
import json
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config"}


def _run(args, env=None, timeout=900):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=timeout, env=e)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_json():
    """--impl reference times the oracle on the host (the tier's reference arm); no GPU needed."""
    d = _run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "1"])
    assert KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "points/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_b200_arm_json_one_and_two_ranks():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    common = ["--photons", "1", "--points", "262144", "--steps", "3", "--warmup", "3", "--no-per-n", "--no-cpu-baseline",
              "--config-shrink", "6"]
    d1 = _run([sys.executable, "bench.py"] + common)
    assert KEYS <= set(d1) and d1["n_gpus"] == 1 and d1["value"] > 0
    r = d1["roofline"]
    assert r["bound"] == "alu" and 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    # ONSHELL | CONSERVE: the 3 momentum rows of 3 of the 4 particles cross PCIe; full_4momenta all 16 rows
    assert d1["e2e"]["h2d_bytes_per_step"] == 262144 * 3 * 3 * 8 and d1["e2e"]["d2h_bytes_per_step"] == 262144 * 8
    assert d1["e2e"]["onshell_3momenta"]["h2d_bytes_per_step"] == 262144 * 4 * 3 * 8
    assert d1["e2e"]["full_4momenta"]["h2d_bytes_per_step"] == 262144 * 4 * 4 * 8 and d1["e2e"]["full_4momenta"]["value"] > 0
    assert d1["gpu_launches"] >= 3 and "sm_mhz" in d1["clocks"]
    assert d1["clocks"]["samples"] >= 3, d1["clocks"]          # NVML polling covers the short timed region
    for key, n, total in (("c3_strong", 3, (1 << 24) >> 6), ("c5_strong", 5, (1 << 26) >> 6)):
        c = d1[key]
        assert c["n"] == n and c["points_total"] == total and c["scaling"] == "strong"
        assert c["cdag"]["value"] > 0 and c["bg"]["value"] > 0
    m = d1["mc"]
    for algo in ("bg", "cdag"):
        assert m[algo]["kernel_ms"] > 0 and m[algo]["allreduce_ms"] >= 0 and m[algo]["host_sum_ms"] > 0
        assert abs(m[algo]["value"] - m["points_total"] / (1e-3 * (m[algo]["kernel_ms"] + m[algo]["allreduce_ms"]))) \
            <= 1e-6 * m[algo]["value"]
    d2 = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
               "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2"] + common,
              env={"QED_BENCH_DIST_BACKEND": "gloo"})
    assert d2["n_gpus"] == 2 and d2["config"]["global_batch"] == 2 * 262144 and d2["scaling"] == "weak"
    for algo in ("bg", "cdag"):
        assert d2["mc"][algo]["sigma"] == d1["mc"][algo]["sigma"]      # chunk-aligned shards: bitwise
        assert d2["mc"][algo]["n_pass"] == d1["mc"][algo]["n_pass"]
    for key in ("c3_strong", "c5_strong"):                             # strong scaling: same total, split
        assert d2[key]["points_total"] == d1[key]["points_total"] and d2[key]["ranks"] == 2
        assert d2[key]["points_this_rank"] == d1[key]["points_total"] // 2
    assert d2["mc"]["ranks"] == 2 and "gloo" in d2["mc"]["collective"]
