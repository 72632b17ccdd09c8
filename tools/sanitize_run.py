"""Small invocation of every kernel family through the C ABI, for compute-sanitizer
(tools/sanitize.sh runs it under memcheck, racecheck, synccheck and initcheck on one GPU).
Sizes are small but ragged so that every code path (tails, multiple groups per warp, two-warp
groups, per-configuration output, MC chunks) is exercised."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_2511_19456_b200 import mc, qed  # noqa: E402

torch.cuda.set_device(0)
cases = [("cdag", n, 37) for n in (1, 2, 3, 4, 5)] + [("bg", n, 19) for n in (1, 2, 3, 4, 5, 6, 7)] + [("bg", 8, 2)]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    # racecheck: shared-memory staging of every kernel shape (two-half joins at bg n = 6, 8)
    cases = [("cdag", 1, 37), ("cdag", 2, 37), ("bg", 2, 37), ("cdag", 3, 21), ("cdag", 4, 5), ("cdag", 5, 3), ("bg", 3, 21), ("bg", 4, 5),
             ("bg", 5, 3), ("bg", 6, 3),
             ("bg", 7, 2), ("bg", 8, 1)]
for algo, n, npts in cases:
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=5 + n)
    soa = synthetic.to_soa(mom).cuda()
    proc = qed.Process(n, algorithm=algo)
    out = torch.empty(npts, dtype=torch.float64, device="cuda")
    proc.eval_msq(soa, out)
    cfg = torch.empty(npts << (n + 3), dtype=torch.float64, device="cuda")
    proc.eval_msq_configs(soa, cfg, npts)
    if n <= 5:
        part = torch.zeros(3 * mc.n_chunks(mc.CHUNK + npts), dtype=torch.float64, device="cuda")
        proc.mc_sum(part, 5.0, 0.25, 3, mc.CHUNK - 5, npts)
    if n <= 2:   # host entry point (pinned staging, two streams)
        hout = torch.empty(npts, dtype=torch.float64).pin_memory()
        proc.eval_msq_host(soa.cpu().pin_memory(), hout, npts)
        # 3-momentum uploads with the on-shell / conservation completion kernel (qed_eval_msq_host_ex)
        proc.eval_msq_host(soa.cpu().pin_memory(), hout, npts, onshell=True)
        proc.eval_msq_host(soa.cpu().pin_memory(), hout, npts, onshell=True, conserve=True)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all(), (algo, n)
    print(algo, n, "ok", flush=True)
# non-default launch plans this round added: CUDA-core joins at n = 3 (CDAG variant 1) and the grouped BG
# tasks (n = 5, variant 7), and the ABC-model kernels (include/abc.h)
for algo, n, npts, v in [("cdag", 3, 21, 1), ("bg", 5, 3, 7), ("bg", 3, 21, 1)]:
    mom = synthetic.rambo_cm(n, npts, sqrt_s=5.0, seed=50 + n)
    soa = synthetic.to_soa(mom).cuda()
    proc = qed.Process(n, algorithm=algo, variant=v)
    out = torch.empty(npts, dtype=torch.float64, device="cuda")
    proc.eval_msq(soa, out)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all(), (algo, n, v)
    print(algo, n, "variant", v, "ok", flush=True)
for algo in ("cdag", "bg"):
    for n in (1, 3, 5):
        npts = 37
        mom = synthetic.abc_cm(n, npts, sqrt_s=5.0, seed=60 + n)
        out = torch.empty(npts, dtype=torch.float64, device="cuda")
        qed.AbcProcess(n, algorithm=algo).eval_msq(synthetic.to_soa(mom).cuda(), out)
        torch.cuda.synchronize()
        assert torch.isfinite(out).all(), ("abc", algo, n)
        print("abc", algo, n, "ok", flush=True)
