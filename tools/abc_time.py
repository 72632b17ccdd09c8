"""Time the ABC-model kernels (include/abc.h) on 2^24 RAMBO points, n = 1, 3, 5, both algorithms (CUDA events)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synthetic  # noqa: E402
from paper_2511_19456_b200 import qed  # noqa: E402

P = 1 << 24
res = {}
for n in (1, 3, 5):
    soa = synthetic.to_soa(synthetic.abc_cm(n, P, sqrt_s=5.0, seed=70 + n, device="cuda"))
    out = torch.empty(P, dtype=torch.float64, device="cuda")
    for algo in ("cdag", "bg"):
        proc = qed.AbcProcess(n, algorithm=algo)
        for _ in range(3):
            proc.eval_msq(soa, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            proc.eval_msq(soa, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl = proc.info()["flops_per_point"]
        res[f"{n}_{algo}"] = {"points_per_s": P / ms * 1e3, "ms": ms, "tflops": fl * P / ms / 1e9}
print(json.dumps(res))
