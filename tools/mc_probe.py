"""One fused MC launch (n, algorithm, points from argv) for ncu: python tools/mc_probe.py 4 cdag 1048576"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2511_19456_b200 import mc, qed  # noqa: E402

n, algo, N = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
proc = qed.Process(n, algorithm=algo)
for _ in range(2):
    part = torch.zeros(3 * mc.n_chunks(N), dtype=torch.float64, device="cuda")
    proc.mc_sum(part, 5.0, 0.25, 4, 0, N)
torch.cuda.synchronize()
print(part.view(-1, 3).sum(0).tolist())
