"""Write oracle-only golden files for process sizes whose oracle is too slow to run inside the GPU
test session (n = 7: ~100 s/point/core, n = 8: ~30 min/point/core).

Every stored value comes from oracle/ (the naive diagram-sum oracle) on seeded synthetic inputs;
nothing here touches the CUDA path.  Output: tests/golden/oracle_n{n}.json with the momenta
(AoS, particle order e-_in, gamma_in, e-_out, gamma_out...) and averaged |M|^2.

    python tools/make_golden.py 7 8 [--points 8] [--threads 8]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synthetic  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("ns", type=int, nargs="+")
ap.add_argument("--points", type=int, default=8)
ap.add_argument("--threads", type=int, default=os.cpu_count())
a = ap.parse_args()
for n in a.ns:
    mom = synthetic.rambo_cm(n, a.points, sqrt_s=5.0, seed=9000 + n).numpy()
    t = time.time()
    msq = oracle.msq(1, n, mom, threads=a.threads)
    out = {"n": n, "sqrt_s": 5.0, "seed": 9000 + n, "generator": "synthetic.rambo_cm", "oracle": "oracle.msq f64",
           "seconds": round(time.time() - t, 1), "momenta": mom.tolist(), "msq": msq.tolist()}
    path = os.path.join(ROOT, "tests", "golden", f"oracle_n{n}.json")
    json.dump(out, open(path, "w"))
    print(n, path, out["seconds"], "s")
