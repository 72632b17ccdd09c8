"""Oracle throughput on the host cores (SURVEY.md §8(d) "Oracle timing"): points/s of oracle.msq
(averaged |M|^2, RAMBO sqrt(s) = 5) at n = 1..5 on 1 core and on all cores.

The samples are the first points of the parity subsample sizes of SURVEY.md §8(d)
(4096 / 4096 / 4096 / 1024 / 256 for n = 1..5), cut down so that each (n, threads) cell takes
about `--budget` seconds: every cell says how many points it timed.  This is the reported
baseline, not a target (the oracle is deliberately naive: dense 4x4 algebra, every diagram
and configuration from scratch).

    python tools/oracle_rates.py [--budget 8] > profiles/oracle_rates_rNN.json
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle      # noqa: E402
import synthetic   # noqa: E402

SUBSAMPLE = {1: 4096, 2: 4096, 3: 4096, 4: 1024, 5: 256}


def cell(n, threads, budget):
    full = synthetic.rambo_cm(n, SUBSAMPLE[n], sqrt_s=5.0, seed=500 + n).numpy()
    k = max(threads, min(SUBSAMPLE[n], 2 * threads))
    while True:
        t = time.perf_counter()
        oracle.msq(1, n, full[:k], threads=threads)
        dt = time.perf_counter() - t
        if dt >= budget / 4 or k == SUBSAMPLE[n]:
            break
        k = min(SUBSAMPLE[n], max(k + threads, int(k * budget / 2 / max(dt, 1e-3))))
    return {"points": k, "seconds": round(dt, 3), "points_per_s": k / dt}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budget", type=float, default=8.0)
    ap.add_argument("--max-n", type=int, default=5)
    a = ap.parse_args()
    cores = oracle.default_threads()
    cpu = "unknown"
    for line in open("/proc/cpuinfo"):
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
    res = {"cpu": cpu, "cores": cores, "kind": "oracle", "workload": "RAMBO sqrt(s)=5, averaged |M|^2",
           "subsample": SUBSAMPLE, "rates": {}}
    for n in range(1, a.max_n + 1):
        res["rates"][str(n)] = {"1_core": cell(n, 1, a.budget), f"{cores}_cores": cell(n, cores, a.budget)}
        print(f"n={n}: {res['rates'][str(n)]}", file=sys.stderr, flush=True)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
