"""Summarise an A/B sweep (tools/ab_sweep.sh): per (algorithm, n, variant) the old / new values of both
repetitions and the mean change.   python tools/ab_report.py gpurun_out/ab_<tag>.jsonl"""
import json
import sys
from collections import defaultdict

d = defaultdict(dict)
for line in open(sys.argv[1]):
    r = json.loads(line)
    d[(r["algorithm"], r["n"], r["variant"])][(r["lib"], r["rep"])] = (r["value"], r["frac"])
for k, v in sorted(d.items()):
    old = [v[("old", i)][0] for i in (1, 2) if ("old", i) in v]
    new = [v[("new", i)][0] for i in (1, 2) if ("new", i) in v]
    o, nn = sum(old) / len(old), sum(new) / len(new)
    fo, fn = v[("old", 1)][1], v[("new", 1)][1]
    print(f"{k[0]:5s} n={k[1]} v{k[2]:<2d} old {' '.join(f'{x:.4g}' for x in old)}  new {' '.join(f'{x:.4g}' for x in new)}"
          f"  {100 * (nn / o - 1):+.2f} %  (frac {fo:.4f} -> {fn:.4f})")
