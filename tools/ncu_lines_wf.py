"""Per CUDA source line: share of stall samples, executed instructions and shared-memory wavefronts
(ncu source page, --print-source=cuda,sass).  usage: python tools/ncu_lines_wf.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, hdr = None, [], None
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {}
        for i, k in enumerate(r):
            hdr.setdefault(k, i)
        continue
    if hdr and r and r[0].isdigit():
        rows.append((fname, r))


def f(r, k):
    try:
        return float(r[hdr[k]].replace(",", ""))
    except Exception:
        return 0.0


keys = ["Warp Stall Sampling (All Samples)", "Instructions Executed", "L1 Wavefronts Shared"]
tot = [sum(f(r, k) for _, r in rows) or 1.0 for k in keys]
print("columns: stall%  inst%  smem-wavefront%   (totals: " + ", ".join(f"{t:.3e}" for t in tot) + ")")
seen = set()
for kk in (2, 1, 0):
    print(f"-- top by {keys[kk]}")
    for fn, r in sorted(rows, key=lambda x: -f(x[1], keys[kk]))[:top]:
        v = [100 * f(r, k) / t for k, t in zip(keys, tot)]
        print(f"{v[0]:5.1f} {v[1]:5.1f} {v[2]:5.1f}  {fn}:{r[0]:>4s}  {r[1].strip()[:70]}")
