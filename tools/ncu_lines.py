"""Stall samples per CUDA source line from an ncu report (--print-source=cuda,sass), top stall reasons each.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
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


tot = sum(f(r, "Warp Stall Sampling (All Samples)") for _, r in rows)
stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
print(f"total stall samples {tot:.0f}")
for fn, r in sorted(rows, key=lambda x: -f(x[1], "Warp Stall Sampling (All Samples)"))[:top]:
    s = f(r, "Warp Stall Sampling (All Samples)")
    tops = sorted(((f(r, k), k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{100 * s / tot:5.1f}%  {fn}:{r[0]:>4s}  [{', '.join(f'{k} {v / max(s, 1) * 100:.0f}%' for v, k in tops)}]  {r[1].strip()[:60]}")
