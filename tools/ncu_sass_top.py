"""Summarise an ncu source page (SASS): top instructions by shared-memory wavefronts and by stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
ix = {k: i for i, k in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", ""))
    except Exception:
        return 0.0


tot_w = sum(f(r, "L1 Wavefronts Shared") for r in data)
tot_i = sum(f(r, "L1 Wavefronts Shared Ideal") for r in data)
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"smem wavefronts {tot_w:.3e} ideal {tot_i:.3e}; stall samples {tot_s:.0f}; instructions {len(data)}")
print("-- top by shared wavefronts")
for r in sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared"))[:12]:
    print(f"{f(r,'L1 Wavefronts Shared'):12.3e} ideal {f(r,'L1 Wavefronts Shared Ideal'):10.3e} exec {f(r,'Instructions Executed'):10.3e}  {r[ix['Source']].strip()[:70]}")
print("-- top by stall samples")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:12]:
    print(f"{f(r,'Warp Stall Sampling (All Samples)'):8.0f}  {r[ix['Source']].strip()[:80]}")
hist = {}
for r in data:
    toks = r[ix["Source"]].strip().split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    hist[op] = hist.get(op, 0) + f(r, "Instructions Executed")
tot = sum(hist.values())
print("-- executed warp instructions by opcode")
for k, v in sorted(hist.items(), key=lambda x: -x[1])[:14]:
    print(f"  {k:10s} {v:12.3e} {100*v/tot:5.1f}%")
