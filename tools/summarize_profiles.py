"""Write the committed profile summaries (profiles/<tag>/) from the gpurun_out/ ncu artefacts.

  python tools/summarize_profiles.py r01
-> profiles/r01/launches.csv      every launch of the default bench command (ncu gpu__time_duration)
   profiles/r01/launch_shares.txt per-kernel share of the device time in that list
   profiles/r01/full_n{2,5}.txt   key `ncu --set full` metrics of the timed kernel + stall reasons + opcode mix
   profiles/ncu_traffic.json      dram bytes per launch for bench.py's roofline.traffic
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles", tag)
os.makedirs(dst, exist_ok=True)

KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.per_cycle_active", "sm__maximum_warps_avg_per_active_cycle",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__inst_executed.sum",
        "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return rows[0], rows[1], rows[2]


def num(x):
    try:
        return float(x.replace(",", ""))
    except Exception:
        return None


traffic = {}
tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
if os.path.exists(tpath):
    traffic = json.load(open(tpath))
for name in sorted(os.listdir(src)):
    if not (name.startswith(f"full_{tag}_") and name.endswith(".ncu-rep")):
        continue
    case = name[len(f"full_{tag}_"):-len(".ncu-rep")]
    h, u, v = raw(os.path.join(src, name))
    lines = [f"# ncu --set full --clock-control none, {name} (kernel {v[h.index('Kernel Name')] if 'Kernel Name' in h else '?'})"]
    vals = {}
    for k in KEYS:
        if k in h:
            i = h.index(k)
            vals[k] = num(v[i])
            lines.append(f"{k:70s} {v[i]:>20s} {u[i]}")
    st = []
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            x = num(v[i])
            if x:
                st.append((x, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
    lines.append("# warp stall reasons per issued instruction (top 8)")
    for x, k in sorted(st)[::-1][:8]:
        lines.append(f"  {k:30s} {x:.3f}")
    sass = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_sass_top.py"), os.path.join(src, name)],
                          capture_output=True, text=True).stdout
    lines.append("# SASS summary (tools/ncu_sass_top.py)")
    lines += sass.splitlines()
    open(os.path.join(dst, f"full_{case}.txt"), "w").write("\n".join(lines) + "\n")
    rd, wr = vals.get("dram__bytes_read.sum"), vals.get("dram__bytes_write.sum")
    # units: ncu prints Mbyte/Gbyte; normalise to bytes
    ui = {k: u[h.index(k)] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in h}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if rd is not None and wr is not None:
        b = rd * scale.get(ui["dram__bytes_read.sum"], 1) + wr * scale.get(ui["dram__bytes_write.sum"], 1)
        log = open(os.path.join(src, name.replace(".ncu-rep", ".log"))).read() if os.path.exists(
            os.path.join(src, name.replace(".ncu-rep", ".log"))) else ""
        pts = {"n2": 4194304, "n5": 262144, "bg5": 1048576}.get(case)
        if pts:
            traffic[f"{case}_points{pts}"] = int(b)
    print("wrote", os.path.join(dst, f"full_{case}.txt"))

lpath = os.path.join(src, f"launches_{tag}.csv")
if os.path.exists(lpath):
    txt = open(lpath).read()
    open(os.path.join(dst, "launches.csv"), "w").write(txt)
    rows = [r for r in csv.reader(l for l in txt.splitlines() if not l.startswith("=="))]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot, per = 0.0, {}
    for r in rows[1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            t = num(r[vi]) or 0.0
            tot += t
            nm = r[ki][:90]
            per[nm] = per.get(nm, (0, 0.0))
            per[nm] = (per[nm][0] + 1, per[nm][1] + t)
    with open(os.path.join(dst, "launch_shares.txt"), "w") as f:
        f.write("# per-kernel share of device time in the launch list of `python bench.py --steps 3 --warmup 3 "
                "--no-per-n --no-cpu-baseline` (cold-cache, serialised)\n")
        for nm, (c, t) in sorted(per.items(), key=lambda x: -x[1][1]):
            f.write(f"{100 * t / tot:6.2f}%  {c:4d} launches  {nm}\n")
    print("wrote launch list")
json.dump(traffic, open(tpath, "w"), indent=1)
print(traffic)
