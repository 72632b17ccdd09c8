"""Summarise `ncu --page raw --csv` exports of tools/prof_var.sh captures (gpurun_out/raw_<tag>.csv) into
profiles/<round>/pipes_<set>.txt and profiles/ncu_l1.json: per kernel the FP64 / tensor (DMMA) pipe
utilisation, the L1 data-pipe wavefront utilisation (shared + global/local, the BG kernels' binding limit)
and the wavefronts per point.

  python tools/summarize_raw.py r03 s3 s3_bg3:2097152 s3_bg4:1048576 s3_bg5:524288 s3_bg6:131072
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {
    "ms": "gpu__time_duration.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "dmma_pipe_pct": "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1_data_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "shared_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "shared_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "shared_wavefronts_ideal": "memory_l1_wavefronts_shared_ideal",
    "shared_ld_st_wavefronts": "memory_l1_wavefronts_shared",
    "sm_lsu_wavefronts_avg": "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg",
    "sm_lgds_wavefronts_avg": "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg",
    "warps_per_sm": "sm__warps_active.avg.per_cycle_active",
    "regs": "launch__registers_per_thread",
    "clock_ghz": "sm__cycles_elapsed.avg.per_second",
}


def load(path):
    rows = list(csv.reader(open(path)))
    return dict(zip(rows[0], rows[2]))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except Exception:
        return None


def main():
    rnd, setname, specs = sys.argv[1], sys.argv[2], sys.argv[3:]
    out_json = os.path.join(ROOT, "profiles", "ncu_l1.json")
    db = json.load(open(out_json)) if os.path.exists(out_json) else {}
    lines = ["# ncu --set full --clock-control none (tools/prof_var.sh), summarised by tools/summarize_raw.py",
             "# tag points | ms | FP64 pipe % | DMMA pipe % | issue % | L1 data pipe % (all LSU wavefronts) | "
             "shared wavefront % | L1 wavefronts/point (shared + global) | shared/ideal | warps/SM | regs"]
    for spec in specs:
        tag, pts = spec.split(":")
        pts = int(pts)
        d = load(os.path.join(ROOT, "gpurun_out", f"raw_{tag}.csv"))
        v = {k: num(d.get(m)) for k, m in KEYS.items()}
        sms = 148
        lsu = v["sm_lsu_wavefronts_avg"] * sms
        lgds = v["sm_lgds_wavefronts_avg"] * sms
        rec = {"points": pts, **{k: v[k] for k in ("ms", "fp64_pipe_pct", "dmma_pipe_pct", "issue_pct",
                                                  "l1_data_pipe_pct", "shared_wavefront_pct", "warps_per_sm", "regs")},
               "l1_wavefronts_per_point": round(lsu / pts, 2), "shared_wavefronts_per_point": round(v["shared_wavefronts"] / pts, 2),
               "global_wavefronts_per_point": round(lgds / pts, 2),
               "shared_conflict_ratio": round(v["shared_ld_st_wavefronts"] / v["shared_wavefronts_ideal"], 4)}
        db[tag] = rec
        lines.append(f"{tag} {pts} | {v['ms']:.3f} | {v['fp64_pipe_pct']:.1f} | {(v['dmma_pipe_pct'] or 0):.1f} | "
                     f"{v['issue_pct']:.1f} | {v['l1_data_pipe_pct']:.1f} | {v['shared_wavefront_pct']:.1f} | "
                     f"{rec['l1_wavefronts_per_point']} ({rec['shared_wavefronts_per_point']} + {rec['global_wavefronts_per_point']}) | "
                     f"{rec['shared_conflict_ratio']} | {v['warps_per_sm']:.1f} | {v['regs']:.0f}")
    json.dump(db, open(out_json, "w"), indent=1, sort_keys=True)
    dst = os.path.join(ROOT, "profiles", rnd, f"pipes_{setname}.txt")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
