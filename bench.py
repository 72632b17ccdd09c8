#!/usr/bin/env python
"""Benchmark: |M|^2 evaluations/s for e- gamma -> e- + n gamma on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--n 2] [--points 4194304]

Default workload = BASELINE.json configs[1]: n = 2 (6 diagrams), 2^22 phase-space
points per GPU, polarisation-summed / initial-averaged |M|^2, RAMBO CM sqrt(s) = 5 m_e.
A step is one qed_eval_msq over the whole batch.
Inputs (2^22 x 160 B = 671 MB) exceed the 126 MB L2, so no flush is needed.
Multi-GPU: one process per GPU (torchrun), weak scaling (2^22 points per rank, no
data-path collective), time = max over ranks of the CUDA-event time.

Prints ONE JSON line (rank 0).  Extra keys: roofline (FP64 ALU bound, DESIGN.md
"Roofline"), cpu_baseline (the oracle on a bounded sample), e2e (public host API
with H2D/D2H inside the timed region), clocks, gpu_launches, per_n (the other
process sizes at their own batch sizes, same timing protocol, fewer steps).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "|M|^2 evals/sec (phase-space pts/s) e-gamma->e-+n gamma"
UNIT = "points/s"
FP64_PEAK_TFLOPS = 148 * 128 * 1.965e9 / 1e12   # 148 SM x 64 DFMA/clk x 2 flop x 1965 MHz
PER_N_POINTS = {1: 1 << 22, 2: 1 << 22, 3: 1 << 21, 4: 1 << 20, 5: 1 << 18, 6: 1 << 18, 7: 1 << 16, 8: 1 << 14}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", "--photons", dest="n", type=int, default=2,
                    help="outgoing photons (--photons under torchrun, whose parser claims --n)")
    ap.add_argument("--points", type=int, default=1 << 22, help="points per GPU")
    ap.add_argument("--sqrt-s", type=float, default=5.0)
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--no-per-n", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-API end-to-end leg (tuning sweeps)")
    ap.add_argument("--no-mc", action="store_true", help="skip the MC cross-section leg (configs[3])")
    ap.add_argument("--algorithm", default="cdag", choices=["cdag", "bg"],
                    help="cdag: the paper's node-reduced diagram DAG (headline); bg: Berends-Giele rewrite")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks during the timed region
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "power_w_max": max(pw) if pw else None, "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------- distributed plumbing
DIST_BACKEND = os.environ.get("QED_BENCH_DIST_BACKEND", "nccl")   # "gloo": multi-rank plumbing test on one GPU
def dist_setup(gpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if DIST_BACKEND == "gloo":
            # plumbing check on a box with fewer GPUs than ranks (tests only: ranks share devices,
            # so the timings are not scaling numbers)
            torch.cuda.set_device(local % torch.cuda.device_count())
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    # device of this rank (== local_rank except in the gloo plumbing test, where ranks share devices)
    return world, rank, (torch.cuda.current_device() if torch.cuda.is_available() else local)


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, x: float) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if DIST_BACKEND == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- timing helpers
def time_device(fn, steps: int, warmup: int, world: int, stream) -> tuple[float, list[float]]:
    """Warm up, then time exactly `steps` calls with CUDA events on `stream` (barrier + sync both sides).
    Returns (total seconds max over ranks, per-step ms on this rank)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(stream)
    for i in range(steps):
        fn()
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    barrier(world)
    per = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    total = evs[0].elapsed_time(evs[-1]) / 1e3
    return max_over_ranks(world, total), per


def measure_fp64_peak() -> dict | None:
    import ctypes
    path = os.path.join(ROOT, "paper_2511_19456_b200", "lib", "libqed_peak.so")
    if not os.path.exists(path):
        return None
    lib = ctypes.CDLL(path)
    tf, ms = ctypes.c_double(), ctypes.c_double()
    rc = lib.qed_dfma_peak(4000, 8, ctypes.byref(tf), ctypes.byref(ms))
    if rc != 0:
        return None
    return {"tflops": round(tf.value, 2), "ms": round(ms.value, 2)}


def traffic_from_profile(n: int, points: int):
    """dram bytes per launch of the timed kernel from the committed ncu --set full summary, or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        return d.get(f"n{n}_points{points}")
    except Exception:
        return None


# ---------------------------------------------------------------- oracle timings (CPU)
def oracle_rate(n: int, target_s: float, sqrt_s: float, seed: int) -> dict:
    import oracle
    import synthetic
    threads = oracle.default_threads()
    cal = {1: 4000, 2: 2000, 3: 200, 4: 16, 5: 2}[n]
    mom = synthetic.rambo_cm(n, cal, sqrt_s=sqrt_s, seed=seed).numpy()
    t = time.perf_counter()
    oracle.msq(1, n, mom, threads=threads)
    dt = time.perf_counter() - t
    npts = max(threads, int(cal * target_s / max(dt, 1e-6)))
    mom = synthetic.rambo_cm(n, npts, sqrt_s=sqrt_s, seed=seed + 17).numpy()
    t = time.perf_counter()
    oracle.msq(1, n, mom, threads=threads)
    dt = time.perf_counter() - t
    return {"value": npts / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{npts} RAMBO points, n={n}, sqrt(s)={sqrt_s}, {dt:.1f} s wall on {threads} threads"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- reference arm: the oracle
def run_reference(args, world, rank):
    if rank != 0:
        return
    import oracle
    import synthetic
    n = args.n
    threads = oracle.default_threads()
    # calibrate one step to ~3 s of CPU work
    cal = {1: 4000, 2: 2000, 3: 200, 4: 16, 5: 2}[n]
    mom = synthetic.rambo_cm(n, cal, sqrt_s=args.sqrt_s, seed=args.seed).numpy()
    t = time.perf_counter()
    oracle.msq(1, n, mom, threads=threads)
    dt = time.perf_counter() - t
    npts = max(threads, int(cal * 3.0 / max(dt, 1e-6)))
    mom = synthetic.rambo_cm(n, npts, sqrt_s=args.sqrt_s, seed=args.seed + 1).numpy()
    for _ in range(args.warmup):
        oracle.msq(1, n, mom, threads=threads)
    t = time.perf_counter()
    for _ in range(args.steps):
        oracle.msq(1, n, mom, threads=threads)
    total = time.perf_counter() - t
    value = npts * args.steps / total
    sample = f"{npts} RAMBO points per step (bounded sample of the {args.points}-point workload), n={n}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"e-gamma->e-+{n}gamma, RAMBO sqrt(s)={args.sqrt_s}, averaged |M|^2",
                   "n": n, "points_per_step": npts},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_mc(args, world, rank, stream, dev) -> dict:
    """BASELINE.json configs[3]: e- gamma -> e- + 4 gamma, 2^24 points in total, Monte-Carlo cross-section:
    each rank generates + evaluates its chunk-aligned share on its GPU (fused qed_mc_sum), then ONE
    all_reduce of the chunk partial sums (NCCL on the GPU box).  Timed with CUDA events around the whole
    step (kernel + all-reduce), max over ranks.  Both algorithms give the same sigma (same points)."""
    import torch

    from paper_2511_19456_b200 import mc, qed
    out = {"n": 4, "points_total": 1 << 24, "sqrt_s": args.sqrt_s, "omega_min": 0.05 * args.sqrt_s}
    for algo in ("bg", "cdag"):
        proc = qed.Process(4, algorithm=algo)
        N = out["points_total"]
        res = {}

        def step():
            res.update(mc.mc_cross_section(proc, args.sqrt_s, 0.05 * args.sqrt_s, 4, N, device=dev, stream=stream))
        step()
        torch.cuda.synchronize()
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        t = max_over_ranks(world, e0.elapsed_time(e1) / 1e3)
        out[algo] = {"value": N / t, "unit": UNIT, "ms": 1e3 * t, "sigma": res["sigma"], "error": res["error"],
                     "n_pass": res["n_pass"]}
    out["sigma_unit"] = "m_e^-2 (natural units)"
    return out


def sweep_per_n(args, world, stream, dev, algorithm: str, paper_direction: bool = False) -> dict:
    """Every process size at its own batch size, same timing protocol, 5 steps.  paper_direction:
    e- gamma^n -> e- gamma (time-reversed RAMBO kinematics), same kernels."""
    import torch

    import synthetic
    from paper_2511_19456_b200 import qed
    out = {}
    for m in range(1, 9 if algorithm == "bg" else 6):
        Pm = PER_N_POINTS[m] * (4 if algorithm == "bg" and 4 <= m <= 5 else 1)
        pm = qed.Process(m, n_in_photons=m if paper_direction else 1, algorithm=algorithm)
        mm = synthetic.rambo_cm(m, Pm, sqrt_s=args.sqrt_s, seed=7 + m, device=dev)
        if paper_direction:   # initial <-> final: e_in' = e_out, gamma_in' = gamma_out..., e_out' = e_in, gamma_out' = gamma_in
            mm = torch.cat([mm[:, 2:3], mm[:, 3:], mm[:, 0:1], mm[:, 1:2]], dim=1)
        sm = synthetic.to_soa(mm)
        del mm
        om = torch.empty(Pm, dtype=torch.float64, device=dev)
        tm, perm = time_device(lambda: pm.eval_msq(sm, om, Pm, stream=stream), 5, 3, world, stream)
        fm = pm.info()["flops_per_point"]
        ks = statistics.mean(perm) / 1e3
        out[str(m)] = {"points_per_gpu": Pm, "value": world * Pm * 5 / tm, "unit": UNIT,
                       "ms_per_step": 1e3 * tm / 5, "flops_per_point": fm,
                       "achieved_tflops": round(fm * Pm / ks / 1e12, 3),
                       "frac_fp64_peak": round(fm * Pm / ks / 1e12 / FP64_PEAK_TFLOPS, 4)}
        del sm, om, pm
    return out


def run_e2e(args, world, proc, soa, P) -> dict:
    """Same metric through the public host-buffer API (qed_eval_msq_host): every step copies the
    step's momenta H2D from pinned memory, evaluates, and copies |M|^2 back D2H."""
    import torch
    h_soa = soa.cpu().pin_memory()
    h_out = torch.empty(P, dtype=torch.float64).pin_memory()
    for _ in range(max(1, args.warmup)):
        proc.eval_msq_host(h_soa, h_out, P)
    barrier(world)
    t = time.perf_counter()
    for _ in range(args.steps):
        proc.eval_msq_host(h_soa, h_out, P)
    e2e_s = max_over_ranks(world, time.perf_counter() - t)
    return {"value": world * P * args.steps / e2e_s, "unit": UNIT,
            "h2d_bytes_per_step": int(h_soa.numel() * 8), "d2h_bytes_per_step": int(h_out.numel() * 8)}

def run_b200(args, world, rank, local):
    import torch

    import synthetic
    from paper_2511_19456_b200 import qed

    n, P = args.n, args.points
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    proc = qed.Process(n, algorithm=args.algorithm)
    info = proc.info()
    # each rank owns its own shard of points (weak scaling): seed depends on the rank
    mom = synthetic.rambo_cm(n, P, sqrt_s=args.sqrt_s, seed=args.seed * 1000 + rank, device=dev)
    soa = synthetic.to_soa(mom)
    del mom
    out = torch.empty(P, dtype=torch.float64, device=dev)
    launches0 = qed.launch_count()
    clocks = ClockSampler(local)

    def step():
        proc.eval_msq(soa, out, P, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    total, per = time_device(step, args.steps, 0, world, stream)
    clk = clocks.stop()
    launches = qed.launch_count() - launches0 - args.warmup
    assert torch.isfinite(out).all().item(), "non-finite |M|^2 in the benchmark batch"

    value = world * P * args.steps / total
    kernel_s = statistics.mean(per) / 1e3
    achieved = info["flops_per_point"] * P / kernel_s / 1e12
    roofline = {"bound": "alu", "achieved": round(achieved, 3), "peak": round(FP64_PEAK_TFLOPS, 2),
                "unit": "TFLOP/s", "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                "traffic": traffic_from_profile(n, P),
                "algorithmic_flops_per_point": info["flops_per_point"],
                "algorithmic_bytes_per_point": info["bytes_per_point"],
                "hbm_gbs": round(info["bytes_per_point"] * P / kernel_s / 1e9, 1),
                "peak_note": "FP64 CUDA-core peak 148 SM x 128 flop/clk x 1965 MHz (DESIGN.md Roofline)"}
    if clk.get("sm_mhz"):
        roofline["frac_at_observed_clock"] = round(
            achieved / (148 * 128 * clk["sm_mhz"] * 1e6 / 1e12), 4)

    # end-to-end through the public host API: H2D momenta + kernel + D2H |M|^2 each step
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, world, proc, soa, P)
    per_n = per_n_bg = per_n_paper = None
    if not args.no_per_n:
        per_n = sweep_per_n(args, world, stream, dev, "cdag")
        per_n_bg = sweep_per_n(args, world, stream, dev, "bg")
        per_n_paper = sweep_per_n(args, world, stream, dev, "cdag", paper_direction=True)

    mc_res = None if args.no_mc else run_mc(args, world, rank, stream, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_rate(n, 12.0, args.sqrt_s, args.seed)
        cpu["cpu"] = cpu_model()
    peak = measure_fp64_peak() if rank == 0 else None

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"algorithm": args.algorithm,
                       "workload": f"BASELINE configs[1]: e-gamma->e-+{n}gamma ({math.factorial(n + 1)} diagrams), "
                                   f"{P} RAMBO points/GPU, sqrt(s)={args.sqrt_s}, pol-summed/averaged |M|^2",
                       "n": n, "global_batch": world * P, "points_per_gpu": P,
                       "parallelism": f"points sharded over {world} GPU(s), no collective",
                       "l2": "inputs > 126 MB L2 (no flush needed)",
                       "kernel": dict({k: info[k] for k in ("lanes_per_point", "warps_per_block", "smem_per_block",
                                                            "grid_blocks")}, variant=os.environ.get("QED_VARIANT", "0"))},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "gpu_launches": launches,
            "fp64_dfma_microbench": peak, "per_n": per_n,
            "per_n_berends_giele": per_n_bg, "per_n_paper_direction": per_n_paper, "mc": mc_res,
        }
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        # the oracle runs on rank 0's host cores only; other ranks exit without work
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    world, rank, local = dist_setup(args.gpus)
    try:
        run_b200(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
