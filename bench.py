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
with H2D/D2H inside the timed region), clocks (NVML polled every 2 ms inside the
timed region), gpu_launches, per_n (the other process sizes at their BASELINE
config sizes, same timing protocol, fewer steps), and one block per multi-GPU config
of BASELINE.json: c3_strong (n = 3, 2^24 points in total split over the ranks),
c4_mc (n = 4, 2^24 points, MC kernel and NCCL all-reduce timed separately) and
c5_strong (n = 5, 2^26 points in total split over the ranks).
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
# per-GPU batch of each size: BASELINE.json configs (C2 n=2 2^22; C3 n=3 2^24; C4 n=4 2^24; C5 n=5 2^26 over
# 8 GPUs = 2^23 per GPU); n = 1 (C1 is 4096 points, too small to time) and BG n = 6..8 sized to ~0.1-0.5 s
PER_N_POINTS = {1: 1 << 22, 2: 1 << 22, 3: 1 << 24, 4: 1 << 24, 5: 1 << 23, 6: 1 << 20, 7: 1 << 18, 8: 1 << 16}
GEN_CHUNK = 1 << 20     # points per generator call for the strong-scaling configs (seed keyed by chunk index)


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
    ap.add_argument("--no-configs", action="store_true", help="skip the c3_strong / c4_mc / c5_strong blocks")
    ap.add_argument("--config-shrink", type=int, default=0,
                    help="divide the c3/c4/c5 totals by 2^k (plumbing tests only; the lines then say so)")
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


class NvmlSampler:
    """SM clock and clock-event reasons polled every `period` s from a thread (NVML), so that even a
    30 ms timed region carries ~15 samples.  Device found by PCI bus id (NVML and CUDA indices can differ)."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, cuda_index: int, period: float = 0.002):
        self.period = period
        self.h = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(cuda_index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = None

    def start(self):
        import threading
        self.samples, self.reasons, self.stop_flag = [], 0, False
        if self.h is None:
            return
        self.max_mhz = self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM)

        def run():
            while not self.stop_flag:
                try:
                    self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                    self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    pass
                time.sleep(self.period)
        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()

    def stop(self) -> dict:
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "source": "nvml"}
        self.stop_flag = True
        self.th.join()
        sm = self.samples
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_min_mhz": min(sm) if sm else None,
                "sm_max_mhz": self.max_mhz, "samples": len(sm),
                "reasons": sorted(k for k, b in self.REASONS.items() if self.reasons & b),
                "source": f"NVML polled every {self.period * 1e3:.0f} ms inside the timed region"}


# ---------------------------------------------------------------- distributed plumbing
DIST_BACKEND = os.environ.get("QED_BENCH_DIST_BACKEND", "nccl")   # "gloo": multi-rank plumbing test on one GPU
def dist_setup(gpus: int):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # communicator set-up lines (ranks, NVLS / NVLink transport) on stderr: stdout carries the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
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


def generic_flops(n: int, algorithm: str, flops: int) -> int:
    """Flops per point of the register kernels (n <= 2) under the generic per-node model (every vertex 40 / 24,
    every propagator 56 flop, as for the lane-group kernels), i.e. without the skipped structural zeros of the
    external spinors (gen/emit_regs.py sparse_*); other kernels: their own count."""
    if n > 2:
        return flops
    from paper_2511_19456_b200.gen import emit_regs as er
    gv = {False: 40 + 56, True: 24 + 56}
    extra_u = sum(gv[lam == 1] - er.sparse_vs(er.ZU[s], lam == 1) for s in range(2) for lam in range(2))
    if n == 1:
        extra_ub = sum({False: 40, True: 24}[lam == 1] - er.sparse_v(er.ZU[s], lam == 1)[0] for s in range(2) for lam in range(2))
        return flops + 2 * extra_u + 2 * extra_ub
    if algorithm == "bg":   # P_out on ubar with the zeros common to both s' (ZUX)
        extra_ub = 2 * sum(gv[lam == 1] - er.sparse_vs(er.ZUX, lam == 1) for lam in range(2))
    else:                   # CDAG: the per-spin specialisation (vs_row_ub)
        extra_ub = sum(gv[lam == 1] - er.sparse_vs(er.ZU[s], lam == 1) for s in range(2) for lam in range(2))
    return flops + 3 * extra_u + 3 * extra_ub


def l1_roofline(algorithm: str, n: int, points: int, seconds: float):
    """Second roofline for the lane-group Berends-Giele kernels, which are bound by the L1 data pipe (shared +
    global LSU wavefronts, 1 per clock per SM; DESIGN.md §6 kernel 2b) rather than by FP64: wavefronts per
    point from the committed ncu --set full summary (profiles/ncu_l1.json, tools/summarize_raw.py) x the points
    of this launch / its live CUDA-event duration, against 148 SM x 1965 MHz wavefronts/s."""
    if algorithm != "bg":
        return None
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "ncu_l1.json"))).get(f"s3_bg{n}")
    except Exception:
        return None
    if not rec:
        return None
    peak = 148 * 1.965e9
    achieved = rec["l1_wavefronts_per_point"] * points / seconds
    return {"bound": "l1", "unit": "wavefronts/s", "wavefronts_per_point": rec["l1_wavefronts_per_point"],
            "achieved": round(achieved, -6), "peak": peak, "frac": round(achieved / peak, 4),
            "ncu_l1_data_pipe_pct": rec["l1_data_pipe_pct"], "source": f"profiles/ncu_l1.json s3_bg{n} ({rec['points']} points)"}


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
def gen_soa_range(n: int, first_chunk: int, n_chunks_: int, chunk: int, sqrt_s: float, seed: int, dev):
    """SoA momenta of global chunks [first_chunk, first_chunk + n_chunks_) of a point set that does not
    depend on how it is split: chunk c comes from its own generator seeded (seed, c)."""
    import torch

    import synthetic
    soa = torch.empty((4 * (n + 3), n_chunks_ * chunk), dtype=torch.float64, device=dev)
    for j in range(n_chunks_):
        m = synthetic.rambo_cm(n, chunk, sqrt_s=sqrt_s, seed=seed * 1000003 + first_chunk + j, device=dev)
        soa[:, j * chunk:(j + 1) * chunk] = synthetic.to_soa(m)
        del m
    return soa


def run_strong(args, world, rank, stream, dev, n: int, total: int, seed: int, algorithms, steps: int,
               warmup: int, label: str) -> dict:
    """Strong scaling: `total` points in all, rank r evaluates its contiguous share of the global chunks;
    time = max over ranks of the CUDA-event time of `steps` calls; value = total / (time per step)."""
    import torch

    from paper_2511_19456_b200 import qed
    chunk = min(GEN_CHUNK, total >> 3)   # independent of the rank count: the point set is fixed
    nch = total // chunk
    c0, c1 = nch * rank // world, nch * (rank + 1) // world
    soa = gen_soa_range(n, c0, c1 - c0, chunk, args.sqrt_s, seed, dev)
    P = soa.shape[1]
    out = torch.empty(max(P, 1), dtype=torch.float64, device=dev)
    res = {"workload": label, "n": n, "points_total": total, "points_this_rank": P, "scaling": "strong",
           "ranks": world, "steps": steps, "warmup": warmup}
    for algo in algorithms:
        proc = qed.Process(n, algorithm=algo)
        fpp = proc.info()["flops_per_point"]
        t, per = time_device(lambda: proc.eval_msq(soa, out[:P], P, stream=stream) if P else None, steps, warmup,
                             world, stream)
        per_rank_s = statistics.mean(per) / 1e3 if per else 0.0
        res[algo] = {"value": total * steps / t, "unit": UNIT, "ms_per_step": 1e3 * t / steps,
                     "flops_per_point": fpp,
                     "frac_fp64_peak_rank0": round(fpp * P / per_rank_s / 1e12 / FP64_PEAK_TFLOPS, 4) if P else None}
        del proc
    del soa, out
    return res


def run_mc(args, world, rank, stream, dev, shrink: int = 0) -> dict:
    """BASELINE.json configs[3]: e- gamma -> e- + 4 gamma, 2^24 points in total, Monte-Carlo cross-section.
    Each rank generates + evaluates its chunk-aligned share on its GPU (fused qed_mc_sum), then ONE
    all_reduce of the zero-padded chunk partial sums (NCCL on the GPU box), then the fixed-order chunk
    sum on the host.  The three phases are timed separately over 5 iterations (after 2 warm-up ones):
    kernel and all-reduce with CUDA events on the launching stream (max over ranks), host sum with
    perf_counter.  Both algorithms give the same sigma (same points, chunk-aligned shards)."""
    import torch
    import torch.distributed as dist

    from paper_2511_19456_b200 import mc, qed
    N = (1 << 24) >> shrink
    om = 0.05 * args.sqrt_s
    out = {"workload": "BASELINE configs[3]: e-gamma->e-+4gamma MC cross-section, all-reduced", "n": 4,
           "points_total": N, "sqrt_s": args.sqrt_s, "omega_min": om, "iterations": 5, "warmup": 2,
           "scaling": "strong", "ranks": world, "sigma_unit": "m_e^-2 (natural units)",
           "collective": "all_reduce(SUM) of 3 x n_chunks doubles" + (" (NCCL)" if world > 1 and DIST_BACKEND == "nccl"
                                                                      else " (gloo)" if world > 1 else " (none, 1 rank)")}
    first, count = mc.shard_range(N, rank, world)
    nch = mc.n_chunks(N)
    for algo in ("bg", "cdag"):
        proc = qed.Process(4, algorithm=algo)
        kern, red, host = [], [], []
        res = None
        for it in range(7):
            with torch.cuda.stream(stream):
                partials = torch.zeros(3 * nch, dtype=torch.float64, device=dev)
                torch.cuda.synchronize()
                barrier(world)
                e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                e[0].record(stream)
                if count:
                    proc.mc_sum(partials, args.sqrt_s, om, 4, first, count, stream=stream)
                e[1].record(stream)
                mc.reduce_partials(partials)
                e[2].record(stream)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = mc.cross_section(partials, N, args.sqrt_s, 4)
                th = time.perf_counter() - t0
            if it >= 2:
                kern.append(e[0].elapsed_time(e[1]) / 1e3)
                red.append(e[1].elapsed_time(e[2]) / 1e3)
                host.append(th)
        k = max_over_ranks(world, statistics.mean(kern))
        r = max_over_ranks(world, statistics.mean(red))
        h = statistics.mean(host)
        out[algo] = {"value": N / (k + r), "unit": UNIT, "kernel_ms": 1e3 * k, "allreduce_ms": 1e3 * r,
                     "host_sum_ms": 1e3 * h, "value_incl_host_sum": N / (k + r + h),
                     "sigma": res["sigma"], "error": res["error"], "n_pass": res["n_pass"]}
    return out


def sweep_per_n(args, world, stream, dev, algorithm: str, paper_direction: bool = False) -> dict:
    """Every process size at its BASELINE config batch size (PER_N_POINTS), same timing protocol: 3 warm-up
    + 5 timed steps, or 1 + 2 when one step takes over 0.5 s (CDAG n = 5).  paper_direction:
    e- gamma^n -> e- gamma (time-reversed RAMBO kinematics), same kernels."""
    import torch

    import synthetic
    from paper_2511_19456_b200 import qed
    out = {}
    for m in range(1, 9 if algorithm == "bg" else 6):
        Pm = PER_N_POINTS[m]
        pm = qed.Process(m, n_in_photons=m if paper_direction else 1, algorithm=algorithm)
        mm = synthetic.rambo_cm(m, Pm, sqrt_s=args.sqrt_s, seed=7 + m, device=dev)
        if paper_direction:   # initial <-> final: e_in' = e_out, gamma_in' = gamma_out..., e_out' = e_in, gamma_out' = gamma_in
            mm = torch.cat([mm[:, 2:3], mm[:, 3:], mm[:, 0:1], mm[:, 1:2]], dim=1)
        sm = synthetic.to_soa(mm)
        del mm
        om = torch.empty(Pm, dtype=torch.float64, device=dev)
        t1, _ = time_device(lambda: pm.eval_msq(sm, om, Pm, stream=stream), 1, 1, world, stream)
        K, W = (2, 0) if t1 > 0.5 else (5, 2)
        tm, perm = time_device(lambda: pm.eval_msq(sm, om, Pm, stream=stream), K, W, world, stream)
        fm = pm.info()["flops_per_point"]
        ks = statistics.mean(perm) / 1e3
        out[str(m)] = {"points_per_gpu": Pm, "value": world * Pm * K / tm, "unit": UNIT, "steps": K,
                       "ms_per_step": 1e3 * tm / K, "flops_per_point": fm,
                       "achieved_tflops": round(fm * Pm / ks / 1e12, 3),
                       "frac_fp64_peak": round(fm * Pm / ks / 1e12 / FP64_PEAK_TFLOPS, 4)}
        l1 = l1_roofline(algorithm, m, Pm, ks)
        if l1:
            out[str(m)]["l1_roofline"] = l1
        del sm, om, pm
    return out


def run_abc(args, world, stream, dev, qed_per_n) -> dict:
    """ABC model (App. F, NEXT #3): A B -> A + n B at n = 1, 3, 5, 2^24 points per GPU, both
    algorithms, same protocol as per_n; roofline per line (HBM when flops/byte is below the FP64 ridge,
    FP64 ALU above it) and the kernel-weight ratio to QED e- gamma -> e- + n gamma of the same n
    (same diagram structure, scalar instead of 4x4 kernels)."""
    import torch

    import synthetic
    from paper_2511_19456_b200 import qed
    hbm = hbm_peak_gbs()
    ridge = FP64_PEAK_TFLOPS * 1e12 / (hbm * 1e9)
    out = {"workload": "A B -> A + n B, RAMBO sqrt(s)=5 m_A, masses (m_A, m_B, m_C) = (1, 0.5, 1.2)",
           "points_per_gpu": 1 << 24, "hbm_peak_gbs": hbm, "ridge_flop_per_byte": round(ridge, 2)}
    P = 1 << 24
    for n in (1, 3, 5):
        mom = synthetic.abc_cm(n, P, sqrt_s=args.sqrt_s, seed=70 + n, device=dev)
        soa = synthetic.to_soa(mom)
        del mom
        o = torch.empty(P, dtype=torch.float64, device=dev)
        row = {}
        for algo in ("cdag", "bg"):
            proc = qed.AbcProcess(n, algorithm=algo)
            inf = proc.info()
            t, per = time_device(lambda: proc.eval_msq(soa, o, P, stream=stream), 10, 3, world, stream)
            ks = statistics.mean(per) / 1e3
            fl, by = inf["flops_per_point"], inf["bytes_per_point"]
            if fl / by < ridge:
                roof = {"bound": "hbm", "achieved": round(by * P / ks / 1e9, 1), "peak": hbm, "unit": "GB/s"}
            else:
                roof = {"bound": "alu", "achieved": round(fl * P / ks / 1e12, 3), "peak": round(FP64_PEAK_TFLOPS, 2),
                        "unit": "TFLOP/s"}
            roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
            row[algo] = {"value": world * P * 10 / t, "unit": UNIT, "ms_per_step": 1e3 * t / 10,
                         "flops_per_point": fl, "bytes_per_point": by, "roofline": roof}
            q = (qed_per_n or {}).get(str(n)) if algo == "cdag" else None
            if q:
                row[algo]["qed_same_n_points_per_s"] = q["value"]
                row[algo]["abc_over_qed"] = round(row[algo]["value"] / q["value"], 1)
            del proc
        out[str(n)] = row
        del soa, o
    return out


def hbm_peak_gbs() -> float:
    """Measured copy bandwidth (MEASURED_PEAKS.json, driver-written), else the profiling guide's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def run_e2e(args, world, proc, soa, P) -> dict:
    """Same metric through the public host-buffer API: every step copies the step's momenta H2D from
    pinned memory, evaluates, and copies |M|^2 back D2H.  The line's value is
    qed_eval_msq_host_ex(QED_HOST_ONSHELL) -- the 3-momenta cross PCIe, the energies are restored on the
    device from the mass shell -- and "full_4momenta" is qed_eval_msq_host (all 4 components uploaded)."""
    import torch
    h_soa = soa.cpu().pin_memory()
    h_out = torch.empty(P, dtype=torch.float64).pin_memory()

    def timed(onshell, conserve):
        for _ in range(max(1, args.warmup)):
            proc.eval_msq_host(h_soa, h_out, P, onshell=onshell, conserve=conserve)
        barrier(world)
        t = time.perf_counter()
        for _ in range(args.steps):
            proc.eval_msq_host(h_soa, h_out, P, onshell=onshell, conserve=conserve)
        return max_over_ranks(world, time.perf_counter() - t)

    full_s = timed(False, False)
    on_s = timed(True, False)
    e2e_s = timed(True, True)
    n_ext = h_soa.shape[0] // 4
    # momentum rows uploaded per step: 3 per particle (energies restored on the device), the outgoing
    # electron's none (momentum conservation)
    return {"value": world * P * args.steps / e2e_s, "unit": UNIT,
            "h2d_bytes_per_step": int(3 * (n_ext - 1) * P * 8), "d2h_bytes_per_step": int(h_out.numel() * 8),
            "api": "qed_eval_msq_host_ex(QED_HOST_ONSHELL | QED_HOST_CONSERVE)",
            "onshell_3momenta": {"value": world * P * args.steps / on_s, "unit": UNIT,
                                 "h2d_bytes_per_step": int(3 * n_ext * P * 8), "api": "qed_eval_msq_host_ex(QED_HOST_ONSHELL)"},
            "full_4momenta": {"value": world * P * args.steps / full_s, "unit": UNIT,
                              "h2d_bytes_per_step": int(h_soa.numel() * 8), "api": "qed_eval_msq_host"}}

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
    clocks = NvmlSampler(local)
    smi = ClockSampler(local)
    smi.start()

    def step():
        proc.eval_msq(soa, out, P, stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.02)
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
    gen_fl = generic_flops(n, args.algorithm, info["flops_per_point"])
    if gen_fl != info["flops_per_point"]:
        # the register kernels skip the structural zeros of u / ubar (csrc/qed_sparse.cuh) and count only the
        # products they need; the per-node model of the lane-group kernels and of round 1 (V 40 / 24, S 56 on
        # every node) is kept beside it for comparison
        roofline["generic_model_flops_per_point"] = gen_fl
        roofline["frac_generic_model"] = round(gen_fl * P / kernel_s / 1e12 / FP64_PEAK_TFLOPS, 4)
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

    abc = None if args.no_per_n else run_abc(args, world, stream, dev, per_n)
    mc_res = None if args.no_mc else run_mc(args, world, rank, stream, dev, args.config_shrink)
    c3 = c5 = None
    if not args.no_configs:
        k = args.config_shrink
        c3 = run_strong(args, world, rank, stream, dev, 3, (1 << 24) >> k, 3, ("cdag", "bg"), 5, 3,
                        "BASELINE configs[2]: e-gamma->e-+3gamma, 2^24 points in total" + (f" >> {k}" if k else ""))
        c5 = run_strong(args, world, rank, stream, dev, 5, (1 << 26) >> k, 5, ("bg", "cdag"), 2, 1,
                        "BASELINE configs[4]: e-gamma->e-+5gamma, 2^26 points in total, all 256 configurations"
                        + (f" >> {k}" if k else ""))
    clk_smi = smi.stop()

    peak = None
    if rank == 0:
        pk = NvmlSampler(local)
        pk.start()
        peak = measure_fp64_peak()
        if peak is not None:
            peak["clocks"] = pk.stop()
            if peak["clocks"].get("sm_mhz"):
                peak["frac_of_nominal_at_observed_clock"] = round(
                    peak["tflops"] / (148 * 128 * peak["clocks"]["sm_mhz"] * 1e6 / 1e12), 4)
        else:
            pk.stop()
    # every collective is done: the other ranks leave, so rank 0's oracle baseline has the host to itself
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = oracle_rate(n, 12.0, args.sqrt_s, args.seed)
        cpu["cpu"] = cpu_model()
        if world > 1:
            cpu["note"] = f"rank 0 after the other {world - 1} ranks finished (host idle otherwise)"

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
                                                            "grid_blocks", "variant")})},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "clocks_whole_run": clk_smi,
            "gpu_launches": launches, "fp64_dfma_microbench": peak, "per_n": per_n,
            "per_n_berends_giele": per_n_bg, "per_n_paper_direction": per_n_paper, "mc": mc_res,
            "c3_strong": c3, "c5_strong": c5, "abc_model": abc,
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
