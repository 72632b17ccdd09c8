"""Monte-Carlo cross-section driver: shard, evaluate on each GPU, one all-reduce.

SURVEY.md §8(a) row a9 and §8(e): points are the unit of parallelism.  Rank r owns a
contiguous, chunk-aligned range of global point indices; its GPU generates and
evaluates them inside the fused kernel (qed_mc_sum: Philox counter = global index,
so the point set does not depend on the number of GPUs) and accumulates per-chunk
partial sums into a zero-padded vector of all chunks.  The only collective is one
all_reduce(SUM) of that vector (NCCL over NVLink on the GPU box; gloo in the CPU
tests).  Because every chunk has exactly one contributing rank, x + 0 is exact and
the final chunk sum (fixed order) is bitwise identical for any number of GPUs.

sigma = sum w |M|^2 / (N_total * F * n!),  F = 2 (s - m^2)  (flux of e- gamma at rest frame
invariant 4 p.k), the 1/n! for n identical final photons; error from sum (w |M|^2)^2.
"""
from __future__ import annotations

import math

import numpy as np
import torch

CHUNK = 1024   # = QED_MC_CHUNK (include/qed.h)


def n_chunks(n_total: int, chunk: int = CHUNK) -> int:
    return (n_total + chunk - 1) // chunk


def shard_range(n_total: int, rank: int, world: int, chunk: int = CHUNK) -> tuple[int, int]:
    """Contiguous chunk-aligned share [first, first + count) of rank `rank`."""
    nc = n_chunks(n_total, chunk)
    c0 = nc * rank // world
    c1 = nc * (rank + 1) // world
    first = min(c0 * chunk, n_total)
    last = min(c1 * chunk, n_total)
    return first, last - first


def reduce_partials(partials: torch.Tensor, group=None) -> torch.Tensor:
    """all_reduce(SUM) of the zero-padded chunk vector (the one collective of the path)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(partials, op=dist.ReduceOp.SUM, group=group)
    return partials


def cross_section(partials: torch.Tensor, n_total: int, sqrt_s: float, n_photons: int) -> dict:
    """sigma and its MC error from the reduced chunk sums (summed in chunk order, on the host)."""
    p = partials.detach().to("cpu", torch.float64).numpy().reshape(-1, 3)
    # fixed order, left to right (a running sum: bitwise the sequential loop, for any number of ranks)
    s0, s1, npass = (float(np.cumsum(p[:, k])[-1]) if p.shape[0] else 0.0 for k in range(3))
    s = sqrt_s * sqrt_s
    norm = 1.0 / (2.0 * (s - 1.0) * math.factorial(n_photons))
    mean = s0 / n_total
    var = max(s1 / n_total - mean * mean, 0.0)
    return {"sigma": norm * mean, "error": norm * math.sqrt(var / n_total), "n_pass": npass,
            "n_total": n_total, "sum_w_msq": s0}


def mc_cross_section(proc, sqrt_s: float, omega_min: float, seed: int, n_total: int, group=None,
                     device=None, stream=None) -> dict:
    """Full multi-GPU MC: this rank's shard on its GPU (qed_mc_sum), one all-reduce, sigma."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    dev = device or torch.device("cuda", torch.cuda.current_device())
    st = stream or torch.cuda.current_stream(dev)
    # zero-fill, kernel, all-reduce and the D2H read all run in order on ONE stream
    with torch.cuda.stream(st):
        partials = torch.zeros(3 * n_chunks(n_total), dtype=torch.float64, device=dev)
        first, count = shard_range(n_total, rank, world)
        if count:
            proc.mc_sum(partials, sqrt_s, omega_min, seed, first, count, stream=st)
        reduce_partials(partials, group)
        return cross_section(partials, n_total, sqrt_s, proc.n)
