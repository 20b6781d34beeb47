"""Multi-GPU coverage maps: one process per GPU over torch.distributed (NCCL).

SURVEY §8e.  The path shards in two stages with exactly two exchange points:
  stage 1  rays: rank r launches the coherence bands b = r mod W of the
           Fibonacci lattice (rt_launch_shard; every rank gets the same mix of
           latitudes, unlike contiguous slot ranges); its candidate trie is local.  all_gather of the (padded) candidate
           rows, then every rank installs the union (sorted + unique on the
           device) so all ranks hold the identical global candidate list.
  stage 2  cells: rank r solves the grid rows iy = r mod W
           (round-robin blocks balance the valid-path density and keep a
           footprint's rows together); other rows stay 0 and a sum all_reduce
           of the [ny, nx] grid assembles the map.
Per-cell merging needs every candidate of that cell, so candidates are never
sharded in stage 2.  The collectives work on any backend (gloo on CPU for
the host-logic tests, NCCL over NVLink on the GPU box).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .channel import coverage_from_candidates
from .tracer import get_candidates, run_launch, set_candidates


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def shard_range(n: int, rank: int, world: int):
    """Contiguous slot range of one rank (balanced to within one)."""
    return (n * rank) // world, (n * (rank + 1)) // world


def band_unit(n: int) -> int:
    """The launch's coherence band size B (b200rt.cu rt_launch: pow2 >= sqrt(32 pi n),
    0 below 32 or above n) or the 4096-slot unit used without bands."""
    b = 1
    while b * b < 100.53 * n and b < (1 << 20):
        b <<= 1
    return 4096 if (b < 32 or b > n) else b


def shard_slots(n: int, rank: int, world: int):
    """Host restatement of rt_launch_shard's slot set: units of band_unit(n)
    slots, unit u belongs to rank u mod world."""
    unit = band_unit(n)
    units = (n + unit - 1) // unit
    out = [np.arange(u * unit, min((u + 1) * unit, n)) for u in range(rank, units, world)]
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


ROW_BLOCK = 1   # solve.cuh RT_ROW_BLOCK


def rows_of_shard(ny: int, rank: int, world: int):
    """Grid rows of one stage-2 shard: blocks of ROW_BLOCK rows round-robin."""
    return [iy for iy in range(ny) if (iy // ROW_BLOCK) % world == rank]


def barrier(world):
    d = _dist()
    if d is not None and world > 1:
        d.barrier()


def max_over_ranks(x: float, world: int) -> float:
    d = _dist()
    if d is None or world == 1:
        return float(x)
    dev = torch.device("cuda", torch.cuda.current_device()) if d.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    d.all_reduce(t, op=d.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, world: int) -> float:
    d = _dist()
    if d is None or world == 1:
        return float(x)
    dev = torch.device("cuda", torch.cuda.current_device()) if d.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    d.all_reduce(t)
    return float(t.item())


def gather_candidates(seq: torch.Tensor, ln: torch.Tensor, world: int):
    """All-gather variable-length candidate lists (rows of seq [C, L], len [C]).

    Returns the concatenation over ranks (duplicates included; the device
    sort/unique of rt_candidates_set removes them)."""
    d = _dist()
    if d is None or world == 1:
        return seq, ln
    dev = seq.device
    L = seq.shape[1]
    n = torch.tensor([seq.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(n) for _ in range(world)]
    d.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    cmax = max(counts + [1])
    pad_s = torch.full((cmax, L), -1, dtype=seq.dtype, device=dev)
    pad_l = torch.zeros(cmax, dtype=torch.int32, device=dev)
    pad_s[:seq.shape[0]] = seq
    pad_l[:seq.shape[0]] = ln.to(torch.int32)
    all_s = [torch.empty_like(pad_s) for _ in range(world)]
    all_l = [torch.empty_like(pad_l) for _ in range(world)]
    d.all_gather(all_s, pad_s)
    d.all_gather(all_l, pad_l)
    s = torch.cat([a[:c] for a, c in zip(all_s, counts)])
    l_ = torch.cat([a[:c] for a, c in zip(all_l, counts)]).to(torch.int8)
    return s, l_


def reduce_grid(g: torch.Tensor, world: int):
    d = _dist()
    if d is not None and world > 1:
        d.all_reduce(g)
    return g


def coverage_step(scene, bvh, tx_dev, grid, max_depth, num_rays, rank=0, world=1, out=None,
                  tx_mode="central"):
    """One sharded coverage map with device-resident inputs.

    Returns (local ray-bounces, stats, gains tensor [ny, nx] on the device)."""
    _, bounces = run_launch(bvh, tx_dev.position, max_depth, num_rays, shard=(rank, world))
    if world > 1:
        seq, ln = get_candidates(bvh)
        seq, ln = gather_candidates(seq, ln, world)
        set_candidates(bvh, seq, ln, seq.shape[1])
    g, stats = coverage_from_candidates(scene, bvh, tx_dev, grid, tx_mode, shard_index=rank,
                                        shard_count=world, out=out)
    reduce_grid(g, world)
    stats["ray_bounces_local"] = bounces
    return bounces, stats, g


def coverage_map(scene, bvh, grid, max_depth, num_rays, rank=0, world=1, tx_mode="central"):
    """Public multi-GPU coverage map: returns (host gains [ny, nx], local ray-bounces)."""
    tx = [d for d in scene.devices if d.kind == "tx"][0]
    bounces, _, g = coverage_step(scene, bvh, tx, grid, max_depth, num_rays, rank, world,
                                  tx_mode=tx_mode)
    return N.d2h(g), bounces


def merge_candidate_rows(rows_per_rank):
    """Host reference of the stage-1 merge: union of candidate tuples (for tests)."""
    out = set()
    for rows in rows_per_rank:
        out |= {tuple(int(x) for x in r if x >= 0) for r in np.asarray(rows)}
    return out
