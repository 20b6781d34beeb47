"""Multi-GPU coverage maps, path sets + CIR and calibration gradients: one
process per GPU over torch.distributed (NCCL).

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
sharded in stage 2.

compute_paths + CIR (the (tx, rx) loop of tracer.py:298-311):
stage 1 as above; stage 2 shards the receivers (rx i -> rank i mod W), every
rank packs the CIR rows of its receivers and an all_gather of the padded
slices assembles the [rx, ...] tensors in receiver order.

Calibration (optim.py:348-360): the records are sharded
round-robin, every rank evaluates its share of the mean NMSE and its gradient
through the adjoint, and one all_reduce sums [loss, grads].  The collectives work on any backend (gloo on CPU for
the host-logic tests, NCCL over NVLink on the GPU box).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .channel import build_cir, coverage_from_candidates
from .em import compute_gains
from .tracer import (PathSet, PathTable, TracerError, get_candidates, paths_to_receivers,
                     prepare_candidates, run_launch, set_candidates)


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _wire(d, t: torch.Tensor) -> torch.Tensor:
    """The tensor a collective runs on: NCCL takes device tensors; gloo (the
    CPU test backend, also used with CUDA tensors on one GPU) gets a host copy."""
    return t.cpu() if (t.is_cuda and d.get_backend() != "nccl") else t


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
    n = _wire(d, torch.tensor([seq.shape[0]], dtype=torch.int64, device=dev))
    counts = [torch.zeros_like(n) for _ in range(world)]
    d.all_gather(counts, n)
    counts = [int(c.item()) for c in counts]
    cmax = max(counts + [1])
    pad_s = torch.full((cmax, L), -1, dtype=seq.dtype, device=dev)
    pad_l = torch.zeros(cmax, dtype=torch.int32, device=dev)
    pad_s[:seq.shape[0]] = seq
    pad_l[:seq.shape[0]] = ln.to(torch.int32)
    pad_s, pad_l = _wire(d, pad_s), _wire(d, pad_l)
    all_s = [torch.empty_like(pad_s) for _ in range(world)]
    all_l = [torch.empty_like(pad_l) for _ in range(world)]
    d.all_gather(all_s, pad_s)
    d.all_gather(all_l, pad_l)
    s = torch.cat([a[:c] for a, c in zip(all_s, counts)]).to(dev)
    l_ = torch.cat([a[:c] for a, c in zip(all_l, counts)]).to(torch.int8).to(dev)
    return s, l_


def reduce_grid(g: torch.Tensor, world: int):
    """Sum all-reduce of the [ny, nx] grid.  Every cell is nonzero on exactly one
    rank (its row's shard), so the sum is exact: the map is bit-identical to
    the single-rank one."""
    d = _dist()
    if d is not None and world > 1:
        w = _wire(d, g)
        d.all_reduce(w)
        if w is not g:
            g.copy_(w)
    return g


def coverage_step(scene, bvh, tx_dev, grid, max_depth, num_rays, rank=0, world=1, out=None,
                  tx_mode="central"):
    """One sharded coverage map with device-resident inputs.

    Returns (local ray-bounces, stats, gains tensor [ny, nx] on the device)."""
    if world == 1 and max_depth >= 1 and bvh.num_prims:   # launch + map in one library call
        from .channel import coverage_fibonacci
        g, stats, bounces = coverage_fibonacci(scene, bvh, tx_dev, grid, max_depth, num_rays, tx_mode, out=out)
        stats["ray_bounces_local"] = bounces
        return bounces, stats, g
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


# ---- compute_paths + CIR with receivers sharded ---------------------------------------------

def rx_of_shard(n_rx: int, rank: int, world: int):
    """Receivers of one stage-2 shard: i = rank, rank + W, ..."""
    return list(range(rank, n_rx, world))


def _shared_candidates(bvh, tx_pos, max_depth, method, num_rays, rank, world):
    """Every rank ends with the global candidate set: a sharded launch plus the
    candidate all_gather for ``fibonacci``; ``exhaustive`` enumerates the same
    set on every rank (no exchange needed)."""
    if method == "fibonacci" and world > 1 and max_depth >= 1 and bvh.num_prims:
        run_launch(bvh, tx_pos, max_depth, num_rays, shard=(rank, world))
        seq, ln = gather_candidates(*get_candidates(bvh), world)
        set_candidates(bvh, seq, ln, seq.shape[1])
    else:
        prepare_candidates(bvh, tx_pos, max_depth, method, num_rays)


def _gather_rows(x: torch.Tensor, rows, n_total: int, world: int, pad_dims):
    """All-gather the receiver-row slices x [len(rows), ...] of every rank into
    the full [n_total, ...] tensor (rank r owns rows r, r + W, ...).  Dims in
    ``pad_dims`` may differ across ranks and are zero-padded to the maximum."""
    d = _dist()
    if d is None or world == 1:
        return x
    dev = x.device
    shape = _wire(d, torch.tensor(list(x.shape), dtype=torch.int64, device=dev))
    d.all_reduce(shape, op=d.ReduceOp.MAX)
    full = [int(v) for v in shape.tolist()]
    full[0] = (n_total + world - 1) // world
    buf = torch.zeros(full, dtype=x.dtype, device=dev)
    buf[tuple(slice(0, n) for n in x.shape)] = x
    real = _wire(d, (torch.view_as_real(buf) if buf.is_complex() else buf).contiguous())
    parts = [torch.empty_like(real) for _ in range(world)]
    d.all_gather(parts, real)
    out_shape = [n_total] + full[1:]
    out = torch.zeros(out_shape, dtype=x.dtype, device=dev)
    for r, part in enumerate(parts):
        part = (torch.view_as_complex(part) if x.is_complex() else part).to(dev)
        idx = rx_of_shard(n_total, r, world)
        if idx:
            out[idx] = part[:len(idx)]
    return out


def compute_paths_cir(scene, bvh, max_depth: int, method: str = "fibonacci", num_rays: int = 4096,
                      rank: int = 0, world: int = 1, los=True, reflection=True,
                      normalize_delays=False, to_host=True):
    """compute_paths + compute_gains + build_cir with rays (stage 1) and
    receivers (stage 2) sharded over the ranks.  Returns (Cir, local PathSet):
    the Cir covers every receiver on every rank; the PathSet holds this rank's
    receivers' paths (receiver indices global)."""
    txs = [d for d in scene.devices if d.kind == "tx"]
    rxs = [d for d in scene.devices if d.kind == "rx"]
    if not txs or not rxs:
        raise TracerError("scene needs at least one transmitter and one receiver")
    mine = rx_of_shard(len(rxs), rank, world)
    dev = bvh.device
    rx_pos = np.array([rxs[i].position for i in mine], dtype=np.float64).reshape(-1, 3)
    to_global = torch.tensor(mine + [0], dtype=torch.int32, device=dev)
    tables = []
    for ti, tx in enumerate(txs):
        _shared_candidates(bvh, tx.position, max_depth, method, num_rays, rank, world)
        T = paths_to_receivers(bvh, tx.position, rx_pos, tx_index=ti) if mine else None
        if T is not None:
            T.rx = to_global[T.rx.long()].contiguous()
            tables.append(T)
    if tables:
        T = PathTable.cat(tables) if len(tables) > 1 else tables[0]
    else:
        T = paths_to_receivers(bvh, txs[0].position, np.zeros((0, 3)), tx_index=0)
    T.tx_names = [t.name for t in txs]
    T.rx_names = [r.name for r in rxs]
    ps = PathSet(scene=scene, max_depth=max_depth, method=method, table=T)
    cir = build_cir(compute_gains(scene, bvh, ps), los, reflection, normalize_delays, to_host=False)
    if world > 1:
        sel = torch.tensor(mine, dtype=torch.int64, device=dev)
        cir.a_dev = _gather_rows(cir.a_dev[sel], mine, len(rxs), world, pad_dims=(4,))
        cir.tau_dev = _gather_rows(cir.tau_dev[sel], mine, len(rxs), world, pad_dims=(2,))
    if to_host:
        cir.a = N.d2h(cir.a_dev)
        cir.tau = N.d2h(cir.tau_dev)
    return cir, ps


# ---- calibration gradients with records sharded --------------------------------------------

def material_loss_and_grad(scene, positions, h_targets, max_depth=2, num_subcarriers=128,
                           spacing=30e3, method="exhaustive", num_rays=4096, rank=0, world=1,
                           bvh=None):
    """optim.material_loss_and_grad with the records sharded round-robin: each
    rank builds the frozen topology of its records, evaluates its part of the
    mean NMSE and its gradient through the adjoint, and one all_reduce (sum)
    of [loss, d/d eps_r, d/d sigma ...] combines them.  Every rank returns the
    global (loss, grads)."""
    from .optim import MaterialProblem, _EPS_KEY, _SIG_KEY
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    h = np.asarray(h_targets)
    n = len(pos)
    from .optim import trainable_material_names
    mine = list(range(rank, n, world))
    names = trainable_material_names(scene)
    dev = bvh.device if bvh is not None else torch.device("cuda", torch.cuda.current_device())
    values = {k: (torch.tensor(float(scene.materials[k].eps_r), dtype=torch.float64, device=dev,
                               requires_grad=True),
                  torch.tensor(float(scene.materials[k].sigma), dtype=torch.float64, device=dev,
                               requires_grad=True)) for k in names}
    if mine:
        prob = MaterialProblem(scene, pos[mine], h[mine], max_depth, num_subcarriers, spacing, method,
                               num_rays, bvh)
        # the local loss is the mean over this rank's records: weight it by its share
        loss = prob.loss(values) * (len(mine) / n)
        loss.backward()
    else:
        loss = torch.zeros((), dtype=torch.float64, device=dev)
    flat = [loss.detach().reshape(1)]
    for k in names:
        for v in values[k]:
            flat.append((v.grad if v.grad is not None else torch.zeros_like(v)).reshape(1))
    vec = torch.cat(flat)
    d = _dist()
    if d is not None and world > 1:
        vec = _wire(d, vec)
        d.all_reduce(vec)
    vals = vec.tolist()
    grads = {}
    i = 1
    for k in names:
        grads[_EPS_KEY.format(k)] = vals[i]
        grads[_SIG_KEY.format(k)] = vals[i + 1]
        i += 2
    return vals[0], grads
