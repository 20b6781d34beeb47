"""Host-side logic on CPU: scene model, array layout, CIR packing, OFDM response,
multi-rank sharding (gloo, world_size 2).  No CUDA calls."""

import math
import os
import socket

import numpy as np
import pytest
import torch

import oracle as O
from conftest import golden_scene


def test_scene_json_roundtrip_and_element_layout(golden):
    from paper_2303_11103_b200.scene import element_layout, scene_from_dict, scene_to_dict
    g = golden("canyon")
    sc = golden_scene(g)
    sc2 = scene_from_dict(scene_to_dict(sc))
    assert scene_to_dict(sc2) == scene_to_dict(sc)
    for arr in (sc.tx_array, sc.rx_array):
        off, sl = element_layout(arr, sc.wavelength)
        ooff, osl = O.element_layout(arr, sc.wavelength)
        assert np.array_equal(off, ooff) and np.array_equal(sl, osl)


def test_gather_order_matches_reference_prim_ids(golden):
    from paper_2303_11103_b200.bvh import gather_meshes
    g = golden("canyon")
    sc = golden_scene(g)
    verts, tris, pobj, ptri, pmat, names = gather_meshes(sc)
    sa = O.SceneArrays(sc)
    assert np.array_equal(verts[tris[:, 0]], sa.v0)
    assert np.array_equal(verts[tris[:, 1]] - verts[tris[:, 0]], sa.e1)
    assert np.array_equal(pobj, sa.prim_object)
    assert np.array_equal(pmat, sa.prim_material)


def test_threaded_gather_equals_serial(monkeypatch):
    """Large scenes gather in row chunks on host threads: same arrays as one pass
    (forced here on a small multi-object scene with uneven chunk boundaries)."""
    from paper_2303_11103_b200 import bvh as B, scenes
    sc = scenes.street_canyon(n_per_row=13, seed=2)
    monkeypatch.setattr(B, "_GATHER_PARALLEL_MIN", 1 << 40)
    serial = B._gather_geometry(sc, tri_dtype=np.int32)
    monkeypatch.setattr(B, "_GATHER_PARALLEL_MIN", 1)
    threaded = B._gather_geometry(sc, tri_dtype=np.int32)
    for a, b in zip(serial, threaded):
        assert np.array_equal(np.asarray(a), np.asarray(b))
    assert threaded[1].dtype == np.int32 and len(threaded[1]) > 0


def _cpu_gains(sc, case_golden):
    """A ChannelGains built on CPU tensors from the golden path table + gains."""
    from paper_2303_11103_b200.em import ChannelGains
    from paper_2303_11103_b200.tracer import PathTable
    g = case_golden
    P = len(g["p_kind"])
    L = g["p_seq"].shape[1]
    txn = [d.name for d in sc.devices if d.kind == "tx"]
    rxn = [d.name for d in sc.devices if d.kind == "rx"]
    t = lambda a, dt=torch.float64: torch.as_tensor(np.asarray(a), dtype=dt)  # noqa: E731
    T = PathTable(L, txn, rxn, tx=t([txn.index(x) for x in g["p_tx"]], torch.int32),
                  rx=t([rxn.index(x) for x in g["p_rx"]], torch.int32),
                  cand=t(np.zeros(P), torch.int32), order=t(g["p_order"], torch.int8),
                  seq=t(g["p_seq"], torch.int32), verts=t(g["p_verts"]), length=t(g["p_length"]),
                  delay=t(g["p_delay"]), kdep=t(g["p_kdep"]), karr=t(g["p_karr"]),
                  normals=t(g["p_normals"]), cos=t(g["p_cos"]))
    return ChannelGains(sc, T, torch.as_tensor(g["gains_a"]), np.zeros(1))


@pytest.mark.parametrize("case", ["box", "canyon", "two_ray"])
def test_build_cir_packing_matches_reference(golden, case):
    from paper_2303_11103_b200.channel import build_cir
    g = golden(case)
    sc = golden_scene(g)
    cir = build_cir(_cpu_gains(sc, g))
    assert np.array_equal(cir.a, g["cir_a"])
    assert np.array_equal(cir.tau, g["cir_tau"])
    los_only = build_cir(_cpu_gains(sc, g), los=True, reflection=False)
    assert los_only.a.shape[4] <= 1


def test_shard_ranges_cover_every_slot_and_row():
    from paper_2303_11103_b200.parallel import rows_of_shard, shard_range
    for n in (1, 7, 100, 10**8 + 3):
        for w in (1, 2, 3, 8):
            rngs = [shard_range(n, r, w) for r in range(w)]
            assert rngs[0][0] == 0 and rngs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rngs, rngs[1:]))
    rows = sorted(sum((rows_of_shard(513, r, 8) for r in range(8)), []))
    assert rows == list(range(513))


def test_band_interleaved_shards_partition_the_lattice():
    """rt_launch_shard's slot sets (host restatement): disjoint, cover every slot,
    whole bands per rank, and balanced latitude mix (mean z equal across ranks)."""
    from paper_2303_11103_b200.parallel import band_unit, shard_slots
    for n in (5, 4096, 100_003, 2_000_000):
        unit = band_unit(n)
        for w in (1, 2, 3, 8):
            parts = [shard_slots(n, r, w) for r in range(w)]
            allv = np.concatenate(parts)
            assert len(allv) == n and np.array_equal(np.sort(allv), np.arange(n))
            for r, p in enumerate(parts):
                assert np.all((p // unit) % w == r)
            if n >= 2_000_000:
                z = [np.mean(1.0 - (2.0 * p + 1.0) / n) for p in parts]
                assert max(abs(v) for v in z) < 0.15, z   # contiguous ranges would give +-0.875


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2303_11103_b200 import parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.RandomState(rank)
        n = 5 + 3 * rank
        seq = torch.full((n, 3), -1, dtype=torch.int32)
        ln = torch.zeros(n, dtype=torch.int8)
        for i in range(n):
            k = rng.randint(1, 4)
            seq[i, :k] = torch.as_tensor(rng.randint(0, 6, k), dtype=torch.int32)
            ln[i] = k
        s, l_ = parallel.gather_candidates(seq, ln, world)
        g = torch.zeros((4, 3), dtype=torch.float64)
        for iy in parallel.rows_of_shard(4, rank, world):
            g[iy] = float(iy + 1)
        parallel.reduce_grid(g, world)
        mx = parallel.max_over_ranks(float(rank + 10), world)
        sm = parallel.sum_over_ranks(float(rank + 1), world)
        q.put((rank, s.numpy().tolist(), l_.numpy().tolist(), g.numpy().tolist(), mx, sm,
               seq.numpy().tolist(), ln.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_candidate_gather_and_grid_reduce():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    local_rows = [np.array(o[6]) for o in out]
    want = sum((len(r) for r in local_rows))
    for rank, s, l_, g, mx, sm, _, _ in out:
        assert len(s) == want and len(l_) == want
        # the gathered rows are rank 0's rows then rank 1's rows
        assert np.array_equal(np.array(s), np.concatenate(local_rows))
        assert np.array_equal(np.array(g)[:, 0], [1.0, 2.0, 3.0, 4.0])
        assert mx == 11.0 and sm == 3.0


def _paper_listing_scene():
    """The PAPER.md listing (tx 8x2 tr38901 VH array, rx dipole cross) on a small city."""
    from paper_2303_11103_b200 import scenes
    from paper_2303_11103_b200.sionna import (PlanarArray, RadioMaterial, Receiver, Scene,
                                              SceneObject, Transmitter)
    city = scenes.city(n_side=3, seed=5)
    sc = Scene(frequency=3.5e9, synthetic_array=True)
    for m in city.materials.values():
        sc.add(RadioMaterial(m.name, m.eps_r, m.sigma))
    for o in city.objects:
        sc.add(SceneObject(o.name, o.vertices, o.triangles, o.material))
    sc.tx_array = PlanarArray(8, 2, 0.7, 0.5, "tr38901", "VH")
    sc.rx_array = PlanarArray(1, 1, 0.5, 0.5, "dipole", "cross")
    tx = Transmitter("tx", position=[2.0, 3.0, 27.0])
    rx = Receiver("rx", position=[21.0, -14.0, 1.5])
    sc.add(tx)
    sc.add(rx)
    tx.look_at(rx)
    return sc


def test_sionna_facade_compiles_to_emtrace_scene():
    sc = _paper_listing_scene()
    em = sc._em
    assert [d.kind for d in em.devices] == ["tx", "rx"]
    assert em.tx_array.num_elements == 32 and em.rx_array.num_elements == 2
    tx = em.devices[0]
    assert abs(tx.orientation[0] - math.atan2(-17.0, 19.0)) < 1e-12
    assert sum(len(o.triangles) for o in em.objects) == 2 + 9 * 10


def _gloo_rows_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2303_11103_b200 import parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n_rx = 7
        rows = parallel.rx_of_shard(n_rx, rank, world)
        P = 2 + rank   # path-slot count differs per rank: padded to the maximum
        x = torch.zeros((len(rows), 2, P), dtype=torch.complex128)
        for j, r in enumerate(rows):
            x[j, :, :P] = complex(r, -r) + torch.arange(P, dtype=torch.float64)[None, :]
        full = parallel._gather_rows(x, rows, n_rx, world, pad_dims=(2,))
        q.put((rank, torch.view_as_real(full).numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_cir_row_gather():
    """Receiver rows r, r+W, ... of every rank land in receiver order, the path
    dimension zero-padded to the largest rank's."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_rows_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=120) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.zeros((7, 2, 3), dtype=np.complex128)
    for r in range(7):
        P = 2 + (r % 2)
        want[r, :, :P] = complex(r, -r) + np.arange(P)[None, :]
    for _, full in out:
        f = np.array(full)
        assert np.array_equal(f[..., 0] + 1j * f[..., 1], want)
