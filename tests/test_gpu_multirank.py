"""The sharded multi-GPU paths (parallel.py) run as 2 ranks on one GPU over gloo.

Each rank is its own process with its own library context on cuda:0; the
exchanges (candidate all_gather, grid all_reduce, CIR row all_gather, gradient
all_reduce) go through gloo with CUDA tensors staged on the host, so no kernel
of one rank waits on another.  Results must equal the single-rank ones: the
coverage map and the CIR bit for bit, the calibration loss and gradients to
1e-12 relative (a different but fixed summation order).
"""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import golden_scene, load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    import paper_2303_11103_b200 as P
    from paper_2303_11103_b200 import scenes
    city = scenes.city(n_side=10, seed=5)
    tx = city.devices[0]
    grid = P.GridSpec((float(tx.position[0]) - 80.0, float(tx.position[1]) - 64.0), 2.5, 64, 48, 1.5)
    canyon = scenes.street_canyon(n_per_row=30, n_rx=(8, 4))
    return city, tx, grid, canyon


def _single():
    import paper_2303_11103_b200 as P
    from paper_2303_11103_b200 import parallel
    city, tx, grid, canyon = _workload()
    b = P.build(city)
    _, _, g = parallel.coverage_step(city, b, tx, grid, 4, 300_000)
    cir, _ = parallel.compute_paths_cir(canyon, P.build(canyon), 3, "fibonacci", 50_000)
    cal = load_golden("calib")
    init = golden_scene(cal, "scene_init")
    loss, grads = parallel.material_loss_and_grad(init, cal["positions"], cal["h"], int(cal["max_depth"]),
                                                  int(cal["num_subcarriers"]), float(cal["spacing"]))
    return g.cpu().numpy(), cir.a, cir.tau, loss, grads


def _rank(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_11103_b200 as P
        from paper_2303_11103_b200 import parallel
        city, tx, grid, canyon = _workload()
        b = P.build(city)
        bounces, _, g = parallel.coverage_step(city, b, tx, grid, 4, 300_000, rank, world)
        cir, ps = parallel.compute_paths_cir(canyon, P.build(canyon), 3, "fibonacci", 50_000, rank, world)
        cal = load_golden("calib")
        init = golden_scene(cal, "scene_init")
        loss, grads = parallel.material_loss_and_grad(init, cal["positions"], cal["h"],
                                                      int(cal["max_depth"]), int(cal["num_subcarriers"]),
                                                      float(cal["spacing"]), rank=rank, world=world)
        q.put((rank, g.cpu().numpy(), cir.a, cir.tau, loss, grads, bounces,
               sorted(set(ps.table.rx.cpu().numpy().tolist()))))
    except Exception as e:   # surface the failure instead of a queue timeout
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_equal_single_rank():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=600) for _ in procs], key=lambda o: o[0])
    for p in procs:
        p.join(timeout=120)
    for o in out:
        assert len(o) > 2, o
    for p in procs:
        assert p.exitcode == 0
    g1, a1, tau1, loss1, grads1 = _single()
    for rank, g, a, tau, loss, grads, bounces, rxs in out:
        assert g.tobytes() == g1.tobytes()
        assert a.shape == a1.shape and a.tobytes() == a1.tobytes()
        assert tau.tobytes() == tau1.tobytes()
        assert abs(loss - loss1) <= 1e-12 * abs(loss1)
        for k, v in grads1.items():
            assert abs(grads[k] - v) <= 1e-12 * abs(v) + 1e-300, k
        assert set(rxs) <= set(range(rank, 32, 2)) and rxs   # this rank's receivers only
        assert bounces > 0
    assert (g1 > 0).sum() > 200
