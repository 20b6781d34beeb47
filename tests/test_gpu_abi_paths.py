"""The C2 host-path entry points against the building blocks they replace.

compute_paths -> compute_gains -> build_cir (E/tracer.py:298-311,
E/em.py:359-422, E/channel.py:40-72) runs on fused entry points of the C ABI
(rt_paths_fibonacci, rt_gains_h, rt_cir_plan with the rt_paths bucket bound,
host-memory receivers staged by the library).  Each is checked here against
the separate calls it replaces, on a reduced street canyon (8x8 tr38901 array,
64 receivers, depth 3): the tables bit for bit, the gains to 1e-12 relative
(the host-side rotation / offset arithmetic moved from numpy to C).
"""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_11103_b200 as P
    assert torch.cuda.is_available()
    return P


@pytest.fixture(scope="module")
def canyon(P):
    from paper_2303_11103_b200 import scenes
    sc = scenes.street_canyon(n_per_row=20, n_rx=(16, 4))
    return sc, P.build(sc)


def _tables_equal(a, b):
    assert a.n == b.n and a.L == b.L
    for f in a.FIELDS:
        assert torch.equal(getattr(a, f), getattr(b, f)), f


def test_paths_fibonacci_equals_launch_then_paths(P, canyon):
    from paper_2303_11103_b200 import _native as N, tracer
    sc, bvh = canyon
    tx = [d for d in sc.devices if d.kind == "tx"][0]
    rx = np.array([d.position for d in sc.devices if d.kind == "rx"], dtype=np.float64)
    fused = tracer.paths_fibonacci(bvh, tx.position, rx, 3, 200_000)
    tracer.prepare_candidates(bvh, tx.position, 3, "fibonacci", 200_000)
    split = tracer.paths_to_receivers(bvh, tx.position, rx)
    assert fused.n > 0
    _tables_equal(fused, split)
    assert fused.max_per_rx == split.max_per_rx
    # receivers given as a device array: the same table
    rx_dev = torch.as_tensor(rx, device=bvh.device)
    n = ctypes.c_int64()
    with torch.cuda.device(bvh.device):
        bvh.ctx.call("rt_paths", N.ptr(tracer._pos3(tx.position)), N.ptr(rx_dev), len(rx),
                     ctypes.byref(n), bvh.ctx.stream)
        dev_table = tracer._path_table(bvh, n.value, 0)
    _tables_equal(dev_table, split)
    counts = np.bincount(split.rx.cpu().numpy(), minlength=len(rx))
    assert split.max_per_rx == counts.max()


def test_gains_native_equals_transfer_and_phasors(P, canyon):
    sc, bvh = canyon
    ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=200_000)
    fast = P.compute_gains(sc, bvh, ps).a                     # rt_gains_h
    rx0 = [d for d in sc.devices if d.kind == "rx"][0]
    # an orientation override (equal to the stored one) takes the per-path
    # row gather + rt_transfer + rt_gains_synthetic route
    ctx = P.EvalContext(sc, orientations={rx0.name: tuple(rx0.orientation)})
    ref = P.compute_gains(sc, bvh, ps, ctx=ctx).a
    assert fast.shape == ref.shape and fast.shape[0] == ps.table.n
    scale = ref.abs().max()
    assert float((fast - ref).abs().max()) <= 1e-12 * float(scale)


def test_cir_plan_bound_from_paths_equals_counted(P, canyon):
    sc, bvh = canyon
    ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=200_000)
    g = P.compute_gains(sc, bvh, ps)
    assert ps.table.max_per_rx is not None
    with_bound = P.build_cir(g)                 # no host round trip in rt_cir_plan
    ps.table.max_per_rx = None
    counted = P.build_cir(g)                    # rt_cir_plan counts the buckets
    assert with_bound.a.shape == counted.a.shape
    assert np.array_equal(with_bound.a, counted.a) and np.array_equal(with_bound.tau, counted.tau)
    # only LOS or only reflections: the bound does not apply, the plan counts
    for los, refl in ((True, False), (False, True)):
        c = P.build_cir(g, los=los, reflection=refl)
        assert c.a.shape[4] <= counted.a.shape[4]


def test_staged_uploads_round_trip(P):
    from paper_2303_11103_b200 import _native as N
    dev = torch.device("cuda", torch.cuda.current_device())
    rng = np.random.RandomState(0)
    for n in (1, 1000, (3 << 20) // 8 + 17):   # below, at and across the 1 MiB slots
        a = rng.randn(n)
        want = a.copy()
        t = N.h2d(a, dev)
        a[:] = 0.0                             # the host array may change right away
        torch.cuda.synchronize()
        assert np.array_equal(t.cpu().numpy(), want)
    b = np.arange(12, dtype=np.int32).reshape(3, 4)
    tb = N.h2d(b, dev)
    assert tb.dtype == torch.int32 and tb.shape == (3, 4) and np.array_equal(tb.cpu().numpy(), b)


def test_fused_entry_points_without_geometry(P, golden):
    """A scene without primitives: rt_paths_fibonacci takes the empty candidate
    set (LOS only, as prepare_candidates does) and coverage_map (fibonacci)
    keeps the launch-free route."""
    from conftest import golden_scene
    fs = golden_scene(golden("criteria"), "free_space")
    bvh = P.build(fs)
    assert bvh.num_prims == 0
    fib = P.compute_paths(fs, bvh, 2, method="fibonacci", num_rays=4096)
    exh = P.compute_paths(fs, bvh, 2, method="exhaustive")
    assert [(p.rx, p.kind, p.seq) for p in fib.paths] == [(p.rx, p.kind, p.seq) for p in exh.paths]
    assert all(p.kind == "los" for p in fib.paths) and len(fib.paths) > 0
    tx = [d for d in fs.devices if d.kind == "tx"][0]
    grid = P.GridSpec((float(tx.position[0]) + 5.0, float(tx.position[1]) - 8.0), 2.0, 8, 8, 1.5)
    a = P.coverage_map(fs, bvh, grid, 2, method="fibonacci", num_rays=4096)
    b = P.coverage_map(fs, bvh, grid, 2, method="exhaustive")
    assert np.array_equal(a.gains, b.gains) and (a.gains > 0).all()
