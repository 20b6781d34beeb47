"""The emtrace function boundary called the way the reference's own callers call it.

``transfer`` (E/em.py:291-312) is used by optim._central_gains
(E/optim.py:249-258) and by channel.point_path_gain's probe loop
(E/channel.py:214-232).  Those call sites are restated here verbatim against
this package; the golden values come from running them in the reference
(tests/golden/make_golden.py transfer_case).
"""

import numpy as np
import pytest
import torch

from conftest import golden_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_11103_b200 as P
    assert torch.cuda.is_available()
    return P


def _central_gains(P, scene, bvh, ctx, tx_dev, probe, paths):
    # E/optim.py:249-258, names rebound to this package
    out = []
    for path in paths:
        mats = P.path_materials(scene, bvh, path)
        geom = P.geometry_from_path(path)
        out.append(P.transfer(ctx, geom, mats, tx_dev, probe,
                              scene.tx_array.pattern, scene.rx_array.pattern,
                              scene.tx_array.slants[0], scene.rx_array.slants[0]))
    return out


def test_transfer_as_reference_callers_use_it(P, golden):
    g = golden("transfer")
    sc = golden_scene(g)
    bvh = P.build(sc)
    tx = sc.transmitters[0]
    seqs, central, probes = [], [], []
    for ri, rx in enumerate(sc.receivers[:3]):
        paths = P.compute_paths_between(sc, bvh, tx, rx, 2, "exhaustive", 4096)
        for p, z in zip(paths, _central_gains(P, sc, bvh, P.EvalContext(sc), tx, rx, paths)):
            assert isinstance(z, P.DiffComplex)
            seqs.append((ri,) + tuple(p.seq) + (-1,) * (2 - p.order))
            central.append(z.to_complex())
        # E/channel.py:214-232 (tx_mode "central")
        probe = P.probe_receiver(np.asarray(rx.position) + np.array([0.5, -0.25, 0.0]))
        ctx = P.EvalContext(sc)
        for p in P.compute_paths_between(sc, bvh, tx, probe, 2, "exhaustive", 4096):
            mats = P.path_materials(sc, bvh, p)
            geom = P.path_geometry(ctx, p, tx, probe)
            for pat in ("_probe_theta", "_probe_phi"):
                probes.append(P.transfer(ctx, geom, mats, tx, probe, sc.tx_array.pattern, pat,
                                         sc.tx_array.slants[0], 0.0).to_complex())
    assert np.array_equal(np.array(seqs, dtype=np.int32), g["seqs"])
    c, pr = np.array(central), np.array(probes)
    assert np.abs(c - g["central"]).max() <= 1e-9 * np.abs(g["central"]).max()
    assert pr.shape == g["probes"].shape
    assert np.abs(pr - g["probes"]).max() <= 1e-9 * np.abs(g["probes"]).max()
    # a PropagationPath is accepted where the PathGeometry is expected
    paths = P.compute_paths_between(sc, bvh, tx, sc.receivers[0], 2, "exhaustive", 4096)
    z = P.transfer(P.EvalContext(sc), paths[-1], P.path_materials(sc, bvh, paths[-1]), tx,
                   sc.receivers[0], sc.tx_array.pattern, sc.rx_array.pattern,
                   sc.tx_array.slants[0], sc.rx_array.slants[0])
    assert abs(z.to_complex() - central[len(paths) - 1]) == 0.0


def test_transfer_material_gradients_vs_reference_tape(P, golden):
    """Tensor leaves in EvalContext.material_values make transfer return a
    differentiable value; backward runs the adjoint (rt_transfer_bwd)."""
    g = golden("transfer")
    sc = golden_scene(g)
    bvh = P.build(sc)
    tx, rx = sc.transmitters[0], sc.receivers[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    leaves = {n: (torch.tensor(float(m.eps_r), dtype=torch.float64, device=dev, requires_grad=True),
                  torch.tensor(float(m.sigma), dtype=torch.float64, device=dev, requires_grad=True))
              for n, m in sc.materials.items()}
    ctx = P.EvalContext(sc, material_values=leaves)
    paths = P.compute_paths_between(sc, bvh, tx, rx, 2, "exhaustive", 4096)
    loss = 0.0
    for z in _central_gains(P, sc, bvh, ctx, tx, rx, paths):
        loss = loss + z.abs() ** 2
    assert abs(float(loss) - float(g["loss"])) <= 1e-9 * float(g["loss"])
    loss.backward()
    for name, ref in zip(g["grad_names"], g["grads"]):
        mat, kind = str(name).rsplit(":", 1)
        got = leaves[mat][0 if kind == "eps_r" else 1].grad
        got = 0.0 if got is None else float(got)
        assert abs(got - ref) <= 1e-6 * abs(ref) + 1e-18, (name, got, ref)
