"""Pin the CPU oracle against golden vectors produced by the reference itself.

The oracle (oracle/) is test infrastructure; these tests prove it reproduces
the reference (tests/golden/make_golden.py ran emtrace to make the .npz files)
before any GPU result is compared with it.
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden_scene

PATH_CASES = ["box", "two_ray", "c1", "corner", "merge", "canyon"]


def test_soup_intersect_and_occlusion_bitwise(golden):
    g = golden("soup")
    sc = golden_scene(g)
    sa = O.SceneArrays(sc)
    assert np.array_equal(sa.normals, g["normals"])
    assert np.array_equal(sa.plane_offset, g["plane_offset"])
    b = O.Bvh(sa)
    t, p = b.trace(g["o"], g["d"], 1e-4, np.inf)
    assert np.array_equal(p, g["prim"])
    assert np.array_equal(t[p >= 0], g["t"][g["prim"] >= 0])
    occ = [b.occluded(a, q) for a, q in zip(g["occ_p"], g["occ_q"])]
    assert np.array_equal(np.array(occ), g["occ"])


@pytest.mark.parametrize("case", PATH_CASES)
def test_paths_gains_cir(golden, case):
    g = golden(case)
    sc = golden_scene(g)
    b = O.Bvh(O.SceneArrays(sc))
    paths = O.compute_paths(sc, b, int(g["max_depth"]), method=str(g["method"]),
                            num_rays=int(g["num_rays"]))
    assert len(paths) == len(g["p_kind"])
    for i, p in enumerate(paths):
        k = int(g["p_order"][i])
        assert p.tx == g["p_tx"][i] and p.rx == g["p_rx"][i]
        assert p.order == k and tuple(g["p_seq"][i, :k]) == p.seq
        assert np.array_equal(p.vertices, g["p_verts"][i, :k + 2])
        assert p.length_m == g["p_length"][i] and p.delay_s == g["p_delay"][i]
        assert np.array_equal(p.normals, g["p_normals"][i, :k])
    gains = O.compute_gains(sc, b, paths)
    if gains:
        assert np.array_equal(np.stack([e.a for e in gains]), g["gains_a"])
    a, tau = O.build_cir(sc, gains)
    assert np.array_equal(a, g["cir_a"]) and np.array_equal(tau, g["cir_tau"])


@pytest.mark.parametrize("case", ["box", "c1", "canyon"])
def test_launch_candidates(golden, case):
    g = golden(case)
    sc = golden_scene(g)
    b = O.Bvh(O.SceneArrays(sc))
    keys = [k for k in g if k.startswith("launch_")]
    assert keys
    for k in keys:
        _, txn, depth, n = k.split("_")
        tx = sc.device(txn)
        got = O.launch_candidates(b, tx.position, int(depth), int(n))
        _, arr, _ = O.pack_candidates(got)
        want = g[k]
        assert arr.shape[0] == want.shape[0]
        assert np.array_equal(arr, want[:, :arr.shape[1]])


@pytest.mark.parametrize("case", ["box", "two_ray", "c1", "canyon"])
def test_coverage(golden, case):
    g = golden(case)
    sc = golden_scene(g)
    b = O.Bvh(O.SceneArrays(sc))
    i = 0
    while f"cov{i}_gains" in g:
        ox, oy, cs, nx, ny, h, depth, nr = g[f"cov{i}_spec"]
        got = O.coverage_map(sc, b, (ox, oy), cs, int(nx), int(ny), h, int(depth),
                             method=str(g[f"cov{i}_method"]), num_rays=int(nr),
                             tx_mode=str(g[f"cov{i}_mode"]))
        assert np.array_equal(got, g[f"cov{i}_gains"]), case
        i += 1
    assert i > 0


def test_transfer_central_gains(golden):
    """Oracle transfer vs the reference's optim._central_gains values."""
    g = golden("transfer")
    sc = golden_scene(g)
    b = O.Bvh(O.SceneArrays(sc))
    eta = b.sa.eta_table(sc, None)
    tx = sc.transmitters[0]
    got, seqs = [], []
    for ri, rx in enumerate(sc.receivers[:3]):
        for p in O.compute_paths_between(sc, b, tx, rx, 2, "exhaustive"):
            seqs.append((ri,) + tuple(p.seq) + (-1,) * (2 - p.order))
            got.append(O.transfer(b, eta, p, sc.tx_array.pattern, sc.tx_array.slants[0],
                                  O.rotation_rows(*tx.orientation), sc.rx_array.pattern,
                                  sc.rx_array.slants[0], O.rotation_rows(*rx.orientation)))
    assert np.array_equal(np.array(seqs, dtype=np.int32), g["seqs"])
    assert np.abs(np.array(got) - g["central"]).max() <= 1e-12 * np.abs(g["central"]).max()
