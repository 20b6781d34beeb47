"""Parity at the BASELINE.json configurations' own sizes (C2, C3, C4, C5).

The other parity tests run reduced versions of the configs; these run the
shapes bench.py measures, against the CPU oracle (pinned to the reference's
golden vectors in tests/test_oracle_golden.py) on the host cores:

* C3 — 201,642-tri city, 1e8 Fibonacci rays, depth 5: the device candidate
  set equals the oracle's launch_candidates (E/tracer.py:217-244) row for row,
  with the same intersect-call count; 1,536 cells of the full 512 x 512 map
  (1,024 uniform + 512 among the lit cells) equal the oracle's per-cell probe
  gain (E/channel.py:190-253) with that candidate set.
* C5 — 2,007,042-tri city, 1e7 rays, depth 5: candidate set + 256 cells of the
  2048 x 2048 map.
* C2 — 2,002-tri canyon, 8x8 tr38901 array, 256 rx, depth 3, 1e6 rays: every
  path (rx, kind, sequence) and the CIR.
* C4 — calibration scene, 400 rx, 128 subcarriers: the NMSE loss vs the
  oracle's, and the 8 gradients vs central differences of the oracle's loss.

Tolerances: sequences / candidate rows / zero cells exact; cells, CIR and
loss 1e-9 relative (north_star: 1e-4); gradients 1e-3 relative (north_star).
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2303_11103_b200 as P
    assert torch.cuda.is_available()
    return P


def _city_case(P, n_side, cells, num_rays, n_uniform, n_lit, seed):
    import oracle as O
    from paper_2303_11103_b200 import scenes
    from paper_2303_11103_b200.tracer import get_candidates
    sc = scenes.city(n_side=n_side, seed=0)
    tx = sc.devices[0]
    half = 0.5 * cells
    grid = P.GridSpec((float(tx.position[0]) - half, float(tx.position[1]) - half), 1.0, cells, cells, 1.5)
    b = P.build(sc)
    cm = P.coverage_map(sc, b, grid, 5, method="fibonacci", num_rays=int(num_rays),
                        cell_cap=grid.num_cells)
    seq, ln = get_candidates(b)
    got_rows = seq.cpu().numpy()
    ob = O.Bvh(O.SceneArrays(sc))
    rows, bounces = O.launch_candidate_rows(ob, tx.position, 5, int(num_rays))
    assert cm.stats["ray_bounces"] == bounces
    assert got_rows.shape[0] == rows.shape[0]
    assert np.array_equal(got_rows, rows[:, :got_rows.shape[1]])
    assert (rows[:, got_rows.shape[1]:] == -1).all()
    # cells: uniform over the map + among the lit ones
    rng = np.random.RandomState(seed)
    idx = list(rng.randint(0, grid.num_cells, n_uniform))
    lit = np.flatnonzero(cm.gains.reshape(-1) > 0)
    idx += list(rng.choice(lit, n_lit, replace=False))
    idx = np.array(idx)
    iy, ix = idx // grid.nx, idx % grid.nx
    pts = np.array([grid.cell_center(int(x), int(y)) for x, y in zip(ix, iy)])
    lens = (rows >= 0).sum(1).astype(np.int8)
    want = O.coverage_map(sc, ob, grid.origin, grid.cell_size, 1, 1, grid.height, 5, points=pts,
                          packed=(range(len(rows)), np.ascontiguousarray(rows), lens))
    got = cm.gains.reshape(-1)[idx]
    assert np.array_equal(got == 0.0, want == 0.0)
    nz = want > 0
    assert nz.sum() >= n_lit
    assert np.all(np.abs(got[nz] - want[nz]) <= 1e-9 * want[nz])


def test_c3_full_size_candidates_and_cells(P):
    _city_case(P, 142, 512, 1e8, 1024, 512, seed=3)


def test_c5_candidates_and_cells(P):
    _city_case(P, 448, 2048, 1e7, 192, 64, seed=5)


def test_c2_full_size_paths_and_cir(P):
    import oracle as O
    from paper_2303_11103_b200 import scenes
    sc = scenes.street_canyon(n_per_row=100)
    b = P.build(sc)
    ps = P.compute_paths(sc, b, 3, method="fibonacci", num_rays=1_000_000)
    ob = O.Bvh(O.SceneArrays(sc))
    want = O.compute_paths(sc, ob, 3, method="fibonacci", num_rays=1_000_000)
    got = ps.paths
    assert len({p.rx for p in got}) == 256
    assert [(p.rx, p.kind, p.seq) for p in got] == [(p.rx, p.kind, p.seq) for p in want]
    for a, w in zip(got, want):
        assert abs(a.delay_s - w.delay_s) <= 1e-12 * w.delay_s
    cir = P.build_cir(P.compute_gains(sc, b, ps))
    oa, otau = O.build_cir(sc, O.compute_gains(sc, ob, want))
    assert cir.a.shape == oa.shape and cir.a.shape[:4] == (256, 1, 1, 64)
    assert np.abs(cir.a - oa).max() <= 1e-9 * np.abs(oa).max()
    assert np.allclose(cir.tau, otau, rtol=1e-12, atol=0)


class _Probe:
    def __init__(self, i, pos):
        self.name = f"rec{i}"
        self.position = np.asarray(pos, dtype=np.float64)


def _oracle_nmse(O, sc, ob, tx, recs, h, freqs, overrides):
    """E/optim.py:305-372 loss restated on the oracle: mean over records of
    ||sum_i a_i e^{-j 2 pi f tau_i} - h||^2 / ||h||^2, a_i the central-element
    gains (E/optim.py:249-258)."""
    eta = ob.sa.eta_table(sc, overrides)
    Rtx = O.rotation_rows(*tx.orientation)
    Rrx = O.rotation_rows(0.0, 0.0, 0.0)
    st = O.array_slants(sc.tx_array)[0]
    sr = O.array_slants(sc.rx_array)[0]
    tot = 0.0
    for r, paths in enumerate(recs):
        H = np.zeros(len(freqs), dtype=np.complex128)
        for p in paths:
            a = O.transfer(ob, eta, p, sc.tx_array.pattern, st, Rtx, sc.rx_array.pattern, sr, Rrx)
            H += a * np.exp(-2j * math.pi * freqs * p.delay_s)
        tot += float(np.sum(np.abs(H - h[r]) ** 2)) / float(np.sum(np.abs(h[r]) ** 2))
    return tot / len(recs)


def test_c4_full_size_loss_and_gradients(P):
    import oracle as O
    from paper_2303_11103_b200 import optim, scenes
    truth, init = scenes.calib_scene(truth=True), scenes.calib_scene(truth=False)
    pos = np.array([d.position for d in truth.devices if d.kind == "rx"], dtype=np.float64)
    assert len(pos) == 400
    ds = optim.generate_dataset(truth, pos, 128, 30e3, max_depth=2)
    h = np.array([r.h for r in ds.records])
    keep = (np.abs(h) ** 2).sum(-1) > 0.0
    pos, h = pos[keep], h[keep]
    loss, grads = optim.material_loss_and_grad(init, pos, h, 2, 128, 30e3)
    # oracle: frozen topology per record (exhaustive, depth 2), then the loss
    ob = O.Bvh(O.SceneArrays(init))
    tx = [d for d in init.devices if d.kind == "tx"][0]
    packed = O.pack_candidates(O.enumerate_candidates(ob.num_prims, 2))
    recs = [O.compute_paths_between(init, ob, tx, _Probe(i, p), 2, packed=packed)
            for i, p in enumerate(pos)]
    freqs = O.subcarrier_frequencies(128, 30e3)
    # the dataset itself: device responses of the truth scene vs the oracle's
    obt = O.Bvh(O.SceneArrays(truth))
    recs_t = [O.compute_paths_between(truth, obt, tx, _Probe(i, p), 2, packed=packed)
              for i, p in enumerate(pos[:40])]
    zero = np.zeros((40, 128), dtype=np.complex128)
    for r, paths in enumerate(recs_t):
        eta = obt.sa.eta_table(truth, None)
        H = sum(O.transfer(obt, eta, p, truth.tx_array.pattern, O.array_slants(truth.tx_array)[0],
                           O.rotation_rows(*tx.orientation), truth.rx_array.pattern,
                           O.array_slants(truth.rx_array)[0], O.rotation_rows(0.0, 0.0, 0.0))
                * np.exp(-2j * math.pi * freqs * p.delay_s) for p in paths) + zero[r]
        assert np.abs(H - h[r]).max() <= 1e-9 * np.abs(h[r]).max()
    want = _oracle_nmse(O, init, ob, tx, recs, h, freqs, None)
    assert abs(loss - want) <= 1e-9 * want
    names = sorted(n for n, m in init.materials.items() if m.trainable)
    assert len(names) == 4
    base = {n: (float(init.materials[n].eps_r), float(init.materials[n].sigma)) for n in names}
    for n in names:
        for k, key in enumerate(("eps_r", "sigma")):
            step = 1e-6 * max(abs(base[n][k]), 1e-2)
            f = []
            for sgn in (1.0, -1.0):
                ov = dict(base)
                v = list(ov[n])
                v[k] += sgn * step
                ov[n] = tuple(v)
                f.append(_oracle_nmse(O, init, ob, tx, recs, h, freqs, ov))
            fd = (f[0] - f[1]) / (2 * step)
            g = grads[f"{n}:{key}"]
            assert abs(g - fd) <= 1e-3 * abs(fd) + 1e-12, (n, key, g, fd)
