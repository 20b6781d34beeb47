"""Generate golden vectors by running the REFERENCE (emtrace) itself.

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

Each case writes ``tests/golden/<case>.npz`` holding the scene (as the
reference's JSON schema, so nothing here depends on /root/reference at test
time) and the reference's outputs.  The GPU box never runs this script; it
only reads the committed .npz files.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import emtrace as E  # noqa: E402  (the reference)
from emtrace import bvh as accel  # noqa: E402
from emtrace.autodiff import Tape  # noqa: E402
from emtrace.channel import GridSpec  # noqa: E402
from emtrace.scene import load_scene, bundled_scene, scene_from_dict  # noqa: E402

from paper_2303_11103_b200 import scenes as S  # noqa: E402
from paper_2303_11103_b200.scene import (AntennaArray, RadioDevice, RadioMaterial,  # noqa: E402
                                         Scene, SceneObject, scene_to_dict)


def to_ref(scene):
    return scene_from_dict(scene_to_dict(scene))


def scene_json(ref_scene):
    return json.dumps(scene_to_dict(ref_scene))


def pack_paths(paths, max_len):
    n = len(paths)
    names = sorted({p.tx for p in paths} | {p.rx for p in paths})
    seq = np.full((n, max_len), -1, dtype=np.int32)
    verts = np.zeros((n, max_len + 2, 3))
    nrm = np.zeros((n, max_len, 3))
    cos = np.zeros((n, max_len))
    out = dict(
        p_tx=np.array([p.tx for p in paths], dtype="U32"),
        p_rx=np.array([p.rx for p in paths], dtype="U32"),
        p_kind=np.array([0 if p.kind == "los" else 1 for p in paths], dtype=np.int8),
        p_order=np.array([p.order for p in paths], dtype=np.int8),
        p_length=np.array([p.length_m for p in paths]),
        p_delay=np.array([p.delay_s for p in paths]),
        p_kdep=np.array([p.k_dep for p in paths]).reshape(n, 3),
        p_karr=np.array([p.k_arr for p in paths]).reshape(n, 3),
    )
    for i, p in enumerate(paths):
        k = p.order
        seq[i, :k] = p.seq
        verts[i, :k + 2] = p.vertices
        if k:
            nrm[i, :k] = p.normals
            cos[i, :k] = p.cos_incidence
    out.update(p_seq=seq, p_verts=verts, p_normals=nrm, p_cos=cos)
    del names
    return out


def cands_array(cands, max_len):
    cl = sorted(cands, key=lambda s: (len(s), s))
    arr = np.full((len(cl), max_len), -1, dtype=np.int32)
    for i, s in enumerate(cl):
        arr[i, :len(s)] = s
    return arr


def paths_case(name, ref_scene, max_depth, method="exhaustive", num_rays=4096, extra=None,
               launch=None, coverage=None, launch_max_len=None):
    t0 = time.time()
    tree = accel.build(ref_scene)
    ps = E.compute_paths(ref_scene, tree, max_depth, method=method, num_rays=num_rays)
    gains = E.compute_gains(ref_scene, tree, ps)
    cir = E.build_cir(gains)
    out = dict(scene=np.array(scene_json(ref_scene)), max_depth=max_depth,
               method=np.array(method), num_rays=num_rays)
    out.update(pack_paths(ps.paths, max(max_depth, 1)))
    out["gains_a"] = (np.stack([e.a for e in gains.entries]) if gains.entries
                      else np.zeros((0, 1, 1, 1), dtype=complex))
    out["cir_a"] = cir.a
    out["cir_tau"] = cir.tau
    for tx in ref_scene.transmitters:
        for depth, n in (launch or []):
            c = E.launch_candidates(ref_scene, tree, tx.position, depth, n)
            out[f"launch_{tx.name}_{depth}_{n}"] = cands_array(c, depth)
    if coverage:
        for i, (grid, depth, meth, nr, mode) in enumerate(coverage):
            cm = E.coverage_map(ref_scene, tree, grid, depth, method=meth, num_rays=nr,
                                tx_mode=mode)
            out[f"cov{i}_gains"] = cm.gains
            out[f"cov{i}_spec"] = np.array([grid.origin[0], grid.origin[1], grid.cell_size,
                                            grid.nx, grid.ny, grid.height, depth, nr])
            out[f"cov{i}_method"] = np.array(meth)
            out[f"cov{i}_mode"] = np.array(mode)
    if extra:
        out.update(extra)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}: {len(ps.paths)} paths, {time.time() - t0:.1f}s", flush=True)


def soup_case():
    sc = to_ref(S.random_soup(2000, seed=2))
    tree = accel.build(sc)
    rng = np.random.RandomState(102)
    o = rng.uniform(-60, 60, (1500, 3))
    d = rng.randn(1500, 3)
    d /= np.linalg.norm(d, axis=1)[:, None]
    t = np.full(1500, np.inf)
    prim = np.full(1500, -1, dtype=np.int64)
    normal = np.zeros((1500, 3))
    point = np.zeros((1500, 3))
    for i in range(1500):
        h = tree.intersect(o[i], d[i])
        if h is not None:
            t[i], prim[i], normal[i], point[i] = h.t, h.prim, h.normal, h.point
    rng = np.random.RandomState(9)
    p = rng.uniform(-60, 60, (600, 3))
    q = rng.uniform(-60, 60, (600, 3))
    occ = np.array([tree.occluded(a, b) for a, b in zip(p, q)])
    np.savez_compressed(os.path.join(HERE, "soup.npz"), scene=np.array(scene_json(sc)),
                        o=o, d=d, t=t, prim=prim, normal=normal, point=point,
                        occ_p=p, occ_q=q, occ=occ, normals=tree.normals,
                        plane_offset=tree.plane_offset)
    print("soup: done", flush=True)


def corner_scene():
    def q(name, c):
        v, t = S.quad(c)
        return SceneObject(name, "metal", v, t)
    return Scene(1e9, [q("wall_a", [(0, 0, 0), (0, 10, 0), (0, 10, 10), (0, 0, 10)]),
                       q("wall_b", [(0, 0, 0), (10, 0, 0), (10, 0, 10), (0, 0, 10)])],
                 {"metal": RadioMaterial("metal", "constant", 1.0, 1e7)},
                 AntennaArray(), AntennaArray(),
                 [RadioDevice("tx", "tx", np.array([4.0, 3.0, 5.0])),
                  RadioDevice("rx", "rx", np.array([3.0, 4.0, 5.0]))])


def ground_scene(tx=(0, 0, 10), rx=(100, 0, 10), L=10000.0, pol="H"):
    v, t = S.quad([(-L, -L, 0), (L, -L, 0), (L, L, 0), (-L, L, 0)])
    arr = AntennaArray(pattern="iso", polarization=pol)
    return Scene(1e9, [SceneObject("ground", "ground", v, t)],
                 {"ground": RadioMaterial("ground", "constant", 15.0, 0.015)}, arr, arr,
                 [RadioDevice("tx", "tx", np.array(tx, dtype=float)),
                  RadioDevice("rx", "rx", np.array(rx, dtype=float))])


def calib_case():
    """C4 gradient golden: NMSE frequency-response loss (optim.py:305-372) at the
    initial guess, differentiated by the reference Tape w.r.t. all 8 leaves."""
    from emtrace.optim import _central_gains, _projected_sq_error, generate_dataset
    from emtrace.channel import probe_receiver, subcarrier_frequencies
    from emtrace.tracer import compute_paths_between
    from emtrace.em import EvalContext
    truth = to_ref(S.calib_scene(n_rx=16, truth=True))
    init = to_ref(S.calib_scene(n_rx=16, truth=False))
    tree = accel.build(truth)
    ds = generate_dataset(truth, num_subcarriers=64, subcarrier_spacing_hz=30e3,
                          max_depth=2, bvh=tree)
    # receivers with no propagation path at all have a zero target (the
    # reference refuses those records, optim.py:347-348): drop them
    ds.records = [r for r in ds.records if float(np.vdot(r.h, r.h).real) > 0.0]
    f = subcarrier_frequencies(64, 30e3)
    tx = init.transmitters[0]
    names = sorted(n for n, m in init.materials.items() if m.trainable)
    tape = Tape()
    leaves = {}
    for n in names:
        leaves[n] = (tape.leaf(init.materials[n].eps_r, f"{n}:eps_r"),
                     tape.leaf(init.materials[n].sigma, f"{n}:sigma"))
    ctx = EvalContext(init, material_values=leaves)
    total = 0.0
    for rec in ds.records:
        probe = probe_receiver(rec.position)
        paths = compute_paths_between(init, tree, tx, probe, 2, "exhaustive", 4096)
        basis = np.exp(-2j * np.pi * f[:, None] * np.array([p.delay_s for p in paths])[None, :])
        g = _central_gains(init, tree, ctx, tx, probe, paths)
        norm2 = float(np.vdot(rec.h, rec.h).real)
        total = total + _projected_sq_error(tape, g, basis, rec.h) / norm2
    loss = total / len(ds.records)
    grads = tape.gradient(loss)
    np.savez_compressed(
        os.path.join(HERE, "calib.npz"), scene_truth=np.array(scene_json(truth)),
        scene_init=np.array(scene_json(init)),
        positions=np.array([r.position for r in ds.records]),
        h=np.array([r.h for r in ds.records]), loss=loss.value,
        grad_names=np.array(sorted(grads)), grads=np.array([grads[k] for k in sorted(grads)]),
        num_subcarriers=64, spacing=30e3, max_depth=2)
    print("calib: loss", loss.value, flush=True)


def geo_grad_case():
    """Orientation + position gradients: for every specular
    path of the small canyon, d|a|^2 / d(tx xyz, rx xyz, tx ypr, rx ypr) of the
    first element pair through the reference Tape, with tracked positions
    (path_geometry -> geometry_for_positions, em.py:258-288)."""
    from emtrace.em import EvalContext, path_geometry, path_materials, transfer
    sc = to_ref(_canyon_small())
    tree = accel.build(sc)
    ps = E.compute_paths(sc, tree, 3, method="fibonacci", num_rays=20000)
    tx, rx = sc.device("tx"), None
    rows = []
    for p in ps.paths:
        rx = sc.device(p.rx)
        tape = Tape()
        tp = tuple(tape.leaf(float(v), f"tx_pos{i}") for i, v in enumerate(tx.position))
        rp = tuple(tape.leaf(float(v), f"rx_pos{i}") for i, v in enumerate(rx.position))
        to = tuple(tape.leaf(float(v), f"tx_ypr{i}") for i, v in enumerate(tx.orientation))
        ro = tuple(tape.leaf(float(v), f"rx_ypr{i}") for i, v in enumerate(rx.orientation))
        ctx = EvalContext(sc, orientations={tx.name: to, rx.name: ro},
                          positions={tx.name: tp, rx.name: rp})
        geom = path_geometry(ctx, p, tx, rx)
        a = transfer(ctx, geom, path_materials(sc, tree, p), tx, rx, sc.tx_array.pattern,
                     sc.rx_array.pattern, sc.tx_array.slants[0], sc.rx_array.slants[0])
        loss = a.abs2()
        g = tape.gradient(loss)
        names = ([f"tx_pos{i}" for i in range(3)] + [f"rx_pos{i}" for i in range(3)]
                 + [f"tx_ypr{i}" for i in range(3)] + [f"rx_ypr{i}" for i in range(3)])
        rows.append((a.to_complex(), loss.value, [g[n] for n in names]))
    out = dict(scene=np.array(scene_json(sc)), num_rays=20000, max_depth=3)
    out.update(pack_paths(ps.paths, 3))
    out["a"] = np.array([r[0] for r in rows])
    out["loss"] = np.array([r[1] for r in rows])
    out["grads"] = np.array([r[2] for r in rows])
    np.savez_compressed(os.path.join(HERE, "geo_grads.npz"), **out)
    print("geo_grads:", len(rows), "paths", flush=True)


def explicit_case():
    """Explicit (non-synthetic) arrays (em.py:425-459) + Doppler (em.py:462-494)."""
    out = {}
    for name, sc in (("ground", to_ref(ground_scene(rx=(200, 0, 10)))), ("canyon", to_ref(_canyon_small()))):
        if name == "ground":
            sc.tx_array = E.AntennaArray(num_rows=8, num_cols=2, vertical_spacing=0.7,
                                         horizontal_spacing=0.5, pattern="iso", polarization="H")
        sc.synthetic_array = False
        tree = accel.build(sc)
        ps = E.compute_paths(sc, tree, 2 if name == "canyon" else 1,
                             method="fibonacci" if name == "canyon" else "exhaustive", num_rays=20000)
        gains = E.compute_gains(sc, tree, ps)
        dop = E.apply_doppler(gains, 1e6, 4, tx_velocities=[3.0, -1.0, 0.5],
                              rx_velocities={sc.receivers[0].name: [0.0, 2.0, 0.0]})
        cir = E.build_cir(gains)
        out[f"{name}_scene"] = np.array(scene_json(sc))
        out[f"{name}_a"] = np.stack([e.a for e in gains.entries])
        out[f"{name}_delay"] = np.array([e.delay for e in gains.entries])
        out[f"{name}_delays"] = np.stack([e.delays for e in gains.entries])
        out[f"{name}_kdep"] = np.stack([e.k_dep for e in gains.entries])
        out[f"{name}_dop_a"] = np.stack([e.a for e in dop.entries])
        out[f"{name}_cir_a"] = cir.a
        out[f"{name}_cir_tau"] = cir.tau
        out[f"{name}_max_depth"] = 2 if name == "canyon" else 1
    np.savez_compressed(os.path.join(HERE, "explicit.npz"), **out)
    print("explicit: done", flush=True)


def drivers_case():
    """Acceptance criteria 6 and 7 (test_acceptance.py:178-231): the reference's
    material-learning and orientation-ascent trajectories."""
    from emtrace.optim import OptimConfig, generate_dataset, learn_materials, optimize_orientation
    truth = load_scene(bundled_scene("calib_truth"))
    init = load_scene(bundled_scene("calib_init"))
    ds = generate_dataset(truth, num_subcarriers=128, subcarrier_spacing_hz=30e3, max_depth=1)
    log6 = learn_materials(init, ds, OptimConfig(iterations=300, max_depth=1))
    sc = load_scene(bundled_scene("orient"))
    c = 70.71067811865476
    region = GridSpec(origin=(c - 2.5, 47.5), cell_size=5.0, nx=1, ny=1, height=50.0)
    log7 = optimize_orientation(sc, region, OptimConfig(iterations=150, max_depth=1))
    np.savez_compressed(
        os.path.join(HERE, "drivers.npz"),
        calib_truth=np.array(scene_json(truth)), calib_init=np.array(scene_json(init)),
        orient=np.array(scene_json(sc)),
        ds_positions=np.array([r.position for r in ds.records]),
        ds_h=np.array([r.h for r in ds.records]),
        learn_names=np.array(log6.leaf_names), learn_losses=np.array(log6.losses),
        learn_final=np.array([log6.final_values[k] for k in log6.leaf_names]),
        learn_values=np.array([[v[k] for k in log6.leaf_names] for _, _, v in log6.rows]),
        orient_names=np.array(log7.leaf_names), orient_losses=np.array(log7.losses),
        orient_final=np.array([log7.final_values[k] for k in log7.leaf_names]),
        region=np.array([region.origin[0], region.origin[1], region.cell_size, region.nx,
                         region.ny, region.height]))
    print("drivers:", len(log6.rows), "learn iters,", len(log7.rows), "orient iters", flush=True)


def artifacts_case():
    """Byte formats of the CLI artifacts: the reference's own
    dump_paths text (tracer.py:314-332), save_cir file (channel.py:75-84) and
    CoverageMap.save_binary file (channel.py:164-171) for C1 and the small canyon."""
    import tempfile
    out = {}
    for name, sc, depth, meth, nr in (("c1", to_ref(S.ground_box_scene()), 1, "fibonacci", 4096),
                                       ("canyon", to_ref(_canyon_small()), 3, "fibonacci", 20000)):
        tree = accel.build(sc)
        ps = E.compute_paths(sc, tree, depth, method=meth, num_rays=nr)
        cir = E.build_cir(E.compute_gains(sc, tree, ps))
        out[f"{name}_scene"] = np.array(scene_json(sc))
        out[f"{name}_spec"] = np.array([depth, nr])
        out[f"{name}_dump"] = np.array(E.dump_paths(ps))
        out[f"{name}_dump_norm"] = np.array(E.dump_paths(ps, normalize_delays=True))
        with tempfile.TemporaryDirectory() as d:
            f = os.path.join(d, "cir.bin")
            E.save_cir(cir, f)
            out[f"{name}_cir_file"] = np.frombuffer(open(f, "rb").read(), dtype=np.uint8)
            if name == "c1":
                grid = GridSpec((-20.0, -40.0), 5.0, 16, 16, 1.5)
                cm = E.coverage_map(sc, tree, grid, 1, method="exhaustive", num_rays=4096)
                f = os.path.join(d, "cov.bin")
                cm.save_binary(f)
                out["c1_cov_file"] = np.frombuffer(open(f, "rb").read(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "artifacts.npz"), **out)
    print("artifacts: done", flush=True)


def transfer_case():
    """The em.py:291-312 ``transfer`` boundary called exactly as the reference's
    own callers do: optim._central_gains (optim.py:249-258: path_materials +
    geometry_from_path + transfer with the arrays' first slants) and
    channel.point_path_gain's probe loop (channel.py:214-232, path_geometry);
    plus the Tape gradient of sum |a|^2 w.r.t. every material leaf."""
    from emtrace.optim import _central_gains
    from emtrace.channel import probe_receiver
    from emtrace.em import EvalContext, path_geometry, path_materials, transfer
    sc = to_ref(_canyon_small())
    tree = accel.build(sc)
    tx = sc.transmitters[0]
    out = {"scene": np.array(scene_json(sc))}
    seqs, central, probes = [], [], []
    for ri, rx in enumerate(sc.receivers[:3]):
        paths = E.compute_paths_between(sc, tree, tx, rx, 2, "exhaustive", 4096)
        g = _central_gains(sc, tree, EvalContext(sc), tx, rx, paths)
        for p, z in zip(paths, g):
            seqs.append((ri,) + tuple(p.seq) + (-1,) * (2 - p.order))
            central.append(z.to_complex())
        probe = probe_receiver(np.asarray(rx.position) + np.array([0.5, -0.25, 0.0]))
        ctx = EvalContext(sc)
        ppaths = E.compute_paths_between(sc, tree, tx, probe, 2, "exhaustive", 4096)
        for p in ppaths:
            mats = path_materials(sc, tree, p)
            geom = path_geometry(ctx, p, tx, probe)
            for pat in ("_probe_theta", "_probe_phi"):
                probes.append(transfer(ctx, geom, mats, tx, probe, sc.tx_array.pattern, pat,
                                       sc.tx_array.slants[0], 0.0).to_complex())
    tape = Tape()
    names = sorted(sc.materials)
    leaves = {n: (tape.leaf(float(sc.materials[n].eps_r), f"{n}:eps_r"),
                  tape.leaf(float(sc.materials[n].sigma), f"{n}:sigma")) for n in names}
    ctx = EvalContext(sc, material_values=leaves)
    rx = sc.receivers[0]
    paths = E.compute_paths_between(sc, tree, tx, rx, 2, "exhaustive", 4096)
    loss = 0.0
    for z in _central_gains(sc, tree, ctx, tx, rx, paths):
        loss = loss + z.abs2()
    grads = tape.gradient(loss)
    out.update(seqs=np.array(seqs, dtype=np.int32), central=np.array(central),
               probes=np.array(probes), loss=loss.value, grad_names=np.array(sorted(grads)),
               grads=np.array([grads[k] for k in sorted(grads)]))
    np.savez_compressed(os.path.join(HERE, "transfer.npz"), **out)
    print("transfer: paths", len(central), "probe transfers", len(probes), flush=True)


def criteria_case():
    """Acceptance criteria 5 and 9 computed by the reference (T/test_acceptance.py
    :122-175, :255-274): Tape gradients of the two-ray reflection power w.r.t.
    (eps_r, sigma) at 5 points and of the region power w.r.t. tx yaw at 5
    points; the moving-tx Doppler phase samples."""
    from emtrace.channel import point_path_gain
    from emtrace.em import (EvalContext, apply_doppler, compute_gains, geometry_from_path,
                            path_materials, transfer)
    sc = load_scene(bundled_scene("two_ray"))
    tree = accel.build(sc)
    ps = E.compute_paths(sc, tree, 1)
    refl = [p for p in ps.paths if p.kind == "specular"][0]
    tx, rx = sc.device("tx"), sc.device("rx")
    mats = path_materials(sc, tree, refl)
    geom = geometry_from_path(refl)
    pts = [(15.0, 0.015), (3.0, 0.1), (5.24, 0.0462), (9.0, 0.3), (22.0, 0.002)]
    mat_out = []
    for eps0, sig0 in pts:
        tape = Tape()
        e, s_ = tape.leaf(eps0, "eps"), tape.leaf(sig0, "sig")
        ctx = EvalContext(sc, material_values={"ground": (e, s_)})
        out = transfer(ctx, geom, mats, tx, rx, "iso", "iso", math.pi / 2, math.pi / 2).abs2()
        g = tape.gradient(out)
        mat_out.append((out.value, g["eps"], g["sig"]))
    sc_dir = to_ref(ground_scene())
    sc_dir.tx_array = E.AntennaArray(pattern="tr38901", polarization="V")
    tree_dir = accel.build(sc_dir)
    cell = GridSpec(origin=(90.0, -5.0), cell_size=10.0, nx=1, ny=1, height=10.0).cell_center(0, 0)
    _, frozen = point_path_gain(sc_dir, tree_dir, sc_dir.device("tx"), cell, 1)
    yaw_out = []
    for yaw0 in (0.2, 0.5, 0.9, 1.3, -0.4):
        tape = Tape()
        y = tape.leaf(yaw0, "yaw")
        ctx = EvalContext(sc_dir, orientations={"tx": (y, 0.0, 0.0)})
        g, _ = point_path_gain(sc_dir, tree_dir, sc_dir.device("tx"), cell, 1, ctx=ctx,
                               frozen_paths=frozen)
        yaw_out.append((g.value, tape.gradient(g)["yaw"]))
    fs = load_scene(bundled_scene("free_space"))
    fs.frequency_hz = 3.5e9
    ftree = accel.build(fs)
    fps = E.compute_paths(fs, ftree, 1)
    moving = apply_doppler(compute_gains(fs, ftree, fps), 1e6, 14, tx_velocities=[3, 0, 0])
    np.savez_compressed(
        os.path.join(HERE, "criteria.npz"), two_ray=np.array(scene_json(sc)),
        mat_points=np.array(pts), mat_out=np.array(mat_out), dir_scene=np.array(scene_json(sc_dir)),
        cell=np.asarray(cell), yaw_points=np.array([0.2, 0.5, 0.9, 1.3, -0.4]),
        yaw_out=np.array(yaw_out), free_space=np.array(scene_json(fs)),
        doppler_a=moving.entries[0].a[0, 0, :], doppler_t=np.asarray(moving.sample_times))
    print("criteria: done", flush=True)


def main(which=None):
    cases = {
        "soup": soup_case,
        "box": lambda: paths_case(
            "box", load_scene(bundled_scene("box")), 3,
            launch=[(2, 4096), (3, 16384)],
            coverage=[(GridSpec((0.5, 0.5), 1.0, 8, 6, 1.5), 2, "exhaustive", 4096, "central")]),
        "two_ray": lambda: paths_case(
            "two_ray", load_scene(bundled_scene("two_ray")), 1,
            coverage=[(GridSpec((20.0, -30.0), 10.0, 6, 6, 1.5), 1, "exhaustive", 4096,
                       "central")]),
        "c1": lambda: paths_case(
            "c1", to_ref(S.ground_box_scene()), 1, method="fibonacci", num_rays=4096,
            launch=[(1, 4096), (2, 4096)],
            coverage=[(GridSpec((-20.0, -40.0), 5.0, 16, 16, 1.5), 1, "exhaustive", 4096,
                       "central"),
                      (GridSpec((0.0, -20.0), 8.0, 8, 6, 1.5), 2, "fibonacci", 3000, "array")]),
        "corner": lambda: paths_case("corner", to_ref(corner_scene()), 2),
        "merge": lambda: paths_case("merge", to_ref(ground_scene(rx=(20, 20, 10))), 1),
        "canyon": lambda: paths_case(
            "canyon", to_ref(_canyon_small()), 3, method="fibonacci", num_rays=20000,
            launch=[(3, 20000)],
            coverage=[(GridSpec((-40.0, -8.0), 10.0, 8, 4, 1.5), 2, "fibonacci", 2000,
                       "central")]),
        "calib": calib_case,
        "geo_grads": geo_grad_case,
        "drivers": drivers_case,
        "explicit": explicit_case,
        "artifacts": artifacts_case,
        "transfer": transfer_case,
        "criteria": criteria_case,
    }
    for k, fn in cases.items():
        if which and k not in which:
            continue
        fn()


def _canyon_small():
    sc = S.street_canyon(n_per_row=10, n_rx=(4, 2),
                         tx_array=AntennaArray(2, 2, 0.5, 0.5, "tr38901", "VH"))
    sc.rx_array = AntennaArray(1, 1, 0.5, 0.5, "dipole", "cross")
    sc.devices[0].orientation = (0.3, 0.1, 0.0)
    sc.devices[2].orientation = (1.0, -0.2, 0.4)
    return sc


if __name__ == "__main__":
    main(sys.argv[1:] or None)
