"""Seeded procedural scenes for the BASELINE.json configurations.

All geometry is built from ``np.random.RandomState(seed)`` so the CUDA path,
the CPU oracle and the reference see identical floats.  Boxes are 4 walls +
roof = 10 triangles (no floor), matching the survey's triangle counts.
"""

from __future__ import annotations

import math

import numpy as np

from .scene import AntennaArray, RadioDevice, RadioMaterial, Scene, SceneObject

# wall quads (0,1,2,3 = bottom ring, 4..7 = top ring) and roof
_BOX_TRIS = np.array([
    [0, 1, 5], [0, 5, 4],      # y = y0 wall
    [1, 2, 6], [1, 6, 5],      # x = x1 wall
    [2, 3, 7], [2, 7, 6],      # y = y1 wall
    [3, 0, 4], [3, 4, 7],      # x = x0 wall
    [4, 5, 6], [4, 6, 7],      # roof
], dtype=np.int64)


def box_vertices(x0, x1, y0, y1, z0, z1):
    return np.array([[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0],
                     [x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]], dtype=np.float64)


def quad(corners):
    return np.asarray(corners, dtype=np.float64), np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int64)


def ground_box_scene(frequency_hz=3.5e9) -> Scene:
    """C1: ground quad over [-100,100]^2 plus one 10x10x10 box; tx/rx iso V."""
    gv, gt = quad([(-100, -100, 0), (100, -100, 0), (100, 100, 0), (-100, 100, 0)])
    objs = [SceneObject("ground", "ground", gv, gt),
            SceneObject("box", "wall", box_vertices(20, 30, 5, 15, 0, 10), _BOX_TRIS.copy())]
    mats = {"ground": RadioMaterial("ground", "constant", 5.24, 0.03),
            "wall": RadioMaterial("wall", "constant", 6.0, 0.05)}
    arr = AntennaArray(pattern="iso", polarization="V")
    devs = [RadioDevice("tx", "tx", np.array([0.0, 0.0, 10.0])),
            RadioDevice("rx", "rx", np.array([50.0, 0.0, 1.5]))]
    sc = Scene(frequency_hz, objs, mats, arr, arr, devs)
    sc.validate()
    return sc


def _boxes_to_objects(boxes, material, name_prefix, merge=True):
    """boxes: [n, 6] (x0, x1, y0, y1, z0, z1) -> SceneObjects (one merged mesh by default)."""
    if merge:
        verts = np.concatenate([box_vertices(*b) for b in boxes]) if len(boxes) else np.zeros((0, 3))
        tris = (np.concatenate([_BOX_TRIS + 8 * i for i in range(len(boxes))])
                if len(boxes) else np.zeros((0, 3), dtype=np.int64))
        return [SceneObject(name_prefix, material, verts, tris)]
    return [SceneObject(f"{name_prefix}{i}", material, box_vertices(*b), _BOX_TRIS.copy())
            for i, b in enumerate(boxes)]


def street_canyon(n_per_row=100, seed=0, n_rx=(32, 8), frequency_hz=3.5e9,
                  tx_array=None, street_half_width=10.0, alley=2.0) -> Scene:
    """C2: ground + 2 rows of boxes along a street on the x axis (2,002 tris at 100/row).

    Footprints U(14,20) m along x by 30 m deep, heights U(10,40) m; 2 m alleys.
    tx at (5, 0, 6) with an 8x8 tr38901 V array; rx on a 32x8 street grid at 1.5 m.
    """
    rng = np.random.RandomState(seed)
    boxes = []
    for side in (1.0, -1.0):
        x = -0.5 * n_per_row * 19.0
        for _ in range(n_per_row):
            w = rng.uniform(14.0, 20.0)
            h = rng.uniform(10.0, 40.0)
            y_in, y_out = side * street_half_width, side * (street_half_width + 30.0)
            boxes.append((x, x + w, min(y_in, y_out), max(y_in, y_out), 0.0, h))
            x += w + alley
    L = 0.5 * n_per_row * 19.0 + 200.0
    gv, gt = quad([(-L, -L, 0), (L, -L, 0), (L, L, 0), (-L, L, 0)])
    objs = [SceneObject("ground", "ground", gv, gt)] + _boxes_to_objects(boxes, "wall", "buildings")
    mats = {"ground": RadioMaterial("ground", "constant", 5.24, 0.03),
            "wall": RadioMaterial("wall", "constant", 6.0, 0.05)}
    tx_arr = tx_array or AntennaArray(8, 8, 0.5, 0.5, "tr38901", "V")
    rx_arr = AntennaArray(pattern="iso", polarization="V")
    devs = [RadioDevice("tx", "tx", np.array([5.0, 0.0, 6.0]))]
    nx, ny = n_rx
    xs = np.linspace(-150.0, 150.0, nx) if nx > 1 else np.array([40.0])
    ys = np.linspace(-0.8 * street_half_width, 0.8 * street_half_width, ny) if ny > 1 else np.array([0.0])
    k = 0
    for y in ys:
        for x in xs:
            devs.append(RadioDevice("rx", f"rx{k:03d}", np.array([float(x) + 0.37, float(y), 1.5])))
            k += 1
    sc = Scene(frequency_hz, objs, mats, tx_arr, rx_arr, devs)
    sc.validate()
    return sc


def city(n_side=142, seed=0, pitch=25.0, street=10.0, frequency_hz=3.5e9,
         tx_height=30.0, materials=None) -> Scene:
    """C3/C5: Manhattan grid of n_side^2 boxes (10 tris each) on a ground quad.

    Block pitch 25 m, streets 10 m, footprints jittered by U(-1.5,1.5) m per
    side, heights U(10,40) m.  n_side=142 gives 201,642 triangles (C3);
    n_side=448 gives 2,007,042 (C5).  tx sits above the central street
    crossing at ``tx_height``.
    """
    rng = np.random.RandomState(seed)
    half = 0.5 * n_side * pitch
    i = np.arange(n_side, dtype=np.float64)
    gx, gy = np.meshgrid(i, i, indexing="xy")
    x0 = -half + gx.ravel() * pitch + 0.5 * street
    y0 = -half + gy.ravel() * pitch + 0.5 * street
    n = n_side * n_side
    jit = rng.uniform(-1.5, 1.5, (n, 4))
    heights = rng.uniform(10.0, 40.0, n)
    bx0 = x0 + np.maximum(jit[:, 0], 0.0)
    bx1 = x0 + (pitch - street) + np.minimum(jit[:, 1], 0.0)
    by0 = y0 + np.maximum(jit[:, 2], 0.0)
    by1 = y0 + (pitch - street) + np.minimum(jit[:, 3], 0.0)
    boxes = np.stack([bx0, bx1, by0, by1, np.zeros(n), heights], axis=1)
    # vectorized mesh: vertices [n, 8, 3]
    X = np.stack([boxes[:, 0], boxes[:, 1], boxes[:, 1], boxes[:, 0]] * 2, axis=1)
    Y = np.stack([boxes[:, 2], boxes[:, 2], boxes[:, 3], boxes[:, 3]] * 2, axis=1)
    Z = np.concatenate([np.zeros((n, 4)), np.repeat(heights[:, None], 4, axis=1)], axis=1)
    verts = np.stack([X, Y, Z], axis=2).reshape(-1, 3)
    tris = (_BOX_TRIS[None, :, :] + 8 * np.arange(n)[:, None, None]).reshape(-1, 3)
    L = half + 100.0
    gv, gt = quad([(-L, -L, 0), (L, -L, 0), (L, L, 0), (-L, L, 0)])
    mats = materials or {"ground": RadioMaterial("ground", "constant", 5.24, 0.03),
                         "wall": RadioMaterial("wall", "constant", 6.0, 0.05)}
    objs = [SceneObject("ground", "ground", gv, gt),
            SceneObject("buildings", "wall", verts, tris)]
    # the central street crossing nearest the origin
    c = -half + round(half / pitch) * pitch
    tx = np.array([c, c, tx_height])
    arr = AntennaArray(pattern="iso", polarization="V")
    devs = [RadioDevice("tx", "tx", tx), RadioDevice("rx", "rx", tx + np.array([37.0, 3.0, -28.5]))]
    sc = Scene(frequency_hz, objs, mats, arr, arr, devs)
    return sc


def calib_scene(n_rx=400, seed=0, frequency_hz=3.5e9, truth=True) -> Scene:
    """C4: ground + 3 wall groups with 4 trainable constant materials.

    Truth eps_r in {5.24, 6.0, 4.0, 7.0}; the initial guess is (3.0, 0.1) for
    every material.  Receivers on a jittered grid at 1.5 m.
    """
    rng = np.random.RandomState(seed)
    truth_vals = {"ground_mat": (5.24, 0.03), "wall_a": (6.0, 0.05),
                  "wall_b": (4.0, 0.02), "wall_c": (7.0, 0.08)}
    mats = {k: RadioMaterial(k, "constant", *(v if truth else (3.0, 0.1)), trainable=True)
            for k, v in truth_vals.items()}
    gv, gt = quad([(-80, -80, 0), (80, -80, 0), (80, 80, 0), (-80, 80, 0)])
    groups = {"wall_a": [(-40, -25, 20, 35, 0, 18), (25, 40, 22, 30, 0, 25)],
              "wall_b": [(-45, -30, -40, -22, 0, 12)],
              "wall_c": [(28, 45, -38, -26, 0, 30)]}
    objs = [SceneObject("ground", "ground_mat", gv, gt)]
    for mat, bxs in groups.items():
        objs += _boxes_to_objects(bxs, mat, mat)
    footprints = [b for bxs in groups.values() for b in bxs]
    arr = AntennaArray(pattern="iso", polarization="V")
    devs = [RadioDevice("tx", "tx", np.array([0.0, -5.0, 12.0]))]
    side = int(math.ceil(math.sqrt(n_rx))) + 2
    k = 0
    for iy in range(side):
        for ix in range(side):
            if k == n_rx:
                break
            x = -60.0 + 120.0 * (ix + 0.5) / side + rng.uniform(-0.5, 0.5)
            y = -60.0 + 120.0 * (iy + 0.5) / side + rng.uniform(-0.5, 0.5)
            if any(b[0] - 1 <= x <= b[1] + 1 and b[2] - 1 <= y <= b[3] + 1 for b in footprints):
                continue
            devs.append(RadioDevice("rx", f"rx{k:03d}", np.array([x, y, 1.5])))
            k += 1
    sc = Scene(frequency_hz, objs, mats, arr, arr, devs)
    sc.validate()
    return sc


def random_soup(n_triangles, seed=0, extent=50.0) -> Scene:
    """Seeded triangle soup (recipe of the reference's tests/test_bvh.py:13-21)."""
    rng = np.random.RandomState(seed)
    centers = rng.uniform(-extent, extent, (n_triangles, 3))
    verts = np.repeat(centers, 3, axis=0) + rng.uniform(-1.5, 1.5, (3 * n_triangles, 3))
    tris = np.arange(3 * n_triangles).reshape(-1, 3)
    sc = Scene(1e9, [SceneObject("soup", "m", verts, tris)],
               {"m": RadioMaterial("m", "constant", eps_r=2.0)},
               AntennaArray(), AntennaArray(),
               [RadioDevice("tx", "tx", np.array([0.0, 0, 100.0])),
                RadioDevice("rx", "rx", np.array([1.0, 0, 100.0]))])
    return sc
