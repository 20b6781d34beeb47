"""numpy/ctypes restatement of emtrace's hot path (parity oracle; test-only).

Every function names the reference lines it restates.  The scalar-heavy
inner loops (BVH traversal, image solve, merge, field transfer) live in
``rt_oracle.c`` and are called through ctypes; the array bookkeeping that the
reference does with numpy (primitive gather, plane precompute, Fibonacci
directions, path assembly, synthetic-array phasors, CIR packing, OFDM
response) is restated here with the same numpy calls so that the floats agree
bit for bit where the reference's discrete decisions depend on them.

The scene is read by duck typing (the reference ``Scene`` or this repo's own
``paper_2303_11103_b200.scene.Scene`` both work): ``objects[i].vertices /
.triangles / .material``, ``materials[name]``, ``tx_array`` / ``rx_array``,
``devices[i]`` and ``frequency_hz``.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading
from dataclasses import dataclass

import numpy as np

SPEED_OF_LIGHT = 299792458.0          # geometry.py:18
VACUUM_PERMITTIVITY = 8.8541878128e-12  # geometry.py:19
_GOLDEN_SQ = (3.0 + math.sqrt(5.0)) / 2.0  # geometry.py:22
TWO_PI = 2.0 * math.pi
RAY_EPS = 1e-4
ENUM_CAP = 10_000_000                 # tracer.py:28
PATTERN_IDS = {"iso": 0, "dipole": 1, "tr38901": 2, "_probe_theta": 3, "_probe_phi": 4}
POLARIZATION_SLANTS = {"V": (0.0,), "H": (math.pi / 2,), "VH": (0.0, math.pi / 2),
                       "cross": (math.pi / 4, -math.pi / 4)}   # scene.py:26-31

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "librt_oracle.so")
_lib = None
_lib_lock = threading.Lock()


class OracleError(ValueError):
    pass


def build_library(force: bool = False) -> str:
    """Compile rt_oracle.c with the committed Makefile (gcc, no GPU needed)."""
    src = os.path.join(_HERE, "rt_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    with _lib_lock:
        if _lib is None:
            build_library()
            L = ctypes.CDLL(_LIB_PATH)
            P = ctypes.c_void_p
            i64, i32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
            L.orc_bvh_build.restype = P
            L.orc_bvh_build.argtypes = [P, P, P, i64]
            L.orc_bvh_free.argtypes = [P]
            L.orc_bvh_num_nodes.restype = i64
            L.orc_bvh_num_nodes.argtypes = [P]
            L.orc_trace.argtypes = [P, P, P, P, P, i64, i32, P, P]
            L.orc_occluded.restype = i32
            L.orc_occluded.argtypes = [P, P, P]
            L.orc_launch.argtypes = [P, P, P, P, i64, i32, P, P]
            L.orc_image_solve.restype = i32
            L.orc_image_solve.argtypes = [P, P, P, P, P, P, i32, P]
            L.orc_paths.argtypes = [P, P, P, P, P, i64, P, P, i64, i32, i32, P, P, P]
            L.orc_transfer.argtypes = [P, P, P, f64, f64, P, P, P, i32, P, i32, f64, P,
                                       i32, f64, P, P]
            L.orc_coverage.argtypes = [P, P, P, P, P, f64, f64, P, P, i32, P, P, i32, i32, P,
                                       P, i64, P, P, i64, i32, i32, P, P]
            L.orc_pset_new.restype = P
            L.orc_pset_new.argtypes = [i32]
            L.orc_pset_free.argtypes = [P]
            L.orc_pset_add.argtypes = [P, P, i64]
            L.orc_pset_size.restype = i64
            L.orc_pset_size.argtypes = [P]
            L.orc_pset_export.argtypes = [P, P]
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


# -- scene model helpers ----------------------------------------------------------

def rotation_rows(yaw, pitch, roll):
    """Intrinsic Z-Y'-X'' rows (geometry.py:50-59), Python-float arithmetic."""
    cy, sy = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    cr, sr = math.cos(roll), math.sin(roll)
    return ((cy * cp, cy * sp * sr - sy * cr, cy * sp * cr + sy * sr),
            (sy * cp, sy * sp * sr + cy * cr, sy * sp * cr - cy * sr),
            (-sp, cp * sr, cp * cr))


def rows_array(rows):
    return np.array(rows, dtype=np.float64).reshape(9)


def material_eta(mat, frequency_hz, eps_override=None, sigma_override=None):
    """Complex relative permittivity (scene.py:79-100)."""
    if mat.model == "constant":
        eps_r, sigma = mat.eps_r, mat.sigma
    else:
        a, b, c, d = mat.coeffs
        f_ghz = frequency_hz / 1e9
        eps_r = a * f_ghz ** b
        sigma = c * f_ghz ** d
    if eps_override is not None:
        eps_r = eps_override
    if sigma_override is not None:
        sigma = sigma_override
    scale = 1.0 / (2.0 * math.pi * frequency_hz * VACUUM_PERMITTIVITY)
    return complex(eps_r, sigma * (-scale))


def array_slants(arr):
    return POLARIZATION_SLANTS[arr.polarization]


def element_layout(arr, wavelength):
    """(offsets [n,3], slants [n]) with index = slant*R*C + r*C + c (scene.py:138-154)."""
    rows, cols = arr.num_rows, arr.num_cols
    dy = arr.horizontal_spacing * wavelength
    dz = arr.vertical_spacing * wavelength
    base = np.zeros((rows * cols, 3))
    for r in range(rows):
        for c in range(cols):
            base[r * cols + c, 1] = (c - (cols - 1) / 2.0) * dy
            base[r * cols + c, 2] = (r - (rows - 1) / 2.0) * dz
    sl = array_slants(arr)
    return np.vstack([base] * len(sl)), np.repeat(sl, rows * cols)


def fibonacci_directions(n: int, begin: int = 0, end: int = None) -> np.ndarray:
    """Spherical Fibonacci lattice (geometry.py:62-76); rows begin..end-1 of the
    n-point lattice (the same elementwise numpy expressions, so a slice equals
    the corresponding rows of the full array)."""
    if n < 1:
        raise OracleError("need at least one direction")
    i = np.arange(begin, n if end is None else end, dtype=np.float64)
    z = 1.0 - (2.0 * i + 1.0) / n
    phi = 2.0 * math.pi * i / _GOLDEN_SQ
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


class SceneArrays:
    """Flattened primitive arrays in global gather order (bvh.py:33-44, 180-197)."""

    def __init__(self, scene):
        v0s, e1s, e2s, objs = [], [], [], []
        for oi, obj in enumerate(scene.objects):
            t = np.asarray(obj.triangles)
            if not len(t):
                continue
            v = np.asarray(obj.vertices, dtype=np.float64)
            v0s.append(v[t[:, 0]])
            e1s.append(v[t[:, 1]] - v[t[:, 0]])
            e2s.append(v[t[:, 2]] - v[t[:, 0]])
            objs.append(np.full(len(t), oi))
        if v0s:
            self.v0 = np.ascontiguousarray(np.vstack(v0s))
            self.e1 = np.ascontiguousarray(np.vstack(e1s))
            self.e2 = np.ascontiguousarray(np.vstack(e2s))
            self.prim_object = np.concatenate(objs)
            n = np.cross(self.e1, self.e2)
            lens = np.linalg.norm(n, axis=1)
            self.normals = np.ascontiguousarray(n / lens[:, None])
            self.plane_offset = np.ascontiguousarray(
                np.einsum("ij,ij->i", self.normals, self.v0))
        else:
            z = np.zeros((0, 3))
            self.v0, self.e1, self.e2, self.normals = z, z.copy(), z.copy(), z.copy()
            self.prim_object = np.zeros(0, dtype=np.int64)
            self.plane_offset = np.zeros(0)
        self.num_prims = len(self.v0)
        self.material_names = list(scene.materials.keys())
        mat_index = {m: i for i, m in enumerate(self.material_names)}
        self.prim_material = np.ascontiguousarray(np.array(
            [mat_index[scene.objects[o].material] for o in self.prim_object], dtype=np.int32))
        self.frequency_hz = float(scene.frequency_hz)
        self.wavelength = SPEED_OF_LIGHT / self.frequency_hz

    def eta_table(self, scene, overrides=None):
        overrides = overrides or {}
        out = np.zeros((max(1, len(self.material_names)), 2))
        for i, name in enumerate(self.material_names):
            ov = overrides.get(name)
            z = material_eta(scene.materials[name], self.frequency_hz,
                             ov[0] if ov else None, ov[1] if ov else None)
            out[i] = (z.real, z.imag)
        return np.ascontiguousarray(out)


class Bvh:
    """Handle to the C restatement of the reference median-split BVH."""

    def __init__(self, sa: SceneArrays):
        self.sa = sa
        self._h = lib().orc_bvh_build(_p(sa.v0), _p(sa.e1), _p(sa.e2), sa.num_prims)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.orc_bvh_free(self._h)
            self._h = None

    @property
    def num_prims(self):
        return self.sa.num_prims

    def trace(self, origins, dirs, t_min, t_max, any_hit=False):
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
        n = len(o)
        tmin = np.ascontiguousarray(np.broadcast_to(np.asarray(t_min, dtype=np.float64), (n,)))
        tmax = np.ascontiguousarray(np.broadcast_to(np.asarray(t_max, dtype=np.float64), (n,)))
        t_out = np.zeros(n)
        p_out = np.zeros(n, dtype=np.int64)
        lib().orc_trace(self._h, _p(o), _p(d), _p(tmin), _p(tmax), n, int(any_hit),
                        _p(t_out), _p(p_out))
        return t_out, p_out

    def intersect(self, origin, direction, t_min=RAY_EPS, t_max=math.inf):
        """bvh.py:83-101 -> (t, prim, point, normal) or None."""
        t, p = self.trace(origin, direction, t_min, t_max)
        if p[0] < 0:
            return None
        o = np.asarray(origin, dtype=np.float64)
        d = np.asarray(direction, dtype=np.float64)
        n = self.sa.normals[p[0]]
        if float(n @ d) > 0.0:
            n = -n
        return float(t[0]), int(p[0]), o + float(t[0]) * d, n

    def occluded(self, p, q):
        """bvh.py:103-115."""
        a = np.ascontiguousarray(p, dtype=np.float64)
        b = np.ascontiguousarray(q, dtype=np.float64)
        r = lib().orc_occluded(self._h, _p(a), _p(b))
        if r < 0:
            raise OracleError("occlusion query endpoints coincide")
        return bool(r)


# -- candidates ----------------------------------------------------------------------

def launch_sequences(bvh: Bvh, tx_pos, max_depth: int, num_rays: int, dirs=None):
    """Per-ray hit sequences and intersect-call counts (tracer.py:217-244)."""
    if dirs is None:
        dirs = fibonacci_directions(num_rays)
    dirs = np.ascontiguousarray(dirs, dtype=np.float64)
    tx = np.ascontiguousarray(tx_pos, dtype=np.float64)
    seq = np.zeros((len(dirs), max_depth), dtype=np.int32)
    bounces = np.zeros(len(dirs), dtype=np.int32)
    lib().orc_launch(bvh._h, _p(bvh.sa.normals), _p(tx), _p(dirs), len(dirs), max_depth,
                     _p(seq), _p(bounces))
    return seq, bounces


def prefixes_from_sequences(seq: np.ndarray) -> set:
    """Every prefix of every ray's hit history as a set of tuples (tracer.py:240-241)."""
    found = set()
    for k in range(1, seq.shape[1] + 1):
        rows = seq[:, :k]
        rows = rows[rows[:, k - 1] >= 0]
        if len(rows):
            for r in np.unique(rows, axis=0):
                found.add(tuple(int(x) for x in r))
    return found


def launch_candidate_rows(bvh: Bvh, tx_pos, max_depth: int, num_rays: int, chunk: int = 1 << 22):
    """launch_candidates for launches too large for Python tuples (C3: 1e8 rays):
    the lattice is traced in chunks of numpy directions and every prefix goes
    into a C hash set.  Returns (rows [C, max_depth] int32 -1 padded, sorted by
    (length, lexicographic), total intersect calls)."""
    h = lib().orc_pset_new(int(max_depth))
    bounces = 0
    try:
        for a in range(0, num_rays, chunk):
            b = min(num_rays, a + chunk)
            seq, nb = launch_sequences(bvh, tx_pos, max_depth, b - a,
                                       dirs=fibonacci_directions(num_rays, a, b))
            bounces += int(nb.sum())
            lib().orc_pset_add(h, _p(np.ascontiguousarray(seq)), b - a)
        n = lib().orc_pset_size(h)
        rows = np.zeros((n, max_depth), dtype=np.int32)
        lib().orc_pset_export(h, _p(rows))
    finally:
        lib().orc_pset_free(h)
    return sort_candidate_rows(rows), bounces


def sort_candidate_rows(rows):
    """Rows (-1 padded) in (length, lexicographic) order."""
    rows = np.asarray(rows, dtype=np.int32)
    if not len(rows):
        return rows
    lens = (rows >= 0).sum(1)
    keys = [rows[:, j] for j in range(rows.shape[1] - 1, -1, -1)] + [lens]
    return rows[np.lexsort(keys)]


def launch_candidates(bvh: Bvh, tx_pos, max_depth: int, num_rays: int = 4096, dirs=None):
    if num_rays < 1 or max_depth < 1:
        raise OracleError("need num_rays >= 1 and max_depth >= 1")
    if bvh.num_prims == 0:
        return set()
    seq, _ = launch_sequences(bvh, tx_pos, max_depth, num_rays, dirs)
    return prefixes_from_sequences(seq)


def enumerate_candidates(num_prims: int, max_depth: int, cap: int = ENUM_CAP):
    """All sequences without immediate repeats (tracer.py:196-214)."""
    if max_depth < 1:
        raise OracleError("max_depth must be >= 1 for candidate enumeration")
    if num_prims == 0:
        return []
    if num_prims ** max_depth > cap:
        raise OracleError("exhaustive enumeration exceeds the cap; use fibonacci")
    out = [(p,) for p in range(num_prims)]
    frontier = list(out)
    for _ in range(max_depth - 1):
        frontier = [s + (p,) for s in frontier for p in range(num_prims) if p != s[-1]]
        out.extend(frontier)
    return out


def pack_candidates(cands):
    """Sequences sorted by (length, lexicographic) as int32 [C, L] (-1 padded)."""
    cl = sorted(set(cands), key=lambda s: (len(s), s))
    L = max((len(s) for s in cl), default=1)
    arr = np.full((len(cl), L), -1, dtype=np.int32)
    lens = np.zeros(len(cl), dtype=np.int8)
    for i, s in enumerate(cl):
        arr[i, :len(s)] = s
        lens[i] = len(s)
    return cl, np.ascontiguousarray(arr), lens


# -- paths -----------------------------------------------------------------------------

@dataclass
class OPath:
    tx: str
    rx: str
    kind: str
    seq: tuple
    vertices: np.ndarray
    length_m: float
    delay_s: float
    k_dep: np.ndarray
    k_arr: np.ndarray
    normals: np.ndarray
    cos_incidence: tuple

    @property
    def order(self):
        return len(self.seq)


def path_from_points(tx_name, rx_name, seq, tx, rx, points, normals):
    """tracer.py:105-133."""
    chain = [np.asarray(tx, dtype=np.float64)]
    chain += [np.asarray(p, dtype=np.float64) for p in points]
    chain.append(np.asarray(rx, dtype=np.float64))
    verts = np.stack(chain)
    segs = verts[1:] - verts[:-1]
    lens = np.linalg.norm(segs, axis=1)
    dirs = segs / lens[:, None]
    nrm = np.zeros((len(seq), 3))
    cosines = []
    for k, prim in enumerate(seq):
        n = normals[prim]
        ci = -float(dirs[k] @ n)
        if ci < 0.0:
            n = -n
            ci = -ci
        nrm[k] = n
        cosines.append(ci)
    total = float(lens.sum())
    return OPath(tx_name, rx_name, "specular" if len(seq) else "los",
                 tuple(int(s) for s in seq), verts, total, total / SPEED_OF_LIGHT,
                 dirs[0], dirs[-1], nrm, tuple(cosines))


def _candidates_for(bvh, tx_pos, max_depth, method, num_rays, dirs=None):
    if max_depth < 1 or bvh.num_prims == 0:
        return []
    if method == "exhaustive":
        return enumerate_candidates(bvh.num_prims, max_depth)
    if method == "fibonacci":
        return launch_candidates(bvh, tx_pos, max_depth, num_rays, dirs)
    raise OracleError(f"unknown path-finding method {method!r}")


def paths_to_points(bvh: Bvh, tx_pos, points, cands_packed, cap=512):
    """Kept (cand index, points) per receiver point (tracer.py:268-295 minus sort)."""
    sa = bvh.sa
    cl, arr, lens = cands_packed
    L = arr.shape[1] if arr.size else 1
    if not arr.size:
        arr = np.zeros((0, L), dtype=np.int32)
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    tx = np.ascontiguousarray(tx_pos, dtype=np.float64)
    R = len(pts)
    cand_out = np.zeros((R, cap), dtype=np.int32)
    pts_out = np.zeros((R, cap, L, 3))
    counts = np.zeros(R, dtype=np.int32)
    lib().orc_paths(bvh._h, _p(sa.normals), _p(sa.plane_offset), _p(tx), _p(pts), R,
                    _p(arr), _p(lens), len(cl), L, cap, _p(cand_out), _p(pts_out), _p(counts))
    if (counts == -2).any():
        raise OracleError("path buffer overflow")
    return cand_out, pts_out, counts


def compute_paths_between(scene, bvh, tx_dev, rx_dev, max_depth, method="exhaustive",
                          num_rays=4096, dirs=None, packed=None):
    if packed is None:
        packed = pack_candidates(_candidates_for(bvh, tx_dev.position, max_depth, method,
                                                 num_rays, dirs))
    cand_out, pts_out, counts = paths_to_points(bvh, tx_dev.position, [rx_dev.position], packed)
    if counts[0] == -1:
        raise OracleError(f"tx {tx_dev.name!r} and rx {rx_dev.name!r} coincide")
    cl = packed[0]
    out = []
    for q in range(counts[0]):
        c = cand_out[0, q]
        seq = () if c < 0 else cl[c]
        out.append(path_from_points(tx_dev.name, rx_dev.name, seq, tx_dev.position,
                                    rx_dev.position, [pts_out[0, q, k] for k in range(len(seq))],
                                    bvh.sa.normals))
    return out


def compute_paths(scene, bvh, max_depth, method="exhaustive", num_rays=4096, dirs=None):
    """All (tx, rx) pairs, tx-major (tracer.py:298-311); launch shared per tx."""
    txs = [d for d in scene.devices if d.kind == "tx"]
    rxs = [d for d in scene.devices if d.kind == "rx"]
    if not txs or not rxs:
        raise OracleError("scene needs at least one transmitter and one receiver")
    out = []
    for tx in txs:
        packed = pack_candidates(_candidates_for(bvh, tx.position, max_depth, method,
                                                 num_rays, dirs))
        cand_out, pts_out, counts = paths_to_points(
            bvh, tx.position, [r.position for r in rxs], packed)
        for r, rx in enumerate(rxs):
            if counts[r] == -1:
                raise OracleError(f"tx {tx.name!r} and rx {rx.name!r} coincide")
            for q in range(counts[r]):
                c = cand_out[r, q]
                seq = () if c < 0 else packed[0][c]
                out.append(path_from_points(tx.name, rx.name, seq, tx.position, rx.position,
                                            [pts_out[r, q, k] for k in range(len(seq))],
                                            bvh.sa.normals))
    return out


# -- transfer / gains / CIR ---------------------------------------------------------------

def transfer(bvh, eta_table, path, tx_pattern, tx_slant, tx_rows, rx_pattern, rx_slant, rx_rows):
    """em.py:291-312 for one path and one element pair -> complex."""
    sa = bvh.sa
    seq = np.ascontiguousarray(np.array(path.seq if path.seq else [0], dtype=np.int32))
    pts = np.ascontiguousarray(path.vertices[1:-1].reshape(-1)) if path.order else np.zeros(3)
    out = np.zeros(2)
    lib().orc_transfer(_p(sa.normals), _p(sa.prim_material), _p(eta_table), sa.wavelength,
                       sa.frequency_hz, _p(np.ascontiguousarray(path.vertices[0])),
                       _p(np.ascontiguousarray(path.vertices[-1])), _p(seq), path.order, _p(pts),
                       PATTERN_IDS[tx_pattern], float(tx_slant), _p(rows_array(tx_rows)),
                       PATTERN_IDS[rx_pattern], float(rx_slant), _p(rows_array(rx_rows)),
                       _p(out))
    return complex(out[0], out[1])


@dataclass
class OGain:
    tx: str
    rx: str
    kind: str
    seq: tuple
    delay: float
    a: np.ndarray  # [rx_el, tx_el, 1]


def compute_gains(scene, bvh, paths, material_overrides=None):
    """Synthetic-array gains (em.py:359-422)."""
    sa = bvh.sa
    lam = sa.wavelength
    eta = sa.eta_table(scene, material_overrides)
    out = []
    tx_arr, rx_arr = scene.tx_array, scene.rx_array
    off_tx, sl_tx = element_layout(tx_arr, lam)
    off_rx, sl_rx = element_layout(rx_arr, lam)
    devs = {d.name: d for d in scene.devices}
    for p in paths:
        txd, rxd = devs[p.tx], devs[p.rx]
        rt, rr = rotation_rows(*txd.orientation), rotation_rows(*rxd.orientation)
        off_tx_w = off_tx @ np.array(rt, dtype=np.float64).T
        off_rx_w = off_rx @ np.array(rr, dtype=np.float64).T
        base = {}
        for st in sorted(set(float(s) for s in sl_tx)):
            for sr in sorted(set(float(s) for s in sl_rx)):
                base[(st, sr)] = transfer(bvh, eta, p, tx_arr.pattern, st, rt,
                                          rx_arr.pattern, sr, rr)
        ph_tx = np.exp(1j * TWO_PI * (off_tx_w @ p.k_dep) / lam)
        ph_rx = np.exp(1j * TWO_PI * (off_rx_w @ -p.k_arr) / lam)
        a = np.empty((len(off_rx_w), len(off_tx_w)), dtype=np.complex128)
        for i in range(len(off_rx_w)):
            for j in range(len(off_tx_w)):
                a[i, j] = base[(float(sl_tx[j]), float(sl_rx[i]))] * ph_rx[i] * ph_tx[j]
        out.append(OGain(p.tx, p.rx, p.kind, p.seq, p.delay_s, a[:, :, None]))
    return out


def build_cir(scene, gains, los=True, reflection=True, normalize_delays=False):
    """channel.py:40-72 -> (a [rx, rx_el, tx, tx_el, path, 1], tau [rx, tx, path])."""
    rx_names = [d.name for d in scene.devices if d.kind == "rx"]
    tx_names = [d.name for d in scene.devices if d.kind == "tx"]
    chosen = [e for e in gains if (los and e.kind == "los") or (reflection and e.kind == "specular")]
    by_pair = {}
    for e in chosen:
        by_pair.setdefault((e.rx, e.tx), []).append(e)
    for v in by_pair.values():
        v.sort(key=lambda e: (e.delay, e.kind, e.seq))
    n_path = max((len(v) for v in by_pair.values()), default=0)
    n_rx_el = scene.rx_array.num_rows * scene.rx_array.num_cols * len(array_slants(scene.rx_array))
    n_tx_el = scene.tx_array.num_rows * scene.tx_array.num_cols * len(array_slants(scene.tx_array))
    a = np.zeros((len(rx_names), n_rx_el, len(tx_names), n_tx_el, n_path, 1), dtype=np.complex128)
    tau = np.zeros((len(rx_names), len(tx_names), n_path))
    for r, rn in enumerate(rx_names):
        for t, tn in enumerate(tx_names):
            ents = by_pair.get((rn, tn), [])
            first = ents[0].delay if (normalize_delays and ents) else 0.0
            for p, e in enumerate(ents):
                a[r, :, t, :, p, :] = e.a
                tau[r, t, p] = e.delay - first
    return a, tau


def subcarrier_frequencies(n, spacing):
    k = np.arange(n, dtype=np.float64)
    return (k - (n - 1) / 2.0) * spacing


def frequency_response(a, tau, n, spacing):
    """channel.py:107-123."""
    f = subcarrier_frequencies(n, spacing)
    phase = np.exp(-2j * np.pi * tau[:, :, :, None] * f[None, None, None, :])
    h = np.einsum("abcdpt,acpk->abcdkt", a, phase)
    nr, nre, nt, nte = a.shape[:4]
    return h.reshape(nr * nre, nt * nte, n, a.shape[-1]), f


# -- coverage ---------------------------------------------------------------------------------

def cell_centers(origin, cell_size, nx, ny, height):
    """GridSpec.cell_center for every cell, row-major [ny, nx] (channel.py:146-149)."""
    pts = np.zeros((ny, nx, 3))
    for iy in range(ny):
        for ix in range(nx):
            pts[iy, ix] = (origin[0] + (ix + 0.5) * cell_size,
                           origin[1] + (iy + 0.5) * cell_size, height)
    return pts


def coverage_map(scene, bvh, origin, cell_size, nx, ny, height, max_depth,
                 method="exhaustive", num_rays=4096, tx_name=None, tx_mode="central",
                 cell_cap=250_000, dirs=None, points=None, cap=512, packed=None):
    """Per-cell probe path gain (channel.py:190-253); returns gains [ny, nx] (or
    [len(points)] when explicit probe points are given)."""
    if points is None and nx * ny > cell_cap:
        raise OracleError(f"grid has {nx * ny} cells, above the cap of {cell_cap}")
    txs = [d for d in scene.devices if d.kind == "tx"]
    if not txs:
        raise OracleError("scene has no transmitter")
    tx = next(d for d in txs if d.name == tx_name) if tx_name else txs[0]
    sa = bvh.sa
    lam = sa.wavelength
    if packed is None:
        packed = pack_candidates(_candidates_for(bvh, tx.position, max_depth, method,
                                                 num_rays, dirs))
    cl, arr, lens = packed
    L = arr.shape[1] if arr.size else 1
    if not arr.size:
        arr = np.zeros((0, L), dtype=np.int32)
    pts = (cell_centers(origin, cell_size, nx, ny, height) if points is None
           else np.asarray(points, dtype=np.float64))
    flat = np.ascontiguousarray(pts.reshape(-1, 3))
    rows = rotation_rows(*tx.orientation)
    off, sl = element_layout(scene.tx_array, lam)
    off_w = np.ascontiguousarray(np.array(
        [[sum_row(rows[r], o) for r in range(3)] for o in off], dtype=np.float64))
    slants = np.ascontiguousarray(np.asarray(sl, dtype=np.float64))
    gains = np.zeros(len(flat))
    counts = np.zeros(len(flat), dtype=np.int32)
    mode = {"central": 0, "array": 1}.get(tx_mode)
    if mode is None:
        raise OracleError(f"unknown tx_mode {tx_mode!r}")
    lib().orc_coverage(bvh._h, _p(sa.normals), _p(sa.plane_offset), _p(sa.prim_material),
                       _p(sa.eta_table(scene)), lam, sa.frequency_hz,
                       _p(np.ascontiguousarray(tx.position, dtype=np.float64)),
                       _p(rows_array(rows)), PATTERN_IDS[scene.tx_array.pattern], _p(slants),
                       _p(off_w), len(off), mode, _p(rows_array(rotation_rows(0.0, 0.0, 0.0))),
                       _p(flat), len(flat), _p(arr), _p(lens), len(cl), L, cap,
                       _p(gains), _p(counts))
    if (counts == -1).any():
        raise OracleError("probe point coincides with the transmitter")
    if (counts == -2).any():
        raise OracleError("path buffer overflow")
    return gains.reshape(pts.shape[:-1])


def sum_row(row, v):
    """t_dot(row, v) in Python-float order (geometry.py mat_vec)."""
    return row[0] * float(v[0]) + row[1] * float(v[1]) + row[2] * float(v[2])
