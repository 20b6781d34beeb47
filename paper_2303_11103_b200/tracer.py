"""Specular paths: candidates, image method, LOS, merge, ordering.

Drop-in for /root/reference/pkg/src/emtrace/tracer.py.  Same public names and
semantics; the work runs in libb200rt.so:

- ``launch_candidates``  (tracer.py:217-244) -> rt_launch (Fibonacci rays +
  LBVH traversal + on-device prefix trie), returns the same ``set`` of tuples.
- ``enumerate_candidates`` (:196-214) -> rt_enumerate.
- ``compute_paths`` / ``compute_paths_between`` (:268-311) -> one launch per
  transmitter shared by every receiver (the reference relaunches per pair;
  the candidate set depends only on the tx) + rt_paths, which image-solves
  every (receiver, candidate) pair, checks LOS, merges coincident paths and
  orders them (los, order, seq).
- ``image_solve`` (:150-183), ``los_path`` (:186-193) for single queries.

``PathSet`` keeps the path table on the device (``PathSet.table``) and
materializes reference-style ``PropagationPath`` objects only when
``PathSet.paths`` is read.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .bvh import RAY_EPS, Bvh

SPEED_OF_LIGHT = 299792458.0
ENUM_CAP = 10_000_000
DEFAULT_NUM_RAYS = 4096
MERGE_TOL = 1e-6


class TracerError(ValueError):
    pass


_TRACER_ERRORS = {N.RT_EINVAL: TracerError, N.RT_ECAP: TracerError, N.RT_ECOINCIDE: TracerError,
                  N.RT_ESTATE: TracerError}


@dataclass(frozen=True)
class PropagationPath:
    """One specular (or LOS) path (tracer.py:39-57)."""

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
    def order(self) -> int:
        return len(self.seq)


class PathTable:
    """Columnar device path table (one row per path)."""

    FIELDS = ("tx", "rx", "cand", "order", "seq", "verts", "length", "delay", "kdep", "karr",
              "normals", "cos")
    # host positions of the devices the table was traced for ([n_tx, 3], [n_rx, 3]),
    # set by compute_paths; None = look them up by name
    tx_pos = None
    rx_pos = None
    tx_ypr = None   # orientations (yaw, pitch, roll) of the same devices
    rx_ypr = None
    max_per_rx = None   # most paths of one (rx, tx) pair (rt_paths); None = unknown

    def __init__(self, L, tx_names, rx_names, **cols):
        self.L = L
        self.tx_names = list(tx_names)
        self.rx_names = list(rx_names)
        for f in self.FIELDS:
            setattr(self, f, cols[f])

    @property
    def n(self):
        return int(self.order.shape[0])

    @staticmethod
    def cat(tables):
        tables = [t for t in tables if t is not None]
        L = max(t.L for t in tables)
        cols = {}
        for f in PathTable.FIELDS:
            parts = []
            for t in tables:
                v = getattr(t, f)
                if f in ("seq", "normals", "cos", "verts") and t.L < L:
                    v = _pad_L(f, v, L, t.L)
                parts.append(v)
            cols[f] = torch.cat(parts, 0)
        T = PathTable(L, tables[0].tx_names, tables[0].rx_names, **cols)
        if all(t.max_per_rx is not None for t in tables):   # one transmitter per part
            T.max_per_rx = max(t.max_per_rx for t in tables)
        return T

    def host(self):
        return {f: getattr(self, f).cpu().numpy() for f in self.FIELDS}


def _pad_L(f, v, L, L0):
    P = v.shape[0]
    if f == "seq":
        out = torch.full((P, L), -1, dtype=v.dtype, device=v.device)
        out[:, :L0] = v
    elif f == "cos":
        out = torch.zeros((P, L), dtype=v.dtype, device=v.device)
        out[:, :L0] = v
    elif f == "normals":
        out = torch.zeros((P, L, 3), dtype=v.dtype, device=v.device)
        out[:, :L0] = v
    else:  # verts [P, L+2, 3]: keep rx as the (order+1)-th vertex, zero tail
        out = torch.zeros((P, L + 2, 3), dtype=v.dtype, device=v.device)
        out[:, :L0 + 2] = v
    return out


@dataclass
class PathSet:
    scene: object
    max_depth: int
    method: str
    table: PathTable = None
    _paths: list = None

    @property
    def paths(self) -> list:
        if self._paths is None:
            self._paths = table_to_paths(self.table) if self.table is not None else []
        return self._paths

    @paths.setter
    def paths(self, v):
        self._paths = list(v)
        self.table = None

    def between(self, tx_name: str, rx_name: str) -> list:
        return [p for p in self.paths if p.tx == tx_name and p.rx == rx_name]


def table_to_paths(T: PathTable) -> list:
    if T is None or T.n == 0:
        return []
    h = T.host()
    out = []
    for i in range(T.n):
        k = int(h["order"][i])
        seq = tuple(int(s) for s in h["seq"][i, :k])
        out.append(PropagationPath(
            tx=T.tx_names[int(h["tx"][i])], rx=T.rx_names[int(h["rx"][i])],
            kind="specular" if k else "los", seq=seq, vertices=h["verts"][i, :k + 2].copy(),
            length_m=float(h["length"][i]), delay_s=float(h["delay"][i]),
            k_dep=h["kdep"][i].copy(), k_arr=h["karr"][i].copy(),
            normals=h["normals"][i, :k].copy(), cos_incidence=tuple(float(c) for c in h["cos"][i, :k])))
    return out


# -- candidates ---------------------------------------------------------------------------

def _pos3(p):
    return np.ascontiguousarray([float(p[0]), float(p[1]), float(p[2])], dtype=np.float64)


def run_launch(bvh: Bvh, tx_pos, max_depth, num_rays, slot_begin=0, slot_end=None, dirs=None,
               shard=None):
    """rt_launch on the device; returns (n_candidates, n_ray_bounces).

    shard=(index, count) launches that rank's band-interleaved share of the
    lattice (rt_launch_shard) instead of the slot range."""
    if num_rays < 1 or max_depth < 1:
        raise TracerError("need num_rays >= 1 and max_depth >= 1")
    slot_end = num_rays if slot_end is None else slot_end
    txh = _pos3(tx_pos)
    nc = ctypes.c_int64()
    nb = ctypes.c_int64()
    d = None
    if dirs is not None:
        d = torch.as_tensor(dirs, dtype=torch.float64, device=bvh.device).reshape(-1, 3).contiguous()
    with torch.cuda.device(bvh.device):
        if shard is not None and int(shard[1]) > 1:
            bvh.ctx.call("rt_launch_shard", N.ptr(txh), int(num_rays), int(shard[0]), int(shard[1]),
                         int(max_depth), N.ptr(d), ctypes.byref(nc), ctypes.byref(nb),
                         bvh.ctx.stream, exc_map=_TRACER_ERRORS)
        else:
            bvh.ctx.call("rt_launch", N.ptr(txh), int(num_rays), int(slot_begin), int(slot_end),
                         int(max_depth), N.ptr(d), ctypes.byref(nc), ctypes.byref(nb), bvh.ctx.stream,
                         exc_map=_TRACER_ERRORS)
    return nc.value, nb.value


def run_enumerate(bvh: Bvh, max_depth, cap=ENUM_CAP):
    nc = ctypes.c_int64()
    with torch.cuda.device(bvh.device):
        bvh.ctx.call("rt_enumerate", int(max_depth), int(cap), ctypes.byref(nc), bvh.ctx.stream,
                     exc_map=_TRACER_ERRORS)
    return nc.value


def set_candidates(bvh: Bvh, seq, lens, max_len):
    """Install a candidate list (device or host arrays); returns the unique count."""
    s = torch.as_tensor(seq, dtype=torch.int32, device=bvh.device).reshape(-1, max_len).contiguous()
    ln = torch.as_tensor(lens, dtype=torch.int8, device=bvh.device).reshape(-1).contiguous()
    nu = ctypes.c_int64()
    with torch.cuda.device(bvh.device):
        bvh.ctx.call("rt_candidates_set", N.ptr(s), N.ptr(ln), s.shape[0], int(max_len),
                     ctypes.byref(nu), bvh.ctx.stream, exc_map=_TRACER_ERRORS)
    return nu.value


def get_candidates(bvh: Bvh):
    """Current candidate list as device tensors (seq [C, L] -1 padded, len [C])."""
    lib = bvh.ctx.lib
    n = lib.rt_num_candidates(bvh.ctx.h)
    L = lib.rt_candidates_max_len(bvh.ctx.h)
    seq = torch.empty((max(n, 0), L), dtype=torch.int32, device=bvh.device)
    ln = torch.empty(max(n, 0), dtype=torch.int8, device=bvh.device)
    if n:
        with torch.cuda.device(bvh.device):
            bvh.ctx.call("rt_candidates_get", N.ptr(seq), N.ptr(ln), L, bvh.ctx.stream)
    return seq, ln


def _cands_to_tuples(seq, ln):
    s = seq.cpu().numpy()
    lens = ln.cpu().numpy()
    return [tuple(int(x) for x in s[i, :lens[i]]) for i in range(len(lens))]


def launch_candidates(scene, bvh: Bvh, tx_pos, max_depth: int, num_rays: int = DEFAULT_NUM_RAYS):
    """Candidate sequences hit by Fibonacci-lattice rays from tx_pos (tracer.py:217-244)."""
    if num_rays < 1 or max_depth < 1:
        raise TracerError("need num_rays >= 1 and max_depth >= 1")
    if bvh.num_prims == 0:
        return set()
    run_launch(bvh, tx_pos, max_depth, num_rays)
    return set(_cands_to_tuples(*get_candidates(bvh)))


def enumerate_candidates(bvh: Bvh, max_depth: int, cap: int = ENUM_CAP):
    """All sequences of length 1..max_depth without immediate repeats (tracer.py:196-214)."""
    if max_depth < 1:
        raise TracerError("max_depth must be >= 1 for candidate enumeration")
    if bvh.num_prims == 0:
        return []
    run_enumerate(bvh, max_depth, cap)
    return _cands_to_tuples(*get_candidates(bvh))


def prepare_candidates(bvh: Bvh, tx_pos, max_depth, method, num_rays):
    """Make the context's candidate set the one compute_paths_between would use."""
    if max_depth >= 1 and bvh.num_prims:
        if method == "exhaustive":
            run_enumerate(bvh, max_depth)
        elif method == "fibonacci":
            run_launch(bvh, tx_pos, max_depth, num_rays)
        else:
            raise TracerError(f"unknown path-finding method {method!r}")
    else:
        set_candidates(bvh, np.zeros((0, 1), dtype=np.int32), np.zeros(0, dtype=np.int8), 1)


# -- paths --------------------------------------------------------------------------------

def paths_to_receivers(bvh: Bvh, tx_pos, rx_pos, tx_index=0) -> PathTable:
    """rt_paths for the current candidate set; returns the device path table."""
    rx = np.ascontiguousarray(np.asarray(rx_pos, dtype=np.float64).reshape(-1, 3))   # staged in by rt_paths
    n = ctypes.c_int64()
    txh = _pos3(tx_pos)
    with torch.cuda.device(bvh.device):
        bvh.ctx.call("rt_paths", N.ptr(txh), N.ptr(rx), rx.shape[0], ctypes.byref(n), bvh.ctx.stream,
                     exc_map=_TRACER_ERRORS)
        return _path_table(bvh, n.value, tx_index)


def paths_fibonacci(bvh: Bvh, tx_pos, rx_pos, max_depth, num_rays, tx_index=0) -> PathTable:
    """prepare_candidates("fibonacci") + paths_to_receivers as one library call
    (rt_paths_fibonacci: no host round trip between the launch and the paths)."""
    if num_rays < 1 or max_depth < 1:
        raise TracerError("need num_rays >= 1 and max_depth >= 1")
    rx = np.ascontiguousarray(np.asarray(rx_pos, dtype=np.float64).reshape(-1, 3))
    nc, nb, n = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    txh = _pos3(tx_pos)
    with torch.cuda.device(bvh.device):
        bvh.ctx.call("rt_paths_fibonacci", N.ptr(txh), int(num_rays), int(max_depth), N.ptr(rx), rx.shape[0],
                     ctypes.byref(nc), ctypes.byref(nb), ctypes.byref(n), bvh.ctx.stream, exc_map=_TRACER_ERRORS)
        return _path_table(bvh, n.value, tx_index)


def _path_table(bvh: Bvh, P, tx_index) -> PathTable:
    """The library's current path table (P rows) as device tensors."""
    dev = bvh.device
    L = bvh.ctx.lib.rt_candidates_max_len(bvh.ctx.h)
    f64 = dict(dtype=torch.float64, device=dev)
    cols = dict(rx=torch.empty(P, dtype=torch.int32, device=dev),
                cand=torch.empty(P, dtype=torch.int32, device=dev),
                order=torch.empty(P, dtype=torch.int8, device=dev),
                seq=torch.empty((P, L), dtype=torch.int32, device=dev),
                verts=torch.empty((P, L + 2, 3), **f64), length=torch.empty(P, **f64),
                delay=torch.empty(P, **f64), kdep=torch.empty((P, 3), **f64),
                karr=torch.empty((P, 3), **f64), normals=torch.empty((P, L, 3), **f64),
                cos=torch.empty((P, L), **f64))
    if P:
        bvh.ctx.call("rt_paths_get", *[N.ptr(cols[k]) for k in
                                       ("rx", "cand", "order", "seq", "verts", "length", "delay",
                                        "kdep", "karr", "normals", "cos")], bvh.ctx.stream)
    cols["tx"] = torch.full((P,), tx_index, dtype=torch.int32, device=dev)
    T = PathTable(L, [], [], **cols)
    T.max_per_rx = int(bvh.ctx.lib.rt_paths_max_per_receiver(bvh.ctx.h))
    return T


def compute_paths_between(scene, bvh: Bvh, tx_dev, rx_dev, max_depth: int,
                          method: str = "exhaustive", num_rays: int = DEFAULT_NUM_RAYS):
    """All valid paths from one tx to one rx, deduplicated and sorted (tracer.py:268-295)."""
    prepare_candidates(bvh, tx_dev.position, max_depth, method, num_rays)
    T = paths_to_receivers(bvh, tx_dev.position, [rx_dev.position])
    T.tx_names, T.rx_names = [tx_dev.name], [rx_dev.name]
    return table_to_paths(T)


def compute_paths(scene, bvh: Bvh, max_depth: int, method: str = "exhaustive",
                  num_rays: int = DEFAULT_NUM_RAYS) -> PathSet:
    """Paths for every (tx, rx) device pair, tx-major then rx (tracer.py:298-311)."""
    txs = [d for d in scene.devices if d.kind == "tx"]
    rxs = [d for d in scene.devices if d.kind == "rx"]
    if not txs or not rxs:
        raise TracerError("scene needs at least one transmitter and one receiver")
    if max_depth < 0:
        raise TracerError("max_depth must be >= 0")
    rx_pos = np.array([r.position for r in rxs], dtype=np.float64).reshape(-1, 3)
    tables = []
    for ti, tx in enumerate(txs):
        if method == "fibonacci" and max_depth >= 1:
            tables.append(paths_fibonacci(bvh, tx.position, rx_pos, max_depth, num_rays, tx_index=ti))
        else:
            prepare_candidates(bvh, tx.position, max_depth, method, num_rays)
            tables.append(paths_to_receivers(bvh, tx.position, rx_pos, tx_index=ti))
    T = PathTable.cat(tables) if len(tables) > 1 else tables[0]
    T.tx_names = [t.name for t in txs]
    T.rx_names = [r.name for r in rxs]
    T.tx_pos = np.array([t.position for t in txs], dtype=np.float64).reshape(-1, 3)
    T.rx_pos = rx_pos
    T.tx_ypr = _orientations(txs)
    T.rx_ypr = _orientations(rxs)
    return PathSet(scene=scene, max_depth=max_depth, method=method, table=T)


def _orientations(devs):
    """[n, 3] (yaw, pitch, roll); devices sharing one orientation object (the
    dataclass default) cost one conversion."""
    o0 = devs[0].orientation
    if all(d.orientation is o0 for d in devs):
        return np.tile(np.asarray(o0, dtype=np.float64).reshape(1, 3), (len(devs), 1))
    return np.array([d.orientation for d in devs], dtype=np.float64).reshape(-1, 3)


def solve_pairs(bvh: Bvh, tx_pos, rx_pos, seqs, lens):
    """Batched image_solve (tracer.py:150-183) of independent (tx, rx, seq) rows
    via rt_solve_pairs; order-0 rows are LOS visibility checks.  Returns
    (valid [n] bool tensor, PathTable with one row per input)."""
    dev = bvh.device
    f64 = dict(dtype=torch.float64, device=dev)
    if isinstance(tx_pos, np.ndarray) and not tx_pos.flags.writeable:
        tx_pos = np.array(tx_pos)
    if isinstance(rx_pos, np.ndarray) and not rx_pos.flags.writeable:
        rx_pos = np.array(rx_pos)
    if not isinstance(tx_pos, torch.Tensor):
        tx_pos = np.asarray(tx_pos, dtype=np.float64)
    if not isinstance(rx_pos, torch.Tensor):
        rx_pos = np.asarray(rx_pos, dtype=np.float64)
    tx = torch.as_tensor(tx_pos, **f64).reshape(-1, 3).contiguous()
    rx = torch.as_tensor(rx_pos, **f64).reshape(-1, 3).contiguous()
    sq = torch.as_tensor(seqs, dtype=torch.int32, device=dev).contiguous()
    n, L = sq.shape[0], max(sq.shape[1] if sq.dim() == 2 else 1, 1)
    sq = sq.reshape(n, L)
    ln = torch.as_tensor(lens, dtype=torch.int8, device=dev).reshape(n).contiguous()
    valid = torch.zeros(n, dtype=torch.uint8, device=dev)
    cols = dict(rx=torch.zeros(n, dtype=torch.int32, device=dev),
                cand=torch.zeros(n, dtype=torch.int32, device=dev),
                order=torch.zeros(n, dtype=torch.int8, device=dev),
                seq=torch.full((n, L), -1, dtype=torch.int32, device=dev),
                verts=torch.zeros((n, L + 2, 3), **f64), length=torch.zeros(n, **f64),
                delay=torch.zeros(n, **f64), kdep=torch.zeros((n, 3), **f64),
                karr=torch.zeros((n, 3), **f64), normals=torch.zeros((n, L, 3), **f64),
                cos=torch.zeros((n, L), **f64), tx=torch.zeros(n, dtype=torch.int32, device=dev))
    if n:
        with torch.cuda.device(dev):
            bvh.ctx.call("rt_solve_pairs", n, L, N.ptr(tx), N.ptr(rx), N.ptr(sq), N.ptr(ln),
                         N.ptr(valid), N.ptr(cols["verts"]), N.ptr(cols["length"]),
                         N.ptr(cols["delay"]), N.ptr(cols["kdep"]), N.ptr(cols["karr"]),
                         N.ptr(cols["normals"]), N.ptr(cols["cos"]), N.ptr(cols["seq"]),
                         N.ptr(cols["order"]), bvh.ctx.stream, exc_map=_TRACER_ERRORS)
    return valid.bool(), PathTable(L, [], [], **cols)


def image_solve(tx_name, rx_name, tx_pos, rx_pos, seq, bvh: Bvh):
    """Image-method solve of one candidate (tracer.py:150-183); None when invalid."""
    seq = tuple(int(s) for s in seq)
    if not seq:
        raise TracerError("image_solve needs a non-empty sequence")
    valid, T = solve_pairs(bvh, [_pos3(tx_pos)], [_pos3(rx_pos)], [list(seq)], [len(seq)])
    if not bool(valid[0]):
        return None
    T.tx_names, T.rx_names = [tx_name], [rx_name]
    return table_to_paths(T)[0]


def los_path(scene, bvh: Bvh, tx_dev, rx_dev):
    """LOS path or None when blocked (tracer.py:186-193)."""
    if np.allclose(tx_dev.position, rx_dev.position):
        raise TracerError(f"tx {tx_dev.name!r} and rx {rx_dev.name!r} coincide")
    set_candidates(bvh, np.zeros((0, 1), dtype=np.int32), np.zeros(0, dtype=np.int8), 1)
    T = paths_to_receivers(bvh, tx_dev.position, [rx_dev.position])
    T.tx_names, T.rx_names = [tx_dev.name], [rx_dev.name]
    ps = table_to_paths(T)
    return ps[0] if ps else None


def dump_paths(pathset: PathSet, normalize_delays: bool = False) -> str:
    """The CLI trace text format (tracer.py:314-332)."""
    first = {}
    if normalize_delays:
        for p in pathset.paths:
            key = (p.tx, p.rx)
            first[key] = min(first.get(key, math.inf), p.delay_s)
    lines = ["# tx rx type order length_m delay_s primitive_ids vertices"]
    for p in pathset.paths:
        verts = ";".join(",".join(repr(float(x)) for x in v) for v in p.vertices)
        prims = ",".join(str(s) for s in p.seq) if p.seq else "-"
        delay = p.delay_s - first.get((p.tx, p.rx), 0.0)
        lines.append(f"{p.tx} {p.rx} {p.kind} {p.order} {p.length_m!r} {delay!r} {prims} {verts}")
    return "\n".join(lines) + "\n"
