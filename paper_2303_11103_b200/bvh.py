"""Acceleration structure: GPU BVH (binned SAH) over the scene triangles.

Drop-in for /root/reference/pkg/src/emtrace/bvh.py: ``build(scene) -> Bvh``
with ``Bvh.intersect`` (:83-101), ``Bvh.occluded`` (:103-115) and the
per-primitive arrays the rest of the reference reads (``num_prims``,
``prim_object``, ``prim_triangle``, ``v0``/``e1``/``e2``, ``normals``,
``plane_offset``; :33-44).  Construction and queries run in libb200rt.so;
the host only flattens the meshes (``_gather`` order, :180-197).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N

RAY_EPS = 1e-4
LEAF_SIZE = 4


@dataclass(frozen=True)
class Hit:
    t: float
    prim: int
    point: np.ndarray
    normal: np.ndarray


class _PinnedStaging:
    """Reusable page-locked host buffers for the scene upload: no page faults on
    refill and truly asynchronous H2D copies (rt_bvh_build returns only after
    the upload has consumed them)."""

    def __init__(self):
        self.bufs = {}

    def get(self, name, shape, dtype):
        n = int(np.prod(shape)) if len(shape) else 1
        tdt = {np.float64: torch.float64, np.int64: torch.int64, np.int32: torch.int32}[dtype]
        b = self.bufs.get(name)
        if b is None or b.numel() < n or b.dtype != tdt:
            b = torch.empty(max(n, 1), dtype=tdt, pin_memory=True)
            self.bufs[name] = b
        return b[:n].numpy().reshape(shape)


_STAGING = {}


def _staging_for(device):
    st = _STAGING.get(device)
    if st is None:
        st = _STAGING[device] = _PinnedStaging()
    return st


def _gather_geometry(scene, alloc=None, tri_dtype=np.int64):
    """One pass over the objects into preallocated arrays: (vertices [V,3] f64,
    tri_vertex [N,3] i64 with global vertex ids, prim_material [N] i32,
    material_names, object index of each non-empty object, its triangle count).
    `alloc(name, shape, dtype)` supplies the output arrays (default np.empty)."""
    objs = []
    nv = nt = 0
    for oi, obj in enumerate(scene.objects):
        t = np.asarray(obj.triangles, dtype=np.int64).reshape(-1, 3)
        if not len(t):
            continue
        v = np.asarray(obj.vertices, dtype=np.float64).reshape(-1, 3)
        objs.append((oi, v, t))
        nv += len(v)
        nt += len(t)
    names = list(scene.materials.keys())
    mindex = {m: i for i, m in enumerate(names)}
    if alloc is None:
        def alloc(name, shape, dtype):
            return np.empty(shape, dtype=dtype)
    if nv >= 2 ** 31:
        raise ValueError("scene has 2^31 or more vertices (vertex ids are 32-bit on the device)")
    verts = alloc("verts", (nv, 3), np.float64)
    tris = alloc("tris", (nt, 3), tri_dtype)
    pmat = alloc("pmat", (nt,), np.int32)
    obj_ids = np.empty(len(objs), dtype=np.int64)
    counts = np.empty(len(objs), dtype=np.int64)
    vb = tb = 0
    jobs = []
    for k, (oi, v, t) in enumerate(objs):
        jobs.append((verts[vb:vb + len(v)], v, tris[tb:tb + len(t)], t, vb, pmat[tb:tb + len(t)],
                     mindex.get(scene.objects[oi].material, -1)))
        obj_ids[k] = oi
        counts[k] = len(t)
        vb += len(v)
        tb += len(t)
    if nv + nt >= _GATHER_PARALLEL_MIN:
        # large scenes: the copies in row chunks on host threads (numpy drops the
        # GIL in them); C5's 2M triangles gather in ~1/4 of the one-thread time
        pool = _gather_pool()
        futs = [pool.submit(_gather_chunk, job, lo, hi) for job in jobs
                for lo, hi in _chunks(max(len(job[1]), len(job[3])), _GATHER_THREADS)]
        for f in futs:
            f.result()
    else:
        for job in jobs:
            _gather_chunk(job, 0, max(len(job[1]), len(job[3])))
    return verts, tris, pmat, names, obj_ids, counts


_GATHER_PARALLEL_MIN = 1 << 20
_GATHER_THREADS = 8
_POOL = None


def _gather_pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(_GATHER_THREADS, thread_name_prefix="b200rt-gather")
    return _POOL


def _chunks(n, k):
    step = max((n + k - 1) // k, 1)
    return [(lo, min(lo + step, n)) for lo in range(0, n, step)]


def _gather_chunk(job, lo, hi):
    """rows [lo, hi) of one object's vertices and triangles (either may be shorter)"""
    vdst, v, tdst, t, vb, pdst, mat = job
    if lo < len(v):
        vdst[lo:min(hi, len(v))] = v[lo:min(hi, len(v))]
    if lo < len(t):
        e = min(hi, len(t))
        np.add(t[lo:e], vb, out=tdst[lo:e], casting="unsafe")
        pdst[lo:e] = mat


def _prim_ids(obj_ids, counts):
    """(prim_object, prim_triangle) of the _gather order from per-object counts."""
    n = int(counts.sum()) if len(counts) else 0
    prim_object = np.repeat(obj_ids, counts)
    starts = np.cumsum(counts) - counts
    prim_triangle = np.arange(n, dtype=np.int64) - np.repeat(starts, counts)
    return prim_object, prim_triangle


def gather_meshes(scene):
    """Flatten objects into (vertices [V,3], tri_vertex [N,3], prim_object, prim_triangle,
    prim_material, material_names) in the reference's global primitive order."""
    verts, tris, pmat, names, obj_ids, counts = _gather_geometry(scene)
    prim_object, prim_triangle = _prim_ids(obj_ids, counts)
    return verts, tris, prim_object, prim_triangle, pmat, names


class Bvh:
    """Device-resident scene + BVH; immutable after build, queries are stream-ordered."""

    def __init__(self, scene, device=None):
        self.ctx = N.acquire_context(device)
        self.device = self.ctx.device
        staging = _staging_for(self.device)
        verts, tris, prim_mat, self.material_names, self._obj_ids, self._obj_counts = \
            _gather_geometry(scene, staging.get, tri_dtype=np.int32)   # 32-bit vertex ids on the device
        self._prim_ids = None
        self.num_prims = len(tris)
        self.frequency_hz = float(scene.frequency_hz)
        dev = self.device
        with torch.cuda.device(dev):
            # rt_scene_upload copies the pinned staging in on the library's stream;
            # rt_bvh_build returns only after those copies, so the staging may be refilled
            s = self.ctx.stream
            self.ctx.call("rt_scene_upload", N.ptr(verts), len(verts), N.ptr(tris), N.ptr(prim_mat),
                          self.num_prims, s)
            self.ctx.call("rt_bvh_build", s)
        self._arrays = None

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None:
            self.ctx = None
            try:
                N.release_context(ctx)
            except Exception:   # interpreter shutdown
                pass

    # -- per-primitive arrays (bit-identical to the reference's numpy ones) ------------
    @property
    def prim_object(self):
        if self._prim_ids is None:
            self._prim_ids = _prim_ids(self._obj_ids, self._obj_counts)
        return self._prim_ids[0]

    @property
    def prim_triangle(self):
        if self._prim_ids is None:
            self._prim_ids = _prim_ids(self._obj_ids, self._obj_counts)
        return self._prim_ids[1]

    def _fetch_arrays(self):
        if self._arrays is None:
            n = max(self.num_prims, 0)
            with torch.cuda.device(self.device):
                outs = [torch.empty((n, 3), dtype=torch.float64, device=self.device) for _ in range(4)]
                poff = torch.empty(n, dtype=torch.float64, device=self.device)
                self.ctx.call("rt_scene_arrays", *[N.ptr(o) for o in outs], N.ptr(poff), self.ctx.stream)
                self._arrays = [o.cpu().numpy() for o in outs] + [poff.cpu().numpy()]
                self.normals_dev = outs[3]
        return self._arrays

    @property
    def v0(self):
        return self._fetch_arrays()[0]

    @property
    def e1(self):
        return self._fetch_arrays()[1]

    @property
    def e2(self):
        return self._fetch_arrays()[2]

    @property
    def normals(self):
        return self._fetch_arrays()[3]

    @property
    def plane_offset(self):
        return self._fetch_arrays()[4]

    # -- queries ----------------------------------------------------------------------
    def trace(self, origins, directions, t_min=RAY_EPS, t_max=math.inf, any_hit=False):
        """Batched closest (or any) hit: returns device tensors (t [n], prim [n], -1 miss)."""
        dev = self.device
        o = torch.as_tensor(np.asarray(origins, dtype=np.float64).reshape(-1, 3) if not
                            isinstance(origins, torch.Tensor) else origins, dtype=torch.float64,
                            device=dev).reshape(-1, 3).contiguous()
        d = torch.as_tensor(np.asarray(directions, dtype=np.float64).reshape(-1, 3) if not
                            isinstance(directions, torch.Tensor) else directions,
                            dtype=torch.float64, device=dev).reshape(-1, 3).contiguous()
        n = o.shape[0]
        tmin = torch.as_tensor(t_min, dtype=torch.float64, device=dev).expand(n).contiguous()
        tmax = torch.as_tensor(t_max, dtype=torch.float64, device=dev).expand(n).contiguous()
        t = torch.empty(n, dtype=torch.float64, device=dev)
        p = torch.empty(n, dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            self.ctx.call("rt_trace", N.ptr(o), N.ptr(d), N.ptr(tmin), N.ptr(tmax), n,
                          int(any_hit), N.ptr(t), N.ptr(p), self.ctx.stream)
        return t, p

    def intersect(self, origin, direction, t_min: float = RAY_EPS, t_max: float = math.inf):
        """Nearest hit with t in (t_min, t_max), or None (bvh.py:83-101)."""
        t, p = self.trace(origin, direction, t_min, t_max)
        prim = int(p[0].item())
        if prim < 0:
            return None
        tt = float(t[0].item())
        o = np.asarray(origin, dtype=np.float64)
        d = np.asarray(direction, dtype=np.float64)
        n = self.normals[prim]
        if float(n @ d) > 0.0:
            n = -n
        return Hit(t=tt, prim=prim, point=o + tt * d, normal=n)

    def occluded(self, p, q, eps: float = RAY_EPS) -> bool:
        """True iff a primitive cuts the open segment p -> q shrunk by eps (bvh.py:103-115)."""
        dx = float(q[0]) - float(p[0])
        dy = float(q[1]) - float(p[1])
        dz = float(q[2]) - float(p[2])
        dist = math.sqrt(dx * dx + dy * dy + dz * dz)
        if dist == 0.0:
            raise ValueError("occlusion query endpoints coincide")
        inv = 1.0 / dist
        _, prim = self.trace([float(p[0]), float(p[1]), float(p[2])], [dx * inv, dy * inv, dz * inv],
                             eps, dist - eps, any_hit=True)
        return bool(prim[0].item() >= 0)

    def occluded_batch(self, p, q):
        """Device batch of Bvh.occluded with eps = RAY_EPS; -1 marks coincident endpoints."""
        dev = self.device
        P = torch.as_tensor(p, dtype=torch.float64, device=dev).reshape(-1, 3).contiguous()
        Q = torch.as_tensor(q, dtype=torch.float64, device=dev).reshape(-1, 3).contiguous()
        out = torch.empty(P.shape[0], dtype=torch.int32, device=dev)
        with torch.cuda.device(dev):
            self.ctx.call("rt_occluded", N.ptr(P), N.ptr(Q), P.shape[0], N.ptr(out), self.ctx.stream)
        return out


def build(scene, device=None) -> Bvh:
    """Build the acceleration structure for a validated scene (bvh.py:200-202)."""
    return Bvh(scene, device)
