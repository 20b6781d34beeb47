"""Polarized channel coefficients along traced paths (+ adjoint).

Drop-in for /root/reference/pkg/src/emtrace/em.py.  ``transfer`` (:291-312)
and ``compute_gains`` (:359-422, synthetic arrays) evaluate every path and
element-slant pair in one rt_transfer launch; the plane-wave array phasors
(:408-415) are applied on the device with torch.  Gradients with respect to
material parameters flow through ``PathCoefficients`` (a
``torch.autograd.Function`` whose backward is the hand-written adjoint
kernel rt_transfer_bwd) — this replaces the reference's scalar Tape.
"""

from __future__ import annotations

import ctypes
import math
import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .scene import (POLARIZATION_SLANTS, SPEED_OF_LIGHT, element_layout, eta_scale,
                    material_params)
from .tracer import PathSet, PathTable

TWO_PI = 2.0 * math.pi


class EmError(ValueError):
    pass


def rotation_entries(yaw, pitch, roll):
    """Intrinsic Z-Y'-X'' rows (geometry.py:50-59)."""
    cy, sy = math.cos(yaw), math.sin(yaw)
    cp, sp = math.cos(pitch), math.sin(pitch)
    cr, sr = math.cos(roll), math.sin(roll)
    return ((cy * cp, cy * sp * sr - sy * cr, cy * sp * cr + sy * sr),
            (sy * cp, sy * sp * sr + cy * cr, sy * sp * cr - cy * sr),
            (-sp, cp * sr, cp * cr))


def pattern_id(name):
    try:
        return N.PATTERN_IDS[name]
    except KeyError:
        raise EmError(f"unknown antenna pattern {name!r}") from None


class EvalContext:
    """Per-evaluation parameter values (em.py:186-227).

    ``material_values`` maps material name -> (eps_r, sigma) (floats or 0-d
    tensors); ``orientations`` maps device name -> (yaw, pitch, roll).
    """

    def __init__(self, scene, material_values=None, orientations=None, positions=None):
        self.scene = scene
        self.material_values = material_values or {}
        self.orientations = orientations or {}
        self.positions = positions or {}

    def rotation_rows(self, device):
        ypr = self.orientations.get(device.name, device.orientation)
        if any(isinstance(v, torch.Tensor) for v in ypr):   # autograd leaves: no memo
            return rotation_entries(*ypr)
        key = (float(ypr[0]), float(ypr[1]), float(ypr[2]))   # many receivers share one
        memo = self.__dict__.setdefault("_rows_memo", {})
        rows = memo.get(key)
        if rows is None:
            rows = memo[key] = rotation_entries(*key)
        return rows

    def rotation_rows_many(self, devices):
        """rotation_rows for a list of devices: one rotation per distinct
        orientation, shared row tuples (receivers mostly share one)."""
        yprs = [self.orientations.get(d.name, d.orientation) for d in devices]
        if yprs and all(y is yprs[0] for y in yprs) and not any(isinstance(v, torch.Tensor) for v in yprs[0]):
            r = self.rotation_rows(devices[0])   # one shared orientation object (the default)
            return [r] * len(devices)
        try:
            arr = np.asarray(yprs, dtype=np.float64)
        except (TypeError, ValueError, RuntimeError):   # tensor leaves: per device, no memo
            return [self.rotation_rows(d) for d in devices]
        if arr.shape != (len(devices), 3):
            return [self.rotation_rows(d) for d in devices]
        uniq, inv = np.unique(arr, axis=0, return_inverse=True)
        memo = self.__dict__.setdefault("_rows_memo", {})
        rows = []
        for u in uniq:
            key = (float(u[0]), float(u[1]), float(u[2]))
            r = memo.get(key)
            if r is None:
                r = memo[key] = rotation_entries(*key)
            rows.append(r)
        return [rows[i] for i in inv.reshape(-1)]

    def eta_table(self, bvh):
        """Complex permittivity per material in the scene's material order, [n_mat, 2]."""
        return torch.tensor(self.eta_values(bvh), dtype=torch.float64, device=bvh.device)

    def tracks(self) -> bool:
        """True when a material / orientation / position value is an autograd leaf."""
        vals = [v for pair in self.material_values.values() for v in pair]
        vals += [v for t in self.orientations.values() for v in t]
        vals += [v for t in self.positions.values() for v in t]
        return any(isinstance(v, torch.Tensor) and v.requires_grad for v in vals)

    def eta_tensor(self, bvh):
        """eta_table as a differentiable tensor [n_mat, 2] (tensor leaves in
        ``material_values`` keep their autograd history)."""
        f = self.scene.frequency_hz
        rows = []
        for name in bvh.material_names:
            ov = self.material_values.get(name)
            e, sg = material_params(self.scene.materials[name], f, None if ov is None else ov[0],
                                    None if ov is None else ov[1])
            e = torch.as_tensor(e, dtype=torch.float64, device=bvh.device)
            sg = torch.as_tensor(sg, dtype=torch.float64, device=bvh.device)
            rows.append(eta_from_params(e, sg, f))
        if not rows:
            return torch.tensor([[1.0, 0.0]], dtype=torch.float64, device=bvh.device)
        return torch.stack(rows)

    def eta_values(self, bvh):
        """eta_table on the host (numpy [n_mat, 2])."""
        vals = []
        for name in bvh.material_names:
            m = self.scene.materials[name]
            ov = self.material_values.get(name)
            e, s = material_params(m, self.scene.frequency_hz,
                                   None if ov is None else float(ov[0]),
                                   None if ov is None else float(ov[1]))
            vals.append((e, s * (-eta_scale(self.scene.frequency_hz))))
        if not vals:
            vals = [(1.0, 0.0)]
        return np.asarray(vals, dtype=np.float64).reshape(-1, 2)


def path_materials(scene, bvh, path) -> tuple:
    """Material name per interaction (em.py:315-317)."""
    return tuple(scene.objects[bvh.prim_object[p]].material for p in path.seq)


def _rows_tensor(rows_list, device):
    return torch.tensor(np.asarray(rows_list, dtype=np.float64).reshape(-1, 9), dtype=torch.float64,
                        device=device).contiguous()


def _table_from_paths(paths, bvh, tx_names, rx_names):
    """Device path table from reference-style PropagationPath objects."""
    L = max([p.order for p in paths] + [1])
    P = len(paths)
    seq = np.full((P, L), -1, dtype=np.int32)
    verts = np.zeros((P, L + 2, 3))
    nrm = np.zeros((P, L, 3))
    cos = np.zeros((P, L))
    for i, p in enumerate(paths):
        k = p.order
        seq[i, :k] = p.seq
        verts[i, :k + 2] = p.vertices
        if k:
            nrm[i, :k] = p.normals
            cos[i, :k] = p.cos_incidence
    dev = bvh.device
    t = lambda a, dt=torch.float64: torch.as_tensor(a, dtype=dt, device=dev).contiguous()  # noqa: E731
    return PathTable(L, tx_names, rx_names,
                     tx=t([tx_names.index(p.tx) for p in paths], torch.int32),
                     rx=t([rx_names.index(p.rx) for p in paths], torch.int32),
                     cand=t(np.zeros(P), torch.int32), order=t([p.order for p in paths], torch.int8),
                     seq=t(seq, torch.int32), verts=t(verts),
                     length=t([p.length_m for p in paths]), delay=t([p.delay_s for p in paths]),
                     kdep=t(np.array([p.k_dep for p in paths]).reshape(P, 3)),
                     karr=t(np.array([p.k_arr for p in paths]).reshape(P, 3)),
                     normals=t(nrm), cos=t(cos))


def _launch_transfer(bvh, T: PathTable, tx_rows, rx_rows, tx_pat, rx_pat, st, sr, eta, wavelength,
                     frequency, slants_dev=None):
    P = T.n
    a = torch.empty((P, len(st), len(sr), 2), dtype=torch.float64, device=bvh.device)
    if P == 0:
        return a
    if slants_dev is not None:   # already on the device (compute_gains' single upload)
        stt, srt = slants_dev
    else:
        stt = torch.tensor(st, dtype=torch.float64, device=bvh.device)
        srt = torch.tensor(sr, dtype=torch.float64, device=bvh.device)
    with torch.cuda.device(bvh.device):
        bvh.ctx.call("rt_transfer", P, T.L, N.ptr(T.order), N.ptr(T.seq),
                     N.ptr(getattr(T, "imat", None)), N.ptr(T.verts),
                     N.ptr(T.normals), N.ptr(T.cos), N.ptr(T.length), N.ptr(T.delay),
                     N.ptr(tx_rows), N.ptr(rx_rows), tx_pat, rx_pat, N.ptr(stt), len(st),
                     N.ptr(srt), len(sr), N.ptr(eta), eta.shape[0], float(wavelength),
                     float(frequency), N.ptr(a), bvh.ctx.stream, exc_map={N.RT_EINVAL: EmError})
    return a


class PathCoefficients(torch.autograd.Function):
    """a[p, s, r] (complex) as a function of eta (real pairs [n_mat, 2]).

    forward = rt_transfer; backward = rt_transfer_bwd (hand-written adjoint
    through the Fresnel / basis-change chain, em.py:123-171)."""

    @staticmethod
    def forward(ctx, eta, bvh, T, tx_rows, rx_rows, tx_pat, rx_pat, st, sr, wavelength, frequency,
                slants_dev=None):
        eta_c = eta.detach().contiguous()
        a = _launch_transfer(bvh, T, tx_rows, rx_rows, tx_pat, rx_pat, st, sr, eta_c, wavelength,
                             frequency, slants_dev)
        ctx.save_for_backward(eta_c)
        ctx.args = (bvh, T, tx_rows, rx_rows, tx_pat, rx_pat, st, sr, wavelength, frequency)
        ctx.slants_dev = slants_dev
        return torch.view_as_complex(a)

    @staticmethod
    def backward(ctx, grad_a):
        (eta,) = ctx.saved_tensors
        bvh, T, tx_rows, rx_rows, tx_pat, rx_pat, st, sr, wavelength, frequency = ctx.args
        g = torch.view_as_real(grad_a.contiguous().to(torch.complex128)).contiguous()
        grad_eta = torch.zeros_like(eta)
        if T.n:
            if getattr(ctx, "slants_dev", None) is not None:   # already on the device
                stt, srt = ctx.slants_dev
            else:
                stt = torch.tensor(st, dtype=torch.float64, device=bvh.device)
                srt = torch.tensor(sr, dtype=torch.float64, device=bvh.device)
            with torch.cuda.device(bvh.device):
                bvh.ctx.call("rt_transfer_bwd", T.n, T.L, N.ptr(T.order), N.ptr(T.seq),
                             N.ptr(getattr(T, "imat", None)), N.ptr(T.verts), N.ptr(T.normals),
                             N.ptr(T.cos), N.ptr(T.length),
                             N.ptr(T.delay), N.ptr(tx_rows), N.ptr(rx_rows), tx_pat, rx_pat,
                             N.ptr(stt), len(st), N.ptr(srt), len(sr), N.ptr(eta), eta.shape[0],
                             float(wavelength), float(frequency), N.ptr(g), N.ptr(grad_eta),
                             bvh.ctx.stream)
        return (grad_eta,) + (None,) * 11


def path_coefficients(bvh, T: PathTable, eta, tx_rows, rx_rows, tx_pattern, rx_pattern,
                      tx_slants, rx_slants, wavelength, frequency, slants_dev=None):
    """Differentiable a[p, s, r] (complex128) for a device path table."""
    if not (torch.is_grad_enabled() and eta.requires_grad):   # no autograd node needed
        st = tuple(float(s) for s in tx_slants)
        sr = tuple(float(s) for s in rx_slants)
        a = _launch_transfer(bvh, T, tx_rows, rx_rows, pattern_id(tx_pattern), pattern_id(rx_pattern),
                             st, sr, eta.detach().contiguous(), wavelength, frequency, slants_dev)
        return torch.view_as_complex(a)
    return PathCoefficients.apply(eta, bvh, T, tx_rows, rx_rows, pattern_id(tx_pattern),
                                  pattern_id(rx_pattern), tuple(float(s) for s in tx_slants),
                                  tuple(float(s) for s in rx_slants), float(wavelength),
                                  float(frequency), slants_dev)


def rows_from_ypr(ypr):
    """rotation_entries (geometry.py:50-59) for a [P, 3] tensor -> [P, 9] (no grad)."""
    y, p, r = ypr.detach()[:, 0], ypr.detach()[:, 1], ypr.detach()[:, 2]
    cy, sy, cp, sp, cr, sr = torch.cos(y), torch.sin(y), torch.cos(p), torch.sin(p), torch.cos(r), torch.sin(r)
    return torch.stack([cy * cp, cy * sp * sr - sy * cr, cy * sp * cr + sy * sr,
                        sy * cp, sy * sp * sr + cy * cr, sy * sp * cr - cy * sr,
                        -sp, cp * sr, cp * cr], dim=1).contiguous()


class PathCoefficientsGeo(torch.autograd.Function):
    """a[p, s, r] (complex) as a function of per-path tx/rx positions and
    yaw/pitch/roll ([P, 3] each) and eta ([n_mat, 2]).

    forward = rt_transfer_jvp (geometry re-derived by mirroring through the
    path's planes, em.py:258-282, and its forward-mode Jacobian w.r.t. the 12
    device parameters); backward contracts the Jacobian with the upstream
    gradient, and runs the hand-written eta adjoint (rt_transfer_bwd)."""

    @staticmethod
    def forward(ctx, tx_pos, rx_pos, tx_ypr, rx_ypr, eta, bvh, T, tx_pat, rx_pat, st, sr,
                wavelength, frequency):
        P = T.n
        dev = bvh.device
        a = torch.empty((P, len(st), len(sr), 2), dtype=torch.float64, device=dev)
        jac = torch.empty((P, len(st), len(sr), 12, 2), dtype=torch.float64, device=dev)
        ins = [t.detach().contiguous().to(torch.float64) for t in (tx_pos, rx_pos, tx_ypr, rx_ypr)]
        eta_c = eta.detach().contiguous()
        if P:
            stt = torch.tensor(st, dtype=torch.float64, device=dev)
            srt = torch.tensor(sr, dtype=torch.float64, device=dev)
            with torch.cuda.device(dev):
                bvh.ctx.call("rt_transfer_jvp", P, T.L, N.ptr(T.order), N.ptr(T.seq), N.ptr(T.verts),
                             N.ptr(T.normals), *[N.ptr(t) for t in ins], tx_pat, rx_pat, N.ptr(stt),
                             len(st), N.ptr(srt), len(sr), N.ptr(eta_c), eta_c.shape[0],
                             float(wavelength), float(frequency), N.ptr(a), N.ptr(jac),
                             bvh.ctx.stream, exc_map={N.RT_EINVAL: EmError})
        ctx.save_for_backward(jac, eta_c, ins[2], ins[3])
        ctx.args = (bvh, T, tx_pat, rx_pat, st, sr, wavelength, frequency)
        return torch.view_as_complex(a)

    @staticmethod
    def backward(ctx, grad_a):
        jac, eta, tx_ypr, rx_ypr = ctx.saved_tensors
        bvh, T, tx_pat, rx_pat, st, sr, wavelength, frequency = ctx.args
        g = torch.view_as_real(grad_a.contiguous().to(torch.complex128))      # [P, S, R, 2]
        gp = (g[:, :, :, None, :] * jac).sum(-1).sum((1, 2))                    # [P, 12]
        grad_eta = None
        if ctx.needs_input_grad[4] and T.n:
            grad_eta = PathCoefficients.backward(
                _EtaCtx(eta, (bvh, T, rows_from_ypr(tx_ypr), rows_from_ypr(rx_ypr), tx_pat, rx_pat,
                              st, sr, wavelength, frequency)), grad_a)[0]
        return (gp[:, 0:3], gp[:, 3:6], gp[:, 6:9], gp[:, 9:12], grad_eta) + (None,) * 8


class _EtaCtx:
    """Minimal stand-in for an autograd ctx to reuse PathCoefficients.backward."""

    def __init__(self, eta, args):
        self.saved_tensors = (eta,)
        self.args = args


def path_coefficients_geo(bvh, T: PathTable, eta, tx_pos, rx_pos, tx_ypr, rx_ypr, tx_pattern,
                          rx_pattern, tx_slants, rx_slants, wavelength, frequency):
    """Differentiable a[p, s, r] w.r.t. per-path positions / orientations ([P, 3]) and eta."""
    return PathCoefficientsGeo.apply(tx_pos, rx_pos, tx_ypr, rx_ypr, eta, bvh, T,
                                     pattern_id(tx_pattern), pattern_id(rx_pattern),
                                     tuple(float(s) for s in tx_slants),
                                     tuple(float(s) for s in rx_slants), float(wavelength),
                                     float(frequency))


def eta_from_params(eps_r, sigma, frequency_hz):
    """eta = eps_r - j sigma / (2 pi f eps0) as real pairs (scene.py:99-100); differentiable."""
    return torch.stack([eps_r, sigma * (-eta_scale(frequency_hz))], dim=-1)


class _DeviceHandle:
    """The library context ``transfer`` runs on (no scene is needed: materials
    arrive per interaction through rt_transfer's interaction_mat)."""

    _by_device = {}

    def __init__(self, device):
        self.device = device
        self.ctx = N.acquire_context(device)

    @classmethod
    def get(cls):
        dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else None
        if dev is None:
            raise N.NativeError("no CUDA device: the B200 path has no CPU fallback")
        h = cls._by_device.get(dev.index)
        if h is None:
            h = cls._by_device[dev.index] = cls(dev)
        return h


def fresnel_batch(eta, cos_theta):
    """Fresnel coefficients of many (eta, cos theta_i) pairs on the device
    (rt_fresnel: the transfer kernels' own device function, em.py:123-141).
    Returns (r_te, r_tm) as complex128 numpy arrays."""
    h = _DeviceHandle.get()
    e = np.ascontiguousarray(np.asarray(eta, dtype=np.complex128).reshape(-1))
    c = np.ascontiguousarray(np.asarray(cos_theta, dtype=np.float64).reshape(-1))
    if e.shape != c.shape:
        raise EmError("eta and cos_theta need the same length")
    dev = h.device
    et = torch.view_as_real(torch.as_tensor(e, device=dev)).contiguous()
    ct = torch.as_tensor(c, device=dev)
    te = torch.empty_like(et)
    tm = torch.empty_like(et)
    with torch.cuda.device(dev):
        h.ctx.call("rt_fresnel", len(c), N.ptr(et), N.ptr(ct), N.ptr(te), N.ptr(tm), h.ctx.stream,
                   exc_map={N.RT_EINVAL: EmError})
    return (torch.view_as_complex(te).cpu().numpy(), torch.view_as_complex(tm).cpu().numpy())


def fresnel(eta, cos_theta):
    """(r_te, r_tm) for one interaction (em.py:123-141), as DiffComplex."""
    te, tm = fresnel_batch([complex(eta)], [float(cos_theta)])
    return DiffComplex(complex(te[0])), DiffComplex(complex(tm[0]))


class DiffComplex(complex):
    """Value type ``transfer`` returns: a Python complex that also carries the
    accessors callers of the reference's DiffComplex use (E/autodiff.py:286-360:
    ``to_complex``, ``abs2``, ``re``/``im``); arithmetic stays in this type."""

    @staticmethod
    def from_complex(z):
        return DiffComplex(z)

    @staticmethod
    def expj(phase):
        return DiffComplex(complex(math.cos(phase), math.sin(phase)))

    def to_complex(self) -> complex:
        return complex(self.real, self.imag)

    @property
    def re(self):
        return self.real

    @property
    def im(self):
        return self.imag

    def abs2(self) -> float:
        return self.real * self.real + self.imag * self.imag

    def conj(self):
        return DiffComplex(complex.conjugate(self))

    def __add__(self, o): return DiffComplex(complex.__add__(self, o))
    def __radd__(self, o): return DiffComplex(complex.__radd__(self, o))
    def __sub__(self, o): return DiffComplex(complex.__sub__(self, o))
    def __rsub__(self, o): return DiffComplex(complex.__rsub__(self, o))
    def __mul__(self, o): return DiffComplex(complex.__mul__(self, o))
    def __rmul__(self, o): return DiffComplex(complex.__rmul__(self, o))
    def __truediv__(self, o): return DiffComplex(complex.__truediv__(self, o))
    def __rtruediv__(self, o): return DiffComplex(complex.__rtruediv__(self, o))
    def __neg__(self): return DiffComplex(complex.__neg__(self))


@dataclass
class PathGeometry:
    """Geometry of one path ready for field transport (E/em.py:232-243)."""

    vertices: list
    seg_dirs: list
    length: float
    delay: float
    k_dep: tuple
    k_arr: tuple
    normals: list
    cos_incidence: list


def _unit(v):
    n = math.sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2])
    return (v[0] / n, v[1] / n, v[2] / n)


def _dirs(verts):
    return [_unit((b[0] - a[0], b[1] - a[1], b[2] - a[2])) for a, b in zip(verts[:-1], verts[1:])]


def geometry_from_path(path) -> PathGeometry:
    """Frozen geometry of a traced path (E/em.py:246-255)."""
    verts = [tuple(float(x) for x in v) for v in path.vertices]
    dirs = _dirs(verts)
    return PathGeometry(verts, dirs, float(path.length_m), float(path.delay_s), dirs[0], dirs[-1],
                        [tuple(float(x) for x in n) for n in path.normals],
                        [float(c) for c in path.cos_incidence])


def _chain_points(tx, rx, planes):
    """Interaction points of a reflection chain (the image construction of
    E/tracer.py:71-102): images of tx through the planes in order, then from rx
    backwards each point is where the line to the next image meets its plane.
    None when a line runs parallel to its plane (|seg . n| < 1e-15)."""
    dot = lambda a, b: a[0] * b[0] + a[1] * b[1] + a[2] * b[2]  # noqa: E731
    img = [tx]
    for n, c in planes:
        p = img[-1]
        k2 = 2.0 * (dot(p, n) - c)
        img.append((p[0] - n[0] * k2, p[1] - n[1] * k2, p[2] - n[2] * k2))
    pts = [None] * len(planes)
    cur = rx
    for k in reversed(range(len(planes))):
        n, c = planes[k]
        tgt = img[k + 1]
        seg = (tgt[0] - cur[0], tgt[1] - cur[1], tgt[2] - cur[2])
        den = dot(seg, n)
        if abs(den) < 1e-15:
            return None
        f = (c - dot(cur, n)) / den
        cur = (cur[0] + seg[0] * f, cur[1] + seg[1] * f, cur[2] + seg[2] * f)
        pts[k] = cur
    return pts


def geometry_for_positions(path, tx_pos, rx_pos) -> PathGeometry:
    """Geometry of the same topology for moved endpoints (E/em.py:258-282):
    interaction points re-mirrored through the path's planes, with the plane
    offset taken at the stored interaction vertex.  Host floats; gradients
    w.r.t. positions go through ``path_coefficients_geo`` (rt_transfer_jvp)."""
    normals = [tuple(float(x) for x in n) for n in path.normals]
    planes = []
    for k, n in enumerate(normals):
        v = path.vertices[k + 1]
        planes.append((n, n[0] * float(v[0]) + n[1] * float(v[1]) + n[2] * float(v[2])))
    tx = tuple(float(x) for x in tx_pos)
    rx = tuple(float(x) for x in rx_pos)
    points = _chain_points(tx, rx, planes)
    if points is None:
        raise EmError("path geometry degenerated while differentiating positions")
    verts = [tx] + [tuple(float(x) for x in p) for p in points] + [rx]
    dirs = _dirs(verts)
    length = 0.0
    for a, b in zip(verts[:-1], verts[1:]):
        d = (b[0] - a[0], b[1] - a[1], b[2] - a[2])
        length = length + math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    cosines = [-(dirs[k][0] * n[0] + dirs[k][1] * n[1] + dirs[k][2] * n[2]) for k, n in enumerate(normals)]
    return PathGeometry(verts, dirs, length, length / SPEED_OF_LIGHT, dirs[0], dirs[-1], normals, cosines)


def path_geometry(ctx: EvalContext, path, tx_dev, rx_dev) -> PathGeometry:
    """E/em.py:285-288: moved endpoints re-derive the geometry, else it is frozen."""
    moved = [ctx.positions.get(d.name) for d in (tx_dev, rx_dev)]
    if any(p is not None for p in moved):
        tp = moved[0] if moved[0] is not None else tx_dev.position
        rp = moved[1] if moved[1] is not None else rx_dev.position
        return geometry_for_positions(path, [float(x) for x in tp], [float(x) for x in rp])
    return geometry_from_path(path)


def transfer(ctx: EvalContext, geom, materials, tx_dev, rx_dev, tx_pattern: str, rx_pattern: str,
             tx_slant: float, rx_slant: float):
    """Complex gain of one path for one element pair — E/em.py:291-312's
    signature and meaning: ``geom`` is the PathGeometry (``geometry_from_path``
    / ``path_geometry``; a PropagationPath is accepted too) and ``materials``
    the material name of each interaction (``path_materials``).

    a = lambda/(4 pi L) * <rx field | prod_k R_k | tx field> * exp(-j 2 pi f tau),
    one rt_transfer launch.  Returns a ``DiffComplex``; when a material value in
    ``ctx.material_values`` is a tensor that requires grad, returns instead a
    0-d complex128 tensor whose backward runs the adjoint (rt_transfer_bwd).
    """
    if hasattr(geom, "length_m"):
        geom = geometry_from_path(geom)
    mats = list(materials)
    k = len(mats)
    if k != len(geom.normals):
        raise EmError("one material per interaction is required")
    h = _DeviceHandle.get()
    dev = h.device
    scene = ctx.scene
    names = list(dict.fromkeys(mats))
    # a context with autograd leaves returns tensors for every path (LOS too)
    track = any(isinstance(v, torch.Tensor) and v.requires_grad
                for pair in ctx.material_values.values() for v in pair)
    rows = []
    for name in names:
        m = scene.materials[name]
        ov = ctx.material_values.get(name)
        e, sg = material_params(m, scene.frequency_hz, None if ov is None else ov[0],
                                None if ov is None else ov[1])
        if isinstance(e, torch.Tensor) or isinstance(sg, torch.Tensor):
            e = torch.as_tensor(e, dtype=torch.float64, device=dev)
            sg = torch.as_tensor(sg, dtype=torch.float64, device=dev)
            rows.append(eta_from_params(e, sg, scene.frequency_hz))
        else:
            rows.append(torch.tensor([float(e), float(sg) * (-eta_scale(scene.frequency_hz))],
                                     dtype=torch.float64, device=dev))
    eta = torch.stack(rows) if rows else torch.tensor([[1.0, 0.0]], dtype=torch.float64, device=dev)
    L = max(k, 1)
    verts = np.zeros((1, L + 2, 3))
    verts[0, :k + 2] = np.asarray(geom.vertices, dtype=np.float64).reshape(k + 2, 3)
    nrm = np.zeros((1, L, 3))
    cos = np.zeros((1, L))
    imat = np.zeros((1, L), dtype=np.int32)
    seq = np.full((1, L), -1, dtype=np.int32)
    if k:
        nrm[0, :k] = np.asarray(geom.normals, dtype=np.float64).reshape(k, 3)
        cos[0, :k] = np.asarray(geom.cos_incidence, dtype=np.float64)
        imat[0, :k] = [names.index(m) for m in mats]
        seq[0, :k] = np.arange(k)
    t = lambda a, dt=torch.float64: torch.as_tensor(a, dtype=dt, device=dev).contiguous()  # noqa: E731
    z3 = t(np.zeros((1, 3)))
    T = PathTable(L, [getattr(tx_dev, "name", "tx")], [getattr(rx_dev, "name", "rx")],
                  tx=t([0], torch.int32), rx=t([0], torch.int32), cand=t([0], torch.int32),
                  order=t([k], torch.int8), seq=t(seq, torch.int32), verts=t(verts),
                  length=t([float(geom.length)]), delay=t([float(geom.delay)]), kdep=z3, karr=z3,
                  normals=t(nrm), cos=t(cos))
    T.imat = t(imat, torch.int32)
    as_float = lambda r: tuple(tuple(float(x) for x in row) for row in r)  # noqa: E731
    tx_rows = _rows_tensor([as_float(ctx.rotation_rows(tx_dev))], dev)
    rx_rows = _rows_tensor([as_float(ctx.rotation_rows(rx_dev))], dev)
    with torch.cuda.device(dev):
        a = path_coefficients(h, T, eta, tx_rows, rx_rows, tx_pattern, rx_pattern, [tx_slant],
                              [rx_slant], scene.wavelength, scene.frequency_hz)[0, 0, 0]
    if track:
        return a
    v = torch.view_as_real(a.detach()).cpu().numpy()
    return DiffComplex(complex(float(v[0]), float(v[1])))


# -- channel gains for full arrays -----------------------------------------------------------

@dataclass
class PathGain:
    tx: str
    rx: str
    kind: str
    seq: tuple
    delay: float
    a: np.ndarray
    delays: np.ndarray
    k_dep: np.ndarray
    k_arr: np.ndarray


class ChannelGains:
    """Columnar gains: a [P, rx_el, tx_el, T] complex128 on the device + path table."""

    def __init__(self, scene, table: PathTable, a, sample_times, delay=None, el_geom=None, ctx=None):
        self.scene = scene
        self.ctx = ctx   # the library context of the device tensors (CIR packing kernels)
        self.table = table
        self.a = a
        self.sample_times = np.asarray(sample_times, dtype=np.float64)
        # per-path delay (explicit arrays: mean over valid element pairs, em.py:456)
        self.delay = delay if delay is not None else (table.delay if table is not None else None)
        # explicit arrays: per element pair (delays, k_dep, k_arr) [P, rx_el, tx_el(, 3)]
        self.el_geom = el_geom
        self._entries = None

    @property
    def entries(self):
        if self._entries is None:
            T = self.table
            if T is None or T.n == 0:
                self._entries = []
            else:
                h = T.host()
                a = N.d2h(self.a)
                dl = self.delay.cpu().numpy()
                eg = [g.cpu().numpy() for g in self.el_geom] if self.el_geom else None
                out = []
                for i in range(T.n):
                    k = int(h["order"][i])
                    nr, nt = a.shape[1], a.shape[2]
                    out.append(PathGain(
                        tx=T.tx_names[int(h["tx"][i])], rx=T.rx_names[int(h["rx"][i])],
                        kind="specular" if k else "los",
                        seq=tuple(int(s) for s in h["seq"][i, :k]), delay=float(dl[i]),
                        a=a[i],
                        delays=eg[0][i] if eg else np.full((nr, nt), float(h["delay"][i])),
                        k_dep=eg[1][i] if eg else np.broadcast_to(h["kdep"][i], (nr, nt, 3)).copy(),
                        k_arr=eg[2][i] if eg else np.broadcast_to(h["karr"][i], (nr, nt, 3)).copy()))
                self._entries = out
        return self._entries


def _rows_array(rows):
    """[n, 3, 3] rotation rows; devices sharing one row object cost one conversion."""
    if rows and all(r is rows[0] for r in rows):
        one = np.asarray(rows[0], dtype=np.float64).reshape(1, 3, 3)
        return np.broadcast_to(one, (len(rows), 3, 3))
    return np.asarray(rows, dtype=np.float64).reshape(len(rows), 3, 3)


_APERTURE_MEMO = {}


def _aperture(off, rows):
    """Largest world-frame extent of an array's element offsets (em.py:344-356);
    memoised on (offset array, rotation values): the layouts are shared
    read-only arrays (scene.element_layout) and most devices share one row."""
    if len(off) <= 1:
        return 0.0
    key = (id(off), tuple(float(x) for x in np.asarray(rows, dtype=np.float64).reshape(-1)))
    hit = _APERTURE_MEMO.get(key)
    if hit is not None and hit[0] is off:
        return hit[1]
    w = off @ np.asarray(rows, dtype=np.float64).reshape(3, 3).T
    v = float(np.linalg.norm(w.max(axis=0) - w.min(axis=0)))
    if len(_APERTURE_MEMO) > 4096:
        _APERTURE_MEMO.clear()
    _APERTURE_MEMO[key] = (off, v)
    return v


def _device_positions(scene, T):
    """[n_tx, 3], [n_rx, 3] positions of the table's devices (the arrays
    compute_paths traced with, else looked up by name)."""
    tp, rp = getattr(T, "tx_pos", None), getattr(T, "rx_pos", None)
    if tp is None or rp is None:
        devs = {d.name: d for d in scene.devices}
        tp = np.array([devs[n].position for n in T.tx_names], dtype=np.float64).reshape(-1, 3)
        rp = np.array([devs[n].position for n in T.rx_names], dtype=np.float64).reshape(-1, 3)
    return tp, rp


def _fraunhofer_warnings(scene, T, off_tx, off_rx, tx_rows, rx_rows):
    """em.py:344-356 for every (tx, rx) pair, vectorized over the path table."""
    def aps(off, rows):   # devices sharing one row object: one aperture
        if rows and all(r is rows[0] for r in rows):
            return np.full(len(rows), _aperture(off, rows[0]))
        return np.array([_aperture(off, r) for r in rows])
    ap_t = aps(off_tx, tx_rows)
    ap_r = aps(off_rx, rx_rows)
    if not (ap_t.any() or ap_r.any()):
        return
    n_rx = len(T.rx_names)
    a_pair = np.maximum(ap_t[:, None], ap_r[None, :]).reshape(-1)
    fr_pair = 2.0 * a_pair * a_pair / scene.wavelength
    # every path is at least as long as the straight tx-rx distance: when that
    # already clears the Fraunhofer distance no path can warn (no read-back)
    tp, rp = _device_positions(scene, T)
    dist = np.linalg.norm(tp[:, None, :] - rp[None, :, :], axis=-1).reshape(-1)
    if not np.any((a_pair > 0.0) & (dist < fr_pair)):
        return
    pair = T.tx.long() * n_rx + T.rx.long()
    mins_d = torch.full((len(T.tx_names) * n_rx,), float("inf"), dtype=torch.float64,
                        device=T.length.device)
    mins_d.scatter_reduce_(0, pair, T.length, reduce="amin")
    mins = mins_d.cpu().numpy()   # shortest path per (tx, rx) pair: one small read-back
    for k in np.flatnonzero(np.isfinite(mins) & (a_pair > 0.0) & (mins < fr_pair)):
        ti, ri = divmod(int(k), n_rx)
        warnings.warn(f"path {T.tx_names[ti]}->{T.rx_names[ri]} at {mins[k]:.1f} m is inside "
                      f"the Fraunhofer distance {fr_pair[k]:.1f} m; the plane-wave synthetic-array "
                      "assumption degrades here", stacklevel=3)


_SLANT_MEMO = {}


def _slant_sets(sl):
    """(distinct slants sorted, int32 index of every element's slant) of a
    memoised element_layout slant array."""
    hit = _SLANT_MEMO.get(id(sl))
    if hit is not None and hit[0] is sl:
        return hit[1], hit[2]
    u = sorted(set(float(s) for s in sl))
    idx = np.array([u.index(float(x)) for x in sl], dtype=np.int32)
    if len(_SLANT_MEMO) > 64:
        _SLANT_MEMO.clear()
    _SLANT_MEMO[id(sl)] = (sl, u, idx)
    return u, idx


def compute_gains(scene, bvh, pathset: PathSet, ctx: EvalContext = None, eta=None) -> ChannelGains:
    """Complex gains for every path and element pair (em.py:359-422)."""
    if ctx is None:
        ctx = EvalContext(scene)
    T = pathset.table
    if T is None:
        txn = [d.name for d in scene.devices if d.kind == "tx"]
        rxn = [d.name for d in scene.devices if d.kind == "rx"]
        T = _table_from_paths(pathset.paths, bvh, txn, rxn) if pathset.paths else None
    lam = scene.wavelength
    tx_arr, rx_arr = scene.tx_array, scene.rx_array
    off_tx, sl_tx = element_layout(tx_arr, lam)
    off_rx, sl_rx = element_layout(rx_arr, lam)
    n_tx_el, n_rx_el = len(off_tx), len(off_rx)
    dev = bvh.device
    if T is None or T.n == 0:
        empty = torch.zeros((0, n_rx_el, n_tx_el, 1), dtype=torch.complex128, device=dev)
        return ChannelGains(scene, T, empty, np.zeros(1))
    if (scene.synthetic_array and eta is None and T.rx_ypr is not None and T.tx_ypr is not None
            and not ctx.orientations):
        return _gains_synthetic_native(scene, bvh, T, ctx, off_tx, sl_tx, off_rx, sl_rx)
    devs = {d.name: d for d in scene.devices}
    tx_rows_dev = ctx.rotation_rows_many([devs[n] for n in T.tx_names])
    rx_rows_dev = ctx.rotation_rows_many([devs[n] for n in T.rx_names])
    if not scene.synthetic_array:
        return _gains_explicit(scene, bvh, T, ctx, off_tx, sl_tx, off_rx, sl_rx, tx_rows_dev,
                               rx_rows_dev, devs, eta)
    st, s_idx = _slant_sets(sl_tx)
    sr, r_idx = _slant_sets(sl_rx)
    # every small host-side parameter in one pinned upload
    n_td, n_rd = len(tx_rows_dev), len(rx_rows_dev)
    # world-frame element offsets per device (em.py:372-379), on the host
    rows_t = _rows_array(tx_rows_dev)
    rows_r = _rows_array(rx_rows_dev)
    off_tx_w = np.einsum("ek,dmk->dem", np.asarray(off_tx, dtype=np.float64), rows_t)   # [n_tx, E, 3]
    off_rx_w = np.einsum("ek,dmk->dem", np.asarray(off_rx, dtype=np.float64), rows_r)
    eta_host = ctx.eta_values(bvh) if eta is None else np.zeros((0, 2))
    parts = [rows_t.reshape(-1), rows_r.reshape(-1), off_tx_w.reshape(-1), off_rx_w.reshape(-1),
             np.asarray(st, dtype=np.float64), np.asarray(sr, dtype=np.float64), eta_host.reshape(-1)]
    cuts = np.cumsum([0] + [len(x) for x in parts])
    # slant indices as int32 behind the doubles: one pinned upload, typed device views
    f64 = np.concatenate(parts)
    blob = N.h2d(np.concatenate([f64.view(np.uint8), s_idx.view(np.uint8), r_idx.view(np.uint8)]), dev)
    allp = blob[:8 * len(f64)].view(torch.float64)
    ints = blob[8 * len(f64):].view(torch.int32)
    seg = [allp[cuts[i]:cuts[i + 1]] for i in range(len(parts))]
    si, ri = ints[:len(s_idx)], ints[len(s_idx):]
    _fraunhofer_warnings(scene, T, off_tx, off_rx, tx_rows_dev, rx_rows_dev)
    if eta is None:
        eta = seg[6].reshape(-1, 2)
    if not (torch.is_grad_enabled() and eta.requires_grad):
        # rt_gains: transfer + element phasors in one call, rows picked per path
        # on the device (no per-path row gather)
        eta_c = eta.detach().contiguous()
        a = torch.empty((T.n, n_rx_el, n_tx_el), dtype=torch.complex128, device=dev)
        with torch.cuda.device(dev):
            bvh.ctx.call("rt_gains", T.n, T.L, N.ptr(T.tx), N.ptr(T.rx), N.ptr(T.order), N.ptr(T.seq),
                         N.ptr(getattr(T, "imat", None)), N.ptr(T.verts), N.ptr(T.normals), N.ptr(T.cos),
                         N.ptr(T.length), N.ptr(T.delay), N.ptr(T.kdep), N.ptr(T.karr), N.ptr(seg[0]),
                         N.ptr(seg[1]), pattern_id(tx_arr.pattern), pattern_id(rx_arr.pattern),
                         N.ptr(seg[4]), len(st), N.ptr(seg[5]), len(sr), N.ptr(eta_c), eta_c.shape[0],
                         n_tx_el, N.ptr(seg[2]), N.ptr(si), n_rx_el, N.ptr(seg[3]), N.ptr(ri), float(lam),
                         float(scene.frequency_hz), N.ptr(a), bvh.ctx.stream,
                         exc_map={N.RT_EINVAL: EmError})
        return ChannelGains(scene, T, a[..., None], np.zeros(1), ctx=bvh.ctx)
    # differentiable w.r.t. eta: per-path rows, autograd node over rt_transfer
    tx_idx = T.tx.long()
    rx_idx = T.rx.long()
    Rt, Rr = seg[0].reshape(n_td, 9), seg[1].reshape(n_rd, 9)
    offw_t, offw_r = seg[2].reshape(n_td, n_tx_el, 3), seg[3].reshape(n_rd, n_rx_el, 3)
    tx_rows = Rt[tx_idx].contiguous()
    rx_rows = Rr[rx_idx].contiguous()
    base = path_coefficients(bvh, T, eta, tx_rows, rx_rows, tx_arr.pattern, rx_arr.pattern, st, sr,
                             lam, scene.frequency_hz, slants_dev=(seg[4], seg[5]))  # [P, S, R]
    s_index, r_index = si.long(), ri.long()
    ph_tx = torch.exp(1j * TWO_PI * torch.einsum("pem,pm->pe", offw_t[tx_idx], T.kdep) / lam)
    ph_rx = torch.exp(1j * TWO_PI * torch.einsum("pem,pm->pe", offw_r[rx_idx], -T.karr) / lam)
    b = base[:, s_index][:, :, r_index].transpose(1, 2)                       # [P, rx_el, tx_el]
    a = b * ph_rx[:, :, None] * ph_tx[:, None, :]
    return ChannelGains(scene, T, a[..., None], np.zeros(1), ctx=bvh.ctx)


def _gains_synthetic_native(scene, bvh, T, ctx, off_tx, sl_tx, off_rx, sl_rx):
    """compute_gains for a synthetic array as one rt_gains_h call: the device
    orientations / positions compute_paths traced with, the memoised element
    layouts and the material table go in as host arrays; rows, world-frame
    offsets and slant sets are formed and uploaded by the library."""
    tx_arr, rx_arr = scene.tx_array, scene.rx_array
    eta_h = np.ascontiguousarray(ctx.eta_values(bvh))
    a = torch.empty((T.n, len(off_rx), len(off_tx)), dtype=torch.complex128, device=bvh.device)
    near = ctypes.c_int(0)
    with torch.cuda.device(bvh.device):
        bvh.ctx.call("rt_gains_h", T.n, T.L, N.ptr(T.tx), N.ptr(T.rx), N.ptr(T.order), N.ptr(T.seq),
                     N.ptr(getattr(T, "imat", None)), N.ptr(T.verts), N.ptr(T.normals), N.ptr(T.cos),
                     N.ptr(T.length), N.ptr(T.delay), N.ptr(T.kdep), N.ptr(T.karr),
                     len(T.tx_ypr), N.ptr(T.tx_ypr), N.ptr(T.tx_pos), len(T.rx_ypr), N.ptr(T.rx_ypr),
                     N.ptr(T.rx_pos), pattern_id(tx_arr.pattern), len(off_tx), N.ptr(off_tx), N.ptr(sl_tx),
                     pattern_id(rx_arr.pattern), len(off_rx), N.ptr(off_rx), N.ptr(sl_rx), N.ptr(eta_h),
                     len(eta_h), float(scene.wavelength), float(scene.frequency_hz), N.ptr(a),
                     ctypes.byref(near), bvh.ctx.stream, exc_map={N.RT_EINVAL: EmError})
    if near.value:   # some pair inside the Fraunhofer distance: check the paths themselves
        _fraunhofer_warnings(scene, T, off_tx, off_rx, [rotation_entries(*y) for y in T.tx_ypr],
                             [rotation_entries(*y) for y in T.rx_ypr])
    return ChannelGains(scene, T, a[..., None], np.zeros(1), ctx=bvh.ctx)


def _gains_explicit(scene, bvh, T, ctx, off_tx, sl_tx, off_rx, sl_rx, tx_rows_dev, rx_rows_dev,
                    devs, eta):
    """Explicit arrays (em.py:425-459): every (path, rx element, tx element) is
    re-solved with displaced endpoints (rt_solve_pairs; LOS rows re-check
    visibility), then transferred with that pair's slants; the path delay is
    the mean over valid pairs."""
    from .tracer import solve_pairs
    dev = bvh.device
    P, L = T.n, T.L
    nr, nt = len(off_rx), len(off_tx)
    h = T.host()
    off_tx_w = [off_tx @ np.array(r, dtype=np.float64).T for r in tx_rows_dev]
    off_rx_w = [off_rx @ np.array(r, dtype=np.float64).T for r in rx_rows_dev]
    tpos = np.array([devs[n].position for n in T.tx_names], dtype=np.float64)
    rpos = np.array([devs[n].position for n in T.rx_names], dtype=np.float64)
    ti, ri = h["tx"].astype(np.int64), h["rx"].astype(np.int64)
    # item (p, i, j): rx element i, tx element j (em.py:433-436)
    txp = tpos[ti][:, None, None, :] + np.stack(off_tx_w)[ti][:, None, :, :]
    rxp = rpos[ri][:, None, None, :] + np.stack(off_rx_w)[ri][:, :, None, :]
    txp = np.array(np.broadcast_to(txp, (P, nr, nt, 3)).reshape(-1, 3))
    rxp = np.array(np.broadcast_to(rxp, (P, nr, nt, 3)).reshape(-1, 3))
    seqs = np.repeat(h["seq"], nr * nt, axis=0)
    lens = np.repeat(h["order"], nr * nt)
    valid, Q = solve_pairs(bvh, txp, rxp, seqs, lens)
    a = torch.zeros((P * nr * nt,), dtype=torch.complex128, device=dev)
    if eta is None:
        eta = ctx.eta_table(bvh)
    tx_rows = _rows_tensor(tx_rows_dev, dev)[torch.as_tensor(np.repeat(ti, nr * nt), device=dev)]
    rx_rows = _rows_tensor(rx_rows_dev, dev)[torch.as_tensor(np.repeat(ri, nr * nt), device=dev)]
    st_item = np.tile(np.repeat(np.asarray(sl_tx, dtype=np.float64)[None, :], nr, 0).reshape(-1), P)
    sr_item = np.tile(np.repeat(np.asarray(sl_rx, dtype=np.float64)[:, None], nt, 1).reshape(-1), P)
    vh = valid.cpu().numpy()
    for st in sorted(set(st_item.tolist())):
        for sr in sorted(set(sr_item.tolist())):
            sel = np.flatnonzero(vh & (st_item == st) & (sr_item == sr))
            if not len(sel):
                continue
            idx = torch.as_tensor(sel, device=dev)
            sub = PathTable(L, [], [], **{f: getattr(Q, f)[idx] for f in PathTable.FIELDS})
            v = _launch_transfer(bvh, sub, tx_rows[idx].contiguous(), rx_rows[idx].contiguous(),
                                 pattern_id(scene.tx_array.pattern), pattern_id(scene.rx_array.pattern),
                                 [st], [sr], eta, scene.wavelength, scene.frequency_hz)
            a[idx] = torch.view_as_complex(v[:, 0, 0].contiguous())
    vm = valid.reshape(P, nr * nt)
    dl = torch.where(valid, Q.delay, torch.zeros_like(Q.delay)).reshape(P, nr * nt)
    cnt = vm.sum(1)
    mean = torch.where(cnt > 0, dl.sum(1) / cnt.clamp(min=1).to(torch.float64), T.delay)
    z3 = torch.zeros_like(Q.kdep)
    el = (torch.where(valid, Q.delay, torch.zeros_like(Q.delay)).reshape(P, nr, nt),
          torch.where(valid[:, None], Q.kdep, z3).reshape(P, nr, nt, 3),
          torch.where(valid[:, None], Q.karr, z3).reshape(P, nr, nt, 3))
    return ChannelGains(scene, T, a.reshape(P, nr, nt, 1), np.zeros(1), delay=mean, el_geom=el,
                        ctx=bvh.ctx)


def apply_doppler(gains: ChannelGains, sampling_frequency: float, num_time_steps: int,
                  tx_velocities=None, rx_velocities=None) -> ChannelGains:
    """a_i(t_n) = a_i e^{j 2 pi f_D t_n}, f_D = (f/c)(k_dep.v_tx - k_arr.v_rx) (em.py:462-494)."""
    if num_time_steps < 1 or sampling_frequency <= 0:
        raise EmError("need num_time_steps >= 1 and a positive sampling frequency")
    if gains.a.shape[-1] != 1:
        raise EmError("doppler already applied to these gains")
    T = gains.table
    t = np.arange(num_time_steps) / sampling_frequency
    if T is None or T.n == 0:
        return ChannelGains(gains.scene, T, gains.a[..., :1].repeat(1, 1, 1, num_time_steps), t,
                            ctx=gains.ctx)
    dev = gains.a.device

    def vel(side, names):
        if side is None:
            return torch.zeros((len(names), 3), dtype=torch.float64, device=dev)
        if isinstance(side, dict):
            return torch.tensor(np.array([np.asarray(side.get(n, np.zeros(3)), dtype=np.float64)
                                          for n in names]), device=dev)
        return torch.tensor(np.tile(np.asarray(side, dtype=np.float64), (len(names), 1)), device=dev)

    vt = vel(tx_velocities, T.tx_names)[T.tx.long()]
    vr = vel(rx_velocities, T.rx_names)[T.rx.long()]
    f_over_c = gains.scene.frequency_hz / SPEED_OF_LIGHT
    tt = torch.tensor(t, dtype=torch.float64, device=dev)
    if gains.el_geom is not None:   # explicit arrays: per element-pair directions
        kd, ka = gains.el_geom[1], gains.el_geom[2]                             # [P, r, t, 3]
        fd = f_over_c * ((kd * vt[:, None, None]).sum(-1) - (ka * vr[:, None, None]).sum(-1))
        ph = torch.exp(1j * TWO_PI * fd[..., None] * tt)                          # [P, r, t, T]
        a = gains.a[..., :1] * ph
    else:
        fd = f_over_c * ((T.kdep * vt).sum(-1) - (T.karr * vr).sum(-1))         # [P]
        ph = torch.exp(1j * TWO_PI * fd[:, None] * tt[None, :])                # [P, T]
        a = gains.a[..., :1] * ph[:, None, None, :]
    return ChannelGains(gains.scene, T, a, t, delay=gains.delay, el_geom=gains.el_geom, ctx=gains.ctx)


def slants_of(arr):
    return POLARIZATION_SLANTS[arr.polarization]
