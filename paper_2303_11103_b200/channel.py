"""CIR packing, OFDM frequency response and coverage maps.

Drop-in for /root/reference/pkg/src/emtrace/channel.py.  ``coverage_map``
(:236-253) computes the candidate set once per transmitter (the reference
relaunches per cell, with identical results) and then runs rt_coverage: the
candidate-major image solve over footprint cells, occlusion, probe-power
transfer and per-cell coincident merge, all on the device.  ``build_cir``
(:40-72) and ``frequency_response`` (:107-123) pack / contract device tensors.
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .em import EvalContext, compute_gains, pattern_id, rotation_entries
from .scene import RadioDevice, element_layout
from .tracer import (DEFAULT_NUM_RAYS, PathTable, TracerError, paths_to_receivers,
                     prepare_candidates, run_enumerate, run_launch, set_candidates)

PROBE_NAME = "__probe__"
COVERAGE_MAGIC = "emtrace-coverage-v1"


class ChannelError(ValueError):
    pass


@dataclass
class Cir:
    """a [rx, rx_ant, tx, tx_ant, path, time] complex128; tau [rx, tx, path] (channel.py:24-37)."""

    a: np.ndarray
    tau: np.ndarray
    rx_names: list
    tx_names: list
    sample_times: np.ndarray
    a_dev: torch.Tensor = None
    tau_dev: torch.Tensor = None


def build_cir(gains, los: bool = True, reflection: bool = True,
              normalize_delays: bool = False, to_host: bool = True) -> Cir:
    """Dense CIR tensors sorted per (rx, tx) by (delay, kind, seq) (channel.py:40-72)."""
    scene = gains.scene
    rx_names = [d.name for d in scene.devices if d.kind == "rx"]
    tx_names = [d.name for d in scene.devices if d.kind == "tx"]
    a_all = gains.a
    T = gains.table
    n_rx_el, n_tx_el = scene.rx_array.num_elements, scene.tx_array.num_elements
    n_t = a_all.shape[-1] if a_all.numel() else 1
    dev = a_all.device
    if T is None or T.n == 0:
        a = torch.zeros((len(rx_names), n_rx_el, len(tx_names), n_tx_el, 0, n_t),
                        dtype=torch.complex128, device=dev)
        tau = torch.zeros((len(rx_names), len(tx_names), 0), dtype=torch.float64, device=dev)
    elif getattr(gains, "ctx", None) is not None and a_all.is_cuda and not a_all.requires_grad:
        delay_all = gains.delay if gains.delay is not None else T.delay
        return _build_cir_device(gains, T, a_all, delay_all, rx_names, tx_names, n_rx_el, n_tx_el, n_t,
                                 los, reflection, normalize_delays, to_host)
    else:
        kind = (T.order > 0).to(torch.int64)
        keep = ((kind == 0) & los) | ((kind == 1) & reflection)
        idx = torch.nonzero(keep).flatten()
        # table name order -> scene order (identity in the common case: no upload)
        if list(T.rx_names) == rx_names:
            rxm = T.rx.long()[idx]
        else:
            rxm = N.h2d(np.array([rx_names.index(n) for n in T.rx_names]), dev)[T.rx.long()[idx]]
        if list(T.tx_names) == tx_names:
            txm = T.tx.long()[idx]
        else:
            txm = N.h2d(np.array([tx_names.index(n) for n in T.tx_names]), dev)[T.tx.long()[idx]]
        pair = rxm * len(tx_names) + txm
        delay = (gains.delay if gains.delay is not None else T.delay)[idx]
        # (pair, delay, kind, seq) lexicographic via stable sorts, least significant first
        order = torch.arange(idx.numel(), device=dev)
        n_prims = sum(len(o.triangles) for o in scene.objects)
        seqrank = _seq_rank(T.seq[idx], T.order[idx], n_prims)
        # (kind, seq) share one key: kind (0 LOS, 1 specular) above the sequence rank,
        # which is < 2^62 packed or < 2^31 as a rank
        ks = kind[idx] * (1 << 62) + seqrank if int(T.L) * int(n_prims + 1).bit_length() <= 62 \
            else None
        keys = (ks, delay, pair) if ks is not None else (seqrank, kind[idx], delay, pair)
        for key in keys:
            k = key[order]
            _, o2 = torch.sort(k, stable=True)
            order = order[o2]
        pair_s = pair[order]
        counts = torch.bincount(pair_s, minlength=len(rx_names) * len(tx_names))
        n_path = int(counts.max().item()) if counts.numel() else 0
        starts = torch.cumsum(counts, 0) - counts
        slot = torch.arange(order.numel(), device=dev) - starts[pair_s]
        a = torch.zeros((len(rx_names), n_rx_el, len(tx_names), n_tx_el, n_path, n_t),
                        dtype=torch.complex128, device=dev)
        tau = torch.zeros((len(rx_names), len(tx_names), n_path), dtype=torch.float64, device=dev)
        src = idx[order]
        r_s, t_s = rxm[order], txm[order]
        d_s = delay[order]
        if normalize_delays:
            first = torch.zeros(len(rx_names) * len(tx_names), dtype=torch.float64, device=dev)
            head = slot == 0
            first[pair_s[head]] = d_s[head]
            d_s = d_s - first[pair_s]
        tau[r_s, t_s, slot] = d_s
        a.permute(0, 2, 4, 1, 3, 5)[r_s, t_s, slot] = a_all[src]
    cir = Cir(a=None, tau=None, rx_names=rx_names, tx_names=tx_names,
              sample_times=gains.sample_times, a_dev=a, tau_dev=tau)
    if to_host:
        cir.a = N.d2h(a)
        cir.tau = N.d2h(tau)
    return cir


def _build_cir_device(gains, T, a_all, delay, rx_names, tx_names, n_rx_el, n_tx_el, n_t, los, reflection,
                      normalize_delays, to_host):
    """build_cir through rt_cir_plan / rt_cir_scatter: bucket by (rx, tx) pair,
    order by (delay, kind, sequence), scatter — one host sync for the path count."""
    dev = a_all.device
    ctx = gains.ctx
    if list(T.rx_names) == rx_names:
        rx_of = T.rx
    else:
        rx_of = N.h2d(np.array([rx_names.index(n) for n in T.rx_names], dtype=np.int32), dev)[T.rx.long()]
    if list(T.tx_names) == tx_names:
        tx_of = T.tx
    else:
        tx_of = N.h2d(np.array([tx_names.index(n) for n in T.tx_names], dtype=np.int32), dev)[T.tx.long()]
    rx_of, tx_of = rx_of.to(torch.int32).contiguous(), tx_of.to(torch.int32).contiguous()
    delay = delay.to(torch.float64).contiguous()
    a_in = a_all.contiguous()
    # the largest (rx, tx) bucket is known when every path is kept and the table
    # is compute_paths' own (rt_paths counted them): no host round trip
    known = T.max_per_rx if (los and reflection and T.max_per_rx is not None) else -1
    n = ctypes.c_int64(known)
    with torch.cuda.device(dev):
        ctx.call("rt_cir_plan", T.n, int(T.L), N.ptr(T.order), N.ptr(T.seq), N.ptr(delay), N.ptr(rx_of),
                 N.ptr(tx_of), len(rx_names), len(tx_names), int(bool(los)), int(bool(reflection)),
                 ctypes.byref(n), ctx.stream, exc_map={N.RT_EINVAL: ChannelError})
        n_path = int(n.value)
        # zero-filled by rt_cir_scatter
        a = torch.empty((len(rx_names), n_rx_el, len(tx_names), n_tx_el, n_path, n_t),
                        dtype=torch.complex128, device=dev)
        tau = torch.empty((len(rx_names), len(tx_names), n_path), dtype=torch.float64, device=dev)
        ctx.call("rt_cir_scatter", T.n, N.ptr(delay), int(bool(normalize_delays)), N.ptr(a_in), n_rx_el,
                 n_tx_el, n_t, n_path, N.ptr(a), N.ptr(tau), ctx.stream, exc_map={N.RT_EINVAL: ChannelError})
    cir = Cir(a=None, tau=None, rx_names=rx_names, tx_names=tx_names, sample_times=gains.sample_times,
              a_dev=a, tau_dev=tau)
    if to_host:
        cir.a, cir.tau = N.d2h_many([a, tau])
    return cir


def _seq_rank(seq, order, n_prims=None):
    """Tuple order of the interaction sequences as an integer key."""
    if seq.numel() == 0:
        return torch.zeros(0, dtype=torch.int64, device=seq.device)
    s = seq.to(torch.int64) + 1
    L = s.shape[1]
    if n_prims is not None and L * int(n_prims + 1).bit_length() <= 63:
        # columns (prim + 1, 0 = padding) packed most significant first: the
        # integer order is the tuple order (a prefix sorts first)
        b = int(n_prims + 1).bit_length()
        key = s[:, 0]
        for j in range(1, L):
            key = (key << b) | s[:, j]
        return key
    key = torch.zeros(s.shape[0], dtype=torch.int64, device=seq.device)
    # lexicographic rank via successive stable sorts on the columns
    ordr = torch.arange(s.shape[0], device=seq.device)
    for j in range(L - 1, -1, -1):
        _, o2 = torch.sort(s[ordr, j], stable=True)
        ordr = ordr[o2]
    key[ordr] = torch.arange(s.shape[0], device=seq.device)
    return key


def save_cir(cir: Cir, path: str):
    header = {"format": "emtrace-cir-v1", "a_shape": list(cir.a.shape),
              "tau_shape": list(cir.tau.shape), "rx": cir.rx_names, "tx": cir.tx_names,
              "sample_times_s": [float(t) for t in cir.sample_times]}
    with open(path, "wb") as fh:
        fh.write(json.dumps(header, sort_keys=True).encode() + b"\n")
        fh.write(cir.a.astype("<c16").tobytes())
        fh.write(cir.tau.astype("<f8").tobytes())


def load_cir(path: str) -> Cir:
    with open(path, "rb") as fh:
        header = json.loads(fh.readline().decode())
        if header.get("format") != "emtrace-cir-v1":
            raise ChannelError(f"{path}: not a CIR file")
        a_shape = tuple(header["a_shape"])
        n_a = int(np.prod(a_shape)) if a_shape else 0
        a = np.frombuffer(fh.read(16 * n_a), dtype="<c16").reshape(a_shape).copy()
        tau = np.frombuffer(fh.read(), dtype="<f8").reshape(tuple(header["tau_shape"])).copy()
    return Cir(a=a, tau=tau, rx_names=header["rx"], tx_names=header["tx"],
               sample_times=np.asarray(header["sample_times_s"]))


@dataclass
class FreqResponse:
    h: np.ndarray
    frequencies: np.ndarray


def subcarrier_frequencies(num_subcarriers: int, spacing: float) -> np.ndarray:
    if num_subcarriers < 1:
        raise ChannelError("need at least one subcarrier")
    k = np.arange(num_subcarriers, dtype=np.float64)
    return (k - (num_subcarriers - 1) / 2.0) * spacing


def frequency_response(cir: Cir, num_subcarriers: int, spacing: float) -> FreqResponse:
    """H(f_k) = sum_i a_i e^{-j 2 pi f_k tau_i} (channel.py:107-123) on the device:
    every (rx, rx element, tx, tx element, time) row of the CIR is one record of
    rt_freq_nmse (paths summed in slot order; a host CIR is uploaded first)."""
    from .em import _DeviceHandle
    f = subcarrier_frequencies(num_subcarriers, spacing)
    h = _DeviceHandle.get()
    dev = cir.a_dev.device if cir.a_dev is not None else h.device
    ctx = h.ctx if dev == h.device else N.acquire_context(dev)
    a = cir.a_dev if cir.a_dev is not None else torch.as_tensor(np.asarray(cir.a), device=dev)
    tau = cir.tau_dev if cir.tau_dev is not None else torch.as_tensor(np.asarray(cir.tau), device=dev)
    nr, nre, nt, nte, P, T = a.shape
    R = nr * nre * nt * nte * T
    a_rec = a.to(torch.complex128).permute(0, 1, 2, 3, 5, 4).reshape(R, P)
    tau_rec = tau.to(torch.float64)[:, None, :, None, None, :].expand(nr, nre, nt, nte, T, P).reshape(R, P)
    ar = torch.view_as_real(a_rec.contiguous()).contiguous()
    tr = tau_rec.contiguous()
    start = torch.arange(R + 1, dtype=torch.int64, device=dev) * P
    ft = torch.as_tensor(f, dtype=torch.float64, device=dev)
    H = torch.zeros((R, num_subcarriers, 2), dtype=torch.float64, device=dev)
    if R and P:
        with torch.cuda.device(dev):
            ctx.call("rt_freq_nmse", R, num_subcarriers, N.ptr(start), N.ptr(ar), N.ptr(tr), N.ptr(ft),
                     None, None, 1.0, N.ptr(H), None, None, ctx.stream,
                     exc_map={N.RT_EINVAL: ChannelError})
    Hc = torch.view_as_complex(H).reshape(nr, nre, nt, nte, T, num_subcarriers)
    Hc = Hc.permute(0, 1, 2, 3, 5, 4).reshape(nr * nre, nt * nte, num_subcarriers, T)
    return FreqResponse(h=N.d2h(Hc.contiguous()), frequencies=f)


# -- coverage ---------------------------------------------------------------------------------

@dataclass(frozen=True)
class GridSpec:
    """nx x ny cells of cell_size meters; origin = lower-left corner (channel.py:128-149)."""

    origin: tuple
    cell_size: float
    nx: int
    ny: int
    height: float = 1.5

    def cell_center(self, ix: int, iy: int) -> np.ndarray:
        return np.array([self.origin[0] + (ix + 0.5) * self.cell_size,
                         self.origin[1] + (iy + 0.5) * self.cell_size, self.height])

    @property
    def num_cells(self) -> int:
        return self.nx * self.ny


@dataclass
class CoverageMap:
    grid: GridSpec
    gains: np.ndarray
    frequency_hz: float
    stats: dict = None
    gains_dev: torch.Tensor = None

    def to_db(self, floor_db: float = -150.0) -> np.ndarray:
        out = np.full(self.gains.shape, floor_db)
        mask = self.gains > 0
        out[mask] = np.maximum(10.0 * np.log10(self.gains[mask]), floor_db)
        return out

    def save_binary(self, path: str):
        header = {"format": COVERAGE_MAGIC, "nx": self.grid.nx, "ny": self.grid.ny,
                  "origin_m": list(self.grid.origin), "cell_m": self.grid.cell_size,
                  "height_m": self.grid.height, "frequency_hz": self.frequency_hz}
        with open(path, "wb") as fh:
            fh.write(json.dumps(header, sort_keys=True).encode() + b"\n")
            fh.write(self.gains.astype("<f8").tobytes())

    @staticmethod
    def load_binary(path: str) -> "CoverageMap":
        with open(path, "rb") as fh:
            header = json.loads(fh.readline().decode())
            if header.get("format") != COVERAGE_MAGIC:
                raise ChannelError(f"{path}: not a coverage map file")
            raw = fh.read()
        grid = GridSpec(origin=tuple(header["origin_m"]), cell_size=header["cell_m"],
                        nx=header["nx"], ny=header["ny"], height=header["height_m"])
        gains = np.frombuffer(raw, dtype="<f8").reshape(grid.ny, grid.nx).copy()
        return CoverageMap(grid=grid, gains=gains, frequency_hz=header["frequency_hz"])


def probe_receiver(point) -> RadioDevice:
    return RadioDevice(kind="rx", name=PROBE_NAME, position=np.asarray(point, dtype=np.float64))


def _tx_antenna(scene, tx_dev, ctx):
    rows = ctx.rotation_rows(tx_dev)
    lam = scene.wavelength
    off, sl = element_layout(scene.tx_array, lam)
    # mat_vec(rows, off) in Python-float order (channel.py:558)
    off_w = np.array([[rows[r][0] * float(o[0]) + rows[r][1] * float(o[1]) + rows[r][2] * float(o[2])
                       for r in range(3)] for o in off], dtype=np.float64)
    return rows, np.asarray(sl, dtype=np.float64), off_w


_COV_ERRORS = {N.RT_EINVAL: ChannelError, N.RT_ECOINCIDE: TracerError, N.RT_ECAP: ChannelError}


def _coverage_params(scene, bvh, tx_dev, tx_mode, ctx):
    """Host-side antenna / material parameters of rt_coverage (eta staged to the device)."""
    if ctx is None:
        ctx = EvalContext(scene)
    mode = {"central": 0, "array": 1}.get(tx_mode)
    if mode is None:
        raise ChannelError(f"unknown tx_mode {tx_mode!r}")
    rows, slants, off_w = _tx_antenna(scene, tx_dev, ctx)
    rows_h, _ = N.host_doubles(rows)
    probe_h, _ = N.host_doubles(rotation_entries(0.0, 0.0, 0.0))
    sl_h, _ = N.host_doubles(slants)
    off_h, _ = N.host_doubles(off_w)
    tx_h, _ = N.host_doubles([float(x) for x in tx_dev.position])
    eta = N.h2d(ctx.eta_values(bvh), bvh.device)   # staged: no blocking pageable copy
    return tx_h, rows_h, probe_h, sl_h, off_h, len(slants), mode, eta


_COV_KEYS = ("work_items", "geometric_pairs", "valid_paths", "cells", "candidates")


def coverage_from_candidates(scene, bvh, tx_dev, grid: GridSpec, tx_mode="central", ctx=None,
                             shard_index=0, shard_count=1, out=None):
    """rt_coverage over the context's current candidate set; returns (gains_dev, stats)."""
    tx_h, rows_h, probe_h, sl_h, off_h, n_el, mode, eta = _coverage_params(scene, bvh, tx_dev, tx_mode, ctx)
    dev = bvh.device
    g = out if out is not None else torch.empty((grid.ny, grid.nx), dtype=torch.float64, device=dev)
    stats = np.zeros(8, dtype=np.int64)
    with torch.cuda.device(dev):
        bvh.ctx.call("rt_coverage", N.ptr(tx_h), float(grid.origin[0]), float(grid.origin[1]),
                     float(grid.cell_size), int(grid.nx), int(grid.ny), float(grid.height),
                     N.ptr(rows_h), N.ptr(probe_h), pattern_id(scene.tx_array.pattern), N.ptr(sl_h),
                     N.ptr(off_h), n_el, mode, N.ptr(eta), eta.shape[0], scene.wavelength,
                     scene.frequency_hz, int(shard_index), int(shard_count), N.ptr(g),
                     N.ptr(stats), bvh.ctx.stream, exc_map=_COV_ERRORS)
    # geometric_pairs: (cell, candidate) pairs that passed the image solve and were not
    # stopped by the receiver-side occluder hint (the fused pass exits there early)
    return g, {k: int(stats[i]) for i, k in enumerate(_COV_KEYS)}


def coverage_fibonacci(scene, bvh, tx_dev, grid: GridSpec, max_depth: int, num_rays: int,
                       tx_mode="central", ctx=None, out=None):
    """launch_candidates (fibonacci) + rt_coverage as one library call
    (rt_coverage_fibonacci: no host round trip between the launch and the map).
    Returns (gains_dev, stats, ray_bounces)."""
    if num_rays < 1 or max_depth < 1:
        raise TracerError("need num_rays >= 1 and max_depth >= 1")
    tx_h, rows_h, probe_h, sl_h, off_h, n_el, mode, eta = _coverage_params(scene, bvh, tx_dev, tx_mode, ctx)
    dev = bvh.device
    g = out if out is not None else torch.empty((grid.ny, grid.nx), dtype=torch.float64, device=dev)
    stats = np.zeros(8, dtype=np.int64)
    nb = ctypes.c_int64()
    with torch.cuda.device(dev):
        bvh.ctx.call("rt_coverage_fibonacci", N.ptr(tx_h), int(num_rays), int(max_depth),
                     float(grid.origin[0]), float(grid.origin[1]), float(grid.cell_size), int(grid.nx),
                     int(grid.ny), float(grid.height), N.ptr(rows_h), N.ptr(probe_h),
                     pattern_id(scene.tx_array.pattern), N.ptr(sl_h), N.ptr(off_h), n_el, mode, N.ptr(eta),
                     eta.shape[0], scene.wavelength, scene.frequency_hz, N.ptr(g), N.ptr(stats),
                     ctypes.byref(nb), bvh.ctx.stream, exc_map=_COV_ERRORS)
    return g, {k: int(stats[i]) for i, k in enumerate(_COV_KEYS)}, int(nb.value)


def coverage_map(scene, bvh, grid: GridSpec, max_depth: int, method: str = "exhaustive",
                 num_rays: int = DEFAULT_NUM_RAYS, tx_name: str | None = None,
                 tx_mode: str = "central", cell_cap: int = 250_000) -> CoverageMap:
    """Deterministic per-cell coverage (channel.py:236-253) on the device."""
    if grid.num_cells > cell_cap:
        raise ChannelError(f"grid has {grid.num_cells} cells, above the cap of {cell_cap}")
    txs = [d for d in scene.devices if d.kind == "tx"]
    if not txs:
        raise ChannelError("scene has no transmitter")
    tx_dev = _device(scene, tx_name) if tx_name else txs[0]
    bounces = 0
    if method == "fibonacci" and max_depth >= 1 and bvh.num_prims:   # one library call
        g, stats, bounces = coverage_fibonacci(scene, bvh, tx_dev, grid, max_depth, num_rays, tx_mode)
        stats["ray_bounces"] = int(bounces)
        return CoverageMap(grid=grid, gains=N.d2h(g), frequency_hz=scene.frequency_hz,
                           stats=stats, gains_dev=g)
    if max_depth >= 1 and bvh.num_prims:
        if method == "exhaustive":
            run_enumerate(bvh, max_depth)
        elif method == "fibonacci":
            _, bounces = run_launch(bvh, tx_dev.position, max_depth, num_rays)
        else:
            raise TracerError(f"unknown path-finding method {method!r}")
    else:
        set_candidates(bvh, np.zeros((0, 1), dtype=np.int32), np.zeros(0, dtype=np.int8), 1)
    g, stats = coverage_from_candidates(scene, bvh, tx_dev, grid, tx_mode)
    stats["ray_bounces"] = int(bounces)
    return CoverageMap(grid=grid, gains=N.d2h(g), frequency_hz=scene.frequency_hz,
                       stats=stats, gains_dev=g)


def _device(scene, name):
    for d in scene.devices:
        if d.name == name:
            return d
    raise ChannelError(f"no device named {name!r}")


def _tracked_gain(scene, bvh, T, tx_dev, probe, ctx, tx_mode):
    """point_path_gain under a context holding autograd leaves (the reference's
    Tape context, E/channel.py:214-232 with E/em.py:285-288): returns a 0-d
    tensor whose backward reaches material (eps_r, sigma), tx orientation and
    tx / probe position leaves through rt_transfer_jvp and rt_transfer_bwd."""
    from .em import path_coefficients_geo, slants_of
    if tx_mode != "central":
        raise ChannelError("gradients are available for tx_mode='central' only")
    dev = bvh.device
    P = T.n

    def vec3(v):
        return torch.stack([torch.as_tensor(x, dtype=torch.float64, device=dev) for x in v])

    ypr = vec3(ctx.orientations.get(tx_dev.name, tx_dev.orientation))
    tp = vec3(ctx.positions.get(tx_dev.name, tx_dev.position))
    rp = vec3(ctx.positions.get(probe.name, probe.position))
    eta = ctx.eta_tensor(bvh)
    slant = float(slants_of(scene.tx_array)[0])
    zero = torch.zeros((P, 3), dtype=torch.float64, device=dev)
    total = torch.zeros((), dtype=torch.float64, device=dev)
    for pat in ("_probe_theta", "_probe_phi"):
        a = path_coefficients_geo(bvh, T, eta, tp[None, :].expand(P, 3), rp[None, :].expand(P, 3),
                                  ypr[None, :].expand(P, 3), zero, scene.tx_array.pattern, pat,
                                  [slant], [0.0], scene.wavelength, scene.frequency_hz)[:, 0, 0]
        total = total + (a.real ** 2 + a.imag ** 2).sum()
    return total


def point_path_gain(scene, bvh, tx_dev, point, max_depth: int, method: str = "exhaustive",
                    num_rays: int = 4096, ctx: EvalContext | None = None, frozen_paths=None,
                    tx_mode: str = "central"):
    """Sum_i |a_i|^2 over both probe polarizations at one point (channel.py:190-233).

    Returns (gain, paths) like the reference; ``frozen_paths`` reuses a topology.
    Under a context with autograd leaves the gain is a differentiable 0-d tensor.
    """
    from .em import _launch_transfer, _rows_tensor, _table_from_paths
    from .tracer import table_to_paths
    if ctx is None:
        ctx = EvalContext(scene)
    probe = probe_receiver(point)
    if frozen_paths is None:
        prepare_candidates(bvh, tx_dev.position, max_depth, method, num_rays)
        T = paths_to_receivers(bvh, tx_dev.position, [probe.position])
        T.tx_names, T.rx_names = [tx_dev.name], [PROBE_NAME]
        paths = table_to_paths(T)
    else:
        paths = list(frozen_paths)
        T = _table_from_paths(paths, bvh, [tx_dev.name], [PROBE_NAME]) if paths else None
    if T is None or T.n == 0:
        return 0.0, paths
    if ctx.tracks():
        return _tracked_gain(scene, bvh, T, tx_dev, probe, ctx, tx_mode), paths
    rows, slants, off_w = _tx_antenna(scene, tx_dev, ctx)
    P = T.n
    dev = bvh.device
    txr = _rows_tensor([rows] * P, dev)
    prr = _rows_tensor([rotation_entries(0.0, 0.0, 0.0)] * P, dev)
    eta = ctx.eta_table(bvh)
    tx_pat = pattern_id(scene.tx_array.pattern)
    gain = 0.0
    if tx_mode == "central":
        at = _launch_transfer(bvh, T, txr, prr, tx_pat, 3, [float(slants[0])], [0.0], eta,
                              scene.wavelength, scene.frequency_hz).cpu().numpy()
        ap = _launch_transfer(bvh, T, txr, prr, tx_pat, 4, [float(slants[0])], [0.0], eta,
                              scene.wavelength, scene.frequency_hz).cpu().numpy()
        for i in range(P):
            gain = gain + (at[i, 0, 0, 0] ** 2 + at[i, 0, 0, 1] ** 2)
            gain = gain + (ap[i, 0, 0, 0] ** 2 + ap[i, 0, 0, 1] ** 2)
    elif tx_mode == "array":
        kdep = T.kdep.cpu().numpy()
        sl_u = sorted(set(float(s) for s in slants))
        at = _launch_transfer(bvh, T, txr, prr, tx_pat, 3, sl_u, [0.0], eta, scene.wavelength,
                              scene.frequency_hz).cpu().numpy()
        ap = _launch_transfer(bvh, T, txr, prr, tx_pat, 4, sl_u, [0.0], eta, scene.wavelength,
                              scene.frequency_hz).cpu().numpy()
        lam = scene.wavelength
        gain = 0.0
        for i in range(P):
            for arr in (at, ap):
                z = 0j
                for e in range(len(slants)):
                    b = arr[i, sl_u.index(float(slants[e])), 0]
                    d = kdep[i]
                    ph = 2.0 * math.pi * (d[0] * off_w[e, 0] + d[1] * off_w[e, 1] + d[2] * off_w[e, 2]) / lam
                    z = z + complex(b[0], b[1]) * complex(math.cos(ph), math.sin(ph))
                gain = gain + (z.real * z.real + z.imag * z.imag)
    else:
        raise ChannelError(f"unknown tx_mode {tx_mode!r}")
    return float(gain), paths
