"""Material calibration loss with gradients through the hand-written adjoint.

Restates the loss of /root/reference/pkg/src/emtrace/optim.py:305-372
(learn_materials' loss_fn: mean over records of ||B a - h||^2 / ||h||^2,
B the fixed delay phasors of the subcarrier grid, a the central-element path
gains, _central_gains :249-258) with PyTorch autograd: the per-path gains
come from ``em.PathCoefficients`` whose backward is rt_transfer_bwd.  The
reference's scalar Tape is replaced by one adjoint launch over all paths.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .bvh import build
from .em import _launch_transfer, eta_from_params, path_coefficients, pattern_id, rotation_entries
from .scene import POLARIZATION_SLANTS, eta_scale, material_params
from .tracer import paths_to_receivers, prepare_candidates

_EPS_KEY = "{}:eps_r"
_SIG_KEY = "{}:sigma"


def trainable_material_names(scene) -> list:
    return sorted(n for n, m in scene.materials.items() if m.trainable)


def subcarrier_frequencies(n, spacing):
    k = np.arange(n, dtype=np.float64)
    return (k - (n - 1) / 2.0) * spacing


class MaterialProblem:
    """Frozen topology (paths per record) + differentiable loss in (eps_r, sigma)."""

    def __init__(self, scene, positions, h_targets, max_depth=2, num_subcarriers=128,
                 spacing=30e3, method="exhaustive", num_rays=4096, bvh=None, check_targets=True):
        self.scene = scene
        self.bvh = bvh or build(scene)
        dev = self.bvh.device
        self.names = trainable_material_names(scene)
        tx = [d for d in scene.devices if d.kind == "tx"][0]
        prepare_candidates(self.bvh, tx.position, max_depth, method, num_rays)
        pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
        self.T = paths_to_receivers(self.bvh, tx.position, pos)
        self.R = len(pos)
        f = torch.tensor(subcarrier_frequencies(num_subcarriers, spacing), device=dev)
        self.basis = torch.exp(-2j * math.pi * f[None, :] * self.T.delay[:, None])   # [P, N]
        self.h = torch.as_tensor(np.asarray(h_targets), dtype=torch.complex128, device=dev)
        self.norm2 = (self.h.abs() ** 2).sum(-1)                                      # [R]
        if check_targets and bool((self.norm2 <= 0.0).any()):
            raise ValueError("dataset record has zero-norm target response")   # optim.py:347-348
        P = self.T.n
        self.tx_rows = torch.tensor(np.tile(np.asarray(rotation_entries(*tx.orientation)).reshape(9),
                                            (P, 1)), dtype=torch.float64, device=dev)
        self.rx_rows = torch.tensor(np.tile(np.asarray(rotation_entries(0.0, 0.0, 0.0)).reshape(9),
                                            (P, 1)), dtype=torch.float64, device=dev)
        self.tx_slant = POLARIZATION_SLANTS[scene.tx_array.polarization][0]
        self.rx_slant = POLARIZATION_SLANTS[scene.rx_array.polarization][0]

        # rows of the path table are grouped by record (rt_paths: rx order): record r
        # owns rows rec_start[r] .. rec_start[r + 1] - 1
        counts = torch.bincount(self.T.rx.long(), minlength=self.R)
        self.rec_start = torch.zeros(self.R + 1, dtype=torch.int64, device=dev)
        self.rec_start[1:] = torch.cumsum(counts, 0)
        self.freqs = f.contiguous()
        self.h_ri = torch.view_as_real(self.h.contiguous()).contiguous()
        # the eta table at the scene's own values (device, once) and the slants as
        # device tensors: a step then uploads nothing
        f_c = scene.frequency_hz
        self._eta_base = torch.tensor([[float(x) for x in eta_from_params(
            *[torch.tensor(float(v), dtype=torch.float64) for v in material_params(scene.materials[n], f_c)], f_c)]
            for n in self.bvh.material_names] or [[1.0, 0.0]], dtype=torch.float64, device=dev)
        self._eta_row = {n: i for i, n in enumerate(self.bvh.material_names)}
        self._eta_mul = torch.tensor([1.0, -eta_scale(f_c)], dtype=torch.float64, device=dev)
        self._index_cache = {}
        self._slants_dev = (torch.tensor([float(self.tx_slant)], dtype=torch.float64, device=dev),
                            torch.tensor([float(self.rx_slant)], dtype=torch.float64, device=dev))

    def eta(self, values):
        """eta table [n_mat, 2] with the entries of ``values`` (material -> (eps_r,
        sigma), tensors or floats) replacing the scene's; differentiable in the
        tensors.  Same numbers as eta_from_params per row: (eps_r, sigma * -scale)."""
        keys = tuple(n for n in self.bvh.material_names if n in values)
        if not keys:
            return self._eta_base
        dev = self.bvh.device
        pairs = [torch.stack([torch.as_tensor(values[n][0], dtype=torch.float64, device=dev),
                              torch.as_tensor(values[n][1], dtype=torch.float64, device=dev)]) for n in keys]
        upd = torch.stack(pairs) * self._eta_mul                                     # [k, 2]
        idx = self._index_cache.get(keys)
        if idx is None:
            idx = self._index_cache[keys] = torch.tensor([self._eta_row[n] for n in keys], device=dev)
        return self._eta_base.index_put((idx,), upd)

    def default_values(self):
        """The scene's own (eps_r, sigma) of every trainable material as tensors."""
        dev = self.bvh.device
        return {n: (torch.tensor(float(self.scene.materials[n].eps_r), dtype=torch.float64, device=dev),
                    torch.tensor(float(self.scene.materials[n].sigma), dtype=torch.float64, device=dev))
                for n in self.names}

    def coefficients(self, values):
        """Central-element gains a_i of every frozen path (differentiable in eta)."""
        sc = self.scene
        return path_coefficients(self.bvh, self.T, self.eta(values), self.tx_rows, self.rx_rows,
                                 sc.tx_array.pattern, sc.rx_array.pattern, [self.tx_slant],
                                 [self.rx_slant], sc.wavelength, sc.frequency_hz,
                                 slants_dev=self._slants_dev)[:, 0, 0]

    def _freq_call(self, a, H=None, loss=None, grad=None, scale=1.0):
        ar = torch.view_as_real(a.detach().contiguous()).contiguous()
        with torch.cuda.device(self.bvh.device):
            self.bvh.ctx.call("rt_freq_nmse", self.R, self.freqs.numel(), N.ptr(self.rec_start),
                              N.ptr(ar), N.ptr(self.T.delay), N.ptr(self.freqs),
                              N.ptr(self.h_ri) if loss is not None or grad is not None else None,
                              N.ptr(self.norm2) if loss is not None or grad is not None else None,
                              float(scale), N.ptr(H), N.ptr(loss), N.ptr(grad), self.bvh.ctx.stream)

    def responses(self, values):
        """H_r(f_k) = sum over record r's paths of a_i e^{-j 2 pi f_k tau_i}  [R, N]
        (rt_freq_nmse, fixed summation order; not differentiable)."""
        a = self.coefficients(values)
        H = torch.empty((self.R, self.freqs.numel(), 2), dtype=torch.float64, device=self.bvh.device)
        if self.R:
            self._freq_call(a, H=H)
        return torch.view_as_complex(H)

    def loss(self, values):
        """mean_r ||H_r - h_r||^2 / ||h_r||^2, differentiable in the tensors of
        ``values`` (material -> (eps_r, sigma)): one autograd node whose forward is
        rt_transfer + rt_freq_nmse (loss and dL/da in one launch) and whose backward
        is the hand-written adjoint rt_transfer_bwd."""
        keys = tuple(n for n in self.bvh.material_names if n in values)
        dev = self.bvh.device
        if not keys:
            return _MaterialLoss.apply(torch.zeros((0, 2), dtype=torch.float64, device=dev), self, keys)
        params = torch.stack([torch.as_tensor(x, dtype=torch.float64, device=dev)
                              for n in keys for x in values[n]]).view(-1, 2)
        return _MaterialLoss.apply(params, self, keys)


class _MaterialLoss(torch.autograd.Function):
    """loss = sum_r (1/R) ||B_r a_r - h_r||^2 / ||h_r||^2 of params [k, 2] =
    (eps_r, sigma) of the materials ``keys``.  forward: eta table (the scene's
    rows with those entries replaced, eta_from_params' arithmetic), rt_transfer,
    rt_freq_nmse (per-record losses + dL/da); the per-record losses are summed by
    torch's fixed-order reduction.  backward: rt_transfer_bwd of dL/da (dL/d eta
    per material, deterministic), then d eta / d (eps_r, sigma) = (1, -scale)."""

    @staticmethod
    def forward(ctx, params, prob, keys):
        dev = prob.bvh.device
        sc = prob.scene
        if keys:
            idx = prob._index_cache.get(keys)
            if idx is None:
                idx = prob._index_cache[keys] = torch.tensor([prob._eta_row[n] for n in keys], device=dev)
            eta = prob._eta_base.index_put((idx,), params.detach() * prob._eta_mul)
        else:
            idx, eta = None, prob._eta_base
        st, sr = (float(prob.tx_slant),), (float(prob.rx_slant),)
        a = _launch_transfer(prob.bvh, prob.T, prob.tx_rows, prob.rx_rows, pattern_id(sc.tx_array.pattern),
                             pattern_id(sc.rx_array.pattern), st, sr, eta, sc.wavelength, sc.frequency_hz,
                             prob._slants_dev)
        loss_r = torch.empty(prob.R, dtype=torch.float64, device=dev)
        grad = torch.empty((prob.T.n, 2), dtype=torch.float64, device=dev)
        if prob.R:   # rt_freq_nmse writes every record's loss and every path's dL/da
            prob._freq_call(torch.view_as_complex(a[:, 0, 0]), loss=loss_r, grad=grad, scale=1.0 / prob.R)
        ctx.prob, ctx.idx, ctx.st, ctx.sr = prob, idx, st, sr
        ctx.save_for_backward(grad, eta)
        return loss_r.sum()

    @staticmethod
    def backward(ctx, g):
        grad, eta = ctx.saved_tensors
        prob, idx = ctx.prob, ctx.idx
        if idx is None:
            return None, None, None
        sc = prob.scene
        T = prob.T
        ga = (grad * g).contiguous()            # dL/da as (re, im) pairs = [P, S=1, R=1, 2]
        grad_eta = torch.zeros_like(eta)
        if T.n:
            stt, srt = prob._slants_dev
            with torch.cuda.device(prob.bvh.device):
                prob.bvh.ctx.call("rt_transfer_bwd", T.n, T.L, N.ptr(T.order), N.ptr(T.seq),
                                  N.ptr(getattr(T, "imat", None)), N.ptr(T.verts), N.ptr(T.normals),
                                  N.ptr(T.cos), N.ptr(T.length), N.ptr(T.delay), N.ptr(prob.tx_rows),
                                  N.ptr(prob.rx_rows), pattern_id(sc.tx_array.pattern),
                                  pattern_id(sc.rx_array.pattern), N.ptr(stt), 1, N.ptr(srt), 1, N.ptr(eta),
                                  eta.shape[0], float(sc.wavelength), float(sc.frequency_hz), N.ptr(ga),
                                  N.ptr(grad_eta), prob.bvh.ctx.stream)
        return grad_eta[idx] * prob._eta_mul, None, None


def material_loss_and_grad(scene, positions, h_targets, max_depth=2, num_subcarriers=128,
                           spacing=30e3, method="exhaustive", num_rays=4096, bvh=None):
    """(loss, {'<mat>:eps_r': d/d eps_r, '<mat>:sigma': d/d sigma}) at the scene's values."""
    prob = MaterialProblem(scene, positions, h_targets, max_depth, num_subcarriers, spacing,
                           method, num_rays, bvh)
    dev = prob.bvh.device
    values = {}
    for n in prob.names:
        m = scene.materials[n]
        values[n] = (torch.tensor(float(m.eps_r), dtype=torch.float64, device=dev, requires_grad=True),
                     torch.tensor(float(m.sigma), dtype=torch.float64, device=dev, requires_grad=True))
    loss = prob.loss(values)
    loss.backward()
    grads = {}
    for n, (e, s) in values.items():
        grads[_EPS_KEY.format(n)] = float(e.grad) if e.grad is not None else 0.0
        grads[_SIG_KEY.format(n)] = float(s.grad) if s.grad is not None else 0.0
    return float(loss.detach()), grads


# ---------------------------------------------------------------------------------------------
# Drivers (optim.py:32-460): dataset generation, material learning, orientation ascent.
# The Armijo step logic, projections, topology refresh and convergence test restate
# the reference; losses and gradients come from the device (adjoint / JVP kernels).

from dataclasses import dataclass  # noqa: E402
import json  # noqa: E402
import warnings  # noqa: E402


class OptimError(ValueError):
    pass


@dataclass
class OptimConfig:
    lr: float = 0.05
    lr_sigma: float = 0.005
    lr_angle: float = 0.2
    iterations: int = 500
    line_search: bool = True
    topology_refresh: int = 10
    rel_tol: float = 1e-6
    tol_window: int = 10
    max_depth: int = 2
    method: str = "exhaustive"
    num_rays: int = 4096


@dataclass
class DatasetRecord:
    position: np.ndarray
    h: np.ndarray


@dataclass
class Dataset:
    frequency_hz: float
    num_subcarriers: int
    subcarrier_spacing_hz: float
    records: list

    def save(self, path: str):
        payload = {"frequency_hz": self.frequency_hz, "num_subcarriers": self.num_subcarriers,
                   "subcarrier_spacing_hz": self.subcarrier_spacing_hz,
                   "records": [{"position_m": [float(x) for x in r.position],
                                "h_re": [float(v) for v in r.h.real],
                                "h_im": [float(v) for v in r.h.imag]} for r in self.records]}
        with open(path, "w") as fh:
            json.dump(payload, fh)
            fh.write("\n")

    @staticmethod
    def load(path: str) -> "Dataset":
        with open(path) as fh:
            d = json.load(fh)
        recs = [DatasetRecord(np.asarray(r["position_m"], dtype=np.float64),
                              np.asarray(r["h_re"]) + 1j * np.asarray(r["h_im"])) for r in d["records"]]
        return Dataset(d["frequency_hz"], d["num_subcarriers"], d["subcarrier_spacing_hz"], recs)


class TrainLog:
    """Per-iteration loss and leaf values; CSV like the reference (optim.py:87-112)."""

    def __init__(self, leaf_names):
        self.leaf_names = list(leaf_names)
        self.rows = []
        self.final_values = {}

    def append(self, iteration, loss, values):
        self.rows.append((iteration, loss, dict(values)))

    @property
    def losses(self):
        return [r[1] for r in self.rows]

    def to_csv(self) -> str:
        lines = [",".join(["iteration", "loss"] + self.leaf_names)]
        for it, loss, vals in self.rows:
            lines.append(",".join([str(it), repr(loss)] + [repr(vals[n]) for n in self.leaf_names]))
        return "\n".join(lines) + "\n"

    def save(self, path):
        with open(path, "w") as fh:
            fh.write(self.to_csv())


def nmse_loss(h_pred, h_true):
    h_true = np.asarray(h_true, dtype=np.complex128)
    norm2 = float(np.vdot(h_true, h_true).real)
    if norm2 <= 0.0:
        raise OptimError("NMSE target has zero norm")
    err = np.asarray(h_pred, dtype=np.complex128) - h_true
    return float(np.vdot(err, err).real) / norm2


_ANGLE_LEAVES = ("yaw", "pitch", "roll")


def _leaf_kind(name):
    return name.rsplit(":", 1)[-1]


def _leaf_rate(name, config):
    """Step size of one leaf: sigma and angle leaves have their own rates."""
    kind = _leaf_kind(name)
    if kind == "sigma":
        return config.lr_sigma
    return config.lr_angle if kind in _ANGLE_LEAVES else config.lr


def _to_feasible(point):
    """Clamp material leaves into their physical range in place: eps_r >= 1,
    sigma >= 0 (the reference's projection, E/optim.py:195-200)."""
    for name, v in point.items():
        kind = _leaf_kind(name)
        if kind == "eps_r" and v < 1.0:
            point[name] = 1.0
        elif kind == "sigma" and v < 0.0:
            point[name] = 0.0
    return point


class ArmijoStep:
    """Projected gradient step with backtracking (semantics of E/optim.py:203-234).

    ``sign`` = -1 minimises, +1 maximises.  The trial scale starts at the
    carried ``scale`` and halves until the objective improves by at least
    1e-4 * scale * (d . g); a step accepted at its first trial doubles the
    carried scale (capped at 1e9).  If no trial above 1e-10 is accepted, the
    point is kept and the scale resets to 1.  Without line search a unit step
    is taken unconditionally.
    """

    ARMIJO_C = 1e-4
    MIN_SCALE = 1e-10
    MAX_SCALE = 1e9

    def __init__(self, config, sign):
        self.config = config
        self.sign = sign

    def __call__(self, point, f0, grads, objective, scale=1.0):
        names = list(point)
        g = [grads.get(n, 0.0) for n in names]
        d = [_leaf_rate(n, self.config) * gi for n, gi in zip(names, g)]
        slope = 0.0
        for di, gi in zip(d, g):   # leaf order, left to right
            slope += di * gi
        if slope == 0.0:
            return dict(point), scale

        def trial(s):
            step = self.sign * s
            return _to_feasible({n: point[n] + step * di for n, di in zip(names, d)})

        if not self.config.line_search:
            return trial(1.0), scale
        s, tries = scale, 0
        while s > self.MIN_SCALE:
            cand = trial(s)
            gain = self.sign * (float(objective(cand)) - f0)
            if gain >= self.ARMIJO_C * s * slope:
                return cand, (min(2.0 * s, self.MAX_SCALE) if tries == 0 else s)
            s *= 0.5
            tries += 1
        return dict(point), 1.0


def _plateaued(history, config):
    """True once the loss moved by less than rel_tol (relative) over the last
    tol_window iterations."""
    w = config.tol_window
    if len(history) < w + 1:
        return False
    then, now = history[-(w + 1)], history[-1]
    if then == 0.0:
        return now == 0.0
    return abs(now - then) / abs(then) < config.rel_tol


def generate_dataset(scene, positions=None, num_subcarriers=128, subcarrier_spacing_hz=30e3,
                     max_depth=2, method="exhaustive", num_rays=4096, bvh=None) -> Dataset:
    """Frequency responses at probe positions with the scene's materials (optim.py:261-288)."""
    bvh = bvh or build(scene)
    txs = [d for d in scene.devices if d.kind == "tx"]
    if not txs:
        raise OptimError("scene has no transmitter")
    if positions is None:
        positions = [d.position for d in scene.devices if d.kind == "rx"]
    if not len(positions):
        raise OptimError("no probe positions to generate data for")
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    zero = np.zeros((len(pos), num_subcarriers), dtype=np.complex128)
    prob = MaterialProblem(scene, pos, zero, max_depth, num_subcarriers, subcarrier_spacing_hz,
                           method, num_rays, bvh, check_targets=False)
    with torch.no_grad():
        h = prob.responses(prob.default_values()).cpu().numpy()
    return Dataset(scene.frequency_hz, num_subcarriers, subcarrier_spacing_hz,
                   [DatasetRecord(pos[i].copy(), h[i].copy()) for i in range(len(pos))])


def learn_materials(scene, dataset: Dataset, config: OptimConfig | None = None,
                    bvh=None) -> TrainLog:
    """Projected gradient descent on the dataset NMSE over trainable materials
    (optim.py:305-380); gradients from the hand-written adjoint."""
    config = config or OptimConfig()
    bvh = bvh or build(scene)
    names = trainable_material_names(scene)
    if not names:
        raise OptimError("scene has no trainable materials")
    if abs(dataset.frequency_hz - scene.frequency_hz) > 1e-6 * scene.frequency_hz:
        raise OptimError("dataset and scene carrier frequencies differ")
    values = {}
    for n in names:
        values[f"mat:{n}:eps_r"] = float(scene.materials[n].eps_r)
        values[f"mat:{n}:sigma"] = float(scene.materials[n].sigma)
    leaf_names = sorted(values)
    pos = np.array([r.position for r in dataset.records], dtype=np.float64)
    h = np.array([r.h for r in dataset.records])
    dev = bvh.device
    prob = None

    def as_tensors(vals, grad):
        return {n: (torch.tensor(vals[f"mat:{n}:eps_r"], dtype=torch.float64, device=dev,
                                 requires_grad=grad),
                    torch.tensor(vals[f"mat:{n}:sigma"], dtype=torch.float64, device=dev,
                                 requires_grad=grad)) for n in names}

    def loss_fn(vals):
        with torch.no_grad():
            return float(prob.loss(as_tensors(vals, False)))

    log = TrainLog(leaf_names)
    scale = 1.0
    for it in range(config.iterations):
        if it % config.topology_refresh == 0:
            prob = MaterialProblem(scene, pos, h, config.max_depth, dataset.num_subcarriers,
                                   dataset.subcarrier_spacing_hz, config.method, config.num_rays, bvh)
        tv = as_tensors(values, True)
        loss = prob.loss(tv)
        loss_val = float(loss.detach())
        if not math.isfinite(loss_val):
            raise OptimError(f"loss diverged (non-finite) at iteration {it}: values {values}")
        loss.backward()
        grads = {}
        for n, (e, s) in tv.items():
            grads[f"mat:{n}:eps_r"] = float(e.grad) if e.grad is not None else 0.0
            grads[f"mat:{n}:sigma"] = float(s.grad) if s.grad is not None else 0.0
        log.append(it, loss_val, values)
        values, scale = ArmijoStep(config, -1.0)(values, loss_val, grads, loss_fn, scale)
        if _plateaued(log.losses, config):
            break
    log.final_values = dict(values)
    return log


def optimize_orientation(scene, region, config: OptimConfig | None = None, tx_name=None, bvh=None,
                         tx_mode="central") -> TrainLog:
    """Gradient ascent of the mean region path gain over tx yaw/pitch/roll
    (optim.py:384-460), log-objective with Armijo steps; the orientation
    gradient comes from the forward-mode kernel (rt_transfer_jvp)."""
    from .channel import PROBE_NAME
    from .em import EvalContext, path_coefficients_geo
    if tx_mode != "central":
        raise OptimError("orientation optimisation supports tx_mode='central'")
    config = config or OptimConfig()
    bvh = bvh or build(scene)
    txs = [d for d in scene.devices if d.kind == "tx"]
    tx = next(d for d in txs if d.name == tx_name) if tx_name else txs[0]
    cells = np.array([region.cell_center(ix, iy) for iy in range(region.ny)
                      for ix in range(region.nx)], dtype=np.float64)
    if not len(cells):
        raise OptimError("empty region")
    keys = [f"dev:{tx.name}:{k}" for k in ("yaw", "pitch", "roll")]
    values = dict(zip(keys, (float(a) for a in tx.orientation)))
    dev = bvh.device
    slant0 = POLARIZATION_SLANTS[scene.tx_array.polarization][0]
    eta = EvalContext(scene).eta_table(bvh)
    state = {}

    def refresh():
        prepare_candidates(bvh, tx.position, config.max_depth, config.method, config.num_rays)
        T = paths_to_receivers(bvh, tx.position, cells)
        T.tx_names, T.rx_names = [tx.name], [PROBE_NAME] * len(cells)
        state["T"] = T
        P = T.n
        state["tp"] = torch.tensor(np.tile(tx.position, (P, 1)), dtype=torch.float64, device=dev)
        state["rp"] = torch.tensor(cells[T.rx.long().cpu().numpy()], dtype=torch.float64, device=dev)
        state["ro"] = torch.zeros((P, 3), dtype=torch.float64, device=dev)

    def objective(vals, grad):
        T = state["T"]
        ypr = torch.tensor([vals[k] for k in keys], dtype=torch.float64, device=dev,
                           requires_grad=grad)
        if T.n == 0:
            return torch.zeros((), dtype=torch.float64, device=dev), ypr
        to = ypr[None, :].expand(T.n, 3)
        tot = 0.0
        for pat in ("_probe_theta", "_probe_phi"):
            a = path_coefficients_geo(bvh, T, eta, state["tp"], state["rp"], to, state["ro"],
                                      scene.tx_array.pattern, pat, [slant0], [0.0],
                                      scene.wavelength, scene.frequency_hz)[:, 0, 0]
            tot = tot + (a.abs() ** 2).sum()
        return tot / len(cells), ypr

    def log_objective(vals):
        with torch.no_grad():
            v = float(objective(vals, False)[0])
        return math.log(v) if v > 0 else -math.inf

    log = TrainLog(keys)
    refresh()
    if state["T"].n == 0:
        warnings.warn("no propagation path reaches the target region; orientation left unchanged")
        log.append(0, 0.0, values)
        log.final_values = dict(values)
        return log
    scale = 1.0
    for it in range(config.iterations):
        if it and it % config.topology_refresh == 0:
            refresh()
        obj, ypr = objective(values, True)
        obj_val = float(obj.detach())
        if not math.isfinite(obj_val) or obj_val <= 0.0:
            raise OptimError(f"objective degenerated at iteration {it}")
        torch.log(obj).backward()
        grads = dict(zip(keys, (float(g) for g in ypr.grad)))
        log.append(it, obj_val, values)
        values, scale = ArmijoStep(config, +1.0)(values, math.log(obj_val), grads, log_objective, scale)
        if _plateaued(log.losses, config):
            break
    log.final_values = dict(values)
    return log
