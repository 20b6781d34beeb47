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

from .bvh import build
from .em import eta_from_params, path_coefficients, rotation_entries
from .scene import POLARIZATION_SLANTS, material_params
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
                 spacing=30e3, method="exhaustive", num_rays=4096, bvh=None):
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
        P = self.T.n
        self.tx_rows = torch.tensor(np.tile(np.asarray(rotation_entries(*tx.orientation)).reshape(9),
                                            (P, 1)), dtype=torch.float64, device=dev)
        self.rx_rows = torch.tensor(np.tile(np.asarray(rotation_entries(0.0, 0.0, 0.0)).reshape(9),
                                            (P, 1)), dtype=torch.float64, device=dev)
        self.tx_slant = POLARIZATION_SLANTS[scene.tx_array.polarization][0]
        self.rx_slant = POLARIZATION_SLANTS[scene.rx_array.polarization][0]

    def eta(self, values):
        """eta table [n_mat, 2] with trainable entries taken from ``values`` (tensors)."""
        rows = []
        f = self.scene.frequency_hz
        for name in self.bvh.material_names:
            if name in values:
                e, s = values[name]
            else:
                e0, s0 = material_params(self.scene.materials[name], f)
                e = torch.tensor(float(e0), dtype=torch.float64, device=self.bvh.device)
                s = torch.tensor(float(s0), dtype=torch.float64, device=self.bvh.device)
            rows.append(eta_from_params(e, s, f))
        return torch.stack(rows)

    def loss(self, values):
        sc = self.scene
        a = path_coefficients(self.bvh, self.T, self.eta(values), self.tx_rows, self.rx_rows,
                              sc.tx_array.pattern, sc.rx_array.pattern, [self.tx_slant],
                              [self.rx_slant], sc.wavelength, sc.frequency_hz)[:, 0, 0]
        pred = torch.zeros_like(self.h)
        pred.index_add_(0, self.T.rx.long(), a[:, None] * self.basis)
        err = ((pred - self.h).abs() ** 2).sum(-1) / self.norm2
        return err.mean()


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
