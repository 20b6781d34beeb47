"""Small C1 / C2-scale workload for compute-sanitizer (memcheck, racecheck).

usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py
Exercises the build, k_launch (trie inserts), k_solve / k_validate (coverage
and paths), k_merge, the transfer and its adjoint, and CIR packing.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import optim, scenes  # noqa: E402


def main():
    torch.cuda.set_device(0)
    # C1: ground + box, depth 1
    sc = scenes.ground_box_scene()
    b = P.build(sc)
    ps = P.compute_paths(sc, b, 1, method="fibonacci", num_rays=4096)
    P.build_cir(P.compute_gains(sc, b, ps))
    grid = P.GridSpec((-20.0, -40.0), 5.0, 16, 16, 1.5)
    P.coverage_map(sc, b, grid, 1, method="fibonacci", num_rays=4096)
    # C2 shape at reduced rays: 2,002-tri canyon, 8x8 tr38901 array, 256 rx, depth 3
    sc = scenes.street_canyon(n_per_row=100)
    b = P.build(sc)
    ps = P.compute_paths(sc, b, 3, method="fibonacci", num_rays=20_000)
    cir = P.build_cir(P.compute_gains(sc, b, ps))
    # city coverage, depth 3 (k_launch, footprints, k_solve, k_validate, k_merge)
    sc = scenes.city(n_side=6, seed=1)
    b = P.build(sc)
    tx = sc.devices[0]
    grid = P.GridSpec((float(tx.position[0]) - 60.0, float(tx.position[1]) - 60.0), 5.0, 24, 24, 1.5)
    cm = P.coverage_map(sc, b, grid, 3, method="fibonacci", num_rays=20_000)
    # adjoint (k_transfer_bwd + k_grad_eta_reduce)
    init = scenes.calib_scene(truth=False)
    pos = np.array([d.position for d in init.devices if d.kind == "rx"], dtype=np.float64)[:16]
    h = np.ones((len(pos), 16), dtype=np.complex128)
    loss, grads = optim.material_loss_and_grad(init, pos, h, 2, 16, 30e3)
    torch.cuda.synchronize()
    print("sanitize cases ok:", len(ps.paths), cir.a.shape, float((cm.gains > 0).sum()), loss, len(grads))


if __name__ == "__main__":
    main()
