"""cProfile of the host side of one C2 step (cumulative, package functions only).
Diagnostic only: python tools/c2_cprofile.py"""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import scenes  # noqa: E402


def step(sc):
    bvh = P.build(sc)
    ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
    cir = P.build_cir(P.compute_gains(sc, bvh, ps))
    torch.cuda.synchronize()
    return cir


sc = scenes.street_canyon(n_per_row=100)
for _ in range(4):
    step(sc)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step(sc)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats("paper_2303_11103_b200", 30)
st.sort_stats("tottime").print_stats(15)
