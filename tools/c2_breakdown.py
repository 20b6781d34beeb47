"""C2 (compute_paths + CIR) latency breakdown; diagnostic: python tools/c2_breakdown.py"""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import scenes  # noqa: E402


def step(sc, marks):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    bvh = P.build(sc)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    gains = P.compute_gains(sc, bvh, ps)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    cir = P.build_cir(gains)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    if marks is not None:
        marks.append([1e3 * (b - a) for a, b in zip(t, t[1:])])
    return cir


def main():
    sc = scenes.street_canyon(n_per_row=100)
    for _ in range(3):
        step(sc, None)
    marks = []
    for _ in range(5):
        step(sc, marks)
    for m in marks:
        print("build %.2f  paths %.2f  gains %.2f  cir %.2f ms" % tuple(m))
    pr = cProfile.Profile()
    pr.enable()
    step(sc, None)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
