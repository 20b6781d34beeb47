"""Where the C2 compute_paths + CIR latency goes: per-phase wall time with the
device synchronised after each phase, plus a cProfile of one un-synchronised
iteration (host-side Python cost).  Diagnostic only."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import scenes  # noqa: E402


def main():
    sc = scenes.street_canyon(n_per_row=100)
    for it in range(8):
        marks = []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bvh = P.build(sc)
        torch.cuda.synchronize()
        marks.append(("build", time.perf_counter()))
        ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
        torch.cuda.synchronize()
        marks.append(("paths", time.perf_counter()))
        g = P.compute_gains(sc, bvh, ps)
        torch.cuda.synchronize()
        marks.append(("gains", time.perf_counter()))
        cir = P.build_cir(g)
        torch.cuda.synchronize()
        marks.append(("cir", time.perf_counter()))
        prev = t0
        out = []
        for name, t in marks:
            out.append(f"{name} {1e3 * (t - prev):.3f}")
            prev = t
        print(f"iter {it}: total {1e3 * (prev - t0):.3f} ms | " + " | ".join(out), cir.a.shape, ps.table.n)
    pr = cProfile.Profile()
    torch.cuda.synchronize()
    pr.enable()
    for _ in range(20):
        bvh = P.build(sc)
        ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
        cir = P.build_cir(P.compute_gains(sc, bvh, ps))
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("cumulative").print_stats(45)


if __name__ == "__main__":
    main()
