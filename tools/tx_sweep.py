"""Launch time / node visits of the C3 city for several transmitter positions
(tree-quality A/B across libraries: python tools/ab_run.py libb200rt_X.so tools/tx_sweep.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200.tracer import run_launch  # noqa: E402


def main():
    args = bench.parse([])
    sc, tx, _ = bench.make_workload(args)
    b = P.build(sc)
    lib = b.ctx.lib
    rng = np.random.RandomState(0)
    pos = [np.asarray(tx.position, dtype=float)]
    for _ in range(5):
        p = pos[0].copy()
        p[:2] += rng.uniform(-400, 400, 2)
        p[2] = rng.uniform(5, 45)
        pos.append(p)
    tot = 0.0
    out = []
    for p in pos:
        run_launch(b, p, 5, 50_000_000)
        lib.rt_set_profiling(b.ctx.h, 1)
        run_launch(b, p, 5, 50_000_000)
        ms, ctr = bench._profile(b)
        lib.rt_set_profiling(b.ctx.h, 0)
        out.append(round(float(ms[0]), 2))
        tot += float(ms[0])
    print(os.path.basename(P._native.LIB_PATH), "launch ms per tx:", out, "sum %.2f" % tot)


if __name__ == "__main__":
    main()
