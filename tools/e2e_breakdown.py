"""Where the end-to-end C3 step spends its time (host gather, upload+build,
coverage map, D2H).  Diagnostic only: python tools/e2e_breakdown.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import parallel  # noqa: E402
from paper_2303_11103_b200.bvh import gather_meshes  # noqa: E402


def main():
    args = bench.parse(sys.argv[1:])
    sc, _, grid = bench.make_workload(args)
    rows = []
    for i in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gather_meshes(sc)
        t1 = time.perf_counter()
        bvh = P.build(sc)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        b2 = P.build(sc)   # second build on a warm pooled context
        torch.cuda.synchronize()
        t2b = time.perf_counter()
        del b2
        g, b = parallel.coverage_map(sc, bvh, grid, args.depth, int(args.rays))
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        rows.append((t1 - t0, t2 - t1, t3 - t2b, t2b - t2))
        del bvh
    for r in rows[2:]:
        print("gather %.2f ms  build(incl. gather) %.2f ms  coverage %.2f ms  2nd build %.2f ms"
              % tuple(1e3 * x for x in r))


if __name__ == "__main__":
    main()
