import sys, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
import bench, paper_2303_11103_b200 as P
from paper_2303_11103_b200.channel import coverage_from_candidates
from paper_2303_11103_b200.tracer import run_launch
args = bench.parse([]); sc, tx, grid = bench.make_workload(args)
b = P.build(sc)
run_launch(b, tx.position, args.depth, int(args.rays))
lib = b.ctx.lib
names = ["launch","cand_sort","footprint","solve","validate","rec_sort","merge","los","trie_seq"]
for W in (1, 8):
    coverage_from_candidates(sc, b, tx, grid, shard_index=0, shard_count=W)
    lib.rt_set_profiling(b.ctx.h, 1)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    coverage_from_candidates(sc, b, tx, grid, shard_index=0, shard_count=W)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ms, ctr = bench._profile(b)
    lib.rt_set_profiling(b.ctx.h, 0)
    print(W, "wall %.2f ms" % (1e3 * (t1 - t0)), {n: round(float(ms[i]), 3) for i, n in enumerate(names) if ms[i] > 0})
