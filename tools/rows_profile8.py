import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench, paper_2303_11103_b200 as P
from paper_2303_11103_b200.channel import coverage_from_candidates
from paper_2303_11103_b200.tracer import run_launch
args = bench.parse([a for a in sys.argv[1:]])
sc, tx, grid = bench.make_workload(args)
b = P.build(sc)
run_launch(b, tx.position, args.depth, int(args.rays))
names = ["launch", "cand_sort", "footprint", "solve", "validate", "rec_sort", "merge", "los", "trie_seq"]
for W in (1, 8):
    for r in range(W):
        coverage_from_candidates(sc, b, tx, grid, shard_index=r, shard_count=W)
    b.ctx.lib.rt_set_profiling(b.ctx.h, 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    coverage_from_candidates(sc, b, tx, grid, shard_index=0, shard_count=W)
    e1.record(); torch.cuda.synchronize()
    ms, _ = bench._profile(b)
    b.ctx.lib.rt_set_profiling(b.ctx.h, 0)
    print(f"W={W} rows shard 0: total {e0.elapsed_time(e1):.3f} ms", {n: round(float(ms[i]), 3) for i, n in enumerate(names)})
