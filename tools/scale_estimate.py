"""Per-rank step time of the two-stage multi-GPU coverage map, measured on one GPU.

For W ranks, rank r's device work is: its band-interleaved launch shard, the
sort/unique of the all-gathered candidate union (replicated), and the solve /
validate / merge of its grid rows.  Each piece is timed with CUDA events on
this GPU, rank by rank; the estimated step is the max over ranks (collectives
excluded: a few MB over NVLink).  usage: python tools/scale_estimate.py [--config c5]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200.channel import coverage_from_candidates  # noqa: E402
from paper_2303_11103_b200.tracer import get_candidates, run_launch, set_candidates  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def main():
    args = bench.parse([a for a in sys.argv[1:] if a != "--ranks"])
    sc, tx, grid = bench.make_workload(args)
    b = P.build(sc)
    n, depth = int(args.rays), args.depth
    for _ in range(2):   # warm-up
        run_launch(b, tx.position, depth, n)
        coverage_from_candidates(sc, b, tx, grid)
    (_, nb), t_launch = timed(lambda: run_launch(b, tx.position, depth, n))
    _, t_cov = timed(lambda: coverage_from_candidates(sc, b, tx, grid))
    t1 = t_launch + t_cov
    print(f"W=1: launch {t_launch:.2f} + coverage {t_cov:.2f} = {t1:.2f} ms")
    for W in (2, 4, 8):
        seqs, lens, t_l = [], [], []
        for r in range(W):
            ts = sorted(timed(lambda: run_launch(b, tx.position, depth, n, shard=(r, W)))[1] for _ in range(3))
            t_l.append(ts[1])
            s, ln = get_candidates(b)
            seqs.append(s.clone())
            lens.append(ln.clone())
        L = max(s.shape[1] for s in seqs)
        cat = torch.cat([torch.nn.functional.pad(s, (0, L - s.shape[1]), value=-1) for s in seqs])
        lc = torch.cat(lens)
        for _ in range(2):   # first call may grow the library's scratch buffers
            _, t_u = timed(lambda: set_candidates(b, cat, lc, L))
        t_c = []
        for r in range(W):   # warm every shard first: a shard may grow the scratch buffers
            coverage_from_candidates(sc, b, tx, grid, shard_index=r, shard_count=W)
        for r in range(W):   # median of 3: one-off hiccups do not decide the max over ranks
            ts = sorted(timed(lambda: coverage_from_candidates(sc, b, tx, grid, shard_index=r,
                                                               shard_count=W))[1] for _ in range(3))
            t_c.append(ts[1])
        per = [a + t_u + c for a, c in zip(t_l, t_c)]
        tw = max(per)
        if "--ranks" in sys.argv:
            print(f"  W={W} per-rank rows ms: " + " ".join(f"{x:.2f}" for x in t_c))
        print(f"W={W}: launch max {max(t_l):.2f} (min {min(t_l):.2f}), union sort {t_u:.2f}, "
              f"rows max {max(t_c):.2f} (min {min(t_c):.2f}) -> step {tw:.2f} ms, "
              f"efficiency {t1 / (W * tw):.3f}")


if __name__ == "__main__":
    main()
