import sys, time, cProfile, pstats
sys.path.insert(0, ".")
import torch
import paper_2303_11103_b200 as P
from paper_2303_11103_b200 import scenes
sc = scenes.street_canyon(n_per_row=100)
bvh = P.build(sc)
ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
for _ in range(3):
    g = P.compute_gains(sc, bvh, ps); c = P.build_cir(g)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    g = P.compute_gains(sc, bvh, ps); c = P.build_cir(g)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
