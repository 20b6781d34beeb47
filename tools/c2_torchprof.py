import sys, time
sys.path.insert(0, ".")
import torch
import paper_2303_11103_b200 as P
from paper_2303_11103_b200 import scenes
sc = scenes.street_canyon(n_per_row=100)
bvh = P.build(sc)
ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
for _ in range(3):
    gains = P.compute_gains(sc, bvh, ps)
    cir = P.build_cir(gains)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    gains = P.compute_gains(sc, bvh, ps)
    cir = P.build_cir(gains)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))
print("a shape", cir.a.shape, cir.a.nbytes)
