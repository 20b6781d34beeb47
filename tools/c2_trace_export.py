import sys, time, json
import torch
sys.path.insert(0, ".")
import paper_2303_11103_b200 as P
from paper_2303_11103_b200 import scenes
from torch.profiler import profile, ProfilerActivity
sc = scenes.street_canyon(n_per_row=100)
for _ in range(5):
    bvh = P.build(sc); ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000); cir = P.build_cir(P.compute_gains(sc, bvh, ps))
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bvh = P.build(sc); ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000); cir = P.build_cir(P.compute_gains(sc, bvh, ps))
        torch.cuda.synchronize()
        print("iter ms", 1e3*(time.perf_counter()-t0))
prof.export_chrome_trace("gpurun_out/c2_trace.json")
