"""C2 compute_paths + CIR device timeline (kernels, copies and the gaps between them)
under the torch profiler; diagnostic only: python tools/c2_timeline.py"""
import sys; sys.path.insert(0, ".")
import torch, time, paper_2303_11103_b200 as P
from paper_2303_11103_b200 import scenes
from torch.profiler import profile, ProfilerActivity
sc = scenes.street_canyon(n_per_row=100)
def step():
    bvh = P.build(sc); ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
    return P.build_cir(P.compute_gains(sc, bvh, ps))
for _ in range(20): step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter(); step(); torch.cuda.synchronize(); t1 = time.perf_counter()
print("wall %.3f ms" % (1e3 * (t1 - t0)))
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
base = ev[0].time_range.start
prev_end = base
busy = 0
for e in ev:
    gap = e.time_range.start - prev_end
    busy += e.time_range.elapsed_us()
    print("%8.1f  gap %6.1f  dur %6.1f  %s" % (e.time_range.start - base, gap, e.time_range.elapsed_us(), e.name[:60]))
    prev_end = max(prev_end, e.time_range.end)
print("device span %.1f us, busy %.1f us" % (prev_end - base, busy))
