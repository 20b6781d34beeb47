import cProfile, pstats, sys, time
import torch
sys.path.insert(0, ".")
import paper_2303_11103_b200 as P
from paper_2303_11103_b200 import scenes
sc = scenes.street_canyon(n_per_row=100)
bvh = P.build(sc)
for _ in range(5):
    ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
    cir = P.build_cir(P.compute_gains(sc, bvh, ps))
torch.cuda.synchronize()
pr = cProfile.Profile()
N = 50
t0 = time.perf_counter()
pr.enable()
for _ in range(N):
    g = P.compute_gains(sc, bvh, ps)
    cir = P.build_cir(g)
torch.cuda.synchronize()
pr.disable()
print("gains+cir ms", 1e3 * (time.perf_counter() - t0) / N)
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(30)
