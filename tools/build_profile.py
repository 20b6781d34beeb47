"""BVH build timing on the C3 (or C5) city; diagnostic: python tools/build_profile.py [c5]
Run under `ncu --metrics gpu__time_duration.sum` for the per-kernel split."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import scenes  # noqa: E402


def main():
    sc = scenes.city(n_side=448 if "c5" in sys.argv[1:] else 142)
    reps = 1 if "once" in sys.argv[1:] else 5
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bvh = P.build(sc)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print("build %.2f ms" % (1e3 * (t1 - t0)))
        del bvh


if __name__ == "__main__":
    main()
