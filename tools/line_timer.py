"""Per-line wall time of chosen Python functions (sys.settrace; diagnostic only).

usage: python tools/line_timer.py   -- times compute_gains / build_cir on the C2 workload
"""
import collections
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import channel, em, scenes, tracer  # noqa: E402


def profile(funcs, run, reps):
    codes = {f.__code__ for f in funcs}
    acc = collections.defaultdict(float)
    state = {}

    def tracer_fn(frame, event, arg):
        if frame.f_code not in codes:
            return None

        def local(frame, event, arg):
            now = time.perf_counter()
            key = state.get(frame)
            if key is not None:
                acc[key] += now - state["t"][frame]
            if event in ("line",):
                state[frame] = (frame.f_code.co_name, frame.f_lineno)
                state.setdefault("t", {})[frame] = time.perf_counter()
            elif event == "return":
                state.pop(frame, None)
            return local
        return local

    sys.settrace(tracer_fn)
    for _ in range(reps):
        run()
    torch.cuda.synchronize()
    sys.settrace(None)
    tot = sum(acc.values())
    for (fn, ln), v in sorted(acc.items(), key=lambda kv: -kv[1])[:25]:
        print(f"{fn}:{ln} {1e6 * v / reps:8.1f} us {100 * v / tot:5.1f}%")


def main():
    sc = scenes.street_canyon(n_per_row=100)
    bvh = P.build(sc)
    ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
    for _ in range(5):
        P.build_cir(P.compute_gains(sc, bvh, ps))
    profile([em.compute_gains, channel.build_cir, channel._build_cir_device],
            lambda: P.build_cir(P.compute_gains(sc, bvh, ps)), 30)
    print("---- compute_paths")
    profile([tracer.compute_paths, tracer.paths_to_receivers, tracer.run_launch, tracer.prepare_candidates],
            lambda: P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000), 30)
    print("---- build")
    from paper_2303_11103_b200 import bvh as B
    profile([B.Bvh.__init__, B._gather_geometry], lambda: P.build(sc), 30)


if __name__ == "__main__":
    main()
