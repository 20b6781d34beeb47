"""C2 (compute_paths + CIR) timeline: torch profiler trace of one step (build + paths +
gains + CIR) -> gpurun_out/c2_trace.json plus a summary of device busy time vs wall.
Diagnostic only: python tools/c2_trace.py"""
import json
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
import paper_2303_11103_b200 as P  # noqa: E402
from paper_2303_11103_b200 import scenes  # noqa: E402


def step(sc):
    bvh = P.build(sc)
    ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
    cir = P.build_cir(P.compute_gains(sc, bvh, ps))
    torch.cuda.synchronize()
    return cir


def main():
    sc = scenes.street_canyon(n_per_row=100)
    for _ in range(4):
        step(sc)
    t0 = time.perf_counter()
    step(sc)
    wall = time.perf_counter() - t0
    os.makedirs("gpurun_out", exist_ok=True)
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        step(sc)
    prof.export_chrome_trace("gpurun_out/c2_trace.json")
    ev = json.load(open("gpurun_out/c2_trace.json"))["traceEvents"]
    dev = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    busy = sum(e["dur"] for e in dev)
    span = (max(e["ts"] + e["dur"] for e in dev) - min(e["ts"] for e in dev)) if dev else 0
    print(f"wall {1e3 * wall:.2f} ms (unprofiled); device busy {busy / 1e3:.2f} ms over a {span / 1e3:.2f} ms span, "
          f"{len(dev)} device ops")
    by = {}
    for e in dev:
        k = e["name"].split("(")[0][:70]
        a = by.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += e["dur"]
    for k, (n, d) in sorted(by.items(), key=lambda x: -x[1][1])[:25]:
        print(f"{d / 1e3:8.3f} ms {n:4d}x  {k}")
    rt = [e for e in ev if e.get("cat") == "cuda_runtime"]
    byr = {}
    for e in rt:
        a = byr.setdefault(e["name"], [0, 0.0])
        a[0] += 1
        a[1] += e["dur"]
    print("runtime API:")
    for k, (n, d) in sorted(byr.items(), key=lambda x: -x[1][1])[:12]:
        print(f"{d / 1e3:8.3f} ms {n:4d}x  {k}")


if __name__ == "__main__":
    main()
