"""Benchmark: coverage-map ray-bounces/s (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[2], "C3"): procedural city of 142 x 142 box
buildings (201,642 triangles), one isotropic transmitter above the central
street crossing, coverage map of 512 x 512 cells of 1 m at 1.5 m height,
max_depth = 5, 1e8 Fibonacci rays.  One step = the whole coverage map:
ray launch + candidate dedup/sort (stage 1), footprint culling, image solve,
occlusion, probe-power transfer, per-cell merge and accumulation (stage 2).

value   = launch ray-bounces of all ranks / max-over-ranks device step time
          (inputs resident in HBM; L2 flushed between timed steps).
e2e     = the same metric through the public API (build(scene) with the
          scene's host arrays + coverage_map returning host numpy gains),
          H2D/D2H inside the timed region.
N > 1   = torchrun, one rank per GPU: rays sharded by slot range (stage 1),
          candidates all-gathered, cell rows sharded round-robin (stage 2),
          grids sum-all-reduced over NCCL.  "scaling": "weak" is not claimed —
          total work is fixed (strong scaling).

Also on the line: c2_paths_cir (BASELINE metric part 2, C2 compute_paths +
CIR latency through the public API) and c4_material_grad (C4: one gradient
step of the material-learning loss through the adjoint).

--impl reference runs the CPU oracle (a restatement of the reference
algorithm, pinned to its golden vectors) on the host cores: each step is a
bounded sample of the same workload (see cpu_baseline.sample).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "coverage-map ray-bounces/s"
UNIT = "ray-bounces/s"
BYTES_PER_NODE = 64    # BNode: two float child boxes + refs (rt_common.cuh)
BYTES_PER_TRI = 80     # TriRec: FP64 v0/e1/e2 + prim id


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--rays", type=float, default=1e8)
    ap.add_argument("--depth", type=int, default=5)
    ap.add_argument("--side", type=int, default=142, help="city boxes per side (142 -> C3)")
    ap.add_argument("--cells", type=int, default=512)
    ap.add_argument("--cell-size", type=float, default=1.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c2", action="store_true")
    ap.add_argument("--cpu-rays", type=float, default=4e6)
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--config", default="c3", choices=["c3", "c5"],
                    help="c3: 200k tris, 512^2 cells, 1e8 rays (default); "
                         "c5: 2M tris, 2048^2 cells, 1e9 rays")
    args = ap.parse_args(argv)
    if args.config == "c5":
        args.side, args.cells = 448, 2048
        if args.rays == 1e8:
            args.rays = 1e9
    return args


def make_workload(args):
    from paper_2303_11103_b200 import scenes
    from paper_2303_11103_b200.channel import GridSpec
    sc = scenes.city(n_side=args.side, seed=0)
    tx = sc.devices[0]
    n = args.cells
    half = 0.5 * n * args.cell_size
    grid = GridSpec((float(tx.position[0]) - half, float(tx.position[1]) - half), args.cell_size,
                    n, n, 1.5)
    return sc, tx, grid


def workload_name(args):
    return (f"{args.config.upper()} coverage_map: city {args.side}x{args.side} boxes, 1 tx, "
            f"{args.cells}x{args.cells} cells @{args.cell_size:g}m")


MICROBENCH = (("fp32_tflops", 0), ("fp64_tflops", 1), ("issue_gwarp_inst_per_s", 2),
              ("l1_read_gbs", 3), ("l2_read_gbs", 4))


def measured_peaks(bvh):
    """Roofline denominators measured live on this GPU (rt_microbench,
    csrc/microbench.cuh): FP32 / FP64 FMA throughput, warp-instruction issue
    rate (imm-form FFMA chains: one instruction per SMSP per cycle), L1- and
    L2-resident read bandwidth.  HBM comes from MEASURED_PEAKS.json."""
    import ctypes
    out = {}
    for name, kind in MICROBENCH:
        v = ctypes.c_double()
        bvh.ctx.call("rt_microbench", kind, ctypes.byref(v), bvh.ctx.stream)
        out[name] = v.value
    return out


TRAFFIC_JSON = "profiles/r02_traffic.json"


def committed_traffic(args, field="dram_bytes_per_launch"):
    """Per-launch k_launch figure (DRAM / L2 / L1 bytes, or warp instructions
    executed with field="warp_instructions_per_launch") from the committed
    `ncu --set full` capture of this same workload (TRAFFIC_JSON holds one
    capture per workload, written by tools/ncu_summary.py full ... <json>);
    None when no capture of this configuration is committed."""
    import json as _json
    path = os.path.join(REPO, TRAFFIC_JSON)
    if not os.path.exists(path):
        return None
    d = _json.load(open(path))
    for cap in d.get("captures", [d]):
        if cap.get("workload") != workload_name(args) or float(cap.get("num_rays", -1)) != float(args.rays) \
                or int(cap.get("max_depth", -1)) != int(args.depth):
            continue
        for k, v in cap.get(field, {}).items():
            if "k_launch" in k:
                return float(v)
    return None


def n_prims(sc):
    return sum(len(o.triangles) for o in sc.objects)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        # NVML in a thread at 5 ms (the timed region lasts ~0.1 s; an nvidia-smi
        # child needs ~0.1 s just to start); nvidia-smi -lms 100 as the fallback
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.th = threading.Thread(target=self._poll_nvml, args=(pynvml, h), daemon=True)
            self.th.start()
            return self
        except Exception:
            pass
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None
        return self

    def _poll_nvml(self, nv, h):
        bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                ("sw_power_cap", 0x4)]
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                break
            self.rows.append([str(sm), str(mx), ""] + ["Active" if rs & b else "Not Active" for _, b in bits])
            self.stop.wait(0.005)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        self.stop.set()
        if getattr(self, "th", None) is not None and self.proc is None:
            self.th.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------------------------
# B200 arm

def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    # BENCH_DIST_BACKEND=gloo is a plumbing check of the sharded legs on a box
    # with fewer GPUs than ranks (ranks share devices round-robin); measurements
    # use NCCL with one GPU per rank
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if backend == "gloo":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")   # rank count visible in the NCCL log
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def run_b200(args):
    import torch
    import paper_2303_11103_b200 as P
    from paper_2303_11103_b200 import _native as N
    from paper_2303_11103_b200 import parallel

    rank, world, local = dist_setup(args)
    dev = torch.device("cuda", local)
    sc, tx, grid = make_workload(args)
    n_rays = int(args.rays)
    bvh = P.build(sc)
    torch.cuda.synchronize()
    flush = torch.empty(int(256e6) // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    gbuf = torch.empty((grid.ny, grid.nx), dtype=torch.float64, device=dev)

    def step():
        b, st, _ = parallel.coverage_step(sc, bvh, tx, grid, args.depth, n_rays, rank, world, out=gbuf)
        return b, st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lib = bvh.ctx.lib
    lib.rt_set_profiling(bvh.ctx.h, 1)
    launches0 = _profile(bvh)[1][15]
    times, bounces_local, stats = [], 0, None
    stage_ms = np.zeros(16)
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            parallel.barrier(world)
            torch.cuda.synchronize()
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            b, stats = step()
            e.record()
            torch.cuda.synchronize()
            parallel.barrier(world)
            times.append(s.elapsed_time(e))
            bounces_local += b
            ms, _ = _profile(bvh)
            stage_ms += np.where(ms > 0, ms, 0.0)
    launches = (_profile(bvh)[1][15] - launches0) / args.steps
    lib.rt_set_profiling(bvh.ctx.h, 0)
    total_ms = parallel.max_over_ranks(float(sum(times)), world)
    bounces_all = parallel.sum_over_ranks(float(bounces_local), world)
    ms_per_step = total_ms / args.steps
    value = bounces_all / (total_ms / 1e3)
    stage_ms /= args.steps

    # traversal counters for the roofline's algorithmic bytes (untimed step)
    lib.rt_set_profiling(bvh.ctx.h, 3)
    step()
    ms_c, ctr = _profile(bvh)
    lib.rt_set_profiling(bvh.ctx.h, 0)
    per_bounce_nodes = ctr[1] / max(ctr[0], 1)
    per_bounce_tris = ctr[2] / max(ctr[0], 1)
    # SIMD efficiency of the launch: bounces per warp bounce-iteration / 32, and
    # node visits per warp traversal / (32 * the warp's longest traversal)
    simd = {"bounce_lanes": float(ctr[0]) / max(32.0 * ctr[10], 1.0),
            "traversal_lanes": float(ctr[1]) / max(32.0 * ctr[11], 1.0)}
    simd["bvh_depth"] = int(ctr[13])
    simd["bvh_sah_node_visits"] = float(ctr[14]) / 1000.0   # 1 + sum internal-child area / root area
    if ctr[12] > 0:   # RT_ORACLE_VISITS builds: node visits had t_max been known in advance
        simd["oracle_nodes_per_bounce"] = float(ctr[12]) / max(ctr[0], 1)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, sc, grid, rank, world, dev, flush)

    peaks_live = measured_peaks(bvh)
    c2 = c4 = None
    if not args.no_c2:
        c2 = c2_latency(args, rank, world)
        c4 = c4_latency(args, rank, world)
    if rank != 0:
        return None
    import json as _json
    peaks = _json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(REPO, "MEASURED_PEAKS.json")) else {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    launch_ms = stage_ms[0]
    bounces_per_launch = bounces_local / args.steps
    bytes_per_bounce = BYTES_PER_NODE * per_bounce_nodes + BYTES_PER_TRI * per_bounce_tris
    t_launch = launch_ms / 1e3 if launch_ms > 0 else None
    names = ["launch", "cand_sort", "footprint", "solve", "validate", "rec_sort", "merge", "los",
             "trie_seq"]
    stage = {n: round(float(stage_ms[i]), 3) for i, n in enumerate(names)}
    roof = roofline(args, peaks_live, hbm_peak, bounces_per_launch, bytes_per_bounce,
                    per_bounce_nodes, per_bounce_tris, t_launch)
    roof.update({"nodes_per_bounce": per_bounce_nodes, "tris_per_bounce": per_bounce_tris,
                 "simd_efficiency": simd, "kernel_ms": launch_ms,
                 "kernel_share": launch_ms / ms_per_step})
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded procedural city, scenes.city(seed=0))",
        "config": {"workload": workload_name(args),
                   "triangles": n_prims(sc), "num_rays": n_rays, "max_depth": args.depth,
                   "cells": grid.num_cells, "cell_m": grid.cell_size, "method": "fibonacci",
                   "tx_mode": "central", "parallelism": f"rays+cell-rows x{world}",
                   "l2": "flushed between timed steps (256 MB write)"},
        "ray_bounces_per_step": bounces_all / args.steps,
        "stage_ms": stage,
        "stats": stats,
        "roofline": roof,
        "peaks_measured": dict(peaks_live, hbm_gbs=hbm_peak,
                               hbm_source="MEASURED_PEAKS.json" if peaks else "fallback"),
        "clocks": clocks.summary(),
        "gpu_launches": int(round(launches)),
    }
    if e2e:
        line["e2e"] = e2e
    if c2 is not None:
        line["c2_paths_cir"] = c2
        line["c4_material_grad"] = c4
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(args, sc, tx, grid, samples=1)
    return line


def roofline(args, pk, hbm_peak, bounces, bytes_per_bounce, nodes_pb, tris_pb, t_launch):
    """Roofline of the dominant kernel (k_launch).

    Primary bound = warp-instruction issue, the one that binds:
    achieved = ncu inst_executed of this workload (committed in TRAFFIC_JSON,
    per bounce) x this run's bounces / this run's kernel time (CUDA events);
    peak = the issue rate measured live by rt_microbench.  Secondary fractions:
    L1 (algorithmic bytes / measured L1-resident read peak), L2 and DRAM (ncu
    lts / dram bytes per launch, committed, / measured peaks), FP32 (box +
    triangle flops / measured FP32 FMA peak) and the north-star traversal
    roofline T* = max(bytes / BW_L2, flops / FP32 peak) / T_kernel."""
    if not t_launch:
        return {"bound": None}
    alg = bounces * bytes_per_bounce
    flops = bounces * (14.0 * nodes_pb * 2 + 40.0 * tris_pb)   # 14 per box test, 2 boxes per node
    insts = committed_traffic(args, "warp_instructions_per_launch")
    lts = committed_traffic(args, "lts_bytes_per_launch")
    dram = committed_traffic(args, "dram_bytes_per_launch")
    out = {}
    sec = {}
    l1 = committed_traffic(args, "l1tex_bytes_per_launch")
    if l1 is not None:
        sec["l1"] = {"achieved": l1 / t_launch / 1e9, "peak": pk["l1_read_gbs"], "unit": "GB/s",
                     "frac": l1 / t_launch / 1e9 / pk["l1_read_gbs"],
                     "bytes": "ncu l1tex global-load sectors x 32 B per launch (" + TRAFFIC_JSON + ")"}
    sec["lane_bytes"] = {"achieved": alg / t_launch / 1e9, "unit": "GB/s",
                         "bytes": "algorithmic, per lane: 64 B per node visit + 80 B per triangle test; "
                                  "coherent lanes share each L1 line, so this exceeds any cache bandwidth"}
    if lts is not None:
        sec["l2"] = {"achieved": lts / t_launch / 1e9, "peak": pk["l2_read_gbs"], "unit": "GB/s",
                     "frac": lts / t_launch / 1e9 / pk["l2_read_gbs"],
                     "bytes": "ncu lts__t_bytes per launch (" + TRAFFIC_JSON + ")"}
    if dram is not None:
        sec["hbm"] = {"achieved": dram / t_launch / 1e9, "peak": hbm_peak, "unit": "GB/s",
                      "frac": dram / t_launch / 1e9 / hbm_peak,
                      "bytes": "ncu dram__bytes read+write per launch (" + TRAFFIC_JSON + ")"}
    sec["fp32"] = {"achieved": flops / t_launch / 1e12, "peak": pk["fp32_tflops"], "unit": "TFLOP/s",
                   "frac": flops / t_launch / 1e12 / pk["fp32_tflops"]}
    t_star = max(alg / (pk["l2_read_gbs"] * 1e9), flops / (pk["fp32_tflops"] * 1e12))
    sec["north_star_traversal"] = {"t_star_ms": 1e3 * t_star, "t_kernel_ms": 1e3 * t_launch,
                                   "frac": t_star / t_launch,
                                   "note": "T* = max(alg bytes / BW_L2, FP32 flops / peak); above 1 "
                                           "because L1 serves ~98% of the node fetches"}
    if insts is not None:
        ach = insts / t_launch / 1e9
        out = {"bound": "issue", "kernel": "k_launch", "achieved": ach,
               "peak": pk["issue_gwarp_inst_per_s"], "unit": "Gwarp-inst/s",
               "frac": ach / pk["issue_gwarp_inst_per_s"], "traffic": dram,
               "warp_instructions_per_launch": insts,
               "warp_instructions_per_bounce": insts / max(bounces, 1.0),
               "achieved_source": TRAFFIC_JSON + " ncu inst_executed of this workload / this run's "
                                                 "k_launch CUDA-event time",
               "peak_source": "rt_microbench kind 2 measured in this run (imm-form FFMA chains)"}
    else:   # no committed capture of this workload: FP32 work vs the measured FP32 peak
        out = dict(sec["fp32"], bound="fp32 (no committed ncu capture of this workload)",
                   kernel="k_launch", traffic=dram, peak_source="rt_microbench kind 0 measured in this run")
    out["traffic_source"] = TRAFFIC_JSON if dram is not None else None
    out["bytes_per_bounce"] = bytes_per_bounce
    out["secondary"] = sec
    return out


def c2_latency(args, rank=0, world=1):
    """BASELINE metric part 2: compute_paths + CIR latency at C2 (street canyon,
    2,002 tris, 8x8 tr38901 array, 256 rx, depth 3, 1e6 rays) through the public
    API, host arrays in, host CIR out (wall clock, device synchronised).  With
    N ranks: rays and receivers sharded, CIR rows all-gathered
    (parallel.compute_paths_cir); the latency is the max over ranks."""
    import torch
    import paper_2303_11103_b200 as P
    from paper_2303_11103_b200 import parallel, scenes
    sc = scenes.street_canyon(n_per_row=100)
    times, t_build = [], []
    out = None
    for i in range(args.warmup + args.steps):
        parallel.barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bvh = P.build(sc)
        if i >= args.warmup:   # split point only: the timed chain is not synchronised here
            t_build.append(time.perf_counter() - t0)
        if world == 1:
            ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
            cir = P.build_cir(P.compute_gains(sc, bvh, ps))
        else:
            cir, ps = parallel.compute_paths_cir(sc, bvh, 3, "fibonacci", 1_000_000, rank, world)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if i >= args.warmup:
            times.append(t1 - t0)
        out = (ps.table.n, list(cir.a.shape), bvh.num_prims)
    med = parallel.max_over_ranks(float(np.median(times)), world)
    paths = int(parallel.sum_over_ranks(float(out[0]), world))
    # compute_paths + CIR alone, on a scene already built (Sionna's compute_paths on
    # a loaded scene): one device build, then the same chain timed per step
    bvh = P.build(sc)
    t_pc = []
    for i in range(args.warmup + args.steps):
        parallel.barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world == 1:
            ps = P.compute_paths(sc, bvh, 3, method="fibonacci", num_rays=1_000_000)
            cir = P.build_cir(P.compute_gains(sc, bvh, ps))
        else:
            cir, ps = parallel.compute_paths_cir(sc, bvh, 3, "fibonacci", 1_000_000, rank, world)
        torch.cuda.synchronize()
        if i >= args.warmup:
            t_pc.append(time.perf_counter() - t0)
    med_pc = parallel.max_over_ranks(float(np.median(t_pc)), world)
    return {"metric": "compute_paths+CIR latency", "value_ms": 1e3 * med,
            "paths_cir_prebuilt_ms": 1e3 * med_pc, "build_submit_ms": 1e3 * float(np.median(t_build)),
            "unit": "ms", "higher_is_better": False, "paths": paths, "cir_a_shape": out[1],
            "triangles": out[2], "rx": 256, "tx_elements": 64, "num_rays": 1_000_000, "max_depth": 3,
            "ranks": world,
            "includes": "value_ms: build(scene) H2D + launch + paths + gains + CIR D2H"
                        + (" + candidate all_gather + CIR row all_gather" if world > 1 else "")
                        + "; paths_cir_prebuilt_ms: the same without build(scene)"}


def c4_latency(args, rank=0, world=1):
    """Config 4 (learning radio materials): one gradient step of the NMSE
    frequency-response loss w.r.t. (eps_r, sigma) of the 4 trainable materials
    through the hand-written adjoint — calib scene, 400 receivers, 128
    subcarriers at 30 kHz, depth 2, paths frozen (optim.MaterialProblem).
    With N ranks the records are sharded and [loss, grads] all-reduced
    (parallel.material_loss_and_grad semantics, timed per step here)."""
    import torch
    from paper_2303_11103_b200 import optim, parallel, scenes
    truth, init = scenes.calib_scene(truth=True), scenes.calib_scene(truth=False)
    pos = np.array([d.position for d in truth.devices if d.kind == "rx"], dtype=np.float64)
    ds = optim.generate_dataset(truth, pos, 128, 30e3, max_depth=2)
    h = np.array([r.h for r in ds.records])
    keep = (np.abs(h) ** 2).sum(-1) > 0.0   # receivers inside buildings have no response
    pos, h = pos[keep], h[keep]
    n_rec = len(pos)
    mine = list(range(rank, n_rec, world))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    prob = optim.MaterialProblem(init, pos[mine], h[mine], 2, 128, 30e3)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    times, grads, loss = [], {}, None
    for i in range(args.warmup + args.steps):
        vals = {n: tuple(torch.tensor(float(getattr(init.materials[n], k)), dtype=torch.float64,
                                      device=prob.bvh.device, requires_grad=True)
                         for k in ("eps_r", "sigma")) for n in prob.names}
        parallel.barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lo = prob.loss(vals) * (len(mine) / n_rec)
        lo.backward()
        vec = torch.stack([lo.detach()] + [v.grad for pair in vals.values() for v in pair])
        if world > 1:
            import torch.distributed as dist
            w = parallel._wire(dist, vec)
            dist.all_reduce(w)
            vec = w
        host = vec.tolist()
        t1 = time.perf_counter()
        loss = host[0]
        names = [f"{n}:{k}" for n in vals for k in ("eps_r", "sigma")]
        grads = dict(zip(names, host[1:]))
        if i >= args.warmup:
            times.append(t1 - t0)
    med = parallel.max_over_ranks(float(np.median(times)), world)
    return {"metric": "material-gradient step latency", "value_ms": 1e3 * med,
            "unit": "ms", "higher_is_better": False, "setup_ms": 1e3 * setup, "records": n_rec,
            "receivers_generated": int(len(keep)), "ranks": world,
            "materials": len(prob.names), "paths_local": int(prob.T.n), "subcarriers": 128,
            "max_depth": 2, "loss": loss, "grads": grads,
            "includes": "forward (rt_transfer + rt_freq_nmse) + backward (rt_transfer_bwd adjoint) "
                        "+ [loss, 8 grads] read-back" + (" after an all_reduce" if world > 1 else "")
                        + "; setup = build + exhaustive candidates + path solve of the records "
                          "(frozen topology)"}


def _profile(bvh):
    import ctypes
    ms = np.zeros(16)
    ctr = np.zeros(16, dtype=np.int64)
    bvh.ctx.lib.rt_get_profile(bvh.ctx.h, ms.ctypes.data_as(ctypes.c_void_p),
                               ctr.ctypes.data_as(ctypes.c_void_p))
    return ms, ctr


def run_e2e(args, sc, grid, rank, world, dev, flush):
    """Public-API step: build(scene) [H2D of the scene arrays] + coverage map
    [D2H gains].  One rank: the emtrace-signature call a drop-in caller makes,
    coverage_map(scene, bvh, grid, max_depth, method, num_rays, cell_cap);
    N ranks: parallel.coverage_map (rays and rows sharded)."""
    import torch
    import paper_2303_11103_b200 as P
    from paper_2303_11103_b200 import parallel
    from paper_2303_11103_b200.bvh import gather_meshes
    verts, tris, _, _, pmat, _ = gather_meshes(sc)
    h2d = verts.nbytes + 4 * tris.size + pmat.nbytes   # vertex ids travel as int32
    d2h = grid.num_cells * 8
    times, bounces = [], 0
    for i in range(args.warmup + args.steps):
        flush.zero_()
        parallel.barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bvh = P.build(sc)
        if world == 1:
            cm = P.coverage_map(sc, bvh, grid, args.depth, method="fibonacci", num_rays=int(args.rays),
                                cell_cap=grid.num_cells)
            g, b = cm.gains, cm.stats["ray_bounces"]
        else:
            g, b = parallel.coverage_map(sc, bvh, grid, args.depth, int(args.rays), rank, world)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        parallel.barrier(world)
        assert g.shape == (grid.ny, grid.nx)
        if i >= args.warmup:
            times.append(t1 - t0)
            bounces += b
        del bvh
    tot = parallel.max_over_ranks(sum(times), world)
    b_all = parallel.sum_over_ranks(float(bounces), world)
    api = ("paper_2303_11103_b200.build + coverage_map(scene, bvh, grid, max_depth, method, num_rays, "
           "cell_cap) (emtrace signature, E/channel.py:236)") if world == 1 else \
        "paper_2303_11103_b200.build + parallel.coverage_map (rays + rows sharded, NCCL)"
    return {"value": b_all / tot, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": 1e3 * tot / args.steps, "api": api}


# ---------------------------------------------------------------------------------------------
# CPU oracle (reference algorithm) arm

def cpu_baseline(args, sc, tx, grid, samples=1, steps=None):
    """Reference algorithm on the host cores: per cell it relaunches the rays
    (channel.py:209-210 -> tracer.py:280-281) and solves every candidate.  A
    bounded sample: launch of --cpu-rays rays at max_depth + one cell's solve."""
    import oracle as O
    t_build0 = time.perf_counter()
    sa = O.SceneArrays(sc)
    ob = O.Bvh(sa)
    t_build = time.perf_counter() - t_build0
    n = int(args.cpu_rays)
    rates, details = [], []
    cell = grid.cell_center(grid.nx // 2 + 7, grid.ny // 2 + 3)
    for _ in range(steps or samples):
        t0 = time.perf_counter()
        seq, bounces = O.launch_sequences(ob, tx.position, args.depth, n)
        cands = O.prefixes_from_sequences(seq)
        packed = O.pack_candidates(cands)
        t1 = time.perf_counter()
        O.coverage_map(sc, ob, grid.origin, grid.cell_size, 1, 1, grid.height, args.depth,
                       points=[cell], packed=packed)
        t2 = time.perf_counter()
        b = int(bounces.sum())
        rates.append(b / (t2 - t0))
        details.append((b, t1 - t0, t2 - t1, len(cands)))
    b, tl, ts, nc = details[-1]
    cores = os.cpu_count()
    job_s = (tl * (args.rays / n) + ts) * grid.num_cells
    return {"value": float(np.mean(rates)), "unit": UNIT, "cores": cores, "kind": "port",
            "sample": (f"oracle (C restatement of emtrace, OpenMP {cores} threads): one cell of the "
                       f"reference algorithm = launch of {n} Fibonacci rays at depth {args.depth} "
                       f"({b} ray-bounces, {tl:.2f}s) + image-solve of {nc} candidates at one cell "
                       f"({ts:.2f}s); BVH build {t_build:.2f}s excluded. The reference relaunches "
                       f"per cell, so the full C3 map would take ~{job_s:.3g}s on this host"),
            "job_seconds_extrapolated": job_s}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    # torchrun sets OMP_NUM_THREADS=1 for every rank; the reference arm runs on
    # rank 0 alone and uses all host cores (read when the oracle's libgomp loads)
    os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
    sc, tx, grid = make_workload(args)
    cb = cpu_baseline(args, sc, tx, grid, steps=args.warmup + args.steps)
    return {"metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded procedural city, scenes.city(seed=0))",
            "config": {"workload": workload_name(args),
                       "triangles": n_prims(sc), "num_rays": int(args.rays),
                       "max_depth": args.depth, "cells": grid.num_cells, "method": "fibonacci"},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def self_launch(args):
    """--gpus N > 1 outside torchrun: start N ranks with torch.distributed.run
    (127.0.0.1, one rank per GPU) and return their exit code."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    line = run_reference(args) if args.impl == "reference" else run_b200(args)
    if args.impl != "reference" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    if line is not None:   # last, after NCCL's own log lines
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
