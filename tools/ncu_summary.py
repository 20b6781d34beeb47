"""Summarise ncu outputs into profiles/ (launch list shares + per-kernel metrics).

usage: python tools/ncu_summary.py launches <launches.csv> <out.md>
       python tools/ncu_summary.py full <report.ncu-rep> <out.md> [<traffic.json> <bench args...>]
The traffic JSON keeps one capture per bench workload (bench.py committed_traffic);
the bench args (e.g. --config c5) name the workload the capture was taken of.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path, out):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    data = [dict(zip(hdr, r)) for r in rows[start + 1:] if len(r) == len(hdr)]
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0,
                 "msecond": 1.0}.get(unit, 1e-6)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    with open(out, "w") as fh:
        fh.write(f"# ncu launch list: {path}\n\n`--metrics gpu__time_duration.sum --clock-control none` "
                 "(cold-cache, serialised per launch: compare shares, not absolutes)\n\n")
        fh.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            fh.write(f"| `{k[:90]}` | {n} | {ms:.3f} | {100 * ms / tot:.1f}% |\n")
        fh.write(f"\ntotal kernel time {tot:.2f} ms over {sum(v[0] for v in agg.values())} launches\n")


KEYS = ["Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput",
        "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "Branch Efficiency", "Executed Instructions"]


def full(path, out, traffic_json=None, *bench_args):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    per = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        k = (d.get("ID"), d.get("Kernel Name", "").split("(")[0])
        if d.get("Metric Name") in KEYS:
            per[k][d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    rh = rr[0]
    units = dict(zip(rh, rr[1])) if len(rr) > 1 else {}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    dram = {}
    stalls = {}
    insts = {}
    lts, l1 = {}, {}
    for r in rr[2:]:
        d = dict(zip(rh, r))
        k = (d.get("ID"), d.get("Kernel Name", "").split("(")[0])
        try:
            insts[k] = float(d["inst_executed"].replace(",", ""))
        except (KeyError, ValueError):
            pass
        # 32-byte sectors through L2 (all sources) and the L1/TEX global loads
        for name, dst in (("lts__t_sectors.sum", lts), ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", l1)):
            try:
                dst[k] = 32.0 * float(d[name].replace(",", ""))
            except (KeyError, ValueError):
                pass
        try:
            dram[k] = sum(float(d[m].replace(",", "")) * scale.get(units.get(m, "byte"), 1.0)
                          for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        except (KeyError, ValueError):
            pass
        st = {}
        for h, v in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v.replace(",", ""))
                except ValueError:
                    pass
        stalls[k] = st
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full: {path}\n\n")
        for k, m in per.items():
            fh.write(f"## {k[1]} (launch id {k[0]})\n\n")
            for key in KEYS:
                if key in m:
                    fh.write(f"- {key}: {m[key]}\n")
            if k in dram:
                fh.write(f"- dram bytes (read+write): {dram[k]:.6g} B\n")
            st = stalls.get(k, {})
            tot = sum(st.values()) or 1.0
            top = sorted(st.items(), key=lambda kv: -kv[1])[:6]
            fh.write("- top stall reasons (share of samples): " +
                     ", ".join(f"{n} {100 * v / tot:.0f}%" for n, v in top) + "\n\n")


    if traffic_json:   # per-kernel figures for bench.py's roofline
        import json
        def per_kernel(m):
            acc = {}
            for k, v in m.items():
                acc.setdefault(k[1], []).append(v)
            return {k: sum(v) / len(v) for k, v in acc.items()}
        import os
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench
        args = bench.parse(list(bench_args))
        cap = {"source": path, "workload": bench.workload_name(args), "num_rays": int(args.rays),
               "max_depth": args.depth,
               "dram_bytes_per_launch": per_kernel(dram), "warp_instructions_per_launch": per_kernel(insts),
               "lts_bytes_per_launch": per_kernel(lts), "l1tex_bytes_per_launch": per_kernel(l1)}
        caps = []
        if os.path.exists(traffic_json):
            old = json.load(open(traffic_json))
            caps = [c for c in old.get("captures", [old]) if c.get("workload") != cap["workload"]]
        json.dump({"captures": caps + [cap]}, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:])
