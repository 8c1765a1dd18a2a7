"""Summarise ncu outputs of a gpurun pass into profiles/<round>/ (tracked).

    python tools/ncu_summary.py gpurun_out/r01b profiles/r01b [tag]

Reads <src>/launches.csv (ncu --metrics gpu__time_duration.sum --csv launch
list) and <src>/full_raw.csv (ncu --set full, --page raw --csv) and writes
launches_<tag>.txt (per-kernel count / mean / min of the cold-cache serialised
launch times, and each kernel's share of the listed library time) and
ncu_full_<tag>.txt (the counters the roofline and DESIGN.md cite, per
captured launch). Also refreshes profiles/traffic.json (dram bytes per launch
of the resampling kernels, used for bench.py's roofline.traffic).
"""
import csv
import json
import os
import statistics
import sys
from collections import OrderedDict, defaultdict

FULL_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
]


def short(name, n=100):
    return name if len(name) <= n else name[:n]


def launches(src, dst, tag, header):
    rows = list(csv.reader(open(os.path.join(src, "launches.csv"))))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[hdr]
    t = defaultdict(list)
    order = []
    for r in rows[hdr + 1:]:
        if len(r) != len(H):
            continue
        d = dict(zip(H, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"]
        if k not in t:
            order.append(k)
        v = float(d["Metric Value"])
        t[k].append(v / 1000.0 if d["Metric Unit"] == "ns" else v)
    mine = sum(sum(v) for k, v in t.items() if "nfftb::" in k or "_kernel" in k and "at::" not in k)
    out = [header, "# cold-cache, serialised per-launch times (compare shares, not absolutes)",
           "# launches  mean_us  min_us  share_of_library_time  kernel"]
    for k in sorted(order, key=lambda k: -sum(t[k])):
        lib = "nfftb::" in k
        share = f"{sum(t[k]) / mine * 100:5.1f}%" if lib and mine else "   -  "
        out.append(f"{len(t[k]):5d} {statistics.mean(t[k]):8.2f} {min(t[k]):8.2f}   {share}   {short(k)}")
    open(os.path.join(dst, f"launches_{tag}.txt"), "w").write("\n".join(out) + "\n")


def full(src, dst, tag):
    rows = list(csv.reader(open(os.path.join(src, "full_raw.csv"))))
    H = rows[0]
    units = rows[1] if len(rows) > 1 and rows[1] and rows[1][0] == "" else None
    data = [dict(zip(H, r)) for r in rows[(2 if units else 1):] if len(r) == len(H)]
    out = []
    traffic = defaultdict(list)
    for d in data:
        out.append(f"--- {short(d['Kernel Name'], 110)}")
        for k in FULL_KEYS:
            if k in d:
                u = units[H.index(k)] if units else ""
                out.append(f"  {k:70s} {d[k]:>16s} {u}")
        try:
            rb = float(d["dram__bytes_read.sum"].replace(",", ""))
            wb = float(d["dram__bytes_write.sum"].replace(",", ""))
            ur = units[H.index("dram__bytes_read.sum")] if units else "byte"
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(ur, 1)
            uw = units[H.index("dram__bytes_write.sum")] if units else "byte"
            scalew = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(uw, 1)
            traffic[d["Kernel Name"]].append(rb * scale + wb * scalew)
        except (KeyError, ValueError):
            pass
    open(os.path.join(dst, f"ncu_full_{tag}.txt"), "w").write("\n".join(out) + "\n")
    return traffic


def main():
    src, dst = sys.argv[1], sys.argv[2]
    tag = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(dst.rstrip("/"))
    cfg = sys.argv[4] if len(sys.argv) > 4 else "cfg2_1d_2e18:m4"
    os.makedirs(dst, exist_ok=True)
    header = ("# ncu --metrics gpu__time_duration.sum --clock-control none -c 600 python bench.py --steps 3 "
              "--warmup 3 --no-sweep --no-e2e --no-cpu --no-configs --no-strategies (tools/gpu_evidence.sh)")
    if os.path.exists(os.path.join(src, "launches.csv")):
        launches(src, dst, tag, header)
    if os.path.exists(os.path.join(src, "full_raw.csv")):
        traffic = full(src, dst, tag)
        tp = os.path.join(os.path.dirname(dst.rstrip("/")), "traffic.json")
        tj = json.load(open(tp)) if os.path.exists(tp) else {}
        for k, v in traffic.items():
            kind = "spread" if "spread" in k else ("interp" if "interp" in k else None)
            if kind:
                tj[f"{cfg}:{kind}"] = int(statistics.mean(v))
        tj["_source"] = (f"dram__bytes_read.sum + dram__bytes_write.sum per launch, ncu --set full, "
                         f"{dst}/ncu_full_{tag}.txt")
        json.dump(tj, open(tp, "w"), indent=1)
    for f in ("bench.log", "pytest_gpu.log", "smoke.log", "lscpu.txt", "smi.txt"):
        p = os.path.join(src, f)
        if os.path.exists(p):
            lines = open(p).read().splitlines()
            keep = [l for l in lines if l.startswith("{") or "passed" in l or "exit" in l or "smoke" in l
                    or "Model name" in l or "NVIDIA" in l or l.strip().isdigit()]
            open(os.path.join(dst, f.replace(".", f"_{tag}.", 1)), "w").write("\n".join(keep) + "\n")


if __name__ == "__main__":
    main()
