"""Summarise ncu outputs (run here, on the CPU box) into profiles/.

    python scripts/ncu_summary.py --rep gpurun_out/prof_fused_c3.ncu-rep --name r01_fused_c3
    python scripts/ncu_summary.py --launches gpurun_out/launches.csv --name r01_launches
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__average_warp_latency_per_inst_issued.ratio",
]


def rep_summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[m] = float(r[i].replace(",", ""))
                except ValueError:
                    d[m] = r[i]
                d[m + ".unit"] = units[i]
        launches.append(d)
    return launches


def launches_summary(path, split_ns=None):
    """Per-kernel launch counts, mean duration and share of GPU time.  With
    split_ns, launches longer than split_ns are reported as a separate group
    (bench.py's zero-copy e2e launches read their inputs over PCIe and run
    ~30x longer than the device-resident steps)."""
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    dur = {r[ii]: float(r[vi].replace(",", "")) for r in rows[1:] if r[mi] == "gpu__time_duration.sum"}
    d = defaultdict(lambda: defaultdict(list))
    units = {}
    for r in rows[1:]:
        name = r[ki]
        if split_ns is not None and dur.get(r[ii], 0.0) > split_ns:
            name += f"  [launches > {split_ns / 1e3:g} us: pinned-host inputs (zero-copy e2e)]"
        d[name][r[mi]].append(float(r[vi].replace(",", "")))
        units[r[mi]] = r[ui]
    total = sum(sum(m.get("gpu__time_duration.sum", [])) for m in d.values())
    out = []
    for k, m in d.items():
        t = m.get("gpu__time_duration.sum", [])
        out.append({"kernel": k[:200], "launches": len(t), "mean_" + units.get("gpu__time_duration.sum", ""):
                    sum(t) / max(len(t), 1), "share_of_time": sum(t) / total if total else None,
                    **{f"mean_{mm}": sum(v) / len(v) for mm, v in m.items() if mm != "gpu__time_duration.sum"}})
    return sorted(out, key=lambda x: -(x["share_of_time"] or 0))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--name", required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("--split-us", type=float, default=None)
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    res = {"note": a.note}
    if a.rep:
        res["source"] = os.path.basename(a.rep)
        res["ncu"] = "ncu --set full --clock-control none --import-source on (cold L2: ncu cache-control all)"
        res["launches"] = rep_summary(a.rep)
    if a.launches:
        res["source"] = os.path.basename(a.launches)
        res["ncu"] = "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
        res["kernels"] = launches_summary(a.launches, None if a.split_us is None else a.split_us * 1e3)
    with open(os.path.join(PROF, a.name + ".json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:3000])
