"""Warp-stall breakdown of one launch in an ncu report (--set full).

    python scripts/ncu_stalls.py gpurun_out/final_prof_fused.ncu-rep [--launch 0]

Prints smsp__average_warp_latency_issue_stalled_* (cycles per issued
instruction spent in each stall reason) sorted, plus a few context metrics.
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--launch", type=int, default=0)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
r = data[a.launch]
print(r[hdr.index("Kernel Name")][:100])
stalls = []
for i, h in enumerate(hdr):
    if "issue_stalled" in h and h.endswith(".ratio") and "not_issued" not in h:
        try:
            stalls.append((float(r[i].replace(",", "")), h))
        except ValueError:
            pass
for v, h in sorted(stalls, reverse=True)[:16]:
    print(f"{v:8.3f}  {h}")
for key in ("gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
            "smsp__inst_executed.sum", "smsp__warps_active.avg.per_cycle_active",
            "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "dram__bytes_read.sum",
            "lts__t_bytes.sum", "sm__ctas_launched.sum"):
    if key in hdr:
        i = hdr.index(key)
        print(f"{key} = {r[i]} {units[i]}")
