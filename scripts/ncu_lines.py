"""Per-source-line summary of an ncu report (warp-stall samples, instructions).

    python scripts/ncu_lines.py gpurun_out/prof.ncu-rep [--kernel attn_tc] [--top 40]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--launch", type=int, default=0, help="which profiled launch (0 = first)")
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
# sections start with "File Path" rows; each launch repeats the set of files
lines, cur_file, launch, seen_files = [], None, -1, set()
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        if r[1] in seen_files or cur_file is None and launch < 0:
            launch += 1 if (r[1] in seen_files or launch < 0) else 0
            seen_files = set()
        seen_files.add(r[1])
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or launch != a.launch or r[0] == "":
        continue
    try:
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        inst = int(r[hdr.index("Instructions Executed")] or 0)
    except (ValueError, IndexError):
        continue
    lines.append((samp, inst, cur_file, r[0], r[1]))
tot_s = sum(x[0] for x in lines) or 1
tot_i = sum(x[1] for x in lines) or 1
print(f"samples {tot_s}  instructions {tot_i}")
for samp, inst, f, ln, src in sorted(lines, reverse=True)[: a.top]:
    print(f"{100 * samp / tot_s:5.1f}% samp {100 * inst / tot_i:5.1f}% inst  {f}:{ln:>4}  {src.strip()[:90]}")
