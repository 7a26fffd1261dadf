"""Per-source-line hotspots of one kernel in an ncu report.

    python tools/ncu_lines.py <rep> <kernel-regex> [--top N]

Aggregates "Instructions Executed" and warp-stall samples per CUDA source
line (needs -lineinfo at build and --import-source on at capture).
"""

import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("kernel")
ap.add_argument("--top", type=int, default=40)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "-k", f"regex:{a.kernel}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = ""
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    d = dict(zip(hdr[2:], r[2:])) if False else None
    try:
        inst = int(r[hdr.index("Instructions Executed")])
        samp = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur_file, int(r[0]), r[1].strip()[:90])
    v = agg.setdefault(key, [0, 0])
    v[0] += inst
    v[1] += samp
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for (f, ln, src), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
    print(f"{i / tot_i * 100:5.1f}% inst {s / tot_s * 100:5.1f}% stall  {f}:{ln}  {src}")
