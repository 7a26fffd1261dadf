"""Summarize an ncu report (or a launch-list CSV) as markdown for profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--cells N]
    python tools/ncu_summary.py --launches gpurun_out/launches.csv

For a --set full report: per kernel duration, DRAM bytes (read+write), DRAM
throughput, fp64-pipe utilisation, achieved occupancy, registers, warp
instructions per cell, and the SASS opcode mix of the heaviest kernel.
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def ncu_csv(args):
    out = subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


BYTE_UNITS = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,
              "GB": 1e9, "MB": 1e6, "KB": 1e3, "B": 1.0}
TIME_MS = {"msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "second": 1e3,
           "ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3}


def short(name: str) -> str:
    base = name.split("(")[0].replace("void ", "").replace("bsq::", "")
    return base


def summary(rep: str, cells: int, mix: str = None) -> str:
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)])
    hdr, units = rows[0], rows[1]
    lines = ["| kernel | ms | DRAM GB (r+w) | bytes/cell | DRAM % peak | fp64 pipe % | warps active % | regs | warp-inst/cell |",
             "|---|---|---|---|---|---|---|---|---|"]
    heavy = None
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        un = dict(zip(hdr, units))
        ms = float(d["gpu__time_duration.sum"]) * TIME_MS.get(un["gpu__time_duration.sum"], 1.0)
        byts = (float(d["dram__bytes_read.sum"]) * BYTE_UNITS.get(un["dram__bytes_read.sum"], 1e9)
                + float(d["dram__bytes_write.sum"]) * BYTE_UNITS.get(un["dram__bytes_write.sum"], 1e9))
        inst = float(d["smsp__inst_executed.sum"])
        lines.append(f"| {short(d['Kernel Name'])} | {ms:.3f} | {byts / 1e9:.3f} | {byts / cells:.1f} | "
                     f"{float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):.1f} | "
                     f"{float(d['sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} | "
                     f"{d['launch__registers_per_thread']} | {inst / cells:.1f} |")
        if heavy is None or ms > heavy[1]:
            heavy = (d["Kernel Name"], ms)
    if heavy:
        k = mix or short(heavy[0]).split("<")[0].split("::")[-1]
        sass = ncu_csv(["-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}",
                        "--print-source", "sass"])
        h = sass[1]
        ie, isrc = h.index("Instructions Executed"), h.index("Source")
        ops = collections.Counter()
        tot = 0
        for r in sass[2:]:
            if len(r) <= ie:
                continue
            try:
                n = int(r[ie])
            except ValueError:
                continue
            toks = r[isrc].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            ops[op.split(".")[0]] += n
            tot += n
        lines.append("")
        lines.append(f"SASS opcode mix of {k} (thread-instructions per cell):")
        lines.append("")
        lines.append("| opcode | per cell | share |")
        lines.append("|---|---|---|")
        for op, n in ops.most_common(16):
            lines.append(f"| {op} | {n * 32 / cells:.1f} | {n / tot * 100:.1f}% |")
    return "\n".join(lines)


def launches(path: str) -> str:
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[start + 1:]:
        if len(r) > mv and r[mv]:
            v = float(r[mv].replace(",", ""))
            tot[short(r[kn])] += v
            cnt[short(r[kn])] += 1
    s = sum(tot.values())
    out = ["| kernel | launches | total | share |", "|---|---|---|---|"]
    for k in sorted(tot, key=lambda x: -tot[x]):
        out.append(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {tot[k] / s * 100:.1f}% |")
    return "\n".join(out)


def traffic_json(rep: str, cells: int, source: str) -> dict:
    """Per-kernel DRAM bytes per launch (first launch of each name) and the
    fp64-pipe utilisation, for bench.py's roofline.traffic."""
    rows = ncu_csv(["-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)])
    hdr, units = rows[0], rows[1]
    un = dict(zip(hdr, units))
    sr = BYTE_UNITS.get(un["dram__bytes_read.sum"], 1e9)
    sw = BYTE_UNITS.get(un["dram__bytes_write.sum"], 1e9)
    tms = TIME_MS.get(un["gpu__time_duration.sum"], 1.0)
    names = {"k_stage": "stage", "k_correct": "correct", "k_final": "final"}
    out, seen_solve = {}, 0
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = short(d["Kernel Name"]).split("<")[0].split("::")[-1]
        if k == "k_solve_tma":
            seen_solve += 1
            key = f"solve{seen_solve}"
        else:
            key = names.get(k)
        if not key or key in out:
            continue
        b = float(d["dram__bytes_read.sum"]) * sr + float(d["dram__bytes_write.sum"]) * sw
        out[key] = {"bytes_per_launch": b, "bytes_per_cell": b / cells,
                    "ms": float(d["gpu__time_duration.sum"]) * tms,
                    "fp64_pipe_pct": float(d["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"])}
    return {"source": source, "cells": cells, "kernels": out}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", nargs="?")
    ap.add_argument("--cells", type=int, default=4096 * 4096)
    ap.add_argument("--launches")
    ap.add_argument("--mix", help="kernel name (regex) for the opcode mix; default the heaviest")
    ap.add_argument("--traffic-json", help="write per-kernel DRAM bytes (for bench.py) here")
    a = ap.parse_args()
    if a.traffic_json:
        import json
        with open(a.traffic_json, "w") as fh:
            json.dump(traffic_json(a.rep, a.cells, a.rep), fh, indent=1)
    if a.launches:
        print(launches(a.launches))
    if a.rep:
        print(summary(a.rep, a.cells, a.mix))
