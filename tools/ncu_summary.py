#!/usr/bin/env python
"""Summarize ncu reports into profiles/: key speed-of-light metrics, DRAM
traffic per launch and the top warp-stall reasons (from the source page)."""
import csv
import io
import os
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Eligible Warps Per Scheduler",
        "L2 Hit Rate", "Waves Per SM", "Grid Size", "Block Size", "Dynamic Shared Memory Per Block"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def summarize(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "details", "--csv"))))
    h = rows[0]
    det = {}
    name = ""
    for r in rows[1:]:
        d = dict(zip(h, r))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in KEYS and d["Metric Name"] not in det:
            det[d["Metric Name"]] = f'{d["Metric Value"]} {d["Metric Unit"]}'.strip()
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    rd = dict(zip(raw[0], raw[2])) if len(raw) > 2 else {}
    ru = dict(zip(raw[0], raw[1])) if len(raw) > 1 else {}
    traffic = {k: f"{rd[k]} {ru.get(k, '')}" for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in rd}
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv"))))
    stalls = {}
    if len(src) > 2:
        sh = src[1]
        for i, c in enumerate(sh):
            if c.startswith("stall_") and "Not Issued" not in c:
                stalls[c] = sum(float(r[i] or 0) for r in src[2:] if len(r) > i)
    tot = sum(stalls.values()) or 1.0
    out = [f"### {name}", "", "| metric | value |", "|---|---|"]
    out += [f"| {k} | {det[k]} |" for k in KEYS if k in det]
    out += [f"| {k} | {v} |" for k, v in traffic.items()]
    out += ["", "Top warp-stall reasons (sampled):", ""]
    out += [f"- {k}: {100 * v / tot:.1f}%" for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]]
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    dst = sys.argv[1]
    with open(dst, "w") as f:
        f.write(f"# ncu summaries ({os.path.basename(dst)})\n\n")
        f.write("Captured with `ncu --set full --clock-control none --import-source on` on one B200 "
                "(profiles/run_ncu.sh); one launch per kernel of the config-2 bench step.\n\n")
        for rep in sys.argv[2:]:
            f.write(summarize(rep) + "\n")
    print(dst)
