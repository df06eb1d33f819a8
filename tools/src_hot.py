"""Aggregate ncu source-page stall samples per CUDA source line.

usage: python tools/src_hot.py REPORT.ncu-rep [top_n]
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res, hdr = "", [], None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            smp = float(r[4] or 0)
        except ValueError:
            continue
        res.append((smp, fname, int(r[0]), r[1].strip()[:90]))
tot = sum(x[0] for x in res) or 1
for smp, f, ln, src in sorted(res, reverse=True)[:top]:
    print(f"{100 * smp / tot:5.1f}%  {f}:{ln}  {src}")
