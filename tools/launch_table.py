#!/usr/bin/env python
"""launches.csv (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv) -> the markdown launch table under profiles/."""
import collections
import csv
import re
import sys


def main(src, dst, round_tag, only=None, max_id=None):
    rows = list(csv.reader(open(src)))
    hdr = None
    per = {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if only and not re.search(only, d["Kernel Name"]):
                continue
            if max_id is not None and int(d["ID"]) > max_id:
                continue
            per.setdefault((d["ID"], d["Kernel Name"]), {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    agg = collections.OrderedDict()
    for (i, k), m in per.items():
        agg.setdefault(k.split("(")[0], []).append(m)
    tot = sum(sum(x["gpu__time_duration.sum"] for x in l) / len(l) for l in agg.values())
    out = [f"# Launch list ({round_tag}; ncu, cold-cache, serialized)", "",
           "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` "
           "over `bench.py --steps 3 --warmup 3 --graph 0` (profiles/run_ncu.sh). Per-launch times are serialized "
           "and cold-cache: compare shares, not absolutes.", "",
           "| kernel | launches | mean us | share of step | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
    for k, l in agg.items():
        us = sum(x["gpu__time_duration.sum"] for x in l) / len(l) / 1e3
        rd = sum(x.get("dram__bytes_read.sum", 0) for x in l) / len(l) / 1e6
        wr = sum(x.get("dram__bytes_write.sum", 0) for x in l) / len(l) / 1e6
        out.append(f"| {k} | {len(l)} | {us:.1f} | {100 * us * 1e3 / tot:.1f}% | {rd:.1f} | {wr:.1f} |")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "r01", sys.argv[4] if len(sys.argv) > 4 else None,
         int(sys.argv[5]) if len(sys.argv) > 5 else None)
