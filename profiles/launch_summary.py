"""Summarise an ncu launch list (gpu__time_duration.sum CSV) by kernel.

    python profiles/launch_summary.py gpurun_out/launches.csv profiles/rN/launches_summary.csv "<command>"
"""

import collections
import csv
import sys

UNIT = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}


def main(src, dst, command=""):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        ns = float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += ns
    total = sum(v[1] for v in agg.values())
    n = sum(v[0] for v in agg.values())
    with open(dst, "w") as f:
        f.write("# ncu launch list summary (gpu__time_duration.sum, --clock-control none)\n")
        f.write(f"# command: {command}  ({n} launches)\n")
        f.write("# unit: ns; cold-cache serialised per-launch times: compare SHARES\n")
        f.write("kernel,launches,total,share\n")
        for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"{k},{c},{t:.1f},{t / total:.4f}\n")


if __name__ == "__main__":
    main(*sys.argv[1:4])
