"""Summarise an ncu --set full report into a small CSV (+ per-class DRAM traffic JSON).

    python profiles/ncu_summary.py gpurun_out/prof.ncu-rep profiles/rN/ncu_full_summary.csv

Columns: kernel, duration, DRAM read/write bytes, DRAM throughput % of peak,
L2 hit rate, registers, achieved occupancy, issue-slot busy.  The traffic JSON
(profiles/ncu_traffic.json) maps bench.py's kernel classes to DRAM bytes per
launch, which bench.py reports as roofline.traffic.
"""

import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("duration_us", "gpu__time_duration.sum"),
    ("dram_read_B", "dram__bytes_read.sum"),
    ("dram_write_B", "dram__bytes_write.sum"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("regs", "launch__registers_per_thread"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("issue_busy_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
]
SCALE = {"usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3, "ns": 1e-3, "byte": 1.0, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0, "": 1.0, "register/thread": 1.0}

CLASS = [("k_front", "sweep_front"), ("k_bcr", "sweep_front"), ("k_part_solve", "sweep_front"), ("k_stencil<", None),
         ("k_block_dot", "krylov_dot"), ("k_block_update", "krylov_update"),
         ("k_restrict", "restrict"), ("k_prolong", "prolong"), ("k_gather", "sweep_gather"),
         ("k_pre2d", "pre_fused"), ("k_post2d", "post_fused"), ("k3_solve", "sweep_front")]
MODE = {"0": "stencil", "1": "residual", "2": "jacobi", "3": "jacobi2z"}


def kclass(name):
    for key, cls in CLASS:
        if key in name:
            if cls is None:   # k_stencil<S, MODE>
                mode = name.split("<")[1].split(">")[0].split(",")[1].strip()
                return MODE.get(mode, "stencil")
            return cls
    return None


def main(rep, out_csv, traffic_json="profiles/ncu_traffic.json", config=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    ki = hdr.index("Kernel Name")
    lines = ["kernel," + ",".join(m for m, _ in METRICS)]
    traffic = {}
    for r in rows[2:]:
        vals = []
        for _, key in METRICS:
            if key not in hdr:
                vals.append("")
                continue
            i = hdr.index(key)
            try:
                v = float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0)
            except ValueError:
                v = float("nan")
            vals.append(f"{v:.4g}")
        name = r[ki].replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        lines.append(f"\"{name}\"," + ",".join(vals))
        cls = kclass(name)
        if cls and "dram__bytes_read.sum" in hdr:
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", "")) * \
                SCALE.get(units[hdr.index("dram__bytes_read.sum")], 1.0)
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", "")) * \
                SCALE.get(units[hdr.index("dram__bytes_write.sum")], 1.0)
            traffic.setdefault(cls, []).append(rd + wr)
    open(out_csv, "w").write("\n".join(lines) + "\n")
    tr = {k: sum(v) / len(v) for k, v in traffic.items()}
    if config is not None:   # BASELINE configs index the capture ran on (bench.py checks it)
        tr["config"] = int(config)
    json.dump(tr, open(traffic_json, "w"), indent=1)
    print("\n".join(lines))
    print(json.dumps(tr, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
