"""Summarise ncu output (read here, no GPU needed) into profiles/<round>/.

    python tools/ncu_summary.py r01 [--config KEY] gpurun_out/launches.csv gpurun_out/prof_*.ncu-rep

--config KEY tags the ncu_traffic.json entries with the bench configuration the
captures ran (bench.config_key: model/tokens/layout/res/page/requests/shard/n);
bench.py only reports roofline.traffic from a capture of its own configuration.

Writes launches.md (per-kernel launch-time shares of the serialized launch
list) and <kernel>.md (key raw metrics + top warp-stall reasons) per report.
"""

from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__occupancy_limit_registers",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > mi:
            agg[r[ki]].append(float(r[mi].replace(",", "")))
    total = sum(sum(v) for v in agg.values())
    with open(out, "w") as fh:
        fh.write("# ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
        fh.write(f"Source: `{os.path.basename(path)}` — serialized, cold-cache; compare shares.\n\n")
        fh.write("| kernel | launches | mean us | total ms | share |\n|---|---|---|---|---|\n")
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            name = k if len(k) < 90 else k[:87] + "..."
            fh.write(f"| `{name}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | "
                     f"{sum(v) / 1e6:.3f} | {sum(v) / total * 100:.1f}% |\n")


def report(path, out, config=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, vals = rows[0], rows[1], rows[2]
    name = vals[h.index("Kernel Name")] if "Kernel Name" in h else os.path.basename(path)
    name = name.replace("(anonymous namespace)::", "")
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full: `{name[:120]}`\n\nReport: `{os.path.basename(path)}`\n\n")
        fh.write("| metric | value | unit |\n|---|---|---|\n")
        for k in KEYS:
            if k in h:
                fh.write(f"| {k} | {vals[h.index(k)]} | {units[h.index(k)]} |\n")
        if "dram__bytes_read.sum" in h:
            def gb(k):
                v = float(vals[h.index(k)].replace(",", ""))
                u = units[h.index(k)]
                return v * {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}.get(u, 1)
            traffic = gb('dram__bytes_read.sum') + gb('dram__bytes_write.sum')
            fh.write(f"\nDRAM traffic per launch: {traffic:.3f} GB\n")
            # a capture of every launch of one step (-c N): the step's traffic
            step_traffic, n_launch = 0.0, 0
            for r in rows[2:]:
                if len(r) == len(h) and r[h.index("Kernel Name")] == vals[h.index("Kernel Name")]:
                    def gbr(k, r=r):
                        v = float(r[h.index(k)].replace(",", ""))
                        u = units[h.index(k)]
                        return v * {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}.get(u, 1)
                    step_traffic += gbr('dram__bytes_read.sum') + gbr('dram__bytes_write.sum')
                    n_launch += 1
            if n_launch > 1:
                fh.write(f"DRAM traffic of the {n_launch} captured launches (one step): "
                         f"{step_traffic:.3f} GB\n")
            # machine-readable: bench.py reports it as roofline.traffic
            tj = os.path.join(os.path.dirname(out), "ncu_traffic.json")
            data = json.load(open(tj)) if os.path.exists(tj) else {}
            short = name.split("(")[0].split("::")[-1].split("<")[0]
            data[short] = {"dram_bytes_per_launch": traffic * 1e9, "report": os.path.basename(path),
                           "config": config, "launches_captured": n_launch,
                           "dram_bytes_captured": step_traffic * 1e9,
                           "duration": vals[h.index("gpu__time_duration.sum")] + " "
                           + units[h.index("gpu__time_duration.sum")]}
            json.dump(data, open(tj, "w"), indent=1, sort_keys=True)
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(vals[i]), k))
                except ValueError:
                    pass
        fh.write("\nTop warp-stall reasons (warps per issue-active cycle):\n\n")
        for v, k in sorted(stalls, reverse=True)[:6]:
            fh.write(f"- {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}: {v:.3f}\n")


def main():
    rnd = sys.argv[1]
    out_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", rnd)
    os.makedirs(out_dir, exist_ok=True)
    args, config = sys.argv[2:], None
    if args and args[0] == "--config":
        config, args = args[1], args[2:]
    for p in args:
        base = os.path.basename(p)
        if p.endswith(".csv"):
            launches(p, os.path.join(out_dir, base.replace(".csv", ".md")))
        elif p.endswith(".ncu-rep"):
            report(p, os.path.join(out_dir, base.replace(".ncu-rep", ".md")), config)


if __name__ == "__main__":
    main()
