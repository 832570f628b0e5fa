"""profiles/walk_traffic.json from an ncu metrics capture of one bench step
(tools/ncu_walk.sh: every walk kernel of one launch of the default workload,
serialised by ncu).

  python tools/traffic_json.py gpurun_out/walk_metrics.csv [round-tag]
Copies the raw csv to profiles/<tag>_walk_metrics_batch4096.csv and writes,
per kernel and summed over the step's kernels, the DRAM traffic bench.py
reports as roofline.traffic.
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "walk_metrics.csv")
tag = sys.argv[2] if len(sys.argv) > 2 else "r02"
rows = [r for r in csv.reader(line for line in open(src) if not line.startswith("=="))]
h = rows[0]
kernels = {}
for r in rows[1:]:
    name = r[h.index("Kernel Name")]
    short = "walk_kernel_wide" if "walk_kernel_wide" in name else (
        "walk_kernel_smem" if "walk_kernel_smem" in name else ("walk_kernel" if "walk_kernel" in name else None))
    if short is None:
        continue
    kernels.setdefault(short, {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))


def summary(m):
    return {
        "bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
        "dram_read": m["dram__bytes_read.sum"],
        "dram_write": m["dram__bytes_write.sum"],
        "duration_ns": m["gpu__time_duration.sum"],
        "l2_bytes": m.get("lts__t_bytes.sum"),
        "l1_hit_pct": m.get("l1tex__t_sector_hit_rate.pct"),
        "l2_hit_pct": m.get("lts__t_sector_hit_rate.pct"),
        "issue_active_pct": m.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": m.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    }


per = {k: summary(m) for k, m in kernels.items()}
raw = f"profiles/{tag}_walk_metrics_batch4096.csv"
out = {
    "bytes_per_launch": sum(v["bytes_per_launch"] for v in per.values()),
    "kernels": per,
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,... --clock-control none on every walk "
              "kernel of one launch of the default 4096-instance workload (tools/walk_profile.py batch:4096; "
              f"ncu serialises walk_kernel_wide and walk_kernel); summed over the step's kernels; raw csv {raw}",
}
shutil.copy(src, os.path.join(ROOT, raw))
json.dump(out, open(os.path.join(ROOT, "profiles", "walk_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
