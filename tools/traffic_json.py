"""profiles/walk_traffic.json from the ncu metrics capture of tools/ncu_walk.sh.

  python tools/traffic_json.py gpurun_out/walk_metrics.csv
Copies the raw csv to profiles/r01_walk_metrics_batch4096.csv and writes the
per-launch DRAM traffic that bench.py reports as roofline.traffic.
"""
import csv
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "walk_metrics.csv")
rows = [r for r in csv.reader(l for l in open(src) if not l.startswith("=="))]
h = rows[0]
m = {}
for r in rows[1:]:
    if "walk_kernel(" not in r[h.index("Kernel Name")]:
        continue
    m[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
out = {
    "bytes_per_launch": m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"],
    "dram_read": m["dram__bytes_read.sum"],
    "dram_write": m["dram__bytes_write.sum"],
    "duration_ns": m["gpu__time_duration.sum"],
    "l2_bytes": m["lts__t_bytes.sum"],
    "l1_hit_pct": m["l1tex__t_sector_hit_rate.pct"],
    "l2_hit_pct": m["lts__t_sector_hit_rate.pct"],
    "issue_active_pct": m["smsp__issue_active.avg.pct_of_peak_sustained_active"],
    "warps_active_pct": m["sm__warps_active.avg.pct_of_peak_sustained_active"],
    "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,... --clock-control none on one "
              "walk_kernel launch of the default 4096-instance workload (tools/walk_profile.py batch:4096; "
              "ncu serialises it behind walk_kernel_wide); raw csv profiles/r01_walk_metrics_batch4096.csv",
}
shutil.copy(src, os.path.join(ROOT, "profiles", "r01_walk_metrics_batch4096.csv"))
json.dump(out, open(os.path.join(ROOT, "profiles", "walk_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
