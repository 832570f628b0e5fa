"""BASELINE.md §3 / SURVEY §8(d) same-run table: the unmodified reference
planner (oracle/_ref/ref_driver, compiled from /root/reference) walks the
named configurations 1-4 in full on this host's cores, next to the B200 walk
of the same instances (discover_frontier end to end, T* -> T_min).

  python tools/cpu_table.py [--out profiles/r02_cpu_table.json] [--configs 1,2,3,4]

CPU, per config:
  * 1 thread  -- one walk (best of 3 for configs 1-2; configs 3-4 take
    4-13 min per walk, so the single-thread figure is the fastest of the
    concurrent walks below, each of which runs on its own core);
  * nproc threads -- nproc concurrent copies of the instance (throughput
    over the whole host; best of 3 for configs 1-2, one run for 3-4).
GPU, per config: one instance alone (latency: the shared-memory-resident
walk) and a batch of copies filling the device (throughput), device-timed
launches (best of 3), plus the same through the C ABI with host buffers.
"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")
STEPS = {1: 264, 2: 936, 3: 3240, 4: 3432}


def ref_bench(threads, specs):
    out = subprocess.run([DRIVER, "bench", str(threads), *specs], capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def cpu_row(k, nproc):
    spec = f"config:{k}"
    reps = 3 if k <= 2 else 1
    one = None
    if k <= 2:
        one = min((ref_bench(1, [spec]) for _ in range(reps)), key=lambda r: r["wall_s"])
    many = min((ref_bench(nproc, [spec] * nproc) for _ in range(reps)), key=lambda r: r["wall_s"])
    if one is None:  # fastest concurrent walk, one per core
        t1 = min(many["instance_s"])
        one = {"points": many["points"] // nproc, "wall_s": t1, "from": "fastest of the concurrent walks"}
    return {
        "config": k, "points_per_walk": one["points"],
        "t1_s": one["wall_s"], "t1_points_per_s": one["points"] / one["wall_s"],
        "t1_source": one.get("from", f"best of {reps}"),
        "threads": nproc, "tn_wall_s": many["wall_s"], "tn_points_per_s": many["points"] / many["wall_s"],
        "tn_source": f"best of {reps}", "instance_s": many["instance_s"],
    }


def gpu_row(k):
    import paper_2312_06902_b200 as pb
    from paper_2312_06902_b200 import g9
    row = {"config": k}
    for label, reps in (("single", 1), ("batch", {1: 4096, 2: 1776, 3: 444, 4: 296}[k])):
        b = pb.FrontierBatch()
        for _ in range(reps):
            b.add_g9(g9.named_config(k))
        b.prepare(0)
        b.launch()
        ms = min(b.launch() for _ in range(3))
        b.fetch()
        st = b.stats()
        pts = sum(b.summary(i).steps + 1 for i in range(len(b)))
        assert all(b.summary(i).status == 0 and b.summary(i).steps == STEPS[k] for i in range(len(b)))
        t0 = time.perf_counter()
        b.run(0)
        e2e = time.perf_counter() - t0
        row[label] = {"instances": reps, "kernel_ms": ms, "points_per_s": pts / (ms / 1e3),
                      "us_per_step": ms * 1e3 / STEPS[k] if reps == 1 else None,
                      "e2e_s": e2e, "e2e_points_per_s": pts / e2e,
                      "mode": "smem" if st.smem_walks else ("wide+walker" if st.wide_walks else "walker"),
                      "smem_region": st.smem_region}
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_cpu_table.json"))
    ap.add_argument("--configs", default="1,2,3,4")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    nproc = os.cpu_count() or 1
    rows = []
    for k in [int(x) for x in args.configs.split(",")]:
        r = {"config": k, "gpu": gpu_row(k)}
        if not args.no_cpu:
            r["cpu"] = cpu_row(k, nproc)
            c, g = r["cpu"], r["gpu"]
            r["gpu_single_over_cpu_1t"] = g["single"]["points_per_s"] / c["t1_points_per_s"]
            r["gpu_batch_over_cpu_nproc"] = g["batch"]["points_per_s"] / c["tn_points_per_s"]
        rows.append(r)
        print(json.dumps(r), flush=True)
    with open(args.out, "w") as f:
        json.dump({"host_cores": nproc, "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0]
                   .strip(" :\t") if os.path.exists("/proc/cpuinfo") else None, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
