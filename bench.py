#!/usr/bin/env python
"""Benchmark: Perseus frontier generation on B200 (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload batch|config1|config2|config3|config4] [--batch 4096]
                  [--scaling strong|weak]

One "step" = one pass of the hot path over one batch: every instance's full
frontier walk (frontier.hpp:166-189) in one launch of the sm_100a walk
kernels.  `value` = frontier points/s over the whole job (sum over instances
of steps + 1, all ranks) with inputs resident in HBM; `e2e` = the same metric
through the C ABI (pb_batch_run: pack + H2D + walk + D2H of the
delta-encoded frontiers, host buffers in and out).  Every instance's results
are digested after the first and the last timed launch and after the e2e run;
any difference fails the run (the minimal min cut is unique, so the output
must not depend on timing).

Multi-GPU: one process per GPU (torchrun).  Instances are independent, so
there is no data-path collective: with --scaling strong (default, the
north_star's split) the one 4096-instance batch is LPT-sharded over the
ranks by estimated work; with --scaling weak rank r walks its own block
[r*B, (r+1)*B) of the config-5 sequence.  Times are device-measured (CUDA
events on the walk kernels' stream) and reduced as the max over ranks.

--impl reference runs the UNMODIFIED reference planner (oracle/_ref/ref_driver,
compiled from /root/reference by `make -C oracle ref`) on the host cores, on
a deterministic sample of the same batch: the 16 stratified instances
i = 0 mod 256, each walked for its first 300 steps (cpu_sample()).  The GPU
arm walks the identical capped sample too and reports both side by side
("same_work"), next to the whole-batch value.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frontier points/sec (min-cut iters/sec) over instance batch at 1/2/4/8 B200 vs CPU"
UNIT = "frontier points/s"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Dist:
    """torch.distributed plumbing (barrier + max-reduce of device times)."""

    def __init__(self, backend="nccl"):
        self.rank, self.world, self.local = dist_env()
        self.pg = None
        if self.world > 1:
            import torch
            import torch.distributed as dist
            ndev = torch.cuda.device_count() if backend == "nccl" else 0
            if backend == "nccl" and self.world > ndev:
                # more ranks than GPUs (a 1-GPU smoke test of the N > 1 path):
                # ranks share devices round-robin and NCCL cannot run two
                # ranks on one device, so the plumbing falls back to gloo
                backend = "gloo"
            if ndev:
                self.local = self.local % ndev
                torch.cuda.set_device(self.local)
            dist.init_process_group(backend=backend)
            self.dist, self.torch = dist, torch
            self.dev = torch.device("cuda", self.local) if backend == "nccl" else torch.device("cpu")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


# ------------------------------------------------------------------ workload

def batch_indices(batch: int, rank: int, world: int, scaling: str):
    """Instances of this rank.  weak: its own block of the config-5 sequence;
    strong: an LPT shard (by estimated work) of instances [0, batch)."""
    if scaling == "weak" or world == 1:
        return list(range(rank * batch, (rank + 1) * batch))
    from paper_2312_06902_b200 import shard
    return shard.lpt_shard([shard.g9_work_estimate(i) for i in range(batch)], world)[rank]


SAMPLE_STRIDE = 256  # stratified sample: instances i = 0 mod 256 of the batch
SAMPLE_STEPS = 300   # each walked for its first 300 steps (tests/golden batch5 prefixes)


def sample_indices(batch: int):
    return list(range(0, batch, SAMPLE_STRIDE))


def build_batch(args, rank, world):
    import paper_2312_06902_b200 as pb
    from paper_2312_06902_b200 import g9
    b = pb.FrontierBatch()
    if args.workload == "batch":
        idx = batch_indices(args.batch, rank, world, args.scaling)
        if idx == list(range(idx[0], idx[0] + len(idx))) if idx else False:
            b.add_g9_batch(idx[0], len(idx))  # contiguous block: built on all host threads
        else:
            b.add_g9_indices(idx)  # LPT shard, built on all host threads
        desc = (f"G9 config-5 batch: {args.batch} heterogeneous 1F1B instances "
                f"{'per GPU' if args.scaling == 'weak' else 'LPT-sharded over the GPUs'} (N 4-16, M 8-256, B=10, "
                f"imbalance 1.0-1.25, straggler phi in 1.0-1.5), full frontiers, tau=1000us")
    else:
        k = int(args.workload[-1])
        reps = max(1, args.reps)
        for _ in range(reps):
            b.add_g9(g9.named_config(k))
        desc = f"G9 config {k} ({g9.named_config(k).stages}x{g9.named_config(k).microbatches} 1F1B) x{reps}"
        idx = list(range(reps))
    return b, desc, idx


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampled DURING the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def loop():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU side

def ref_driver_path():
    return os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def cpu_sample(args, threads: int):
    """The reference planner on the deterministic sample of the batch: the
    instances i = 0 mod 256 (stratified over the mix), each walked from its
    seed with the reference's public API for its first SAMPLE_STEPS steps,
    one instance per host thread (ref_driver capped).  Early steps are the
    cheapest ones (the critical sub-DAG grows along the walk), so this
    overstates the reference's whole-batch throughput."""
    specs = sample_specs(args)
    out = subprocess.run([ref_driver_path(), "capped", str(SAMPLE_STEPS), str(threads), *specs],
                         capture_output=True, text=True, check=True)
    r = json.loads(out.stdout.strip().splitlines()[-1])
    r["sample"] = (f"{len(specs)} instances ({sample_desc(args)}), each walked from T* for its first "
                   f"{SAMPLE_STEPS} steps with the reference API, {threads} threads")
    return r


def sample_specs(args):
    if args.workload == "batch":
        return [f"batch:{i}" for i in sample_indices(args.batch)]
    return [f"config:{args.workload[-1]}"] * 16


def sample_desc(args):
    return ("every 256th of the config-5 batch" if args.workload == "batch"
            else f"16 copies of config {args.workload[-1]}")


# ------------------------------------------------------------------ arms

def run_reference(args):
    """The reference arm: no product code is imported or loaded here."""
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    if not os.path.exists(ref_driver_path()):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/ref_driver not built (needs /root/reference)"}))
        return 0
    threads = min(os.cpu_count() or 1, len(sample_specs(args)))
    for _ in range(args.warmup):
        cpu_sample(args, threads)
    pts = steps = 0
    wall = 0.0
    last = None
    for _ in range(args.steps):
        r = cpu_sample(args, threads)
        pts += r["points"]
        steps += r["steps"]
        wall += r["wall_s"]
        last = r
    value = pts / wall
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (G9 generator, SURVEY.md §8d)",
        "config": {"workload": f"{workload_desc(args)}; sampled: {last['sample']}",
                   "sample": last["sample"]},
        "iterations_per_s": steps / wall,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": last["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def workload_desc(args):
    if args.workload == "batch":
        return f"G9 config-5 batch: {args.batch} heterogeneous 1F1B instances"
    return f"G9 config {args.workload[-1]}"


def load_traffic():
    """dram read+write bytes per launch of the walk kernel from the committed
    ncu --set full capture of the default workload (profiles/), if any."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "walk_traffic.json")))
    except Exception:
        return None


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def digests(b):
    return [b.digest(k) for k in range(len(b))]


def flow_share(prof):
    """Share of the walk spent in the max-flow phases (phase A repair +
    phase B augmentation and the final reachability BFS = §8(d)'s K4), from
    the device cycle counters of the same launch (pb_batch_profile slots:
    2 phase A, 3 phase B, 7 whole walk; summed over walks)."""
    return (prof[2] + prof[3]) / prof[7] if prof[7] else 0.0


def run_sample_gpu(args, device):
    """The CPU arm's exact sample on the GPU: same instances, same step cap,
    one launch, device-timed (a latency measurement: 16 walks on 148 SMs)."""
    import paper_2312_06902_b200 as pb
    b = pb.FrontierBatch()
    if args.workload == "batch":
        b.add_g9_indices(sample_indices(args.batch))
    else:
        from paper_2312_06902_b200 import g9
        for _ in range(16):
            b.add_g9(g9.named_config(int(args.workload[-1])))
    b.set_max_steps(SAMPLE_STEPS)
    b.prepare(device)
    b.launch()
    ms = min(b.launch() for _ in range(3))
    b.fetch()
    pts = sum(b.summary(k).steps + 1 for k in range(len(b)))
    return pts / (ms / 1e3), ms


def run_ours(args):
    import paper_2312_06902_b200 as pb  # noqa: F401  (loads the CUDA library; fails loudly if absent)
    D = Dist("nccl")
    rank, world = D.rank, D.world
    device = D.local if world > 1 else 0
    b, desc, idx = build_batch(args, rank, world)
    b.prepare(device)
    # warm-up (untimed)
    for _ in range(args.warmup):
        b.launch()
    D.barrier()
    launches0 = b.stats().kernel_launches
    kernel_ms = []
    ref_digest = None
    with ClockSampler(device) as clk:
        for step in range(args.steps):
            D.barrier()
            kernel_ms.append(b.launch())  # device time (CUDA events), its stream synchronized on both sides
            D.barrier()
            if step == 0 or step == args.steps - 1:
                b.fetch()  # outside the device-timed region
                d = digests(b)
                if ref_digest is None:
                    ref_digest = d
                elif d != ref_digest:
                    bad = sum(x != y for x, y in zip(d, ref_digest))
                    raise RuntimeError(f"{bad} instances differ between timed launches on rank {rank}")
    st = b.stats()
    prof = b.profile()
    timed_launches = st.kernel_launches - launches0  # walker + cooperative kernels per step
    points = steps = 0
    bad = 0
    for k in range(len(b)):
        s = b.summary(k)
        bad += s.status != 0 or s.n_table_misses != 0
        points += s.steps + 1
        steps += s.steps
    if bad:
        raise RuntimeError(f"{bad} instances failed on rank {rank}")
    t_dev = D.max(sum(kernel_ms) / 1e3)
    total_points = D.sum(points)
    total_steps = D.sum(steps)
    value = total_points * args.steps / t_dev
    # e2e through the C ABI with host buffers: pack + H2D + kernel + D2H
    e2e_times = []
    for _ in range(max(1, args.e2e_steps)):
        D.barrier()
        t0 = time.perf_counter()
        b.run(device)
        _ = [b.summary(k).steps for k in range(len(b))]
        e2e_times.append(time.perf_counter() - t0)
        D.barrier()
    if digests(b) != ref_digest:
        raise RuntimeError(f"e2e results differ from the device-timed launches on rank {rank}")
    st_e2e = b.stats()
    t_e2e = D.max(sum(e2e_times))
    e2e_value = total_points * len(e2e_times) / t_e2e
    # Roofline.  SURVEY §8(d) K4 bytes -- 16 B per arc
    # scan + 24 B per node update -- over the time the launch spends in the
    # max-flow phases (device cycle counters); also the same bytes over the
    # whole launch, and the implementation's own per-unit bytes.
    launch_s = st.kernel_ms / 1e3
    share = flow_share(prof)
    k4_bytes = 16 * st.arc_scans + 24 * st.node_updates
    impl_bytes = 24 * st.arc_scans + 16 * st.node_updates + 48 * st.comp_visits
    peaks = load_peaks()
    peak = peaks.get("hbm_gbs", 6650.0)
    gbs = lambda by, t: by / t / 1e9 if t > 0 else 0.0  # noqa: E731
    achieved = gbs(k4_bytes, launch_s * share)
    traffic = load_traffic()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "int64",
        "data": "synthetic (G9 generator, SURVEY.md §8d)",
        "config": {"workload": desc, "instances_per_rank": len(b), "tau_us": 1000,
                   "l2": "no flush: per-walker workspaces + instance data exceed the 126 MB L2",
                   "parallelism": (f"instances LPT-ordered over {world} GPU(s): " + (
                       f"every walk shared-memory resident, one 1-warp CTA each ({st.smem_region} B region)"
                       if st.smem_walks else
                       f"{st.wide_walks} longest walks on 2-warp cooperative CTAs, one warp per walk for the rest"))},
        "iterations_per_s": total_steps * args.steps / t_dev,
        "points_per_step": int(total_points),  # frontier points of the whole batch, all ranks
        "deterministic": True,  # digests equal after the first / last timed launch and the e2e run
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(st_e2e.h2d_bytes),
                "d2h_bytes_per_step": int(st_e2e.d2h_bytes),
                "breakdown_ms": {"wall": 1e3 * t_e2e / len(e2e_times), "pack": st_e2e.pack_ms,
                                 "h2d": st_e2e.h2d_ms, "kernel": st_e2e.kernel_ms, "d2h": st_e2e.d2h_ms}},
        "gpu_launches": int(timed_launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None,
                     "traffic": traffic.get("bytes_per_launch") if traffic else None,
                     "traffic_source": traffic.get("source") if traffic else None,
                     "model": "SURVEY §8(d) K4: 16 B x arc_scans + 24 B x node_updates over the launch time "
                              "x the max-flow phases' cycle share",
                     "algorithmic_bytes_per_launch": k4_bytes,
                     "flow_phase_share": share,
                     "frac_whole_launch": gbs(k4_bytes, launch_s) / peak if peak else None,
                     "impl_bytes_per_launch": impl_bytes,
                     "impl_frac_whole_launch": gbs(impl_bytes, launch_s) / peak if peak else None,
                     "counters": {"arc_scans": st.arc_scans, "node_updates": st.node_updates,
                                  "comp_visits": st.comp_visits, "bfs_levels": st.rounds},
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)" if "hbm_gbs" in peaks
                     else "fallback 6650 GB/s"},
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu and os.path.exists(ref_driver_path()):
        threads = min(os.cpu_count() or 1, len(sample_specs(args)))
        r = cpu_sample(args, threads)
        cpu_v = r["points"] / r["wall_s"]
        line["cpu_baseline"] = {"value": cpu_v, "unit": UNIT, "cores": r["threads"], "kind": "reference",
                                "sample": r["sample"]}
        gpu_v, gpu_ms = run_sample_gpu(args, device)
        line["same_work"] = {"same_config": True, "sample": r["sample"], "unit": UNIT,
                             "gpu_value": gpu_v, "gpu_ms": gpu_ms, "cpu_value": cpu_v,
                             "cpu_ms": 1e3 * r["wall_s"], "cpu_threads": r["threads"],
                             "gpu_over_cpu": gpu_v / cpu_v if cpu_v else None}
    if rank == 0:
        print(json.dumps(line))
    D.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="batch",
                    choices=["batch", "config1", "config2", "config3", "config4"])
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
