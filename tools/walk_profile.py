"""Per-phase device profile of the frontier-walk kernel (pb_batch_profile).

  python tools/walk_profile.py config2 [config4 ...] [config1*1776] [batch:N]
"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_06902_b200 as pb  # noqa: E402
from paper_2312_06902_b200 import _native as N, g9  # noqa: E402

NAMES = ["lp", "cap", "phaseA", "phaseB", "bfs", "augment", "update", "walk", "bfs_A", "bfs_B",
         "bfs_levels", "paths", "path_hops", "steps", "imbalanced", "lp_levels"]


def profile(name):
    b = pb.FrontierBatch()
    if name.startswith("config"):
        k, _, reps = name[len("config"):].partition("*")
        for _ in range(int(reps or 1)):
            b.add_g9(g9.named_config(int(k)))
    elif name.startswith("rep:"):  # rep:3284:148 = 148 copies of config-5 instance 3284
        _, i, r = name.split(":")
        for _ in range(int(r)):
            b.add_g9(g9.batch_params(int(i)))
    elif name.startswith("inst:"):  # single config-5 instances: inst:3284[,1580...]
        for i in name.split(":")[1].split(","):
            b.add_g9(g9.batch_params(int(i)))
    elif name.startswith("shard:"):  # shard:R:W = rank R's LPT shard of the 4096 batch over W GPUs
        from paper_2312_06902_b200 import shard
        _, r, w = name.split(":")
        b.add_g9_indices(shard.lpt_shard([shard.g9_work_estimate(i) for i in range(4096)], int(w))[int(r)])
    elif name.startswith("batch:"):
        for i in range(int(name.split(":")[1])):
            b.add_g9(g9.batch_params(i))
    if os.environ.get("PB_PROFILE_MAX_STEPS"):  # step-capped walks (short ncu captures)
        b.set_max_steps(int(os.environ["PB_PROFILE_MAX_STEPS"]))
    t = time.time()
    b.prepare(0)
    ms = b.launch()
    b.fetch()
    prof = np.zeros(16, np.int64)
    N.check(N.lib.pb_batch_profile(b._h, N.ptr(prof, C.c_int64), 16))
    st = b.stats()
    steps = sum(b.summary(k).steps for k in range(len(b)))
    bad = [(k, b.summary(k).status, b.summary(k).n_table_misses, b.summary(k).steps) for k in range(len(b)) if b.summary(k).status]
    walk = max(prof[7], 1)
    print(f"== {name}: kernel {ms:.1f} ms, {steps} steps, {ms * 1e3 / max(steps, 1):.1f} us/step, wall {time.time() - t:.1f}s")
    print("   cycles share: " + ", ".join(f"{NAMES[i]} {prof[i] / walk:.1%}" for i in range(7)))
    S = max(prof[13], 1)
    print("   per step: " + ", ".join(f"{NAMES[i]} {prof[i] / S:.2f}" for i in range(8, 16)))
    print(f"   cycles/step {prof[7] / S:.0f}, cycles per bfs level {prof[4] / max(prof[10], 1):.0f}")
    print(f"   arc_scans/step {st.arc_scans / S:.0f}, node_updates/step {st.node_updates / S:.0f}; "
          f"smem walks {st.smem_walks} (region {st.smem_region} B), cooperative walks {st.wide_walks}")
    walks = sorted(((b.summary(k).walk_us, k) for k in range(len(b))), reverse=True)
    t0 = min(b.summary(k).start_us for k in range(len(b)))
    if len(walks) > 1:
        import heapq
        slots = [0.0] * min(len(walks), int(os.environ.get("PB_SLOTS", "1776")))
        heapq.heapify(slots)
        for us, _ in walks:  # LPT order approximates the device's queue order
            t = heapq.heappop(slots)
            heapq.heappush(slots, t + us)
        print(f"   walks: longest {walks[0][0] / 1e3:.1f} ms, median {walks[len(walks) // 2][0] / 1e3:.2f} ms, "
              f"sum {sum(w for w, _ in walks) / 1e6:.1f} s; LPT replay makespan {max(slots) / 1e3:.1f} ms")
        ends = sorted(((b.summary(k).start_us - t0 + b.summary(k).walk_us, k) for k in range(len(b))), reverse=True)
        print("   last to finish (end ms, start ms, walk ms, index, steps, warps): " + ", ".join(
            f"{e / 1e3:.0f}/{(b.summary(k).start_us - t0) / 1e3:.0f}/{b.summary(k).walk_us / 1e3:.0f}/{k}/"
            f"{b.summary(k).steps}/{b.summary(k).warps}" for e, k in ends[:8]))
        print("   top walks (ms, index, steps): " + ", ".join(
            f"{us / 1e3:.0f}/{k}/{b.summary(k).steps}" for us, k in walks[:8]))
    if os.environ.get("PB_PROFILE_DUMP"):  # per-walk table for work-model fits
        import json as _j
        with open(os.environ["PB_PROFILE_DUMP"], "w") as f:
            for k in range(len(b)):
                sm = b.summary(k)
                pp = None
                if name.startswith("batch:"):
                    q = g9.batch_params(k)
                    pp = [q.stages, q.microbatches]
                f.write(_j.dumps({"k": k, "steps": sm.steps, "walk_us": sm.walk_us, "start_us": sm.start_us - t0,
                                  "warps": sm.warps, "n": b._packed[k].n, "shape": pp}) + "\n")
    if bad:
        print("   FAILED (index, status, detail, steps):", bad[:10])


for name in sys.argv[1:]:
    profile(name)
