"""Host/device breakdown of single-instance calls (the drop-in's
get_next_schedule / discover_frontier path): add (validate + derive), run
(pack + H2D + kernel + D2H), schedule expansion.

  python tools/call_profile.py [config1 config2 ...] [--calls 50]
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2312_06902_b200 as pb  # noqa: E402
from paper_2312_06902_b200 import g9  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["config1", "config2"])
    ap.add_argument("--calls", type=int, default=50)
    args = ap.parse_args()
    for case in args.cases:
        p = g9.named_config(int(case[-1]))
        dag, model = g9.instance(p)
        seed = pb.min_energy_schedule(dag, model)
        b = pb.FrontierBatch()
        rows = []
        planned = list(seed.planned_t)
        for call in range(args.calls + 3):
            t0 = time.perf_counter()
            b.clear()
            b.add(dag, model, g9.TAU, start_planned_t=planned, max_steps=1)
            t1 = time.perf_counter()
            b.run(0)
            t2 = time.perf_counter()
            nxt = b.schedule(0, 1)
            t3 = time.perf_counter()
            st = b.stats()
            rows.append((t1 - t0, t2 - t1, t3 - t2, st.h2d_ms / 1e3, st.kernel_ms / 1e3, st.d2h_ms / 1e3))
            planned = nxt.planned_t
        r = np.array(rows[3:]) * 1e3
        med = np.median(r, axis=0)
        print(f"{case}: median per call (ms): add {med[0]:.3f}, run {med[1]:.3f} "
              f"(h2d {med[3]:.3f}, kernel {med[4]:.3f}, d2h {med[5]:.3f}, host rest "
              f"{med[1] - med[3] - med[4] - med[5]:.3f}), schedule {med[2]:.3f}, mode smem={st.smem_walks}")


if __name__ == "__main__":
    main()
