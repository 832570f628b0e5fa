"""Regenerates the golden fixtures in tests/golden/ by running the UNMODIFIED
reference (oracle/_ref/ref_driver, built from /root/reference by
`make -C oracle ref`).  Run in the build container:

    python tests/golden/make_golden.py

Fixtures (JSON lines, gzip):
  walks.jsonl.gz      frontier walks: the reference's own golden instances
                      (diamond, lone, clip, ten-tau), G9 configs 1-2, random
                      grid-profile walks (testutil::grid_profiles) and random
                      cubic-profile walks (infeasible / infinite-cut stops)
  flow424242.jsonl.gz acceptance gate 3 corpus: 1000 random bounded graphs,
                      seed 424242, <= 12 nodes (acceptance.cpp:137-157)
  flow7302.jsonl.gz   test_flow.cpp:90-114 corpus: 600 graphs, seed 7302
  slack7102.jsonl.gz  annotate_slack on random DAGs (test_dag.cpp:244-263 style)
  savings.jsonl.gz    straggler_savings rows (baselines.hpp:162-188) on the
                      reference frontier, 8 pipelines, the config-4 factor sweep

  artifacts.jsonl.gz  frontier.csv + schedule_<k>.json bytes (serde.hpp:194-257)
  brute.jsonl.gz      brute_force_frontier exact frontiers (oracle.hpp:47-114)
  getnext.jsonl.gz    get_next_schedule from caller schedules outside the
                      curve intervals (tables widened around the start)
  batch5.jsonl.gz     config-5 batch instances: the largest 16x256 walks and
                      mid-size walks in full, 300-step prefixes of the 16
                      stratified samples ("batch5", opt-in: ~2 h on 6 cores;
                      BATCH5_FROM=dir collects the outputs of earlier runs)
  walks_large.jsonl.gz  full-size reference walks of G9 configs 3 (8x128) and
                      4 (16x128) -- ~30 min of reference CPU time ("large")
  walks_phi.jsonl.gz  the config-4 straggler sweep (16x128, stage 8 slowed by
                      phi in 1.05, 1.1, 1.2, 1.3, 1.5), full walks, instance
                      dumps stripped (rebuilt by the native G9 builder) --
                      ~15 min on 5 cores ("phi", opt-in)
  savings_c4.jsonl.gz straggler_savings rows of configs 4 and 3 at the sweep
                      factors (baselines.hpp:162-188) ("phi")

    python tests/golden/make_golden.py [walks|flow|slack|savings|artifacts ...]
  batch_small.jsonl.gz  small config-5 style G9 instances (summaries only)
"""
import gzip
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "ref_driver")


def run(*args):
    out = subprocess.run([DRIVER, *args], check=True, capture_output=True, text=True)
    return [line for line in out.stdout.splitlines() if line.strip()]


def write(name, lines):
    path = os.path.join(HERE, name)
    with gzip.open(path, "wt") as f:
        for line in lines:
            f.write(line + "\n")
    print(f"{name}: {len(lines)} records, {os.path.getsize(path)} bytes")


SAVINGS_FACTORS = "1.0,1.05,1.1,1.2,1.3,1.5"  # SURVEY §8d config-4 straggler sweep
PHI_SWEEP = ["1.05", "1.1", "1.2", "1.3", "1.5"]


def main():
    if not os.path.exists(DRIVER):
        sys.exit("build the reference driver first: make -C oracle ref")
    parts = set(sys.argv[1:]) or {"walks", "flow", "slack", "savings", "artifacts", "brute"}  # "large": opt-in
    walk_specs = ["diamond", "lone:1000:9000:3000:5000", "lone:1000:9000:3000:5000:800",
                  "lone:1000:5000:11000:800", "config:1", "config:2"]
    walk_specs += [f"grid:{s}:{1 + s % 3}:{1 + s % 4}" for s in range(1, 41)]
    walk_specs += [f"grid:{s}:{2 + s % 3}:{2 + s % 5}:4" for s in range(100, 120)]
    walk_specs += [f"cubic:{s}:{1 + s % 4}:{1 + s % 6}" for s in range(1, 41)]
    walk_specs += [f"g9:{2 + s % 5}:{2 + s % 7}:{8 + s % 4}:1.2:{s}:{s % 3 - 1}:1.5" for s in range(1, 21)]
    if "walks" in parts:
        write("walks.jsonl.gz", run("walkcheck", *walk_specs))
    if "flow" in parts:
        write("flow424242.jsonl.gz", run("flow", "424242", "1000", "12", "30"))
        write("flow7302.jsonl.gz", run("flow", "7302", "600", "8", "30"))
    if "slack" in parts:
        write("slack7102.jsonl.gz", run("slack", "7102", "200"))
    if "savings" in parts:
        sav = [w for w in walk_specs if not w.startswith("cubic")]  # cubic walks stop early (infeasible)
        sav += [f"g9:4:{8 + s}:10:1.1:{s}:{s % 4}:{[1.0, 1.1, 1.3, 1.5][s % 4]}" for s in range(6)]
        write("savings.jsonl.gz", run("savings", "8", SAVINGS_FACTORS, *sav))
    if "artifacts" in parts:
        art = ["diamond", "lone:1000:9000:3000:5000", "config:1", "grid:3:1:4", "grid:101:4:3:4", "g9:3:5:9:1.2:7:1:1.5"]
        write("artifacts.jsonl.gz", run("artifacts", "1", *art) + run("artifacts", "10", "config:1", "diamond"))
    if "large" in parts:
        write("walks_large.jsonl.gz", run("walkcheck", "config:3") + run("walkcheck", "config:4"))
    if "phi" in parts:  # opt-in: ~15 min on 6 cores
        procs = [subprocess.Popen([DRIVER, "walk", f"config:4:{p}"], stdout=subprocess.PIPE, text=True)
                 for p in PHI_SWEEP]
        sav = subprocess.Popen([DRIVER, "savings", "8", SAVINGS_FACTORS, "config:4", "config:3"],
                               stdout=subprocess.PIPE, text=True)
        lines = []
        for p in procs:
            out, _ = p.communicate()
            lines += [strip_instance(x) for x in out.splitlines() if x.strip()]
        write("walks_phi.jsonl.gz", lines)
        write("savings_c4.jsonl.gz", [x for x in sav.communicate()[0].splitlines() if x.strip()])
    if "batch5" in parts:  # opt-in: hours of reference CPU time
        batch5(os.environ.get("BATCH5_FROM"))
    if "getnext" in parts:
        write("getnext.jsonl.gz", run("getnext", "1000", *getnext_cases(walk_specs)))
    if "brute" in parts:
        small = [w for w in walk_specs if w.startswith(("grid:", "diamond", "lone", "cubic:"))][:60]
        write("brute.jsonl.gz", run("brute", *small, "config:1"))


# Config-5 goldens (the headline batch): the two largest
# 16x256 walks in full (~1.5-2 h of reference CPU each), three mid-size walks
# in full, the first 300 steps of the 16 stratified sample instances.
BATCH5_FULL = ["batch:3284", "batch:2404", "batch:2641", "batch:150", "batch:3496"]
BATCH5_PREFIX = [f"batch:{i}" for i in range(0, 4096, 256)]


def strip_instance(line):
    """The batch instances are rebuilt natively (pb_batch_add_g9_batch, whose
    generator test_g9_generator_matches_reference_instances pins): drop the
    instance dump and curves to keep the fixture small."""
    w = json.loads(line)
    w.pop("instance", None)
    w.pop("curves", None)
    w.pop("wall_s", None)
    return json.dumps(w, separators=(",", ":"))


def batch5(from_dir=None):
    """Runs the reference on every config-5 golden in parallel (or collects
    outputs of earlier runs, one JSON line per walk, from from_dir/*.jsonl)."""
    lines = []
    if from_dir:
        import glob
        for path in sorted(glob.glob(os.path.join(from_dir, "*.jsonl"))):
            lines += [strip_instance(x) for x in open(path) if x.startswith('{"spec":"batch:')]
    else:
        procs = [subprocess.Popen([DRIVER, "walk", s], stdout=subprocess.PIPE, text=True) for s in BATCH5_FULL]
        procs.append(subprocess.Popen([DRIVER, "walkprefix", "300", *BATCH5_PREFIX], stdout=subprocess.PIPE, text=True))
        for p in procs:
            out, _ = p.communicate()
            lines += [strip_instance(x) for x in out.splitlines() if x.strip()]
    order = {s: i for i, s in enumerate(BATCH5_FULL + BATCH5_PREFIX)}
    lines.sort(key=lambda x: order.get(json.loads(x)["spec"], 99))
    write("batch5.jsonl.gz", lines)


def getnext_cases(walk_specs):
    """get_next_schedule from caller schedules whose planned times lie
    anywhere in [t_min - 3 tau, t_max + 3 tau] (also off the tau grid): the
    curve is evaluated outside its fitted interval (costmodel.hpp:47)."""
    import random
    rng = random.Random(2312)
    specs = ["diamond", "lone:1000:9000:3000:5000", "config:1"]
    specs += [w for w in walk_specs if w.startswith(("grid:", "cubic:", "g9:"))][::3]
    with gzip.open(os.path.join(HERE, "walks.jsonl.gz"), "rt") as f:
        walks = {w["spec"]: w for w in map(json.loads, f)}
    args = []
    for spec in specs:
        w = walks[spec]
        cls = {(c["stage"], c["kind"]): c for c in w["curves"]}
        comps = w["instance"]["comps"]
        rng_lo_hi = []
        for stage, kind, _ in comps:
            c = cls[(stage, kind)]
            rng_lo_hi.append((c["pareto"][0][1],) * 2 if c["constant"] else (c["t_min"], c["t_max"]))
        for rep in range(6):
            # rep 0-1: every computation shifted above t_max; rep 2-5: the
            # seed (t_max) with a few computations moved below t_min or
            # above t_max; odd reps off the tau grid
            if rep < 2:
                k = rng.randint(1, 3)
                start = [hi + k * 1000 for lo, hi in rng_lo_hi]
            else:
                start = [hi for lo, hi in rng_lo_hi]
                for i in rng.sample(range(len(comps)), min(len(comps), rng.randint(1, 3))):
                    lo, hi = rng_lo_hi[i]
                    start[i] = lo - rng.randint(1, 3) * 1000 if rng.random() < 0.6 else hi + rng.randint(1, 3) * 1000
            if rep % 2:
                start = [t + rng.randint(-400, 400) for t in start]
            args += [spec, ",".join(str(max(1, t)) for t in start)]
    return args


if __name__ == "__main__":
    main()
