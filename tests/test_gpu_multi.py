"""The N > 1 bench path with real walks: bench.py under torchrun with 2
ranks (on one GPU both ranks share the device and the plumbing falls back to
gloo -- NCCL needs one device per rank).  Strong scaling LPT-shards one batch,
so the 2-rank run must walk exactly the points of the 1-rank run; every
rank's results are digest-checked inside bench.py."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _bench(nproc, *args):
    base = [sys.executable, "bench.py", "--steps", "1", "--warmup", "1", "--no-cpu", *args]
    if nproc > 1:
        base = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
                "--master-addr", "127.0.0.1", "--master-port", str(_port()), *base[1:], "--gpus", str(nproc)]
    out = subprocess.run(base, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return lines[0]


@pytest.mark.parametrize("scaling", ["strong", "weak"])
def test_two_rank_bench_walks_the_sharded_batch(scaling):
    one = _bench(1, "--batch", "96")
    two = _bench(2, "--batch", "96", "--scaling", scaling)
    assert two["n_gpus"] == 2 and two["scaling"] == scaling
    assert two["deterministic"] is True and two["value"] > 0 and two["e2e"]["value"] > 0
    if scaling == "strong":  # one batch split over the ranks: the same points
        assert two["points_per_step"] == one["points_per_step"]
    else:  # each rank its own block of the config-5 sequence: more points
        assert two["points_per_step"] > one["points_per_step"]
