"""N > 1 host path on CPU: the bench's per-rank sharding (weak: disjoint
blocks of the config-5 sequence; strong: LPT shards of one batch) and its
torch.distributed plumbing (barrier, max / sum of per-rank figures) under
world_size 2 with the gloo backend -- the same code bench.py runs over NCCL,
one process per GPU.  Instances are independent, so there is no data-path
collective to test."""
import os
import socket

import pytest
import torch.multiprocessing as mp

import bench
from paper_2312_06902_b200 import shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, scaling, batch, out):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import paper_2312_06902_b200 as pb
    from paper_2312_06902_b200 import g9
    D = bench.Dist("gloo")
    idx = bench.batch_indices(batch, rank, world, scaling)
    b = pb.FrontierBatch()  # host-side packing only: no device needed
    for i in idx:
        b.add_g9(g9.batch_params(i))
    work = float(sum(shard.g9_work_estimate(i) for i in idx))
    D.barrier()
    out[rank] = (idx, len(b), D.sum(float(len(idx))), D.max(work), D.sum(work))
    D.close()


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_two_rank_sharding_over_gloo(scaling):
    world, batch = 2, 12
    out = mp.Manager().dict()
    mp.spawn(_rank_main, args=(world, _free_port(), scaling, batch, out), nprocs=world, join=True)
    idx0, idx1 = out[0][0], out[1][0]
    assert out[0][1] == len(idx0) and out[1][1] == len(idx1)
    assert not set(idx0) & set(idx1)
    if scaling == "weak":
        assert idx0 == list(range(batch)) and idx1 == list(range(batch, 2 * batch))
    else:
        assert sorted(idx0 + idx1) == list(range(batch))
    # collectives agree on every rank
    for k in (2, 3, 4):
        assert out[0][k] == out[1][k]
    assert out[0][2] == len(idx0) + len(idx1)
    w = [sum(shard.g9_work_estimate(i) for i in ix) for ix in (idx0, idx1)]
    assert out[0][3] == max(w) and out[0][4] == sum(w)


def test_lpt_shard_is_a_balanced_partition():
    works = [shard.g9_work_estimate(i) for i in range(64)]
    for parts in (1, 2, 4, 8):
        sh = shard.lpt_shard(works, parts)
        assert sorted(i for p in sh for i in p) == list(range(64))
        loads = [sum(works[i] for i in p) for p in sh]
        # Graham's LPT bound: makespan <= (4/3 - 1/(3m)) OPT <= (4/3) * max(avg, max item)
        assert max(loads) <= (4 / 3) * max(sum(works) / parts, max(works)) + 1
