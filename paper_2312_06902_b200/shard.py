"""Host-side sharding of independent frontier walks over GPUs:
LPT (longest processing time first) by estimated walk time -- the same model
as the native scheduler (pb_host.cpp walk_work): steps x per-step time, the
per-step time growing with the DAG's width and edge count."""
from __future__ import annotations

import heapq
from typing import List, Sequence


def g9_work_estimate(i: int) -> int:
    """Estimated walk time of config-5 instance i (SURVEY.md §8a shapes: a 1F1B
    N x M DAG has n = 2NM computations on 2(N + M - 1) levels, E = 6NM - 2M +
    N + 1 edge-centric edges incl. the return arc, 24(N + M - 1) steps)."""
    from . import g9
    p = g9.batch_params(i)
    n_st, m = p.stages, p.microbatches
    n = 2 * n_st * m
    levels = 2 * (n_st + m - 1)
    e_ec = 6 * n_st * m - 2 * m + n_st + 1
    per_step = max(10.0, 79.0 * n / levels + 0.0223 * e_ec - 226.0)
    return int(per_step * 1000.0) * 24 * (n_st + m - 1)


def lpt_shard(works: Sequence[int], parts: int) -> List[List[int]]:
    """Greedy LPT: heaviest item to the least-loaded part; deterministic ties."""
    heap = [(0, p) for p in range(parts)]
    out: List[List[int]] = [[] for _ in range(parts)]
    for i in sorted(range(len(works)), key=lambda k: (-works[k], k)):
        load, p = heapq.heappop(heap)
        out[p].append(i)
        heapq.heappush(heap, (load + works[i], p))
    for p in out:
        p.sort()
    return out
