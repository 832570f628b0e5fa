"""Host-side sharding of independent frontier walks over GPUs:
LPT (longest processing time first) by estimated work = edges x steps."""
from __future__ import annotations

import heapq
from typing import List, Sequence


def g9_work_estimate(i: int) -> int:
    """Edge-centric edges x expected steps of config-5 instance i."""
    from . import g9
    p = g9.batch_params(i)
    n, m = p.stages, p.microbatches
    e_ec = 2 * n * m + 4 * n * m - 2 * m + n
    return e_ec * 24 * (n + m - 1)


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
