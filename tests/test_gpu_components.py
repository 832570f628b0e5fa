"""GPU parity of the component kernels behind the walk: the BFS-augmentation
min cut with lower bounds on arbitrary FlowGraphs (max_flow_lower_bounds +
min_cut_from_flow, flow.hpp:167-278) and the level-synchronous slack pass
(annotate_slack, dag.hpp:233-286), against reference-produced corpora."""
import ctypes as C

import numpy as np
import pytest

from paper_2312_06902_b200 import _native as N

pytestmark = pytest.mark.gpu


def run_flow(graphs):
    cnt = len(graphs)
    nodes = np.array([g["nodes"] for g in graphs], np.int32)
    src = np.array([g["source"] for g in graphs], np.int32)
    snk = np.array([g["sink"] for g in graphs], np.int32)
    m = np.array([len(g["edges"]) for g in graphs], np.int32)
    E = [e for g in graphs for e in g["edges"]]
    arr = np.array(E, np.int64).reshape(-1, 5) if E else np.zeros((0, 5), np.int64)
    tl = np.ascontiguousarray(arr[:, 0].astype(np.int32))
    hd = np.ascontiguousarray(arr[:, 1].astype(np.int32))
    lo = np.ascontiguousarray(arr[:, 2])
    up = np.ascontiguousarray(arr[:, 3])
    inf = np.ascontiguousarray(arr[:, 4].astype(np.uint8))
    st = np.zeros(cnt, np.int32)
    fe = np.zeros(cnt, np.uint8)
    val, sen, cost = (np.zeros(cnt, np.int64) for _ in range(3))
    side = np.zeros(int(nodes.sum()), np.uint8)
    cd = np.zeros(max(len(E), 1), np.int8)
    N.check(N.lib.pb_flow_min_cut_batch(0, cnt, N.ptr(nodes, C.c_int32), N.ptr(src, C.c_int32),
                                        N.ptr(snk, C.c_int32), N.ptr(m, C.c_int32), N.ptr(tl, C.c_int32),
                                        N.ptr(hd, C.c_int32), N.ptr(lo, C.c_int64), N.ptr(up, C.c_int64),
                                        N.ptr(inf, C.c_uint8), N.ptr(st, C.c_int32), N.ptr(fe, C.c_uint8),
                                        N.ptr(val, C.c_int64), N.ptr(sen, C.c_int64), N.ptr(cost, C.c_int64),
                                        N.ptr(side, C.c_uint8), N.ptr(cd, C.c_int8)))
    out = []
    no = eo = 0
    for g in range(cnt):
        dirs = cd[eo:eo + m[g]].tolist()
        out.append({"status": int(st[g]), "feasible": bool(fe[g]), "value": int(val[g]),
                    "sentinel": int(sen[g]), "cost": int(cost[g]),
                    "source_side": side[no:no + nodes[g]].tolist(),
                    "speed_up": [i for i, d in enumerate(dirs) if d == 1],
                    "slow_down": [i for i, d in enumerate(dirs) if d == -1]})
        no += nodes[g]
        eo += m[g]
    return out


def test_flow_corpus_matches_reference(flow_corpus):
    """Acceptance gate 3 (1000 graphs, seed 424242) + test_flow.cpp 7302 corpus."""
    res = run_flow([r["graph"] for r in flow_corpus])
    feasible = 0
    for rec, r in zip(flow_corpus, res):
        assert r["status"] == 0
        assert r["feasible"] == rec["feasible"], rec["graph"]
        if not rec["feasible"]:
            continue
        feasible += 1
        assert r["value"] == rec["value"], rec["graph"]
        assert r["sentinel"] == rec["sentinel"]
        assert r["source_side"] == rec["source_side"], rec["graph"]
        assert r["speed_up"] == rec["speed_up"] and r["slow_down"] == rec["slow_down"]
        assert r["cost"] == rec["cost"] == rec["value"]
    assert feasible > 500


def test_flow_named_cases():
    g = lambda n, s, t, e: {"nodes": n, "source": s, "sink": t, "edges": e}  # noqa: E731
    res = run_flow([
        g(4, 0, 3, [(0, 1, 0, 9, 0), (0, 2, 0, 9, 0), (1, 3, 0, 2, 0), (2, 3, 0, 3, 0)]),
        g(4, 0, 3, [(0, 1, 0, 20, 0), (1, 3, 0, 3, 0), (2, 1, 5, 5, 0), (0, 2, 0, 4, 0), (2, 3, 0, 20, 0),
                    (1, 2, 0, 20, 0)]),
        g(4, 0, 3, [(0, 1, 0, 1, 0), (1, 3, 2, 5, 0), (0, 2, 0, 4, 0), (2, 3, 0, 4, 0)]),
        g(2, 0, 1, [(0, 1, 1, 3, 0)]),
        g(4, 0, 3, [(0, 1, 1, 1, 0), (1, 2, 1, 3, 0), (2, 3, 0, 5, 0), (0, 2, 0, 2, 0)]),
        g(3, 0, 2, []),
    ])
    assert res[0]["value"] == 5 and res[0]["speed_up"] == [2, 3] and res[0]["cost"] == 5  # test_flow.cpp:179-193
    assert res[1]["value"] == 22 and res[1]["slow_down"] == [2] and res[1]["speed_up"] == [1, 3, 5]
    assert not res[2]["feasible"]  # test_flow.cpp:45-53
    assert res[3]["value"] == 3  # test_flow.cpp:36-43
    assert res[4]["value"] == 3  # test_flow.cpp:55-66
    assert res[5]["feasible"] and res[5]["value"] == 0


def test_flow_overflow_checks():
    big = (2**63 - 1) // 4
    res = run_flow([{"nodes": 2, "source": 0, "sink": 1, "edges": [(0, 1, 0, big, 0)]},
                    {"nodes": 3, "source": 0, "sink": 2, "edges": [(0, 1, 0, 2**60, 0), (1, 2, 0, 0, 1),
                                                                  (0, 2, 0, 0, 1), (0, 1, 0, 0, 1)]}])
    assert res[0]["status"] == N.PB_ERR_OVERFLOW  # flow.hpp:65-66
    assert res[1]["status"] == N.PB_ERR_OVERFLOW  # flow.hpp:196-197


def test_slack_corpus_matches_reference(slack_corpus):
    cnt = len(slack_corpus)
    n = np.array([r["n"] for r in slack_corpus], np.int32)
    ne = np.array([len(r["edges"]) for r in slack_corpus], np.int32)
    E = np.array([e for r in slack_corpus for e in r["edges"]], np.int32).reshape(-1, 2)
    tl, hd = np.ascontiguousarray(E[:, 0]), np.ascontiguousarray(E[:, 1])
    dur = np.array([d for r in slack_corpus for d in r["durations"]], np.int64)
    V = int((2 * n + 2).sum())
    ea, la = np.zeros(V, np.int64), np.zeros(V, np.int64)
    cr = np.zeros(int((n + ne).sum()), np.uint8)
    ms = np.zeros(cnt, np.int64)
    N.check(N.lib.pb_annotate_slack_batch(0, cnt, N.ptr(n, C.c_int32), N.ptr(ne, C.c_int32),
                                          N.ptr(tl, C.c_int32), N.ptr(hd, C.c_int32), N.ptr(dur, C.c_int64),
                                          N.ptr(ea, C.c_int64), N.ptr(la, C.c_int64), N.ptr(cr, C.c_uint8),
                                          N.ptr(ms, C.c_int64)))
    vo = eo = 0
    for g, r in enumerate(slack_corpus):
        v = 2 * r["n"] + 2
        m = r["n"] + len(r["edges"])
        assert ms[g] == r["makespan"]
        assert ea[vo:vo + v].tolist() == r["earliest"]
        assert la[vo:vo + v].tolist() == r["latest"]
        assert cr[eo:eo + m].tolist() == r["critical"]
        vo += v
        eo += m
