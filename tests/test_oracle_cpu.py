"""Pins the CPU oracle (oracle/perseus_oracle.c) before it is trusted as the
checker: against the reference's own golden vectors (test_frontier.cpp,
test_flow.cpp) and against fixtures produced by the unmodified reference
(tests/golden/, oracle/_ref/ref_driver)."""
import struct

import pytest

from fixtures import instance_from_golden
from oracle import port
from paper_2312_06902_b200.model import PackedInstance


def oracle_walk(w):
    dag, model, tau = instance_from_golden(w)
    return port.discover_frontier(PackedInstance(dag, model, tau), tau)


FIELDS = ["t_min", "t_star", "steps", "reason", "t_planned", "t_realized", "eff_planned", "eff_realized",
          "sum_planned_e", "sum_realized_e", "hash", "cut_cost", "step_size", "sped", "slowed"]


# ---- test_frontier.cpp golden integers -------------------------------------

def test_diamond_walk_matches_test_frontier_cpp(walks):
    r = oracle_walk(walks["diamond"])
    # test_frontier.cpp:188-193
    assert r["cut_cost"] == [300, 375, 1875, 3900]
    assert r["sped"] == [[1, 3, 4], [1, 3, 4], [0, 2], [0, 2]]
    assert r["slowed"] == [[], [], [1], [1]]
    # test_frontier.cpp:217-242
    assert r["steps"] == 4 and r["t_star"] == 9000 and r["t_min"] == 5000
    assert r["t_planned"] == [9000, 8000, 7000, 6000, 5000]
    assert r["t_realized"] == [9000, 7000, 7000, 5000, 5000]
    assert r["sum_planned_e"] == [3200, 3500, 3875, 5750, 9650]
    assert r["eff_planned"] == pytest.approx([1625, 2150, 2750, 4700, 8675])


def test_lone_steps_match_test_frontier_cpp(walks):
    r = oracle_walk(walks["lone:1000:9000:3000:5000"])
    # test_frontier.cpp:120-144: e(2000) = sqrt(9000 * 5000) -> 6708; cuts 1708, 2292
    assert r["t_planned"] == [3000, 2000, 1000]
    assert r["sum_planned_e"] == [5000, 6708, 9000]
    assert r["cut_cost"] == [1708, 2292]
    assert r["sped"] == [[0], [0]]


def test_clip_and_ten_tau(walks):
    r = oracle_walk(walks["lone:1000:9000:3000:5000:800"])
    assert r["t_planned"] == [3000, 2200, 1400, 1000]  # test_frontier.cpp:154-164
    r = oracle_walk(walks["lone:1000:5000:11000:800"])
    assert r["steps"] == 10  # test_frontier.cpp:166-173
    assert all(a - b == 1000 for a, b in zip(r["t_planned"], r["t_planned"][1:]))


# ---- every reference-produced walk fixture ----------------------------------

def test_oracle_reproduces_every_reference_walk(walks):
    for spec, w in walks.items():
        if spec == "config:2":
            continue  # covered (slowly) below
        r = oracle_walk(w)
        for f in FIELDS:
            assert r[f] == w[f], (spec, f)


def test_oracle_reproduces_config2_walk(walks):
    w = walks["config:2"]
    r = oracle_walk(w)
    for f in FIELDS:
        assert r[f] == w[f], f


def test_fixtures_cover_all_terminations(walks):
    reasons = {w["reason"] for w in walks.values()}
    assert {"at_t_min", "infeasible", "infinite_cut"} <= reasons


def test_g9_step_count_formula(walks):
    # G9 walks take 24 (N + M - 1) steps
    assert walks["config:1"]["steps"] == 24 * (4 + 8 - 1)
    assert walks["config:2"]["steps"] == 24 * (8 + 32 - 1)


# ---- cost model ------------------------------------------------------------

def test_oracle_fit_matches_reference_curve_bits(walks):
    for w in walks.values():
        for c in w["curves"]:
            if c["constant"]:
                continue
            times = [p[1] for p in c["pareto"]]
            energies = [p[2] for p in c["pareto"]]
            rc, abc = port.fit_exp(times, energies)
            assert rc == 0
            bits = [struct.pack(">d", x).hex() for x in abc]
            assert bits == c["curve_bits"]


# ---- flow -------------------------------------------------------------------

def test_oracle_flow_corpus(flow_corpus):
    feasible = infeasible = 0
    for rec in flow_corpus:
        g = rec["graph"]
        r = port.flow_min_cut(g["nodes"], g["source"], g["sink"], g["edges"])
        assert r["rc"] == 0
        assert r["feasible"] == rec["feasible"]
        if not rec["feasible"]:
            infeasible += 1
            continue
        feasible += 1
        assert r["value"] == rec["value"]
        assert r["cost"] == rec["cost"]
        assert r["source_side"] == rec["source_side"]
        assert r["speed_up"] == rec["speed_up"]
        assert r["slow_down"] == rec["slow_down"]
    assert feasible > 50 and infeasible > 50


def test_oracle_flow_named_cases():
    # test_flow.cpp:179-193
    r = port.flow_min_cut(4, 0, 3, [(0, 1, 0, 9, 0), (0, 2, 0, 9, 0), (1, 3, 0, 2, 0), (2, 3, 0, 3, 0)])
    assert r["value"] == 5 and r["speed_up"] == [2, 3] and r["slow_down"] == [] and r["cost"] == 5
    # test_flow.cpp:195-213
    r = port.flow_min_cut(4, 0, 3, [(0, 1, 0, 20, 0), (1, 3, 0, 3, 0), (2, 1, 5, 5, 0), (0, 2, 0, 4, 0),
                                    (2, 3, 0, 20, 0), (1, 2, 0, 20, 0)])
    assert r["value"] == 22 and r["slow_down"] == [2] and r["speed_up"] == [1, 3, 5] and r["cost"] == 22
    # test_flow.cpp:45-53
    r = port.flow_min_cut(4, 0, 3, [(0, 1, 0, 1, 0), (1, 3, 2, 5, 0), (0, 2, 0, 4, 0), (2, 3, 0, 4, 0)])
    assert not r["feasible"]
    # test_flow.cpp:25-32
    r = port.flow_min_cut(4, 0, 3, [(0, 1, 2, 10, 0), (1, 3, 0, 7, 0), (0, 2, 3, 0, 1), (2, 3, 1, 4, 0)])
    assert r["sentinel"] == 2 + 10 + 7 + 3 + 1 + 4 + 1


def test_oracle_slack_corpus(slack_corpus):
    for rec in slack_corpus:
        rc, ea, la, cr, ms = port.annotate_slack(rec["n"], rec["edges"], rec["durations"])
        assert rc == 0
        assert ms == rec["makespan"]
        assert ea.tolist() == rec["earliest"]
        assert la.tolist() == rec["latest"]
        assert cr.tolist() == rec["critical"]


def test_oracle_lookup_matches_test_frontier_cpp():
    # test_frontier.cpp:250-265 on the diamond grid 9000..5000
    tp = [9000, 8000, 7000, 6000, 5000]
    import numpy as np
    arr = np.array(tp, np.int64)
    L = port.lib()
    look = lambda t: L.or_lookup(5, arr.ctypes.data_as(port.i64p), 9000, t)  # noqa: E731
    assert [look(t) for t in (9000, 250000, 8999, 7500, 7000, 5000, 4999, 0)] == [0, 0, 1, 2, 2, 4, 4, 4]
