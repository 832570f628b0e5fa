"""GPU parity: the sm_100a frontier walk (through the C ABI) against the
reference's outputs (golden fixtures from the unmodified reference) and the
CPU oracle.  Bit-exact for every integer field; energies within 1e-9
relative (north_star) -- and bit-exact when materialized through
pb_batch_schedule, which sums in reference order."""
import numpy as np
import pytest

import paper_2312_06902_b200 as pb
from paper_2312_06902_b200 import _native as N, g9
from paper_2312_06902_b200.model import (ClassKey, Computation, CostModel, FrequencyProfile, Kind,
                                         PackedInstance, ProfilePoint, ProfileSet, finalize_custom_dag)
from oracle import port

from fixtures import instance_from_golden

pytestmark = pytest.mark.gpu

REL = 1e-9  # north_star energy tolerance


def _eff(sum_e, sum_t, watts, q):
    return float(sum_e) - watts * float(sum_t) * float(q) * 1e-3


def check_walk_against(batch, k, w, watts, q, full=True, hash_points=None):
    """Instance k of a run batch against reference walk w (ref_driver walk
    JSON).  A prefix golden (reason "max_steps", ref_driver walkprefix) is
    compared on its steps only.  full: the schedule hash of every point;
    else of hash_points (if given)."""
    s = batch.summary(k)
    assert s.status == 0
    assert s.n_table_misses == 0, w["spec"]  # every curve value came from the host (libm) tables
    assert (s.t_min, s.t_star) == (w["t_min"], w["t_star"]), w["spec"]
    nst = w["steps"]
    if w["reason"] == "max_steps":
        assert s.steps >= nst, (w["spec"], s.steps, nst)
    else:
        assert pb.STOP_NAMES[s.stop] == w["reason"], (w["spec"], pb.STOP_NAMES[s.stop], w["reason"])
        assert s.steps == nst, w["spec"]
    pts = batch.points(k)[:nst + 1]
    assert pts["t_planned"].tolist() == w["t_planned"], w["spec"]
    assert pts["t_realized"].tolist() == w["t_realized"], w["spec"]
    assert pts["sum_planned_e"].tolist() == w["sum_planned_e"], w["spec"]
    assert pts["sum_realized_e"].tolist() == w["sum_realized_e"], w["spec"]
    assert pts["cut_cost"][1:].tolist() == w["cut_cost"], w["spec"]
    assert pts["step_size"][1:].tolist() == w["step_size"], w["spec"]
    ids, _ = batch.deltas(k)
    for j in range(1, nst + 1):
        p = pts[j]
        seg = ids[p["id_begin"]:p["id_begin"] + p["n_sped"] + p["n_slowed"]]
        assert [int(x) - 1 for x in seg if x > 0] == w["sped"][j - 1], (w["spec"], j)
        assert [int(-x) - 1 for x in seg if x < 0] == w["slowed"][j - 1], (w["spec"], j)
    for j in range(nst + 1):
        ep = _eff(pts["sum_planned_e"][j], pts["sum_planned_t"][j], watts, q)
        er = _eff(pts["sum_realized_e"][j], pts["sum_realized_t"][j], watts, q)
        assert abs(ep - w["eff_planned"][j]) <= REL * max(1.0, abs(w["eff_planned"][j]))
        assert abs(er - w["eff_realized"][j]) <= REL * max(1.0, abs(w["eff_realized"][j]))
    if full:
        hash_points = range(nst + 1)
    for j in hash_points or ():
        d = batch.schedule(k, j)
        h = port.schedule_hash(d.planned_t, d.planned_e, d.freq_mhz, d.realized_t, d.realized_e)
        assert h == w["hash"][j], (w["spec"], j)
        assert d.eff_planned_mj == w["eff_planned"][j]
        assert d.eff_realized_mj == w["eff_realized"][j]


@pytest.mark.parametrize("smem,region", [("-1", None), ("0", None), ("1", "6000"), ("1", "0")])
def test_every_golden_walk_in_one_batch(walks, monkeypatch, smem, region):
    """All 126 reference walks (golden instances, G9 configs 1-2, random grid
    and cubic profiles with infeasible / infinite-cut stops) as ONE batch:
    shared-memory-resident walks (the automatic choice for a batch this
    size), the global-memory walker, and shared-memory walks whose region
    holds only part of the arrays (6000 B) or none of them."""
    monkeypatch.setenv("PB_SMEM", smem)
    if smem == "0":
        monkeypatch.setenv("PB_WIDE", "0")  # the global-memory walker kernel only
    if region is not None:
        monkeypatch.setenv("PB_SMEM_REGION", region)
    b = pb.FrontierBatch()
    meta = []
    for spec, w in walks.items():
        dag, model, tau = instance_from_golden(w)
        b.add(dag, model, tau)
        meta.append((spec, model))
    b.run(0)
    st = b.stats()
    assert st.smem_walks == (0 if smem == "0" else len(meta)), (smem, st.smem_walks)
    if region is not None:
        assert st.smem_region <= int(region)
    for k, (spec, model) in enumerate(meta):
        check_walk_against(b, k, walks[spec], model.blocking_watts, model.quantum_us, full=spec != "config:2")


@pytest.mark.parametrize("warps,shared_parents", [(2, True), (4, True), (2, False)])
def test_golden_walks_through_the_cooperative_bfs(walks, monkeypatch, warps, shared_parents):
    """The same 126 walks with every instance on the wide (multi-warp BFS)
    kernel, and with the wide kernel sharing the batch with the walker; with
    the augment chase through shared-memory parent links and through the
    global log (the fallback for instances too large for shared memory)."""
    monkeypatch.setenv("PB_WIDE_WARPS", str(warps))
    if not shared_parents:
        monkeypatch.setenv("PB_WIDE_NO_SHARED_PARENTS", "1")
    monkeypatch.setenv("PB_WIDE_CTAS", "7")
    for wide in ("100000", "9"):
        monkeypatch.setenv("PB_WIDE", wide)
        b = pb.FrontierBatch()
        meta = []
        for spec, w in walks.items():
            dag, model, tau = instance_from_golden(w)
            b.add(dag, model, tau)
            meta.append((spec, model))
        b.run(0)
        for k, (spec, model) in enumerate(meta):
            check_walk_against(b, k, walks[spec], model.blocking_watts, model.quantum_us, full=False)


def test_config2_every_point_bit_exact(walks):
    w = walks["config:2"]
    dag, model, tau = instance_from_golden(w)
    b = pb.FrontierBatch()
    b.add(dag, model, tau)
    b.run(0)
    check_walk_against(b, 0, w, model.blocking_watts, model.quantum_us, full=True)


def test_walks_individually_match_batched(walks):
    specs = [s for s in walks if s.startswith("cubic")][:6]
    for spec in specs:
        w = walks[spec]
        dag, model, tau = instance_from_golden(w)
        b = pb.FrontierBatch()
        b.add(dag, model, tau)
        b.run(0)
        check_walk_against(b, 0, w, model.blocking_watts, model.quantum_us)


def test_random_g9_instances_vs_oracle():
    """Small G9 instances drawn like config 5, checked against the C oracle."""
    b = pb.FrontierBatch()
    packs = []
    rng = np.random.default_rng(11)
    for i in range(24):
        p = g9.G9Params(int(rng.integers(2, 6)), int(rng.integers(2, 12)), int(rng.integers(8, 12)),
                        float(rng.uniform(1.0, 1.25)), int(rng.integers(0, 2**31)),
                        int(rng.integers(-1, 3)), float(rng.choice([1.0, 1.05, 1.1, 1.2, 1.3, 1.5])))
        if p.straggler_stage >= p.stages:
            p.straggler_stage = -1
        dag, model = g9.instance(p)
        b.add(dag, model, g9.TAU)
        packs.append(PackedInstance(dag, model, g9.TAU))
    b.run(0)
    for k, P in enumerate(packs):
        ref = port.discover_frontier(P, g9.TAU)
        s = b.summary(k)
        pts = b.points(k)
        assert s.steps == ref["steps"] and pb.STOP_NAMES[s.stop] == ref["reason"]
        assert pts["t_planned"].tolist() == ref["t_planned"]
        assert pts["t_realized"].tolist() == ref["t_realized"]
        assert pts["cut_cost"][1:].tolist() == ref["cut_cost"]
        last = b.schedule(k, s.steps)
        assert last.planned_t == ref["final_planned_t"] and last.freq_mhz == ref["final_freq"]


def _layered_dag(rng, levels, max_width, stages):
    """Random layered DAG: levels wider than 16, up to 6 predecessors (some
    more than 3 levels back) and computations without successors at every
    level, so the sweep's overflow rows, far neighbours and the makespan over
    sinks below an incremental forward range are all exercised."""
    comps, edges, by_level = [], [], []
    for lev in range(levels):
        ids = []
        for _ in range(int(rng.integers(1, max_width + 1))):
            i = len(comps)
            comps.append(Computation(i, int(rng.integers(0, stages)), i, Kind(int(rng.integers(0, 2)))))
            ids.append(i)
            if lev:
                preds = {int(rng.choice(by_level[lev - 1]))}
                for _ in range(int(rng.integers(0, 6))):
                    lv = int(rng.integers(max(0, lev - 8), lev))
                    preds.add(int(rng.choice(by_level[lv])))
                edges += [(u, i) for u in sorted(preds)]
        by_level.append(ids)
    ps = ProfileSet(75.0, [])
    for s in range(stages):
        b = int(rng.integers(8, 13))
        ps.profiles.append(FrequencyProfile(ClassKey(s, int(Kind.Forward)), g9.stage_profile(b, False)))
        ps.profiles.append(FrequencyProfile(ClassKey(s, int(Kind.Backward)), g9.stage_profile(b, True)))
    return finalize_custom_dag(comps, edges), CostModel.build(ps)


def test_layered_dags_incremental_sweep_vs_oracle():
    """Walks on irregular DAGs (wide levels, deep fan-in, early sinks) against
    the C oracle: every makespan, cut cost and the final plan bit-exact."""
    rng = np.random.default_rng(2024)
    b = pb.FrontierBatch()
    packs = []
    for k in range(12):
        dag, model = _layered_dag(rng, int(rng.integers(4, 30)), 24 if k % 2 else 6, 3)
        b.add(dag, model, g9.TAU)
        packs.append(PackedInstance(dag, model, g9.TAU))
    b.run(0)
    sinks = 0
    for k, P in enumerate(packs):
        ref = port.discover_frontier(P, g9.TAU)
        s = b.summary(k)
        pts = b.points(k)
        assert s.status == 0
        assert s.steps == ref["steps"] and pb.STOP_NAMES[s.stop] == ref["reason"]
        assert pts["t_planned"].tolist() == ref["t_planned"]
        assert pts["t_realized"].tolist() == ref["t_realized"]
        assert pts["cut_cost"][1:].tolist() == ref["cut_cost"]
        last = b.schedule(k, s.steps)
        assert last.planned_t == ref["final_planned_t"] and last.freq_mhz == ref["final_freq"]
        sinks += int(np.count_nonzero(P.edge_head == P.n + 1) > 1)
    assert sinks >= 6  # several sink computations per DAG
    assert sum(b.summary(k).steps for k in range(len(packs))) > 100


# ---- the reference API, test_frontier.cpp style -----------------------------

def _lone(ft, fe, st, se):
    dag = finalize_custom_dag([Computation(0, 0, 0, Kind.Forward)], [])
    m = CostModel.build(ProfileSet(75.0, [FrequencyProfile(ClassKey(0, 0), [ProfilePoint(1400, ft, fe),
                                                                            ProfilePoint(1000, st, se)])]))
    return dag, m


def _diamond():
    comps = [Computation(i, i, 0, Kind.Forward) for i in range(5)]
    dag = finalize_custom_dag(comps, [(0, 1), (1, 2), (0, 3), (4, 2)])

    def two(stage, t0, e0, t1, e1):
        return FrequencyProfile(ClassKey(stage, 0), [ProfilePoint(1400, t0, e0), ProfilePoint(1000, t1, e1)])
    m = CostModel.build(ProfileSet(75.0, [two(0, 1000, 4000, 3000, 1000), two(1, 1000, 625, 3000, 400),
                                          two(2, 1000, 4000, 3000, 1000), two(3, 4000, 625, 6000, 400),
                                          two(4, 4000, 625, 6000, 400)]))
    return dag, m


def test_min_energy_seed():
    dag, m = _lone(1000, 9000, 2000, 5000)
    s = pb.min_energy_schedule(dag, m)  # test_frontier.cpp:70-78
    assert s.planned_t == [2000] and s.planned_e == [5000] and s.t_planned == 2000
    assert s.eff_planned_mj == pytest.approx(5000 - 0.075 * 2000)
    assert not s.discretized()


def test_all_max_schedule():
    dag, m = _diamond()
    s = pb.all_max_schedule(dag, m)  # test_frontier.cpp:80-90
    assert s.schedule_id == -1 and s.freq_mhz == [1400] * 5
    assert s.planned_t == [1000, 1000, 1000, 4000, 4000] and s.realized_t == s.planned_t
    assert s.t_planned == 5000 and s.t_realized == 5000
    assert s.eff_planned_mj == pytest.approx(9875 - 0.075 * 11000)


def test_lone_get_next_schedule():
    dag, m = _lone(1000, 9000, 3000, 5000)
    seed = pb.min_energy_schedule(dag, m)
    info = pb.StepInfo()
    mid = pb.get_next_schedule(dag, seed, m, 1000, info)  # test_frontier.cpp:120-144
    assert mid.t_planned == 2000 and mid.planned_t == [2000] and mid.planned_e == [6708]
    assert info.cut_cost == 1708 and info.sped_up == [0] and info.slowed_down == []
    fast = pb.get_next_schedule(dag, mid, m, 1000, info)
    assert fast.t_planned == 1000 and fast.planned_e == [9000] and info.cut_cost == 2292
    assert pb.get_next_schedule(dag, fast, m, 1000) is None
    with pytest.raises(ValueError):
        pb.get_next_schedule(dag, seed, m, 0)
    with pytest.raises(ValueError):
        pb.discover_frontier(dag, m, 0)


def test_get_next_from_schedules_outside_the_curve_interval(walks):
    """get_next_schedule (frontier.hpp:90-135) from caller schedules with
    planned times below t_min / above t_max, on and off the tau grid: the
    reference evaluates ExpCurve::eval there (costmodel.hpp:47); the device
    reads the host tables, widened around the start schedule, and must
    reproduce the step exactly (golden: ref_driver getnext)."""
    from conftest import load_golden
    cases = load_golden("getnext.jsonl.gz")
    assert sum("cut_cost" in c for c in cases) > 100
    for c in cases:
        dag, model, _ = instance_from_golden(walks[c["spec"]])
        cur = pb.EnergySchedule(0, list(c["start"]), list(c["start_e"]))
        info = pb.StepInfo()
        nxt = pb.get_next_schedule(dag, cur, model, c["tau"], info)
        if "cut_cost" not in c:
            assert nxt is None, c
            continue
        assert nxt is not None, c
        assert (info.cut_cost, info.sped_up, info.slowed_down) == (c["cut_cost"], c["sped"], c["slowed"]), c
        assert nxt.planned_t == c["planned_t"] and nxt.planned_e == c["planned_e"], c
        assert nxt.t_planned == c["t_planned"] and nxt.eff_planned_mj == c["eff_planned"], c


def test_diamond_step_by_step():
    dag, m = _diamond()
    cur = pb.min_energy_schedule(dag, m)
    assert cur.t_planned == 9000 and cur.planned_t == [3000, 3000, 3000, 6000, 6000]
    walk = [(300, [1, 3, 4], [], [3000, 2000, 3000, 5000, 5000]),
            (375, [1, 3, 4], [], [3000, 1000, 3000, 4000, 4000]),
            (1875, [0, 2], [1], [2000, 2000, 2000, 4000, 4000]),
            (3900, [0, 2], [1], [1000, 3000, 1000, 4000, 4000])]
    for cut, sped, slowed, planned in walk:  # test_frontier.cpp:177-212
        info = pb.StepInfo()
        nxt = pb.get_next_schedule(dag, cur, m, 1000, info)
        assert (info.cut_cost, info.sped_up, info.slowed_down, nxt.planned_t) == (cut, sped, slowed, planned)
        assert nxt.t_planned == cur.t_planned - 1000
        assert sum(nxt.planned_e) - sum(cur.planned_e) == cut
        cur = nxt
    assert pb.get_next_schedule(dag, cur, m, 1000) is None


def test_diamond_frontier_and_lookup():
    dag, m = _diamond()
    f = pb.discover_frontier(dag, m, 1000)  # test_frontier.cpp:214-265
    assert len(f.schedules) == 5 and f.steps == 4 and f.t_star == 9000 and f.t_min == 5000
    assert [s.t_planned for s in f.schedules] == [9000, 8000, 7000, 6000, 5000]
    assert [s.t_realized for s in f.schedules] == [9000, 7000, 7000, 5000, 5000]
    assert [sum(s.planned_e) for s in f.schedules] == [3200, 3500, 3875, 5750, 9650]
    assert [s.eff_planned_mj for s in f.schedules] == pytest.approx([1625, 2150, 2750, 4700, 8675])
    assert f.schedules[1].freq_mhz == f.schedules[2].freq_mhz
    for s in f.schedules:
        assert all(r <= p for r, p in zip(s.realized_t, s.planned_t))
    am = pb.all_max_schedule(dag, m)
    assert f.schedules[-1].t_realized == am.t_realized
    assert f.schedules[-1].eff_realized_mj < am.eff_realized_mj
    ids = [pb.lookup(f, t).schedule_id for t in (9000, 250000, 8999, 7500, 7000, 5000, 4999, 0)]
    assert ids == [0, 0, 1, 2, 2, 4, 4, 4]
    with pytest.raises(pb.LogicError):
        pb.lookup(pb.Frontier(), 1000)


def test_all_constant_classes_single_point():
    dag = finalize_custom_dag([Computation(0, 0, 0, Kind.Forward), Computation(1, 1, 0, Kind.Forward)], [(0, 1)])
    m = CostModel.build(ProfileSet(75.0, [
        FrequencyProfile(ClassKey(0, 0), [ProfilePoint(1400, 2000, 3000), ProfilePoint(1200, 2500, 3100)]),
        FrequencyProfile(ClassKey(1, 0), [ProfilePoint(1400, 1500, 2000), ProfilePoint(1200, 1600, 2400)])]))
    seed = pb.min_energy_schedule(dag, m)  # test_frontier.cpp:92-116
    assert seed.planned_t == pb.all_max_schedule(dag, m).planned_t
    assert pb.get_next_schedule(dag, seed, m, 1000) is None
    f = pb.discover_frontier(dag, m, 1000)
    assert len(f.schedules) == 1 and f.steps == 0 and f.t_star == f.t_min == 3500
    assert pb.lookup(f, 0) is f.schedules[0] and pb.lookup(f, 100000) is f.schedules[0]


def test_discretize_cases():
    dag = finalize_custom_dag([Computation(0, 0, 0, Kind.Forward)], [])
    m = CostModel.build(ProfileSet(75.0, [FrequencyProfile(ClassKey(0, 0), [
        ProfilePoint(1410, 1900, 900), ProfilePoint(1200, 2300, 700), ProfilePoint(1000, 2800, 500)])]))
    for planned, freq, rt in [(2400, 1200, 2300), (2300, 1200, 2300), (1500, 1410, 1900), (5000, 1000, 2800)]:
        s = pb.EnergySchedule(planned_t=[planned], planned_e=[700], t_planned=planned)
        d = pb.discretize(s, dag, m)  # test_frontier.cpp:269-309
        assert d.freq_mhz == [freq] and d.realized_t == [rt] and d.t_realized == rt


# ---- full-size properties (BASELINE configs 3 and 4 shapes) -----------------

@pytest.mark.parametrize("cfg,phi", [(3, 1.0), (4, 1.2)])
def test_full_size_walk_properties(cfg, phi):
    p = g9.named_config(cfg, phi)
    dag, model = g9.instance(p)
    b = pb.FrontierBatch()
    b.add(dag, model, g9.TAU)
    b.run(0)
    s = b.summary(0)
    assert s.status == 0 and pb.STOP_NAMES[s.stop] == "at_t_min"
    assert s.steps == 24 * (p.stages + p.microbatches - 1)
    pts = b.points(0)
    tp = pts["t_planned"]
    assert tp[0] == s.t_star and tp[-1] == s.t_min
    assert np.all(tp[:-1] - tp[1:] == pts["step_size"][1:])
    assert np.all(pts["t_realized"] <= tp)
    # the relaxed energy moves by the cut cost within 1 mJ per touched computation
    d = np.diff(pts["sum_planned_e"])
    touched = pts["n_sped"][1:] + pts["n_slowed"][1:]
    assert np.all(np.abs(d - pts["cut_cost"][1:]) <= touched)
    # replaying the delta log reproduces the device's running sums
    last = b.schedule(0, s.steps)
    assert sum(last.planned_t) == pts["sum_planned_t"][-1]
    assert sum(last.realized_e) == pts["sum_realized_e"][-1]


def test_straggler_sweep_matches_reference(walks):
    """pb_batch_straggler (device lookup + Eq. 3 energy) against the unmodified
    reference's straggler_savings on its own frontier (tests/golden/savings):
    the looked-up point is identical; energies within 1e-9 relative to the
    all-max energy (the reference sums per-stage blocking terms one by one)."""
    from conftest import load_golden
    from fixtures import instance_from_golden
    recs = load_golden("savings.jsonl.gz")
    b = pb.FrontierBatch()
    for r in recs:
        spec = r["spec"]
        if spec in walks:
            dag, model, tau = instance_from_golden(walks[spec])
            b.add(dag, model, tau)
        else:  # g9:N:M:B:imb:seed:straggler:phi
            _, N_, M_, B_, imb, seed, st, phi = spec.split(":")
            b.add_g9(g9.G9Params(int(N_), int(M_), int(B_), float(imb), int(seed), int(st), float(phi)))
    b.run(0)
    factors = [row["factor"] for row in recs[0]["rows"]]
    P = recs[0]["pipelines"]
    out = b.straggler(factors, P, [r["num_stages"] for r in recs])
    for k, r in enumerate(recs):
        for j, ref in enumerate(r["rows"]):
            got = out[k, j]
            assert got["status"] == 0, r["spec"]
            assert got["point"] == ref["point"], (r["spec"], ref["factor"])
            scale = (P - 1) * abs(got["all_max_mj"])
            assert abs(got["savings_mj"] - ref["savings_mj"]) <= 1e-9 * scale, (r["spec"], ref, got)
            assert abs(got["savings_pct"] - ref["savings_pct"]) <= 1e-9 * 100, (r["spec"], ref, got)


def test_artifacts_byte_identical_to_reference_writer(walks):
    """frontier.csv and schedules/schedule_<k>.json expanded from the delta log
    (pb_batch_frontier_csv / pb_batch_schedule_json) against the bytes the
    reference writer produces (serde.hpp:194-257, 304-316), quantum 1 and 10."""
    from conftest import load_golden
    recs = load_golden("artifacts.jsonl.gz")
    b = pb.FrontierBatch()
    for r in recs:
        spec = r["spec"]
        if spec in walks:
            dag, model, tau = instance_from_golden(walks[spec])
            b.add(dag, model, tau)
        else:
            _, N_, M_, B_, imb, seed, st, phi = spec.split(":")
            b.add_g9(g9.G9Params(int(N_), int(M_), int(B_), float(imb), int(seed), int(st), float(phi)))
    b.run(0)
    for k, r in enumerate(recs):
        assert b.frontier_csv(k, r["quantum"]) == r["csv"], r["spec"]
        for which, text in r["schedules"].items():
            assert b.schedule_json(k, int(which), r["quantum"]) == text, (r["spec"], which)


def test_lone_artifacts_match_test_serde_cpp():
    """test_serde.cpp:252-259 golden CSV of the lone walk."""
    dag, model = _lone(1000, 9000, 3000, 5000)
    b = pb.FrontierBatch()
    b.add(dag, model, 1000)
    b.run(0)
    assert b.frontier_csv(0) == ("t_planned_us,t_realized_us,energy_planned_mj,energy_realized_mj,schedule_id\n"
                                 "3000,3000,4775.000,4775.000,0\n"
                                 "2000,1000,6558.000,8925.000,1\n"
                                 "1000,1000,8925.000,8925.000,2\n")
    assert "30000,30000,4775.000" in b.frontier_csv(0, 10)
    assert b.schedule_json(0, 1).replace("\n", "").replace(" ", "") == (
        '{"schedule_id":1,"t_planned_us":2000,"eff_planned_mj":6558.0,'
        '"t_realized_us":1000,"eff_realized_mj":8925.0,'
        '"computations":[{"id":0,"freq_mhz":1400,"t_planned_us":2000,"e_planned_mj":6708,'
        '"t_realized_us":1000,"e_realized_mj":9000}]}')


def test_brute_force_oracle_matches_reference(walks):
    """pb_batch_brute_force (GPU enumeration) against the reference's
    brute_force_frontier (tests/golden/brute): identical times, bit-identical
    effective energies and frequency plans; BudgetExceeded where the reference
    throws.  Also acceptance gate 1 on the same instances: every frontier
    point's lookup within 2% of the exact optimum (acceptance.cpp:79-112)."""
    import struct
    from conftest import load_golden
    recs = load_golden("brute.jsonl.gz")
    b = pb.FrontierBatch()
    for r in recs:
        dag, model, tau = instance_from_golden(walks[r["spec"]])
        b.add(dag, model, tau)
    b.run(0)
    checked = 0
    for k, r in enumerate(recs):
        if r.get("budget_exceeded"):
            with pytest.raises(N.BudgetExceeded):
                b.brute_force(k)
            continue
        pts, fr = b.brute_force(k)
        assert len(pts) == len(r["points"]), r["spec"]
        for j, ref in enumerate(r["points"]):
            assert int(pts[j]["time"]) == ref["time"], r["spec"]
            bits = struct.unpack("<Q", struct.pack("<d", float(pts[j]["eff_energy_mj"])))[0]
            assert bits == int(ref["eff_bits"]), (r["spec"], j)
            assert fr[j].tolist() == ref["freq_mhz"], (r["spec"], j)
        # gate 1: lookup(frontier, exact time) within 2% of the exact optimum
        s = b.summary(k)
        tp = b.points(k)["t_planned"]
        for p in pts:
            target = min(s.t_star, int(p["time"]))
            idx = next((q for q in range(s.steps + 1) if tp[q] <= target), s.steps)
            sched = b.schedule(k, idx)
            gap = (sched.eff_realized_mj - p["eff_energy_mj"]) / p["eff_energy_mj"]
            assert gap <= 0.02 + 1e-12, (r["spec"], gap)
        checked += 1
    assert checked >= 30


def test_parallel_batch_builder_matches_serial_adds():
    """pb_batch_add_g9_batch (instances built on all host threads) walks
    exactly like the same instances added one by one."""
    a = pb.FrontierBatch()
    a.add_g9_batch(100, 24)
    c = pb.FrontierBatch()
    for i in range(100, 124):
        c.add_g9(g9.batch_params(i))
    a.run(0)
    c.run(0)
    for k in range(24):
        sa, sc = a.summary(k), c.summary(k)
        assert (sa.t_min, sa.t_star, sa.steps, sa.stop) == (sc.t_min, sc.t_star, sc.steps, sc.stop)
        pa, pc = a.points(k), c.points(k)
        assert pa["t_planned"].tolist() == pc["t_planned"].tolist()
        assert pa["sum_realized_e"].tolist() == pc["sum_realized_e"].tolist()


def test_batch_scale_invariants():
    """Size-independent properties on 256 instances of the config-5 batch
    (N 4-16, M 8-256) in one launch: every G9 walk stops AT_TMIN after
    ceil((T* - T_min) / tau) steps of exactly tau (last one clipped,
    acceptance gate 2); the delta log reproduces every point's planned-time
    sum; ids inside a step are ascending (sped, then slowed); realized
    iteration times never undercut T_min; the host replay of the last point
    agrees with the device totals."""
    b = pb.FrontierBatch()
    b.add_g9_batch(0, 256)
    b.run(0)
    for k in range(len(b)):
        s = b.summary(k)
        assert s.status == 0 and pb.STOP_NAMES[s.stop] == "at_t_min", k
        assert s.steps == -(-(s.t_star - s.t_min) // 1000), k
        pts = b.points(k)
        tp = pts["t_planned"]
        assert tp[0] == s.t_star and tp[-1] == s.t_min
        assert all(tp[q] - tp[q + 1] == min(1000, tp[q] - s.t_min) for q in range(s.steps)), k
        assert (pts["t_realized"] >= s.t_min).all()
        ids, _ = b.deltas(k)
        for q in range(1, s.steps + 1):
            p = pts[q]
            seg = ids[p["id_begin"]:p["id_begin"] + p["n_sped"] + p["n_slowed"]]
            sp, sl = seg[:p["n_sped"]], -seg[p["n_sped"]:]
            assert (sp > 0).all() and (sl > 0).all()
            assert (np.diff(sp) > 0).all() and (np.diff(sl) > 0).all()
            dt = int(p["sum_planned_t"]) - int(pts[q - 1]["sum_planned_t"])
            assert dt == int(p["step_size"]) * (len(sl) - len(sp)), (k, q)
        if k % 32 == 0:
            last = b.schedule(k, s.steps)
            assert sum(last.planned_t) == int(pts[-1]["sum_planned_t"])
            assert sum(last.realized_e) == int(pts[-1]["sum_realized_e"])


def test_full_size_configs_3_and_4_bit_exact():
    """The named full-size configurations against the unmodified reference
    (tests/golden/walks_large: 8x128 with 3240 steps, 16x128 with 3432 steps;
    ~30 min of reference CPU time to regenerate): every point's times, cut
    cost, sped/slowed ids and energies, and every schedule's hash."""
    from conftest import load_golden
    recs = load_golden("walks_large.jsonl.gz")
    b = pb.FrontierBatch()
    meta = []
    for w in recs:
        dag, model, tau = instance_from_golden(w)
        b.add(dag, model, tau)
        meta.append(model)
    b.run(0)
    for k, (w, model) in enumerate(zip(recs, meta)):
        check_walk_against(b, k, w, model.blocking_watts, model.quantum_us, full=True)


@pytest.fixture(scope="module")
def batch5():
    """The headline workload: the whole config-5 batch (4096 instances), as
    bench.py runs it -- the LPT head on the cooperative kernel, the rest on
    walker warps, one launch."""
    b = pb.FrontierBatch()
    b.add_g9_batch(0, 4096)
    b.run(0)
    return b


def test_config5_batch_bit_exact_vs_reference(batch5):
    """Config-5 instances against the unmodified reference (golden
    batch5.jsonl.gz, ref_driver walk / walkprefix): the largest 16x256 walks
    in full (they run on the cooperative kernel with shared-memory parent
    links and the split capacity pass), mid-size walks in full, and the first
    300 steps of the 16 stratified sample instances (i = 0 mod 256)."""
    from conftest import load_golden
    gold = load_golden("batch5.jsonl.gz")
    coop = 0
    for w in gold:
        k = int(w["spec"].split(":")[1])
        n = len(w["t_planned"]) - 1
        sample = sorted({0, 1, n // 3, n // 2, (2 * n) // 3, n})
        check_walk_against(batch5, k, w, 75.0, 1, full=False, hash_points=sample)
        if w["reason"] != "max_steps" and batch5.summary(k).warps > 1:
            coop += 1
    heavy = [w for w in gold if w["reason"] != "max_steps" and len(w["t_planned"]) > 6000]
    assert all(batch5.summary(int(w["spec"].split(":")[1])).warps > 1 for w in heavy)
    assert sum(w["reason"] == "max_steps" for w in gold) >= 16


def test_config5_batch_is_deterministic(batch5):
    """Every instance of the 4096 batch: status ok, no table miss, and the
    same results (digest of points + delta records) on a second launch --
    the minimal min cut is unique, so the walk must not depend on timing."""
    n = len(batch5)
    first = [batch5.digest(k) for k in range(n)]
    for k in range(n):
        s = batch5.summary(k)
        assert s.status == 0 and s.n_table_misses == 0, k
    batch5.launch()
    batch5.fetch()
    assert [batch5.digest(k) for k in range(n)] == first


def test_run_multi_two_devices_matches_single(walks):
    """pb_batch_run_multi LPT-shards a batch over a device list (here device
    0 twice, two host threads): results stitched back in caller order, delta
    pools and curve-table offsets rebased -- bit-identical to one device."""
    specs = ["diamond", "config:1", "config:2"] + [s for s in walks if s.startswith(("grid:", "g9:"))][:30]

    def build():
        b = pb.FrontierBatch()
        for s in specs:
            dag, model, tau = instance_from_golden(walks[s])
            b.add(dag, model, tau)
        b.add_g9_indices([7, 300, 1234, 4000])
        return b

    one, two = build().run(0), build().run_multi([0, 0])
    for k in range(len(specs) + 4):
        assert two.summary(k).status == 0
        assert two.digest(k) == one.digest(k), k
        last = one.summary(k).steps
        for j in {0, last // 2, last}:
            a, c = one.schedule(k, j), two.schedule(k, j)
            assert (a.planned_t, a.planned_e, a.freq_mhz, a.eff_planned_mj, a.eff_realized_mj) == \
                (c.planned_t, c.planned_e, c.freq_mhz, c.eff_planned_mj, c.eff_realized_mj), (k, j)
    for k, s in enumerate(specs):
        check_walk_against(two, k, walks[s], walks[s]["instance"]["blocking_watts"],
                           walks[s]["instance"]["quantum_us"], full=False, hash_points=[0])
    assert two.frontier_csv(1) == one.frontier_csv(1)


def test_config4_straggler_sweep_bit_exact_vs_reference():
    """The config-4 straggler sweep (Bloom-like 16x128, stage 8
    slowed by phi in 1.05 ... 1.5, each a separate instance) walked in full
    against the unmodified reference (golden walks_phi: every point's times,
    cut costs, ids and energies; schedule hashes at sampled points), and
    straggler_savings (baselines.hpp:162-188) of configs 4 and 3 at the sweep
    factors (golden savings_c4) on the device frontiers."""
    from conftest import load_golden
    walks_phi = load_golden("walks_phi.jsonl.gz")
    sav = load_golden("savings_c4.jsonl.gz")
    b = pb.FrontierBatch()
    for w in walks_phi:
        phi = float(w["spec"].split(":")[2])
        b.add_g9(g9.named_config(4, phi))
    b.add_g9(g9.named_config(4))
    b.add_g9(g9.named_config(3))
    b.run(0)
    for k, w in enumerate(walks_phi):
        n = w["steps"]
        check_walk_against(b, k, w, 75.0, 1, full=False, hash_points=sorted({0, 1, n // 4, n // 2, n - 1, n}))
    factors = [row["factor"] for row in sav[0]["rows"]]
    P = sav[0]["pipelines"]
    out = b.straggler(factors, P, [16] * len(walks_phi) + [16, 8])
    for r, k in zip(sav, (len(walks_phi), len(walks_phi) + 1)):
        assert r["spec"] == ("config:4", "config:3")[k - len(walks_phi)]
        for j, ref in enumerate(r["rows"]):
            got = out[k, j]
            assert got["status"] == 0 and got["point"] == ref["point"], (r["spec"], ref["factor"])
            scale = (P - 1) * abs(got["all_max_mj"])
            assert abs(got["savings_mj"] - ref["savings_mj"]) <= 1e-9 * scale, (r["spec"], ref, got)
            assert abs(got["savings_pct"] - ref["savings_pct"]) <= 1e-9 * 100, (r["spec"], ref, got)


def test_schedules_range_matches_single_schedules(walks):
    """pb_batch_schedules (one incremental replay for a range of points)
    returns exactly what pb_batch_schedule returns point by point."""
    w = walks["config:2"]
    dag, model, tau = instance_from_golden(w)
    b = pb.FrontierBatch()
    b.add(dag, model, tau)
    b.run(0)
    s = b.summary(0)
    rng = b.schedules(0, 5, 40)
    for q, got in enumerate(rng):
        assert got == b.schedule(0, 5 + q)
    full = b.frontier(0).schedules
    assert len(full) == s.steps + 1
    for j in (0, s.steps // 2, s.steps):
        assert full[j] == b.schedule(0, j)


def test_cleared_handle_walks_new_instances(walks):
    """pb_batch_clear keeps the device context but drops every instance and
    result: a handle reused for a different DAG, then for the first DAG again
    with a start schedule (the derived-layout cache path), walks each exactly
    as a fresh handle does."""
    b = pb.FrontierBatch()
    for spec in ("config:1", "diamond", "config:1"):
        w = walks[spec]
        dag, model, tau = instance_from_golden(w)
        b.clear()
        b.add(dag, model, tau)
        b.run(0)
        check_walk_against(b, 0, w, model.blocking_watts, model.quantum_us, full=False, hash_points=[0, 1])
    # get-next from the frontier's point 5 on the cleared handle
    w = walks["config:1"]
    dag, model, tau = instance_from_golden(w)
    start = b.schedule(0, 5)
    b.clear()
    b.add(dag, model, tau, start_planned_t=start.planned_t, max_steps=1)
    b.run(0)
    nxt = b.schedule(0, 1)
    assert nxt.t_planned == w["t_planned"][6]
    assert b.step_info(0, 1).sped_up == w["sped"][5]


def test_config4_alone_on_the_cooperative_kernel():
    """A lone wide DAG that does not fit a shared-memory region (config 4,
    16x128: width n / levels = 14) is walked by a 2-warp cooperative CTA:
    bit-exact against the reference walk, every point and schedule hash."""
    from conftest import load_golden
    w = next(r for r in load_golden("walks_large.jsonl.gz") if r["spec"] == "config:4")
    dag, model, tau = instance_from_golden(w)
    b = pb.FrontierBatch()
    b.add(dag, model, tau)
    b.run(0)
    st = b.stats()
    assert st.wide_walks == 1 and st.smem_walks == 0
    check_walk_against(b, 0, w, model.blocking_watts, model.quantum_us, full=True)


@pytest.mark.parametrize("shape", [(32, 512), (24, 300)])
def test_very_large_instance_agrees_across_kernels(monkeypatch, shape):
    """A DAG far beyond the config-5 sizes (32x512: 32,768 computations,
    ~98k edge-centric edges; the cooperative kernel's parent links no longer
    fit shared memory) walked for 200 steps by each kernel: the single-warp
    walker, the cooperative CTA and the shared-memory kernel (partial
    placement).  The minimal min cut is unique, so every point and delta
    record must agree bit for bit (size-independent parity property)."""
    N_, M_ = shape
    p = g9.G9Params(N_, M_, 10, 1.1, 77, N_ // 2, 1.2)
    digests = {}
    for mode in ({"PB_SMEM": "0", "PB_WIDE": "0"}, {"PB_WIDE": "1"}, {"PB_SMEM": "1"}):
        for k in ("PB_SMEM", "PB_WIDE"):
            monkeypatch.delenv(k, raising=False)
        for k, v in mode.items():
            monkeypatch.setenv(k, v)
        b = pb.FrontierBatch()
        b.add_g9(p)
        b.set_max_steps(200)
        b.run(0)
        s = b.summary(0)
        assert s.status == 0 and s.n_table_misses == 0 and s.steps == 200, (mode, s.status, s.steps)
        digests[tuple(mode.items())] = b.digest(0)
    assert len(set(digests.values())) == 1, digests


@pytest.mark.parametrize("carry", [True, False])
def test_get_next_chain_warm_start_matches_the_walk(walks, monkeypatch, carry):
    """A loop of single get_next calls on one handle (the drop-in's pattern)
    resumes each call from the flow state the previous one ended in (the
    device carry buffer), instead of a cold max flow: every step's cut cost,
    sped/slowed ids and planned times must equal the reference walk's, with
    and without the warm start (PB_NO_CARRY), and the warm path must be taken."""
    if not carry:
        monkeypatch.setenv("PB_NO_CARRY", "1")
    w = walks["config:2"]
    dag, model, tau = instance_from_golden(w)
    b = pb.FrontierBatch()
    b.add(dag, model, tau, max_steps=-1)  # the seed (zero-step walk)
    b.run(0)
    planned = b.schedule(0, 0).planned_t
    warm = 0
    for k in range(300):
        b.clear()
        b.add(dag, model, tau, start_planned_t=planned, max_steps=1)
        b.run(0)
        warm += b.stats().warm_starts
        s = b.summary(0)
        assert s.status == 0 and s.steps == 1
        info = b.step_info(0, 1)
        assert info.cut_cost == w["cut_cost"][k], k
        assert info.sped_up == w["sped"][k] and info.slowed_down == w["slowed"][k], k
        nxt = b.schedule(0, 1)
        assert nxt.t_planned == w["t_planned"][k + 1], k
        planned = nxt.planned_t
        if k % 50 == 7:  # a discretize (zero-step walk) in between must not break the chain
            b.clear()
            b.add(dag, model, tau, start_planned_t=planned, max_steps=-1)
            b.run(0)
    assert warm == (299 if carry else 0)
