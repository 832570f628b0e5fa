"""CPU-side checks of the product library (no GPU needed): the C ABI loads
and exports every symbol include/perseus_b200.h declares, the native cost
model reproduces the reference's curve bits, the G9 generator and the 1F1B
builder reproduce the reference's instances, and invalid inputs raise the
reference's exception classes at add time."""
import os
import re
import struct

import numpy as np
import pytest

import paper_2312_06902_b200 as pb
from paper_2312_06902_b200 import _native as N
from paper_2312_06902_b200 import g9
from paper_2312_06902_b200.model import (ClassKey, Computation, CostModel, FrequencyProfile, Kind,
                                         ProfilePoint, ProfileSet, build_1f1b, finalize_custom_dag)

from conftest import ROOT
from fixtures import instance_from_golden


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "perseus_b200.h")).read()
    declared = set(re.findall(r"\b(pb_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(N.lib, name), name
    assert declared == set(N.EXPORTED)
    assert b"sm_100a" in N.lib.pb_version()


def test_library_contains_sm100a_cubin():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_native_fit_matches_reference_curve_bits(walks):
    checked = 0
    for w in walks.values():
        for c in w["curves"]:
            if c["constant"]:
                continue
            pts = [ProfilePoint(*p) for p in c["pareto"]]
            curve = pb.fit_exp(pts)
            assert [struct.pack(">d", x).hex() for x in (curve.a, curve.b, curve.c)] == c["curve_bits"]
            assert (curve.t_min, curve.t_max) == (c["t_min"], c["t_max"])
            checked += 1
    assert checked > 100


def test_cost_model_build_matches_reference(walks):
    for w in walks.values():
        _, model, _ = instance_from_golden(w)
        keys = sorted(model.classes)
        assert len(keys) == len(w["curves"])
        for k, c in zip(keys, w["curves"]):
            cm = model.classes[k]
            assert (k.stage, k.kind) == (c["stage"], c["kind"])
            assert cm.is_constant == c["constant"]
            assert [[p.freq_mhz, p.time, p.energy] for p in cm.pareto] == c["pareto"]


def test_g9_generator_matches_reference_instances(walks):
    for cfg in (1, 2):
        w = walks[f"config:{cfg}"]
        p = g9.named_config(cfg)
        dag, model = g9.instance(p)
        ref_dag, ref_model, _ = instance_from_golden(w)
        assert [(c.stage, int(c.kind), c.microbatch) for c in dag.computations] == \
               [(c.stage, int(c.kind), c.microbatch) for c in ref_dag.computations]
        assert dag.edges == ref_dag.edges
        ps = g9.profile_set(p)
        ref_ps = w["instance"]["profiles"]
        assert [[[q.freq_mhz, q.time, q.energy] for q in f.points] for f in ps.profiles] == \
               [f["points"] for f in ref_ps]


def test_g9_batch_params_are_deterministic():
    a = [g9.batch_params(i) for i in range(16)]
    b = [g9.batch_params(i) for i in range(16)]
    assert a == b
    for p in a:
        assert 4 <= p.stages <= 16 and 8 <= p.microbatches <= 256
        assert 1.0 <= p.imbalance <= 1.25 and p.phi in (1.0, 1.05, 1.1, 1.2, 1.3, 1.5)
        assert 0 <= p.straggler_stage < p.stages


def test_1f1b_edge_count():
    # test_dag.cpp:111-136: 4NM - 2M + N edges
    for n, m in [(1, 1), (2, 3), (4, 8), (8, 32)]:
        dag = build_1f1b(n, m)
        assert len(dag.edges) == 4 * n * m - 2 * m + n
        assert len(dag.computations) == 2 * n * m


def _diamond_model():
    def two(stage, t0, e0, t1, e1):
        return FrequencyProfile(ClassKey(stage, 0), [ProfilePoint(1400, t0, e0), ProfilePoint(1000, t1, e1)])
    return CostModel.build(ProfileSet(75.0, [two(0, 1000, 4000, 3000, 1000), two(1, 1000, 625, 3000, 400),
                                             two(2, 1000, 4000, 3000, 1000), two(3, 4000, 625, 6000, 400),
                                             two(4, 4000, 625, 6000, 400)]))


def test_invalid_inputs_raise_reference_exceptions():
    comps = [Computation(i, i, 0, Kind.Forward) for i in range(5)]
    dag = finalize_custom_dag(comps, [(0, 1), (1, 2), (0, 3), (4, 2)])
    model = _diamond_model()
    b = pb.FrontierBatch()
    with pytest.raises(ValueError):
        b.add(dag, model, 0)  # frontier.hpp:168
    with pytest.raises(ValueError):
        b.add(dag, model, -5)
    bad = CostModel(dict(list(model.classes.items())[:4]))
    with pytest.raises(ValueError):
        b.add(dag, bad, 1000)  # costmodel.hpp:209-213 missing class
    with pytest.raises(ValueError):
        finalize_custom_dag(comps, [(0, 1), (1, 0)])  # cycle
    with pytest.raises(ValueError):
        build_1f1b(0, 3)
    # a cyclic NodeDag that bypassed finalize_custom_dag is rejected by the ABI
    cyc = finalize_custom_dag(comps, [(0, 1)])
    cyc.edges.append((1, 0))
    with pytest.raises(ValueError):
        b.add(cyc, model, 1000)
    assert len(b) == 0


def test_degenerate_fit_collapses_to_constant():
    # costmodel.hpp:225-233: equal energies -> DegenerateFit -> constant class
    m = CostModel.build(ProfileSet(75.0, [FrequencyProfile(ClassKey(0, 0), [ProfilePoint(1400, 1000, 500),
                                                                            ProfilePoint(1000, 2000, 500)])]))
    cm = m.classes[ClassKey(0, 0)]
    assert cm.is_constant and len(cm.pareto) == 1
    with pytest.raises(pb.DegenerateFit):
        pb.fit_exp([ProfilePoint(1400, 1000, 500), ProfilePoint(1000, 2000, 500)])


def test_pareto_filter_matches_oracle():
    from oracle import port
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = int(rng.integers(1, 10))
        f = sorted(rng.choice(np.arange(500, 2000), n, replace=False).tolist(), reverse=True)
        t = rng.integers(1, 20, n).tolist()
        e = rng.integers(1, 20, n).tolist()
        mine = pb.pareto_filter([ProfilePoint(a, b, c) for a, b, c in zip(f, t, e)])
        of, ot, oe = port.pareto_filter(f, t, e)
        assert [(p.freq_mhz, p.time, p.energy) for p in mine] == list(zip(of, ot, oe))


def test_parallel_batch_builder_counts_and_order():
    import paper_2312_06902_b200 as pb
    a = pb.FrontierBatch()
    a.add_g9_batch(0, 40, threads=3)
    assert len(a) == 40 and N.lib.pb_batch_size(a._h) == 40
    with pytest.raises(ValueError):
        N.check(N.lib.pb_batch_add_g9_batch(a._h, -1, 2, 1000, 0))
