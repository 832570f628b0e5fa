"""Reference-shaped data model: NodeDag and CostModel.

Mirrors /root/reference/proj/include/perseus/dag.hpp (NodeDag, Computation,
Kind, build_1f1b/build_gpipe, finalize_custom_dag, to_edge_centric) and
costmodel.hpp (ProfilePoint, ClassKey, FrequencyProfile, ExpCurve,
CostModel::build with pareto_filter/fit_exp done by the native library).
These are input containers; all frontier compute happens on the device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N


class Kind(IntEnum):
    """perseus::Kind (dag.hpp:18)."""
    Forward = 0
    Backward = 1
    Constant = 2


@dataclass
class Computation:
    """perseus::Computation (dag.hpp:36-41)."""
    id: int = 0
    stage: int = 0
    microbatch: Optional[int] = None
    kind: Kind = Kind.Constant


@dataclass
class NodeDag:
    """perseus::NodeDag (dag.hpp:50-58): virtual source n, sink n+1."""
    computations: List[Computation] = field(default_factory=list)
    edges: List[Tuple[int, int]] = field(default_factory=list)
    num_stages: int = 0

    def source_id(self) -> int:
        return len(self.computations)

    def sink_id(self) -> int:
        return len(self.computations) + 1

    def node_count(self) -> int:
        return len(self.computations) + 2


def _topo_check(node_count: int, edges: Sequence[Tuple[int, int]]) -> None:
    # Kahn (dag.hpp:64-86): only used to reject cycles at construction time.
    indeg = [0] * node_count
    adj: List[List[int]] = [[] for _ in range(node_count)]
    for u, v in edges:
        adj[u].append(v)
        indeg[v] += 1
    ready = [v for v in range(node_count) if indeg[v] == 0]
    seen = 0
    while ready:
        u = ready.pop()
        seen += 1
        for v in adj[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                ready.append(v)
    if seen != node_count:
        raise ValueError("dependency graph contains a cycle")


def one_f_one_b_stage_stream(num_stages: int, microbatches: int, stage: int) -> List[Tuple[Kind, int]]:
    """dag.hpp:91-103: min(M, N-s) warm-up forwards, then 1B1F pairs, then the rest."""
    seq: List[Tuple[Kind, int]] = []
    warmup = min(microbatches, num_stages - stage)
    fwd = bwd = 0
    while fwd < warmup:
        seq.append((Kind.Forward, fwd))
        fwd += 1
    while fwd < microbatches:
        seq.append((Kind.Backward, bwd))
        bwd += 1
        seq.append((Kind.Forward, fwd))
        fwd += 1
    while bwd < microbatches:
        seq.append((Kind.Backward, bwd))
        bwd += 1
    return seq


def all_f_all_b_stage_stream(microbatches: int) -> List[Tuple[Kind, int]]:
    """dag.hpp:105-110."""
    return [(Kind.Forward, m) for m in range(microbatches)] + [(Kind.Backward, m) for m in range(microbatches)]


def build_pipeline(num_stages: int, microbatches: int, one_f_one_b: bool) -> NodeDag:
    """dag.hpp:112-143: stage-major ids in stream order; chain, cross-stage, endpoint edges."""
    if num_stages < 1:
        raise ValueError("pipeline needs at least one stage")
    if microbatches < 1:
        raise ValueError("pipeline needs at least one microbatch")
    dag = NodeDag(num_stages=num_stages)
    ids: Dict[Tuple[int, int, int], int] = {}
    order: List[List[int]] = [[] for _ in range(num_stages)]
    for s in range(num_stages):
        seq = one_f_one_b_stage_stream(num_stages, microbatches, s) if one_f_one_b else all_f_all_b_stage_stream(microbatches)
        for kind, m in seq:
            cid = len(dag.computations)
            dag.computations.append(Computation(cid, s, m, kind))
            ids[(s, int(kind), m)] = cid
            order[s].append(cid)
    for s in range(num_stages):
        for a, b in zip(order[s], order[s][1:]):
            dag.edges.append((a, b))
    for s in range(num_stages - 1):
        for m in range(microbatches):
            dag.edges.append((ids[(s, Kind.Forward, m)], ids[(s + 1, Kind.Forward, m)]))
            dag.edges.append((ids[(s + 1, Kind.Backward, m)], ids[(s, Kind.Backward, m)]))
    for s in range(num_stages):
        dag.edges.append((dag.source_id(), order[s][0]))
        dag.edges.append((order[s][-1], dag.sink_id()))
    _topo_check(dag.node_count(), dag.edges)
    return dag


def build_1f1b(num_stages: int, microbatches: int) -> NodeDag:
    return build_pipeline(num_stages, microbatches, True)


def build_gpipe(num_stages: int, microbatches: int) -> NodeDag:
    return build_pipeline(num_stages, microbatches, False)


def finalize_custom_dag(computations: Sequence[Computation], edges: Sequence[Tuple[int, int]]) -> NodeDag:
    """dag.hpp:158-191: validate, sort by id, attach virtual endpoints."""
    n = len(computations)
    if n == 0:
        raise ValueError("dag needs at least one computation")
    seen = [False] * n
    for c in computations:
        if c.id < 0 or c.id >= n or seen[c.id]:
            raise ValueError("computation ids must be dense and unique")
        seen[c.id] = True
        if c.stage < 0:
            raise ValueError("stage must be non-negative")
        if c.kind != Kind.Constant and c.microbatch is None:
            raise ValueError("forward/backward computations need a microbatch index")
        if c.microbatch is not None and c.microbatch < 0:
            raise ValueError("microbatch must be non-negative")
    comps = sorted(computations, key=lambda c: c.id)
    indeg = [0] * n
    outdeg = [0] * n
    for u, v in edges:
        if u < 0 or u >= n or v < 0 or v >= n:
            raise ValueError("edge references unknown computation")
        if u == v:
            raise ValueError("self-dependency")
        outdeg[u] += 1
        indeg[v] += 1
    dag = NodeDag(list(comps), list(edges), 0)
    dag.num_stages = max(c.stage + 1 for c in comps)
    for v in range(n):
        if indeg[v] == 0:
            dag.edges.append((dag.source_id(), v))
        if outdeg[v] == 0:
            dag.edges.append((v, dag.sink_id()))
    _topo_check(dag.node_count(), dag.edges)
    return dag


# ----------------------------------------------------------------- cost model

@dataclass
class ProfilePoint:
    """costmodel.hpp:17-21."""
    freq_mhz: int = 0
    time: int = 0
    energy: int = 0


@dataclass(frozen=True, order=True)
class ClassKey:
    """costmodel.hpp:24-28: computations sharing (stage, kind) share a profile."""
    stage: int = 0
    kind: int = int(Kind.Forward)


def class_of(c: Computation) -> ClassKey:
    return ClassKey(c.stage, int(c.kind))


@dataclass
class FrequencyProfile:
    key: ClassKey
    points: List[ProfilePoint]


@dataclass
class ProfileSet:
    p_blocking_watts: float = 75.0
    profiles: List[FrequencyProfile] = field(default_factory=list)


@dataclass
class ExpCurve:
    """e(t) = a exp(b t) + c on [t_min, t_max] (costmodel.hpp:39-48)."""
    a: float = 0.0
    b: float = 0.0
    c: float = 0.0
    t_min: int = 0
    t_max: int = 0
    rmse: float = 0.0


@dataclass
class ClassModel:
    is_constant: bool = False
    raw: List[ProfilePoint] = field(default_factory=list)
    pareto: List[ProfilePoint] = field(default_factory=list)
    curve: Optional[ExpCurve] = None

    def fastest(self) -> ProfilePoint:
        return self.pareto[0]

    def min_energy(self) -> ProfilePoint:
        return self.pareto[-1]


def validate_profile(p: FrequencyProfile) -> None:
    """costmodel.hpp:54-66."""
    if not p.points:
        raise ValueError("profile has no points")
    for pt in p.points:
        if pt.freq_mhz <= 0 or pt.time <= 0 or pt.energy <= 0:
            raise ValueError("profile points must have positive frequency, time, and energy")
    for a, b in zip(p.points, p.points[1:]):
        if a.freq_mhz <= b.freq_mhz:
            raise ValueError("profile frequencies must be strictly decreasing")
    if p.key.kind == Kind.Constant and len(p.points) != 1:
        raise ValueError("constant classes have exactly one operating point")
    if p.key.kind != Kind.Constant and len(p.points) < 2:
        raise ValueError("variable-frequency classes need at least two points")


def pareto_filter(points: Sequence[ProfilePoint]) -> List[ProfilePoint]:
    """costmodel.hpp:70-81, computed by the native library."""
    n = len(points)
    f = np.array([p.freq_mhz for p in points], dtype=np.int32)
    t = np.array([p.time for p in points], dtype=np.int64)
    e = np.array([p.energy for p in points], dtype=np.int64)
    of, ot, oe = np.zeros(n, np.int32), np.zeros(n, np.int64), np.zeros(n, np.int64)
    k = N.lib.pb_pareto_filter(n, N.ptr(f, C.c_int32), N.ptr(t, C.c_int64), N.ptr(e, C.c_int64),
                               N.ptr(of, C.c_int32), N.ptr(ot, C.c_int64), N.ptr(oe, C.c_int64))
    return [ProfilePoint(int(of[i]), int(ot[i]), int(oe[i])) for i in range(k)]


def fit_exp(pareto: Sequence[ProfilePoint]) -> ExpCurve:
    """costmodel.hpp:87-149, computed by the native library (bit-exact libm)."""
    n = len(pareto)
    t = np.array([p.time for p in pareto], dtype=np.int64)
    e = np.array([p.energy for p in pareto], dtype=np.int64)
    out = np.zeros(4, np.float64)
    N.check(N.lib.pb_fit_exp(n, N.ptr(t, C.c_int64), N.ptr(e, C.c_int64), N.ptr(out, C.c_double)))
    return ExpCurve(float(out[0]), float(out[1]), float(out[2]), int(t.min()), int(t.max()), float(out[3]))


@dataclass
class CostModel:
    """costmodel.hpp:194-239."""
    classes: Dict[ClassKey, ClassModel] = field(default_factory=dict)
    blocking_watts: float = 75.0
    quantum_us: int = 1

    def require(self, key: ClassKey) -> ClassModel:
        if key not in self.classes:
            raise ValueError("missing profile for a computation class")
        return self.classes[key]

    @staticmethod
    def build(pset: ProfileSet, quantum_us: int = 1) -> "CostModel":
        model = CostModel(blocking_watts=pset.p_blocking_watts, quantum_us=quantum_us)
        for prof in pset.profiles:
            validate_profile(prof)
            if prof.key in model.classes:
                raise ValueError("duplicate profile class")
            cm = ClassModel(raw=list(prof.points), pareto=pareto_filter(prof.points))
            if prof.key.kind == Kind.Constant or len(cm.pareto) == 1:
                cm.is_constant = True
            else:
                try:
                    cm.curve = fit_exp(cm.pareto)
                except N.DegenerateFit:
                    cm.is_constant = True
                    cm.pareto = [cm.pareto[0]]
            model.classes[prof.key] = cm
        return model


# ------------------------------------------------------------ flat packing

class PackedInstance:
    """Flat arrays of pb_instance_desc (include/perseus_b200.h) for one
    (NodeDag, CostModel, tau); owns the numpy buffers the desc points into."""

    def __init__(self, dag: NodeDag, model: CostModel, tau: int,
                 start_planned_t: Optional[Sequence[int]] = None, max_steps: int = 0):
        keys = sorted(model.classes.keys())
        index = {k: i for i, k in enumerate(keys)}
        n = len(dag.computations)
        cls = np.zeros(n, np.int32)
        for c in dag.computations:
            k = class_of(c)
            if k not in index:
                raise ValueError("missing profile for a computation class")
            cls[c.id] = index[k]
        self.n = n
        self.comp_class = cls
        e = np.array(dag.edges, dtype=np.int32).reshape(-1, 2)
        self.edge_tail = np.ascontiguousarray(e[:, 0])
        self.edge_head = np.ascontiguousarray(e[:, 1])
        nc = len(keys)
        self.cls_const = np.zeros(max(nc, 1), np.uint8)
        off = [0]
        freq: List[int] = []
        time: List[int] = []
        energy: List[int] = []
        curve = np.zeros(3 * max(nc, 1), np.float64)
        trange = np.zeros(2 * max(nc, 1), np.int64)
        for i, k in enumerate(keys):
            cm = model.classes[k]
            self.cls_const[i] = 1 if cm.is_constant else 0
            for p in cm.pareto:
                freq.append(p.freq_mhz)
                time.append(p.time)
                energy.append(p.energy)
            off.append(len(time))
            if not cm.is_constant:
                curve[3 * i:3 * i + 3] = (cm.curve.a, cm.curve.b, cm.curve.c)
                trange[2 * i:2 * i + 2] = (cm.curve.t_min, cm.curve.t_max)
        self.n_classes = nc
        self.cls_pt_off = np.array(off, np.int32)
        self.pt_freq = np.array(freq or [0], np.int32)
        self.pt_time = np.array(time or [0], np.int64)
        self.pt_energy = np.array(energy or [0], np.int64)
        self.curve = curve
        self.trange = trange
        self.start = None if start_planned_t is None else np.array(start_planned_t, np.int64)
        d = N.InstanceDesc()
        d.n = n
        d.comp_class = N.ptr(self.comp_class, C.c_int32)
        d.n_edges = len(self.edge_tail)
        d.edge_tail = N.ptr(self.edge_tail, C.c_int32)
        d.edge_head = N.ptr(self.edge_head, C.c_int32)
        d.n_classes = nc
        d.class_is_constant = N.ptr(self.cls_const, C.c_uint8)
        d.class_point_off = N.ptr(self.cls_pt_off, C.c_int32)
        d.point_freq = N.ptr(self.pt_freq, C.c_int32)
        d.point_time = N.ptr(self.pt_time, C.c_int64)
        d.point_energy = N.ptr(self.pt_energy, C.c_int64)
        d.class_curve = N.ptr(self.curve, C.c_double)
        d.class_t_range = N.ptr(self.trange, C.c_int64)
        d.blocking_watts = float(model.blocking_watts)
        d.quantum_us = int(model.quantum_us)
        d.tau = int(tau)
        d.start_planned_t = N.ptr(self.start, C.c_int64) if self.start is not None else None
        d.max_steps = int(max_steps)
        self.desc = d
