"""The frontier API, mirroring /root/reference/proj/include/perseus/frontier.hpp.

``discover_frontier`` (frontier.hpp:166-189), ``get_next_schedule``
(:90-135), ``discretize`` (:140-161), ``min_energy_schedule`` (:73-83),
``all_max_schedule`` (:193-206) and ``lookup`` (:212-220) keep the
reference's names, argument meaning and error behaviour; every walk runs on
the GPU through the C ABI (``FrontierBatch``).  ``FrontierBatch`` is the
batched form that the benchmark and the multi-instance callers use: one CTA
per instance, a delta-encoded frontier per instance.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _native as N
from .model import CostModel, NodeDag, PackedInstance, class_of


@dataclass
class EnergySchedule:
    """frontier.hpp:20-33."""
    schedule_id: int = 0
    planned_t: List[int] = field(default_factory=list)
    planned_e: List[int] = field(default_factory=list)
    freq_mhz: List[int] = field(default_factory=list)
    realized_t: List[int] = field(default_factory=list)
    realized_e: List[int] = field(default_factory=list)
    t_planned: int = 0
    t_realized: int = 0
    eff_planned_mj: float = 0.0
    eff_realized_mj: float = 0.0

    def discretized(self) -> bool:
        return len(self.freq_mhz) > 0


@dataclass
class Frontier:
    """frontier.hpp:35-40 (+ the terminal reason, which the reference does not expose)."""
    schedules: List[EnergySchedule] = field(default_factory=list)
    t_min: int = 0
    t_star: int = 0
    steps: int = 0
    stop: str = "at_t_min"


@dataclass
class StepInfo:
    """frontier.hpp:43-47."""
    cut_cost: int = 0
    sped_up: List[int] = field(default_factory=list)
    slowed_down: List[int] = field(default_factory=list)


class _G9Meta:
    def __init__(self, n: int):
        self.n = n


class FrontierBatch:
    """A batch of independent frontier walks on one device (pb_batch)."""

    def __init__(self):
        h = C.c_void_p()
        N.check(N.lib.pb_batch_create(C.byref(h)))
        self._h = h
        self._packed: List[PackedInstance] = []
        self._ran = False

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib.pb_batch_destroy(h)
            self._h = None

    def __len__(self) -> int:
        return len(self._packed)

    def add(self, dag: NodeDag, model: CostModel, tau: int = 1000,
            start_planned_t: Optional[Sequence[int]] = None, max_steps: int = 0) -> int:
        if tau <= 0:
            raise ValueError("tau must be positive")
        p = PackedInstance(dag, model, tau, start_planned_t, max_steps)
        idx = C.c_int32()
        N.check(N.lib.pb_batch_add(self._h, C.byref(p.desc), C.byref(idx)))
        self._packed.append(p)
        return idx.value

    def clear(self) -> None:
        """Drops every instance and result; the device context is kept
        (pb_batch_clear)."""
        N.check(N.lib.pb_batch_clear(self._h))
        self._packed = []
        self._ran = False

    def add_g9(self, p, tau: int = 1000) -> int:
        """Appends a G9 instance built natively (pb_batch_add_g9)."""
        idx = C.c_int32()
        N.check(N.lib.pb_batch_add_g9(self._h, p.stages, p.microbatches, p.base, p.imbalance, p.seed,
                                      p.straggler_stage, p.phi, tau, C.byref(idx)))
        self._packed.append(_G9Meta(2 * p.stages * p.microbatches))
        return idx.value

    def add_packed(self, p: PackedInstance) -> int:
        idx = C.c_int32()
        N.check(N.lib.pb_batch_add(self._h, C.byref(p.desc), C.byref(idx)))
        self._packed.append(p)
        return idx.value

    # -- execution
    def run(self, device: int = 0) -> "FrontierBatch":
        N.check(N.lib.pb_batch_run(self._h, device))
        self._ran = True
        return self

    def run_multi(self, devices: Sequence[int]) -> "FrontierBatch":
        arr = np.array(list(devices), np.int32)
        N.check(N.lib.pb_batch_run_multi(self._h, len(arr), N.ptr(arr, C.c_int32)))
        self._ran = True
        return self

    def prepare(self, device: int = 0) -> None:
        N.check(N.lib.pb_batch_prepare(self._h, device))

    def launch(self) -> float:
        ms = C.c_double()
        N.check(N.lib.pb_batch_launch(self._h, C.byref(ms)))
        return ms.value

    def fetch(self) -> None:
        N.check(N.lib.pb_batch_fetch(self._h))
        self._ran = True

    def stats(self) -> N.RunStats:
        s = N.RunStats()
        N.check(N.lib.pb_batch_stats(self._h, C.byref(s)))
        return s

    def profile(self) -> np.ndarray:
        """Per-phase device profile of the last launch (pb_batch_profile, 16 slots)."""
        out = np.zeros(16, np.int64)
        N.check(N.lib.pb_batch_profile(self._h, N.ptr(out, C.c_int64), 16))
        return out

    def straggler(self, factors, pipelines: int, num_stages) -> np.ndarray:
        """straggler_savings (baselines.hpp:162-188) of every instance on the
        device-resident frontiers of the last run: rows[k, j] for factors[j]."""
        f = np.ascontiguousarray(factors, np.float64)
        st = np.ascontiguousarray(num_stages, np.int32)
        buf = (N.SavingsRow * (len(self) * len(f)))()
        N.check(N.lib.pb_batch_straggler(self._h, len(f), N.ptr(f, C.c_double), pipelines,
                                         N.ptr(st, C.c_int32), buf))
        return np.ctypeslib.as_array(buf).copy().reshape(len(self), len(f))

    def add_g9_batch(self, first: int, count: int, tau: int = 1000, threads: int = 0) -> None:
        """Config-5 instances [first, first + count), built on all host threads."""
        from . import g9
        N.check(N.lib.pb_batch_add_g9_batch(self._h, first, count, tau, threads))
        for i in range(first, first + count):
            p = g9.batch_params(i)
            self._packed.append(_G9Meta(2 * p.stages * p.microbatches))

    def add_g9_indices(self, indices, tau: int = 1000, threads: int = 0) -> None:
        """Config-5 instances ``indices`` (e.g. an LPT shard), built on all host threads."""
        from . import g9
        idx = np.ascontiguousarray(list(indices), np.int32)
        N.check(N.lib.pb_batch_add_g9_indices(self._h, N.ptr(idx, C.c_int32), len(idx), tau, threads))
        for i in idx.tolist():
            p = g9.batch_params(i)
            self._packed.append(_G9Meta(2 * p.stages * p.microbatches))

    def set_max_steps(self, max_steps: int) -> None:
        """Caps every instance's walk at max_steps steps (pb_batch_set_max_steps)."""
        N.check(N.lib.pb_batch_set_max_steps(self._h, max_steps))

    def digest(self, k: int) -> int:
        """64-bit digest of instance k's results (pb_batch_digest)."""
        d = C.c_uint64()
        N.check(N.lib.pb_batch_digest(self._h, k, C.byref(d)))
        return d.value

    def brute_force(self, k: int, budget: float = 1e7, device: int = 0):
        """brute_force_frontier (oracle.hpp:47-114) of instance k on the GPU:
        (points[time, eff_energy_mj, code], freq_mhz[point, computation])."""
        n = self._packed[k].n
        cnt = C.c_int32()
        N.check(N.lib.pb_batch_brute_force(self._h, k, budget, device, None, None, 0, C.byref(cnt)))
        pts = (N.ExactPoint * max(cnt.value, 1))()
        fr = np.zeros(max(cnt.value, 1) * n, np.int32)
        N.check(N.lib.pb_batch_brute_force(self._h, k, budget, device, pts, N.ptr(fr, C.c_int32), cnt.value,
                                           C.byref(cnt)))
        return np.ctypeslib.as_array(pts)[:cnt.value].copy(), fr[:cnt.value * n].reshape(cnt.value, n)

    def _text(self, fn, *args) -> str:
        n = C.c_int64()
        N.check(fn(self._h, *args, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        N.check(fn(self._h, *args, buf, n.value, C.byref(n)))
        return buf.raw[:n.value].decode()

    def frontier_csv(self, k: int, quantum_us: int = 1) -> str:
        """frontier.csv of instance k (serde.hpp frontier_csv)."""
        return self._text(N.lib.pb_batch_frontier_csv, k, quantum_us)

    def schedule_json(self, k: int, which: int, quantum_us: int = 1) -> str:
        """schedules/schedule_<which>.json of instance k (serde.hpp write_frontier_artifacts)."""
        return self._text(N.lib.pb_batch_schedule_json, k, which, quantum_us)

    # -- results
    def summary(self, k: int) -> N.FrontierSummary:
        s = N.FrontierSummary()
        N.check(N.lib.pb_batch_summary(self._h, k, C.byref(s)))
        return s

    def points(self, k: int) -> np.ndarray:
        s = self.summary(k)
        buf = (N.Point * (s.steps + 1))()
        N.check(N.lib.pb_batch_points(self._h, k, buf, s.steps + 1))
        return np.ctypeslib.as_array(buf).copy()

    def deltas(self, k: int):
        s = self.summary(k)
        ids = np.zeros(max(s.n_ids, 1), np.int32)
        ch = np.zeros(max(s.n_ids, 1), np.uint8)
        N.check(N.lib.pb_batch_deltas(self._h, k, N.ptr(ids, C.c_int32), N.ptr(ch, C.c_uint8), len(ids)))
        return ids[:s.n_ids], ch[:s.n_ids]

    def schedule(self, k: int, which: int) -> EnergySchedule:
        n = self._packed[k].n
        pt, pe, rt, re = (np.zeros(n, np.int64) for _ in range(4))
        fr = np.zeros(n, np.int32)
        ep, er = C.c_double(), C.c_double()
        N.check(N.lib.pb_batch_schedule(self._h, k, which, N.ptr(pt, C.c_int64), N.ptr(pe, C.c_int64),
                                        N.ptr(fr, C.c_int32), N.ptr(rt, C.c_int64), N.ptr(re, C.c_int64),
                                        C.byref(ep), C.byref(er)))
        pts = self.points(k) if which else None
        p = pts[which] if pts is not None else self.points(k)[0]
        return EnergySchedule(which, pt.tolist(), pe.tolist(), fr.tolist(), rt.tolist(), re.tolist(),
                              int(p["t_planned"]), int(p["t_realized"]), ep.value, er.value)

    def step_info(self, k: int, step: int) -> StepInfo:
        """StepInfo of step ``step`` (1-based: the step producing point ``step``)."""
        pts = self.points(k)
        ids, _ = self.deltas(k)
        p = pts[step]
        seg = ids[p["id_begin"]:p["id_begin"] + p["n_sped"] + p["n_slowed"]]
        return StepInfo(int(p["cut_cost"]), [int(x) - 1 for x in seg if x > 0],
                        [int(-x) - 1 for x in seg if x < 0])

    def schedules(self, k: int, first: int = 0, count: int | None = None) -> list:
        """Schedules first .. first + count - 1 of instance k in ONE incremental
        replay of the delta log (pb_batch_schedules)."""
        s = self.summary(k)
        if count is None:
            count = s.steps + 1 - first
        n = self._packed[k].n
        pt, pe, rt, re = (np.zeros((count, n), np.int64) for _ in range(4))
        fr = np.zeros((count, n), np.int32)
        ep, er = np.zeros(count), np.zeros(count)
        N.check(N.lib.pb_batch_schedules(self._h, k, first, count, N.ptr(pt, C.c_int64), N.ptr(pe, C.c_int64),
                                         N.ptr(fr, C.c_int32), N.ptr(rt, C.c_int64), N.ptr(re, C.c_int64),
                                         N.ptr(ep, C.c_double), N.ptr(er, C.c_double)))
        pts = self.points(k)
        return [EnergySchedule(first + q, pt[q].tolist(), pe[q].tolist(), fr[q].tolist(), rt[q].tolist(),
                               re[q].tolist(), int(pts[first + q]["t_planned"]), int(pts[first + q]["t_realized"]),
                               float(ep[q]), float(er[q])) for q in range(count)]

    def frontier(self, k: int) -> Frontier:
        s = self.summary(k)
        N.raise_for_instance_status(s.status)
        f = Frontier(t_min=int(s.t_min), t_star=int(s.t_star), steps=int(s.steps),
                     stop=N.STOP_NAMES.get(s.stop, str(s.stop)))
        f.schedules = self.schedules(k)
        return f


# ------------------------------------------------------------------ the API

_local = threading.local()


def _handle() -> FrontierBatch:
    """The calling thread's persistent handle, emptied for each call (its
    stream and device / pinned buffers are reused), as the C++ drop-in does."""
    b = getattr(_local, "batch", None)
    if b is None:
        b = _local.batch = FrontierBatch()
    b.clear()
    return b


def discover_frontier(dag: NodeDag, model: CostModel, tau: int = 1000) -> Frontier:
    """frontier.hpp:166-189 on the device."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    b = _handle()
    b.add(dag, model, tau)
    b.run()
    return b.frontier(0)


def _single(dag, model, tau, planned, max_steps):
    b = _handle()
    b.add(dag, model, tau, start_planned_t=planned, max_steps=max_steps)
    b.run()
    s = b.summary(0)
    N.raise_for_instance_status(s.status)
    return b, s


def get_next_schedule(dag: NodeDag, schedule: EnergySchedule, model: CostModel, tau: int,
                      info: Optional[StepInfo] = None) -> Optional[EnergySchedule]:
    """frontier.hpp:90-135: one device step from ``schedule``; None when no finite cut exists."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    b, s = _single(dag, model, tau, schedule.planned_t, 1)
    if s.steps == 0:
        return None
    nxt = b.schedule(0, 1)
    step = b.step_info(0, 1)
    # planned_e carries over from the input except for touched computations
    pe = list(schedule.planned_e) if schedule.planned_e else list(nxt.planned_e)
    for c in step.sped_up + step.slowed_down:
        pe[c] = nxt.planned_e[c]
    out = EnergySchedule(schedule.schedule_id, nxt.planned_t, pe, [], [], [], nxt.t_planned, 0,
                         _eff(pe, nxt.planned_t, model), 0.0)
    if info is not None:
        info.cut_cost, info.sped_up, info.slowed_down = step.cut_cost, step.sped_up, step.slowed_down
    return out


def _eff(energies, times, model: CostModel) -> float:
    # detail::effective_total (frontier.hpp:51-57), index order
    total = 0.0
    for e, t in zip(energies, times):
        total += float(e) - model.blocking_watts * float(t) * float(model.quantum_us) * 1e-3
    return total


def discretize(schedule: EnergySchedule, dag: NodeDag, model: CostModel) -> EnergySchedule:
    """frontier.hpp:140-161 on the device (a zero-step walk from ``schedule``)."""
    b, _ = _single(dag, model, 1, schedule.planned_t, -1)
    d = b.schedule(0, 0)
    return EnergySchedule(schedule.schedule_id, list(schedule.planned_t), list(schedule.planned_e),
                          d.freq_mhz, d.realized_t, d.realized_e, schedule.t_planned, d.t_realized,
                          schedule.eff_planned_mj, d.eff_realized_mj)


def min_energy_schedule(dag: NodeDag, model: CostModel) -> EnergySchedule:
    """frontier.hpp:73-83 (not yet discretized)."""
    b = _handle()
    b.add(dag, model, 1, max_steps=-1)
    b.run()
    N.raise_for_instance_status(b.summary(0).status)
    d = b.schedule(0, 0)
    return EnergySchedule(0, d.planned_t, d.planned_e, [], [], [], d.t_planned, 0, d.eff_planned_mj, 0.0)


def all_max_schedule(dag: NodeDag, model: CostModel) -> EnergySchedule:
    """frontier.hpp:193-206: planned == realized at every class's fastest point."""
    fast = [model.require(class_of(c)).fastest() for c in dag.computations]
    b, _ = _single(dag, model, 1, [p.time for p in fast], -1)
    d = b.schedule(0, 0)
    e = [p.energy for p in fast]
    t = [p.time for p in fast]
    eff = _eff(e, t, model)
    return EnergySchedule(-1, t, e, [p.freq_mhz for p in fast], list(t), list(e), d.t_realized,
                          d.t_realized, eff, eff)


def lookup(frontier: Frontier, straggler_time: int) -> EnergySchedule:
    """frontier.hpp:212-220: first schedule with planned time <= min(T*, T')."""
    if not frontier.schedules:
        raise N.LogicError("frontier is empty")
    target = min(frontier.t_star, straggler_time)
    lo, hi = 0, len(frontier.schedules)
    while lo < hi:
        mid = (lo + hi) // 2
        if frontier.schedules[mid].t_planned > target:
            lo = mid + 1
        else:
            hi = mid
    return frontier.schedules[-1] if lo == len(frontier.schedules) else frontier.schedules[lo]
