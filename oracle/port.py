"""TEST INFRASTRUCTURE -- ctypes wrapper of the C restatement
(oracle/perseus_oracle.c -> oracle/_build/libperseus_oracle.so) and of the
reference driver binary (oracle/_ref/ref_driver).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from typing import Dict, List

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "libperseus_oracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ref_driver")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)
f64p = C.POINTER(C.c_double)
u64p = C.POINTER(C.c_uint64)

STOP = {0: "at_t_min", 1: "infeasible", 2: "infinite_cut", 3: "no_progress"}


class OrInstance(C.Structure):
    _fields_ = [("n", C.c_int), ("cls", i32p), ("ne", C.c_int), ("et", i32p), ("eh", i32p),
                ("ncls", C.c_int), ("is_const", u8p), ("pt_off", i32p), ("pt_freq", i32p),
                ("pt_time", i64p), ("pt_energy", i64p), ("curve", f64p), ("t_range", i64p),
                ("watts", C.c_double), ("quantum", C.c_int64)]


class OrWalkOut(C.Structure):
    _fields_ = [("t_min", C.c_int64), ("t_star", C.c_int64), ("steps", C.c_int32), ("stop", C.c_int32),
                ("t_planned", i64p), ("t_realized", i64p), ("eff_planned", f64p), ("eff_realized", f64p),
                ("sum_planned_e", i64p), ("sum_realized_e", i64p), ("hash", u64p), ("cut_cost", i64p),
                ("step_size", i64p), ("id_off", i32p), ("ids", i32p), ("final_planned_t", i64p),
                ("final_freq", i32p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(PORT_LIB):
            raise ImportError(f"{PORT_LIB} missing: run `make -C oracle port`")
        L = C.CDLL(PORT_LIB)
        L.or_pareto_filter.argtypes = [C.c_int, i32p, i64p, i64p, i32p, i64p, i64p]
        L.or_pareto_filter.restype = C.c_int
        L.or_fit_exp.argtypes = [C.c_int, i64p, i64p, f64p]
        L.or_fit_exp.restype = C.c_int
        L.or_annotate_slack.argtypes = [C.c_int, C.c_int, i32p, i32p, i64p, i64p, i64p, u8p, i64p]
        L.or_annotate_slack.restype = C.c_int
        L.or_flow_min_cut.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p, i64p, i64p, u8p,
                                      C.POINTER(C.c_int), i64p, i64p, u8p, i32p, C.POINTER(C.c_int), i32p,
                                      C.POINTER(C.c_int), i64p]
        L.or_flow_min_cut.restype = C.c_int
        L.or_discover_frontier.argtypes = [C.POINTER(OrInstance), C.c_int64, C.c_int, C.c_int,
                                           C.POINTER(OrWalkOut), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.or_discover_frontier.restype = C.c_int
        L.or_lookup.argtypes = [C.c_int, i64p, C.c_int64, C.c_int64]
        L.or_lookup.restype = C.c_int
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def fit_exp(times, energies):
    t = np.asarray(times, np.int64)
    e = np.asarray(energies, np.int64)
    out = np.zeros(3, np.float64)
    rc = lib().or_fit_exp(len(t), _p(t, C.c_int64), _p(e, C.c_int64), _p(out, C.c_double))
    return rc, out


def pareto_filter(freq, time, energy):
    n = len(freq)
    f = np.asarray(freq, np.int32)
    t = np.asarray(time, np.int64)
    e = np.asarray(energy, np.int64)
    of, ot, oe = np.zeros(n, np.int32), np.zeros(n, np.int64), np.zeros(n, np.int64)
    k = lib().or_pareto_filter(n, _p(f, C.c_int32), _p(t, C.c_int64), _p(e, C.c_int64),
                               _p(of, C.c_int32), _p(ot, C.c_int64), _p(oe, C.c_int64))
    return of[:k].tolist(), ot[:k].tolist(), oe[:k].tolist()


def annotate_slack(n, edges, durations):
    e = np.asarray(edges, np.int32).reshape(-1, 2)
    et = np.ascontiguousarray(e[:, 0])
    eh = np.ascontiguousarray(e[:, 1])
    d = np.asarray(durations, np.int64)
    V, E = 2 * n + 2, n + len(et)
    ea, la = np.zeros(V, np.int64), np.zeros(V, np.int64)
    cr = np.zeros(E, np.uint8)
    ms = np.zeros(1, np.int64)
    rc = lib().or_annotate_slack(n, len(et), _p(et, C.c_int32), _p(eh, C.c_int32), _p(d, C.c_int64),
                                 _p(ea, C.c_int64), _p(la, C.c_int64), _p(cr, C.c_uint8), _p(ms, C.c_int64))
    return rc, ea, la, cr, int(ms[0])


def flow_min_cut(nodes, s, t, edges):
    """edges: list of (tail, head, lower, upper, infinite)."""
    m = len(edges)
    arr = np.array(edges, dtype=np.int64).reshape(-1, 5)
    tl = np.ascontiguousarray(arr[:, 0].astype(np.int32))
    hd = np.ascontiguousarray(arr[:, 1].astype(np.int32))
    lo = np.ascontiguousarray(arr[:, 2])
    up = np.ascontiguousarray(arr[:, 3])
    inf = np.ascontiguousarray(arr[:, 4].astype(np.uint8))
    feas = C.c_int()
    val = np.zeros(1, np.int64)
    sent = np.zeros(1, np.int64)
    side = np.zeros(nodes, np.uint8)
    sp = np.zeros(max(m, 1), np.int32)
    sl = np.zeros(max(m, 1), np.int32)
    nsp, nsl = C.c_int(), C.c_int()
    cost = np.zeros(1, np.int64)
    rc = lib().or_flow_min_cut(nodes, s, t, m, _p(tl, C.c_int32), _p(hd, C.c_int32), _p(lo, C.c_int64),
                               _p(up, C.c_int64), _p(inf, C.c_uint8), C.byref(feas), _p(val, C.c_int64),
                               _p(sent, C.c_int64), _p(side, C.c_uint8), _p(sp, C.c_int32), C.byref(nsp),
                               _p(sl, C.c_int32), C.byref(nsl), _p(cost, C.c_int64))
    return {"rc": rc, "feasible": bool(feas.value), "value": int(val[0]), "sentinel": int(sent[0]),
            "source_side": side.tolist(), "speed_up": sp[:nsp.value].tolist(),
            "slow_down": sl[:nsl.value].tolist(), "cost": int(cost[0])}


class _Keep:
    pass


def _instance(packed):
    """OrInstance view of a product PackedInstance (same flat arrays)."""
    k = _Keep()
    k.cls = packed.comp_class
    k.et = packed.edge_tail
    k.eh = packed.edge_head
    k.isc = packed.cls_const
    k.off = packed.cls_pt_off
    k.f = packed.pt_freq
    k.t = packed.pt_time
    k.e = packed.pt_energy
    k.curve = packed.curve
    k.tr = packed.trange
    I = OrInstance(packed.n, _p(k.cls, C.c_int32), len(k.et), _p(k.et, C.c_int32), _p(k.eh, C.c_int32),
                   packed.n_classes, _p(k.isc, C.c_uint8), _p(k.off, C.c_int32), _p(k.f, C.c_int32),
                   _p(k.t, C.c_int64), _p(k.e, C.c_int64), _p(k.curve, C.c_double), _p(k.tr, C.c_int64),
                   float(packed.desc.blocking_watts), int(packed.desc.quantum_us))
    return I, k


def discover_frontier(packed, tau: int, max_points: int = 0) -> Dict:
    """The restated walk (frontier.hpp:166-189) over a PackedInstance's arrays."""
    I, keep = _instance(packed)
    cap = max_points or 64
    while True:
        ids_cap = cap * 16 + packed.n + 16
        bufs = {
            "t_planned": np.zeros(cap, np.int64), "t_realized": np.zeros(cap, np.int64),
            "eff_planned": np.zeros(cap, np.float64), "eff_realized": np.zeros(cap, np.float64),
            "sum_planned_e": np.zeros(cap, np.int64), "sum_realized_e": np.zeros(cap, np.int64),
            "hash": np.zeros(cap, np.uint64), "cut_cost": np.zeros(cap, np.int64),
            "step_size": np.zeros(cap, np.int64), "id_off": np.zeros(cap + 1, np.int32),
            "ids": np.zeros(ids_cap, np.int32), "final_planned_t": np.zeros(packed.n, np.int64),
            "final_freq": np.zeros(packed.n, np.int32),
        }
        out = OrWalkOut()
        types = {np.int64: C.c_int64, np.float64: C.c_double, np.uint64: C.c_uint64, np.int32: C.c_int32}
        for name, arr in bufs.items():
            setattr(out, name, _p(arr, types[arr.dtype.type]))
        npts, nids = C.c_int(), C.c_int()
        rc = lib().or_discover_frontier(C.byref(I), tau, cap, ids_cap, C.byref(out), C.byref(npts),
                                        C.byref(nids))
        if rc == 4:  # OR_CAPACITY
            cap = max(cap * 2, npts.value + 1)
            continue
        if rc != 0:
            return {"rc": rc}
        P = npts.value
        steps = out.steps
        res = {"rc": 0, "t_min": out.t_min, "t_star": out.t_star, "steps": steps, "reason": STOP[out.stop]}
        for name in ("t_planned", "t_realized", "eff_planned", "eff_realized", "sum_planned_e",
                     "sum_realized_e"):
            res[name] = bufs[name][:P].tolist()
        res["hash"] = [f"{int(h):016x}" for h in bufs["hash"][:P]]
        res["cut_cost"] = bufs["cut_cost"][:steps].tolist()
        res["step_size"] = bufs["step_size"][:steps].tolist()
        off = bufs["id_off"][:steps + 1]
        ids = bufs["ids"]
        res["sped"] = [[int(x) - 1 for x in ids[off[k]:off[k + 1]] if x > 0] for k in range(steps)]
        res["slowed"] = [[int(-x) - 1 for x in ids[off[k]:off[k + 1]] if x < 0] for k in range(steps)]
        res["final_planned_t"] = bufs["final_planned_t"].tolist()
        res["final_freq"] = bufs["final_freq"].tolist()
        return res


def have_ref_driver() -> bool:
    return os.path.exists(REF_DRIVER)


def ref_driver(*args: str, timeout: float = 3600) -> List[Dict]:
    """Runs the reference driver and parses its JSON lines."""
    out = subprocess.run([REF_DRIVER, *args], check=True, capture_output=True, text=True, timeout=timeout)
    return [json.loads(line) for line in out.stdout.splitlines() if line.strip()]


def schedule_hash(planned_t, planned_e, freq, realized_t, realized_e) -> str:
    """FNV-1a over int64 words (ref_driver.cpp schedule_hash)."""
    h = 1469598103934665603
    M = (1 << 64) - 1
    for seq in (planned_t, planned_e, freq, realized_t, realized_e):
        for v in seq:
            u = int(v) & M
            for i in range(8):
                h ^= (u >> (8 * i)) & 0xFF
                h = (h * 1099511628211) & M
    return f"{h:016x}"
