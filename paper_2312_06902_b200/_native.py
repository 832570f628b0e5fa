"""ctypes binding of the product library ``_lib/libperseus_b200.so``.

The library is the C ABI declared in ``include/perseus_b200.h`` (CUDA kernels
for sm_100a + the native host packer).  There is no fallback: importing the
package on a machine where the library is missing raises immediately, and
every compute entry point needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PB_LIB_VARIANT selects an experimental build (_lib/libperseus_b200<variant>.so) for A/B timing.
LIB_PATH = os.path.join(_HERE, "_lib", f"libperseus_b200{os.environ.get('PB_LIB_VARIANT', '')}.so")

PB_OK = 0
PB_ERR_INVALID_ARGUMENT = 1
PB_ERR_OVERFLOW = 2
PB_ERR_LOGIC = 3
PB_ERR_DOMAIN = 4
PB_ERR_CUDA = 5
PB_ERR_UNSUPPORTED = 6
PB_ERR_BUDGET = 7

STOP_AT_TMIN = 0
STOP_INFEASIBLE = 1
STOP_INFINITE_CUT = 2
STOP_NO_PROGRESS = 3
STOP_STEP_LIMIT = 4
STOP_NAMES = {0: "at_t_min", 1: "infeasible", 2: "infinite_cut", 3: "no_progress", 4: "step_limit"}


class LogicError(RuntimeError):
    """std::logic_error (flow.hpp:265, frontier.hpp:213)."""


class DegenerateFit(ArithmeticError):
    """perseus::DegenerateFit, a std::domain_error (costmodel.hpp:50-52)."""


class CudaError(RuntimeError):
    """A device failure; no reference counterpart."""


class UnsupportedInput(NotImplementedError):
    """Documented divergence: a curve evaluated outside its profiled interval."""


class BudgetExceeded(RuntimeError):
    """perseus::BudgetExceeded (oracle.hpp:17-19)."""


_EXC = {
    PB_ERR_INVALID_ARGUMENT: ValueError,
    PB_ERR_OVERFLOW: OverflowError,
    PB_ERR_LOGIC: LogicError,
    PB_ERR_DOMAIN: DegenerateFit,
    PB_ERR_CUDA: CudaError,
    PB_ERR_UNSUPPORTED: UnsupportedInput,
    PB_ERR_BUDGET: BudgetExceeded,
}

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)
i8p = C.POINTER(C.c_int8)
f64p = C.POINTER(C.c_double)


class InstanceDesc(C.Structure):
    _fields_ = [
        ("n", C.c_int32),
        ("comp_class", i32p),
        ("n_edges", C.c_int32),
        ("edge_tail", i32p),
        ("edge_head", i32p),
        ("n_classes", C.c_int32),
        ("class_is_constant", u8p),
        ("class_point_off", i32p),
        ("point_freq", i32p),
        ("point_time", i64p),
        ("point_energy", i64p),
        ("class_curve", f64p),
        ("class_t_range", i64p),
        ("blocking_watts", C.c_double),
        ("quantum_us", C.c_int64),
        ("tau", C.c_int64),
        ("start_planned_t", i64p),
        ("max_steps", C.c_int32),
    ]


class FrontierSummary(C.Structure):
    _fields_ = [
        ("t_min", C.c_int64),
        ("t_star", C.c_int64),
        ("steps", C.c_int32),
        ("stop", C.c_int32),
        ("status", C.c_int32),
        ("n_ids", C.c_int32),
        ("n_table_misses", C.c_int32),
        ("walk_us", C.c_int32),
        ("warps", C.c_int32),
        ("start_us", C.c_int32),
    ]


class Point(C.Structure):
    _fields_ = [
        ("t_planned", C.c_int64),
        ("t_realized", C.c_int64),
        ("sum_planned_e", C.c_int64),
        ("sum_planned_t", C.c_int64),
        ("sum_realized_e", C.c_int64),
        ("sum_realized_t", C.c_int64),
        ("cut_cost", C.c_int64),
        ("step_size", C.c_int64),
        ("id_begin", C.c_int32),
        ("n_sped", C.c_int32),
        ("n_slowed", C.c_int32),
        ("pad", C.c_int32),
    ]


class RunStats(C.Structure):
    _fields_ = [
        ("kernel_ms", C.c_double),
        ("h2d_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("h2d_bytes", C.c_int64),
        ("d2h_bytes", C.c_int64),
        ("arc_scans", C.c_int64),
        ("node_updates", C.c_int64),
        ("rounds", C.c_int64),
        ("kernel_launches", C.c_int64),
        ("comp_visits", C.c_int64),
        ("smem_walks", C.c_int64),
        ("wide_walks", C.c_int64),
        ("smem_region", C.c_int64),
        ("pack_ms", C.c_double),
        ("warm_starts", C.c_int64),
    ]


class SavingsRow(C.Structure):
    _fields_ = [
        ("factor", C.c_double),
        ("savings_pct", C.c_double),
        ("savings_mj", C.c_double),
        ("all_max_mj", C.c_double),
        ("tuned_mj", C.c_double),
        ("point", C.c_int32),
        ("status", C.c_int32),
    ]


class ExactPoint(C.Structure):
    _fields_ = [("time", C.c_int64), ("eff_energy_mj", C.c_double), ("code", C.c_int64)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sig = {
        "pb_last_error": (C.c_char_p, []),
        "pb_version": (C.c_char_p, []),
        "pb_pareto_filter": (C.c_int32, [C.c_int32, i32p, i64p, i64p, i32p, i64p, i64p]),
        "pb_fit_exp": (C.c_int, [C.c_int32, i64p, i64p, f64p]),
        "pb_batch_create": (C.c_int, [C.POINTER(P)]),
        "pb_batch_add": (C.c_int, [P, C.POINTER(InstanceDesc), i32p]),
        "pb_batch_run": (C.c_int, [P, C.c_int32]),
        "pb_batch_prepare": (C.c_int, [P, C.c_int32]),
        "pb_batch_launch": (C.c_int, [P, f64p]),
        "pb_batch_fetch": (C.c_int, [P]),
        "pb_batch_size": (C.c_int32, [P]),
        "pb_batch_run_multi": (C.c_int, [P, C.c_int32, i32p]),
        "pb_batch_summary": (C.c_int, [P, C.c_int32, C.POINTER(FrontierSummary)]),
        "pb_batch_points": (C.c_int, [P, C.c_int32, C.POINTER(Point), C.c_int32]),
        "pb_batch_deltas": (C.c_int, [P, C.c_int32, i32p, u8p, C.c_int32]),
        "pb_batch_schedule": (C.c_int, [P, C.c_int32, C.c_int32, i64p, i64p, i32p, i64p, i64p, f64p, f64p]),
        "pb_batch_stats": (C.c_int, [P, C.POINTER(RunStats)]),
        "pb_batch_profile": (C.c_int, [P, i64p, C.c_int32]),
        "pb_batch_straggler": (C.c_int, [P, C.c_int32, f64p, C.c_int32, i32p, C.POINTER(SavingsRow)]),
        "pb_batch_frontier_csv": (C.c_int, [P, C.c_int32, C.c_int64, C.c_char_p, C.c_int64, i64p]),
        "pb_batch_add_g9_batch": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int64, C.c_int32]),
        "pb_batch_add_g9_indices": (C.c_int, [P, i32p, C.c_int32, C.c_int64, C.c_int32]),
        "pb_batch_digest": (C.c_int, [P, C.c_int32, C.POINTER(C.c_uint64)]),
        "pb_batch_set_max_steps": (C.c_int, [P, C.c_int32]),
        "pb_batch_brute_force": (C.c_int, [P, C.c_int32, C.c_double, C.c_int32, C.POINTER(ExactPoint), i32p,
                                           C.c_int32, i32p]),
        "pb_batch_schedule_json": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int64, C.c_char_p, C.c_int64, i64p]),
        "pb_batch_destroy": (None, [P]),
        "pb_batch_clear": (C.c_int, [P]),
        "pb_batch_schedules": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, i64p, i64p, i32p, i64p, i64p, f64p,
                                         f64p]),
        "pb_annotate_slack_batch": (C.c_int, [C.c_int32, C.c_int32, i32p, i32p, i32p, i32p, i64p,
                                              i64p, i64p, u8p, i64p]),
        "pb_flow_min_cut_batch": (C.c_int, [C.c_int32, C.c_int32, i32p, i32p, i32p, i32p, i32p, i32p,
                                            i64p, i64p, u8p, i32p, u8p, i64p, i64p, i64p, u8p, i8p]),
        "pb_g9_stage_bases": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_uint32, C.c_int32,
                                        C.c_double, i32p]),
        "pb_g9_batch_params": (C.c_int, [C.c_int32, i32p, i32p, f64p, f64p, i32p, C.POINTER(C.c_uint32)]),
        "pb_g9_profile": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, i32p, i64p, i64p]),
        "pb_batch_add_g9": (C.c_int, [P, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_uint32, C.c_int32,
                                      C.c_double, C.c_int64, i32p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

# Every symbol the public header declares; tests check the library exports them.
EXPORTED = (
    "pb_last_error", "pb_version", "pb_pareto_filter", "pb_fit_exp", "pb_batch_create", "pb_batch_add",
    "pb_batch_run", "pb_batch_prepare", "pb_batch_launch", "pb_batch_fetch", "pb_batch_size",
    "pb_batch_run_multi", "pb_batch_summary", "pb_batch_points", "pb_batch_deltas", "pb_batch_schedule",
    "pb_batch_stats", "pb_batch_profile", "pb_batch_destroy", "pb_batch_clear", "pb_batch_schedules",
    "pb_annotate_slack_batch", "pb_flow_min_cut_batch",
    "pb_g9_stage_bases", "pb_g9_batch_params", "pb_g9_profile", "pb_batch_add_g9", "pb_batch_straggler",
    "pb_batch_frontier_csv", "pb_batch_schedule_json", "pb_batch_brute_force",
    "pb_batch_add_g9_batch", "pb_batch_add_g9_indices", "pb_batch_digest", "pb_batch_set_max_steps",
)


def check(status: int) -> None:
    if status == PB_OK:
        return
    msg = lib.pb_last_error().decode() or f"pb status {status}"
    raise _EXC.get(status, RuntimeError)(msg)


def raise_for_instance_status(status: int) -> None:
    if status == PB_OK:
        return
    raise _EXC.get(status, RuntimeError)(f"frontier walk failed with status {status}")


def ptr(arr, ctype):
    """ctypes pointer to a contiguous numpy array (kept alive by the caller)."""
    return arr.ctypes.data_as(C.POINTER(ctype))
