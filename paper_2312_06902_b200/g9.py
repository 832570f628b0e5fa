"""G9 synthetic workloads, drawn by the native generator
(``csrc/g9.hpp``) so that the reference driver and this package see
bit-identical instances."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List

import numpy as np

from . import _native as N
from .model import ClassKey, CostModel, FrequencyProfile, Kind, NodeDag, ProfilePoint, ProfileSet, build_1f1b

TAU = 1000


@dataclass
class G9Params:
    stages: int = 4
    microbatches: int = 8
    base: int = 10
    imbalance: float = 1.2
    seed: int = 1234
    straggler_stage: int = -1
    phi: float = 1.0

    def spec(self) -> str:
        """The reference driver's instance spec (oracle/ref_driver.cpp)."""
        return (f"g9:{self.stages}:{self.microbatches}:{self.base}:{self.imbalance!r}:{self.seed}:"
                f"{self.straggler_stage}:{self.phi!r}")


NAMED = {
    1: G9Params(4, 8, 10, 1.2, 1234),
    2: G9Params(8, 32, 10, 1.2, 1234),
    3: G9Params(8, 128, 33, 1.03, 1234),
    4: G9Params(16, 128, 10, 1.10, 1234),
}


def named_config(k: int, phi: float = 1.0) -> G9Params:
    p = NAMED[k]
    q = G9Params(p.stages, p.microbatches, p.base, p.imbalance, p.seed)
    if k == 4 and phi != 1.0:
        q.straggler_stage, q.phi = 8, phi
    return q


def batch_params(i: int) -> G9Params:
    s, m, st = C.c_int32(), C.c_int32(), C.c_int32()
    imb, phi = C.c_double(), C.c_double()
    seed = C.c_uint32()
    N.check(N.lib.pb_g9_batch_params(i, C.byref(s), C.byref(m), C.byref(imb), C.byref(phi),
                                     C.byref(st), C.byref(seed)))
    return G9Params(s.value, m.value, 10, imb.value, seed.value, st.value, phi.value)


def stage_bases(p: G9Params) -> List[int]:
    out = np.zeros(p.stages, np.int32)
    N.check(N.lib.pb_g9_stage_bases(p.stages, p.base, p.imbalance, p.seed, p.straggler_stage, p.phi,
                                    N.ptr(out, C.c_int32)))
    return out.tolist()


def stage_profile(b: int, backward: bool, tau: int = TAU) -> List[ProfilePoint]:
    f = np.zeros(9, np.int32)
    t = np.zeros(9, np.int64)
    e = np.zeros(9, np.int64)
    N.check(N.lib.pb_g9_profile(b, 1 if backward else 0, tau, N.ptr(f, C.c_int32), N.ptr(t, C.c_int64),
                                N.ptr(e, C.c_int64)))
    return [ProfilePoint(int(f[j]), int(t[j]), int(e[j])) for j in range(9)]


def profile_set(p: G9Params) -> ProfileSet:
    ps = ProfileSet(75.0, [])
    for s, b in enumerate(stage_bases(p)):
        ps.profiles.append(FrequencyProfile(ClassKey(s, int(Kind.Forward)), stage_profile(b, False)))
        ps.profiles.append(FrequencyProfile(ClassKey(s, int(Kind.Backward)), stage_profile(b, True)))
    return ps


_MODEL_CACHE: dict = {}


def instance(p: G9Params):
    """(NodeDag, CostModel) of a G9 instance; cost models are cached by stage bases."""
    dag = build_1f1b(p.stages, p.microbatches)
    key = tuple(stage_bases(p))
    model = _MODEL_CACHE.get(key)
    if model is None:
        model = CostModel.build(profile_set(p))
        _MODEL_CACHE[key] = model
    return dag, model
