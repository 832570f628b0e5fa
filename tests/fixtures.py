"""Builds product-side inputs from the golden fixtures' instance dumps."""
from paper_2312_06902_b200.model import (ClassKey, Computation, CostModel, FrequencyProfile, Kind,
                                         NodeDag, ProfilePoint, ProfileSet)


def instance_from_golden(w):
    """(NodeDag, CostModel, tau) exactly as the reference driver built them."""
    inst = w["instance"]
    comps = [Computation(i, s, None if m < 0 else m, Kind(k)) for i, (s, k, m) in enumerate(inst["comps"])]
    dag = NodeDag(comps, [tuple(e) for e in inst["edges"]], max(c.stage for c in comps) + 1)
    ps = ProfileSet(inst["blocking_watts"], [
        FrequencyProfile(ClassKey(p["stage"], p["kind"]), [ProfilePoint(*pt) for pt in p["points"]])
        for p in inst["profiles"]])
    return dag, CostModel.build(ps, inst["quantum_us"]), inst["tau"]
