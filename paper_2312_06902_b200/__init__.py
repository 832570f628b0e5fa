"""B200-native Perseus frontier generator (arXiv 2312.06902).

Python mirror of the reference planner API (perseus/frontier.hpp) over the C
ABI in include/perseus_b200.h; all frontier compute runs in hand-written
sm_100a CUDA kernels (csrc/pb_kernels.cu).  No CPU fallback.
"""
from ._native import (CudaError, DegenerateFit, LogicError, UnsupportedInput, LIB_PATH,  # noqa: F401
                      STOP_NAMES)
from .model import (ClassKey, ClassModel, Computation, CostModel, ExpCurve, FrequencyProfile,  # noqa: F401
                    Kind, NodeDag, PackedInstance, ProfilePoint, ProfileSet, build_1f1b, build_gpipe,
                    class_of, finalize_custom_dag, fit_exp, pareto_filter)
from .frontier import (EnergySchedule, Frontier, FrontierBatch, StepInfo, all_max_schedule,  # noqa: F401
                       discover_frontier, discretize, get_next_schedule, lookup, min_energy_schedule)

__version__ = "0.1.0"
