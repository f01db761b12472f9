"""B200-native state-vector executor for centrality-partitioned circuits.

Drop-in for the simulation path of the reference package ``svpart``
(``svpart/executor.py``): ``run_plan``, ``gather``, ``scatter``, ``compare``,
``sample``, ``oracle_simulate`` and the result/exception types keep the
reference's names and meaning.  Plans come from the reference's partitioner
unchanged (an ``svpart.plan.ExecutionPlan`` is accepted as is) or from its
JSON wire format (``plan.from_json``).

Execution is CUDA only (sm_100a kernels in ``libsvb200.so``, driven through
a C ABI, see ``include/svb200.h``); there is no CPU fallback.
"""

from .errors import (
    DimensionMismatch,
    ExecutorError,
    NativeError,
    NonUnitaryDrift,
    PlanInvalid,
    TooLarge,
)
from .executor import (
    DistState,
    RunResult,
    RunStats,
    compare,
    fidelity,
    gather,
    gather_device,
    oracle_simulate,
    run_plan,
    sample,
    scatter,
)
from .gates import GATE_SIGNATURES, Gate, gate, gate_tensor
from .plan import ExecutionPlan, Task, from_json, to_json

__version__ = "0.1.0"

__all__ = [
    "DimensionMismatch", "DistState", "ExecutionPlan", "ExecutorError", "GATE_SIGNATURES",
    "Gate", "NativeError", "NonUnitaryDrift", "PlanInvalid", "RunResult", "RunStats", "Task",
    "TooLarge", "compare", "fidelity", "from_json", "gate", "gate_tensor", "gather",
    "gather_device", "oracle_simulate", "run_plan", "sample", "scatter", "to_json",
    "__version__",
]
