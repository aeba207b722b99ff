"""B200-native execution backend for TimeRL recurrent-tensor / PDG programs.

Drop-in replacement for the reference executor `recten.runtime.reference_execute`
(reference pkg/src/recten/runtime.py:460-475): hand-written sm_100a kernels
behind a C ABI (include/rtb200.h), driven by a loop-nest planner.
"""

from .executor import (EvaluationError, OracleError, RuntimeError_, execute,  # noqa: F401
                       get_executable)
from .ir import Graph, from_pdg  # noqa: F401

__all__ = ["execute", "get_executable", "Graph", "from_pdg", "RuntimeError_", "OracleError",
           "EvaluationError"]
