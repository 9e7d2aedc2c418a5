"""paper_1810_08061_b200 — B200 (sm_100a) execution backend for staged
control-flow graphs produced by the stagekit conversion API (arXiv 1810.08061).

Public API (drop-in for the reference CPU executor, graph/execute.py:27):

    from paper_1810_08061_b200 import execute
    result = execute(graph, feeds)          # ExecutionResult(outputs, print_log)

plus ``gradient`` (reverse mode through While/Cond/FuncCall, autodiff.py),
``execute_many`` (many feed sets, one launch), the IR mirror with its JSON
(``ir``) and s-expression (``from_sexpr``/``to_sexpr``) wire formats, and the
error classes (``errors``).
"""

from .errors import (BackendUnavailable, DeviceError, IterationLimitExceeded, LoweringError,
                     RuntimeGraphError, SkbError, ValidationError)
from .executor import (ExecutionResult, PrecisionRangeError, RnnExecutable, bind_feeds, execute,
                       execute_many, lower)
from .autodiff import NotDifferentiable, gradient
from .sexpr import SexprError, from_sexpr, to_sexpr
from .values import DeviceTensor, TensorValue, allclose, max_rel_error

__version__ = "0.1.0"

__all__ = [
    "BackendUnavailable", "DeviceError", "DeviceTensor", "ExecutionResult", "IterationLimitExceeded",
    "LoweringError", "NotDifferentiable", "PrecisionRangeError", "SexprError", "RnnExecutable", "RuntimeGraphError", "SkbError",
    "TensorValue", "ValidationError", "allclose", "bind_feeds", "execute", "execute_many", "from_sexpr", "gradient", "lower",
    "max_rel_error", "to_sexpr",
]
