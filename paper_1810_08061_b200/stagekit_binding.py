"""The stagekit-side binding of skb (what INTEGRATION.md §1 asks a stagekit
maintainer to add): an ``execute(graph, feeds, check)`` with the reference's
exact contract — reference ``ExecutionResult`` / ``TensorValue`` /
``ListValue`` / ``Tree`` results and reference exception classes — that runs
the graph on the B200 through ``paper_1810_08061_b200.execute``.

Rebinding it into the reference's own harness is the parity seam SURVEY §8(f)1
names (reference harness/diff.py:20 imports ``execute`` at module level and
calls it at :156 and :337)::

    import stagekit.harness.diff as diff
    from paper_1810_08061_b200 import stagekit_binding
    diff.execute = stagekit_binding.execute      # every staged run now hits the GPU

``tools/run_reference_harness.py`` does exactly that for the 1000-seed
differential sweep and the golden corpus.  Importing this module requires the
reference package (``stagekit``) on ``sys.path``; the skb product itself never
imports it.
"""

from __future__ import annotations

import numpy as np

from . import errors as E
from . import executor
from .values import ListValue, Tree


def _sk():
    import importlib
    sk_errors = importlib.import_module("stagekit.errors")
    # (stagekit.graph re-exports the function `execute`, which shadows the module attribute)
    sk_execute = importlib.import_module("stagekit.graph.execute")
    sk_tensor = importlib.import_module("stagekit.graph.tensor")
    return sk_errors, sk_execute, sk_tensor


def _to_reference(value, sk_tensor):
    """skb result -> the reference's value classes (tensor.py:23-87)."""
    if value is None:
        return None
    if isinstance(value, ListValue) or type(value).__name__ == "ListValue" and hasattr(value, "items"):
        return sk_tensor.ListValue([_to_reference(v, sk_tensor) for v in value.items],
                                   getattr(value, "elem_dtype", None), getattr(value, "elem_shape", None))
    if isinstance(value, Tree) or (hasattr(value, "is_empty") and not hasattr(value, "dtype")):
        if value.is_empty:
            return sk_tensor.Tree()
        return sk_tensor.Tree(float(value.value), _to_reference(value.left, sk_tensor),
                              _to_reference(value.right, sk_tensor))
    if hasattr(value, "dtype") and hasattr(value, "shape"):
        arr = np.asarray(value.array if hasattr(value, "array") else value)
        dtype = value.dtype
        flat = arr.reshape(-1)
        if dtype == "f64":
            data = tuple(float(v) for v in flat.astype(np.float64))
        elif dtype == "i64":
            data = tuple(int(v) for v in flat.astype(np.int64))
        else:
            data = tuple(bool(v) for v in flat)
        return sk_tensor.TensorValue(dtype, tuple(int(d) for d in value.shape), data)
    return value


def execute(graph, feeds=None, check: bool = True):
    """Reference signature and result (graph/execute.py:27-36) on the B200.
    Precision policy: env SKB_PRECISION (see executor.execute); the harness
    tool sets "f64" so floats meet the harness's own 1e-9 (diff.py:31)."""
    sk_errors, sk_execute, sk_tensor = _sk()
    try:
        res = executor.execute(graph, feeds or {}, check)
    except E.ValidationError as exc:
        raise sk_errors.ValidationError(exc.violations) from exc
    except E.IterationLimitExceeded as exc:
        raise sk_errors.IterationLimitExceeded(str(exc), getattr(exc, "span", None)) from exc
    except E.RuntimeGraphError as exc:
        raise sk_errors.RuntimeGraphError(getattr(exc, "message", str(exc)), getattr(exc, "span", None),
                                          exc.cause_kind) from exc
    return sk_execute.ExecutionResult([_to_reference(v, sk_tensor) for v in res.outputs], list(res.print_log))
