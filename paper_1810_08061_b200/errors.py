"""Error classes of the B200 executor, mirroring the reference's runtime error
contract (reference pkg/src/stagekit/errors.py:13-17, :155-174).

`execute()` failures carry the failing node's origin span and the class name
of the underlying failure as ``cause_kind`` exactly like the reference's
``RuntimeGraphError(message, span, cause_kind)`` built in
graph/execute.py:86-93, so callers (the differential harness compares
``cause_kind`` strings, harness/diff.py:159-164) see identical failures.
"""

from __future__ import annotations

# cause_kind strings produced by the reference executor on the hot path
INDEX_OUT_OF_RANGE = "IndexOutOfRange"
EMPTY_POP = "EmptyPop"
SHAPE_MISMATCH = "ShapeMismatch"
DTYPE_MISMATCH = "DtypeMismatch"
DIVISION_BY_ZERO = "DivisionByZero"
ITERATION_LIMIT = "IterationLimitExceeded"
ASSERTION_FAILED = "AssertionFailed"
MISSING_FEED = "MissingFeed"


class SkbError(Exception):
    """Base class (reference: StagekitError, errors.py:13-17)."""

    def __init__(self, message: str, span=None):
        super().__init__(message)
        self.message = message
        self.span = span


class RuntimeGraphError(SkbError):
    """Execution-time failure tagged with the node span and the reference's
    cause_kind (reference errors.py:155-161)."""

    def __init__(self, message: str, span=None, cause_kind: str = ""):
        super().__init__(message, span)
        self.cause_kind = cause_kind or type(self).__name__


class IterationLimitExceeded(RuntimeGraphError):
    """reference errors.py:164-166"""

    def __init__(self, message: str, span=None):
        super().__init__(message, span, cause_kind=ITERATION_LIMIT)


class ValidationError(SkbError):
    """Structural graph problem (reference errors.py:148-152)."""

    def __init__(self, violations):
        super().__init__("; ".join(violations))
        self.violations = list(violations)


class LoweringError(SkbError):
    """The graph contains a region this backend has no device lowering for.

    The backend never falls back to a CPU interpreter: unsupported regions
    fail loudly (north star: "no CPU fallback")."""


class BackendUnavailable(SkbError):
    """libskb.so is missing or no CUDA device is visible."""


class DeviceError(SkbError):
    """A CUDA-level failure inside libskb (launch/configuration)."""


# skb_status codes of include/skb.h -> reference cause_kind
STATUS_TO_CAUSE = {
    10: INDEX_OUT_OF_RANGE,
    11: EMPTY_POP,
    12: SHAPE_MISMATCH,
    13: DIVISION_BY_ZERO,
    14: ITERATION_LIMIT,
    15: ASSERTION_FAILED,
}
SKB_ERR_FP16_RANGE = 20
SKB_ERR_HANDOFF = 21   # internal: a concurrent-kernel handoff timed out (never expected)


class IntegerOverflow(SkbError):
    """An i64 result outside int64.  The reference's integers are unbounded
    Python ints (graph/tensor.py); the device computes in int64 and reports
    the overflow instead of wrapping."""
