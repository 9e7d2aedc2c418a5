"""Values at the executor boundary.

Feeds may be the reference's own ``TensorValue`` (reference
pkg/src/stagekit/graph/tensor.py:23-48: dtype string, shape tuple, row-major
``data`` tuple), the host ``TensorValue`` below (same attributes, numpy
storage), numpy arrays, Python scalars / nested lists, or torch tensors
(CPU or already resident on the GPU: zero-copy).

Results are ``DeviceTensor`` objects: they keep the device buffer and expose
the reference's ``TensorValue`` surface (``dtype``/``shape``/``data``/
``item()``/``rank``) lazily, copying to the host only when the host view is
asked for.
"""

from __future__ import annotations

import math
from typing import Optional

import numpy as np

DTYPES = ("i64", "f64", "bool")
NP_DTYPE = {"f64": np.float64, "i64": np.int64, "bool": np.bool_}


def _format_scalar(v) -> str:
    # reference tensor.py:90-95
    if isinstance(v, (bool, np.bool_)):
        return "True" if v else "False"
    if isinstance(v, (float, np.floating)):
        return repr(float(v))
    return str(int(v))


class TensorValue:
    """Host tensor with the reference TensorValue surface (numpy storage)."""

    __slots__ = ("dtype", "shape", "_arr", "_tuple")

    def __init__(self, dtype: str, shape: tuple, data):
        if dtype not in DTYPES:
            raise ValueError(f"bad dtype {dtype!r}")
        self.dtype = dtype
        self.shape = tuple(int(d) for d in shape)
        arr = np.asarray(data, dtype=NP_DTYPE[dtype])
        if arr.size != int(np.prod(self.shape, dtype=np.int64)):
            raise ValueError(f"buffer of {arr.size} elements does not fill {self.shape}")
        self._arr = arr.reshape(self.shape)
        self._tuple = None

    @property
    def array(self) -> np.ndarray:
        return self._arr

    @property
    def data(self) -> tuple:
        if self._tuple is None:
            self._tuple = tuple(self._arr.reshape(-1).tolist())
        return self._tuple

    @property
    def rank(self) -> int:
        return len(self.shape)

    def item(self):
        if self.shape != ():
            raise ValueError(f"item() on non-scalar shape {self.shape}")
        return self._arr.reshape(-1)[0].item()

    def __eq__(self, other):
        return (hasattr(other, "dtype") and other.dtype == self.dtype
                and tuple(other.shape) == self.shape
                and np.array_equal(self._arr, as_numpy(other)))

    __hash__ = None

    def __str__(self):
        payload = ",".join(_format_scalar(v) for v in self._arr.reshape(-1))
        return f"{self.dtype}[{','.join(str(d) for d in self.shape)}]:{payload}"

    def __repr__(self):
        return f"TensorValue({self.dtype}, {self.shape})"


class DeviceTensor:
    """An execution result resident in device memory.

    ``tensor`` is the torch view of the device buffer (zero-copy); ``dtype``
    is the reference dtype string of the graph output (``f64`` for float
    outputs); ``precision`` says what the float values actually carry — e.g.
    "fp16 tensor-core operands, fp32 accumulate/state (bound 3e-3)" for the
    fast tier of the fused recurrent loop, "float64" for the region VM —
    so a caller can tell reduced-precision results apart; ``array``/``data``/
    ``item()`` copy to the host on first use.
    """

    __slots__ = ("dtype", "shape", "tensor", "_arr", "_tuple", "precision")

    def __init__(self, dtype: str, tensor, host: Optional[np.ndarray] = None, precision: Optional[str] = None):
        self.dtype = dtype
        self.precision = precision or ("float64" if str(getattr(tensor, "dtype", "")) == "torch.float64" else None)
        self.tensor = tensor
        self.shape = tuple(int(d) for d in tensor.shape)
        self._arr = host
        self._tuple = None

    @property
    def array(self) -> np.ndarray:
        if self._arr is None:
            self._arr = self.tensor.detach().to("cpu").numpy().astype(NP_DTYPE[self.dtype])
        return self._arr

    @property
    def data(self) -> tuple:
        if self._tuple is None:
            self._tuple = tuple(self.array.reshape(-1).tolist())
        return self._tuple

    @property
    def rank(self) -> int:
        return len(self.shape)

    def item(self):
        if self.shape != ():
            raise ValueError(f"item() on non-scalar shape {self.shape}")
        return self.array.reshape(-1)[0].item()

    def __repr__(self):
        return f"DeviceTensor({self.dtype}, {self.shape}, device={self.tensor.device})"


class Tree:
    """reference tensor.py:51-79"""

    def __init__(self, value: Optional[float] = None, left=None, right=None):
        self.value = value
        self.left = left
        self.right = right

    @property
    def is_empty(self) -> bool:
        return self.value is None


class ListValue:
    """reference tensor.py:82-87"""

    def __init__(self, items, elem_dtype=None, elem_shape=None):
        self.items = list(items)
        self.elem_dtype = elem_dtype
        self.elem_shape = elem_shape


# ------------------------------------------------------------------ coercion
def _torch_mod():
    global _TORCH
    if _TORCH is None:
        try:
            import torch
            _TORCH = torch
        except ImportError:  # pragma: no cover
            _TORCH = False
    return _TORCH


_TORCH = None


def infer_dtype(v) -> str:
    """Reference dtype string of a feed (reference tensor.py:105-147)."""
    torch = _torch_mod()
    if torch and isinstance(v, torch.Tensor):
        if v.dtype == torch.bool:
            return "bool"
        return "f64" if v.dtype.is_floating_point else "i64"
    if hasattr(v, "dtype") and isinstance(getattr(v, "dtype"), str):
        return v.dtype
    if isinstance(v, (np.ndarray, np.generic)):
        if v.dtype == np.bool_:
            return "bool"
        return "f64" if np.issubdtype(v.dtype, np.floating) else "i64"
    if isinstance(v, bool):
        return "bool"
    if isinstance(v, int):
        return "i64"
    if isinstance(v, float):
        return "f64"
    arr = np.asarray(v)
    if arr.dtype == np.bool_:
        return "bool"
    return "f64" if np.issubdtype(arr.dtype, np.floating) else "i64"


def shape_of(v) -> tuple:
    torch = _torch_mod()
    if torch and isinstance(v, torch.Tensor):
        return tuple(v.shape)
    s = getattr(v, "shape", None)
    if s is not None:
        return tuple(int(d) for d in s)
    return tuple(np.asarray(v).shape)


def as_numpy(v) -> np.ndarray:
    """Host numpy view of a feed (copies only when it must)."""
    if isinstance(v, (TensorValue, DeviceTensor)):
        return v.array
    try:
        import torch
        if isinstance(v, torch.Tensor):
            return v.detach().to("cpu").numpy()
    except ImportError:  # pragma: no cover
        pass
    if isinstance(v, np.ndarray):
        return v
    if isinstance(v, np.generic):
        return np.asarray(v)
    try:
        if hasattr(v, "dtype") and hasattr(v, "shape") and hasattr(v, "data"):
            # the reference's TensorValue: row-major tuple
            return np.asarray(v.data, dtype=NP_DTYPE[v.dtype]).reshape(tuple(v.shape))
        return np.asarray(v)
    except OverflowError:   # a Python int beyond int64 (the reference's ints are unbounded)
        from .errors import IntegerOverflow
        raise IntegerOverflow("an integer value exceeds int64, the device's integer type") from None


def allclose(a, b, rel: float) -> bool:
    """The reference's comparison rule (tensor.py:433-449) with tolerance
    ``rel``: |x - y| <= rel * max(1, |x|, |y|), NaNs equal, infinities exact,
    integers and bools exact."""
    if a.dtype != b.dtype or tuple(a.shape) != tuple(b.shape):
        return False
    x, y = as_numpy(a), as_numpy(b)
    if a.dtype != "f64":
        return bool(np.array_equal(x, y))
    x = x.astype(np.float64)
    y = y.astype(np.float64)
    both_nan = np.isnan(x) & np.isnan(y)
    inf = np.isinf(x) | np.isinf(y)
    if np.any(inf & ~both_nan & (x != y)):
        return False
    fin = ~both_nan & ~inf
    scale = np.maximum(1.0, np.maximum(np.abs(x[fin]), np.abs(y[fin])))
    return bool(np.all(np.abs(x[fin] - y[fin]) <= rel * scale))


def max_rel_error(a, b) -> float:
    """max |x - y| / max(1, |x|, |y|) — the quantity allclose bounds."""
    x = as_numpy(a).astype(np.float64)
    y = as_numpy(b).astype(np.float64)
    if x.size == 0:
        return 0.0
    return float(np.max(np.abs(x - y) / np.maximum(1.0, np.maximum(np.abs(x), np.abs(y)))))


def is_finite_scalar(v) -> bool:
    return isinstance(v, float) and math.isfinite(v)
