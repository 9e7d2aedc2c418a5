"""`execute(graph, feeds)` — drop-in replacement for the reference CPU graph
executor (reference pkg/src/stagekit/graph/execute.py:27-36) on the B200.

Same signature and result shape: ``ExecutionResult(outputs, print_log)``;
same feed binding errors (MissingFeed / DtypeMismatch / ShapeMismatch,
execute.py:39-65); same runtime failures with the failing node's span and the
reference ``cause_kind`` (IndexOutOfRange, EmptyPop, ShapeMismatch,
IterationLimitExceeded).  ``execute_many`` runs many independent feed sets of
one graph in a single device launch (throughput mode).

The graph is lowered once per graph object (``lowering.py``) and cached; the
packed weights are cached per weight-feed identity.  Everything numeric runs
in libskb kernels; PyTorch only allocates device memory and moves bytes.
"""

from __future__ import annotations

import os
import threading
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import errors as E
from .errors import IterationLimitExceeded, LoweringError, RuntimeGraphError
from .lowering import CELL_LSTM, RnnProgram, lower_rnn_program
from .validate import shapes_compatible, validate
from .values import DeviceTensor, as_numpy, infer_dtype, shape_of


@dataclass
class ExecutionResult:
    """reference execute.py:21-24"""
    outputs: list
    print_log: list = field(default_factory=list)


class PrecisionRangeError(E.SkbError):
    """A value exceeds the fp16 range of the tensor-core path (|v| > 65504)."""


_plans: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
_plans_lock = threading.Lock()


def lower(graph) -> RnnProgram:
    """Lowered program for `graph` (cached per graph object)."""
    with _plans_lock:
        plan = _plans.get(graph)
    if plan is None:
        plan = lower_rnn_program(graph)
        with _plans_lock:
            _plans[graph] = plan
    return plan


# ------------------------------------------------------------------ feeds
def bind_feeds(graph, feeds: dict, memo: Optional[dict] = None) -> dict:
    """Check every main-frame parameter against its feed (reference
    execute.py:39-65): missing -> MissingFeed, dtype -> DtypeMismatch,
    incompatible declared shape -> ShapeMismatch.  `memo` (one dict per
    execute_many call) checks a value object shared by many feed sets once."""
    out = {}
    for param in graph.main.params:
        name = param.attrs.get("name")
        if name not in feeds:
            raise RuntimeGraphError(f"missing feed for parameter {name!r}", param.origin, E.MISSING_FEED)
        value = feeds[name]
        if memo is not None:
            key = (id(param), id(value))
            if key in memo:
                out[name] = value
                continue
            memo[key] = value   # keeps the object alive, so its id is not reused during the call
        spec = param.out_types[0]
        if spec.dtype == "tree":
            if not hasattr(value, "is_empty"):
                raise RuntimeGraphError(f"feed {name!r} must be a tree", param.origin, E.DTYPE_MISMATCH)
            out[name] = value
            continue
        dtype = infer_dtype(value)
        if dtype != spec.dtype:
            raise RuntimeGraphError(f"feed {name!r} has dtype {dtype}, parameter wants {spec.dtype}",
                                    param.origin, E.DTYPE_MISMATCH)
        shape = shape_of(value)
        if spec.shape is not None and not shapes_compatible(tuple(spec.shape), shape):
            raise RuntimeGraphError(f"feed {name!r} has shape {list(shape)}, parameter wants "
                                    f"{_render(spec)}", param.origin, E.SHAPE_MISMATCH)
        out[name] = value
    return out


def _render(spec) -> str:
    return spec.render() if hasattr(spec, "render") else str(spec)


def _source_value(src, feeds):
    if src is None:   # an all-zero weight block (GRU n_x has no U, n_h no W)
        return None
    return feeds[src.name] if src.kind == "param" else src.value


# ------------------------------------------------------------------ device plumbing
def _torch():
    import torch
    return torch


def _to_device(v, dtype, device, stream=None):
    """Feed -> contiguous device tensor of `dtype` (zero-copy when it already is)."""
    torch = _torch()
    if isinstance(v, torch.Tensor):
        t = v
    elif isinstance(v, DeviceTensor):
        t = v.tensor
    else:
        arr = np.ascontiguousarray(as_numpy(v))
        t = torch.from_numpy(arr)
    if t.device != device or t.dtype != dtype or not t.is_contiguous():
        t = t.to(device=device, dtype=dtype, non_blocking=True).contiguous()
    return t


def _fingerprint(w):
    """What must be unchanged for a cached packing of weight feed `w` to stay
    valid.  torch tensors: storage address + in-place version counter;
    writeable numpy arrays: a snapshot of the contents (compared on reuse);
    immutable feeds (reference TensorValue tuples, read-only arrays): identity."""
    torch = _torch()
    if isinstance(w, DeviceTensor):
        w = w.tensor
    if isinstance(w, torch.Tensor):
        return ("t", w.data_ptr(), w._version, tuple(w.shape), w.dtype)
    if isinstance(w, np.ndarray) and w.flags.writeable:
        return ("a", w.copy())
    if hasattr(w, "array") and isinstance(getattr(w, "array"), np.ndarray) and w.array.flags.writeable:
        return ("a", w.array.copy())
    return ("o",)


def _same_fingerprint(w, fp) -> bool:
    cur = _fingerprint(w) if fp[0] != "a" else None
    if fp[0] == "a":
        arr = w.array if hasattr(w, "array") and not isinstance(w, np.ndarray) else w
        return isinstance(arr, np.ndarray) and arr.shape == fp[1].shape and np.array_equal(arr, fp[1])
    return cur == fp


class _WeightCache:
    """Packed tensor-core weight slabs, keyed by the identity of the weight
    feeds (the objects are kept alive so identities stay valid) and validated
    on every reuse against a content fingerprint (`_fingerprint`), so a weight
    changed in place between calls (an SGD step, then an eval) is re-packed
    instead of silently served stale."""

    def __init__(self, capacity: int = 8):
        self.capacity = capacity
        self.entries: list = []   # (key, keepalive, fingerprints, packed)
        self.lock = threading.Lock()

    def get(self, key, weights):
        with self.lock:
            for i, (k, keep, fps, packed) in enumerate(self.entries):
                if k == key:
                    flat = [w for trip in weights for w in trip]
                    if all(_same_fingerprint(w, fp) for w, fp in zip(flat, fps)):
                        return packed
                    self.entries.pop(i)   # stale: re-pack
                    return None
        return None

    def put(self, key, keep, packed):
        fps = [_fingerprint(w) for trip in keep for w in trip]
        with self.lock:
            self.entries.append((key, keep, fps, packed))
            if len(self.entries) > self.capacity:
                self.entries.pop(0)


_weights = _WeightCache()


class RnnExecutable:
    """A lowered recurrent program bound to one weight set and problem shape:
    owns the packed weights and device scratch so repeated launches allocate
    nothing.  ``run`` is the device-resident hot path (inputs already in HBM)."""

    def __init__(self, prog: RnnProgram, weights: list, B: int, T: int, F: int, H: int, P: int,
                 device=None, stream=None, tier: str = "f16"):
        from . import runtime as rt
        torch = _torch()
        self.rt = rt
        self.lib = rt.lib()
        self.prog = prog
        self.tier = tier   # "f16": tcgen05 fp16-operand kernel (csrc/rnn.cu); "f32": FFMA kernel (csrc/rnn_f32.cu)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.B, self.T, self.F, self.H, self.P = B, T, F, H, P
        self.shape = rt.RnnShape(prog.cell, H, F, T, B, P)
        if tier == "f32":
            nb = self.lib.skb_rnn_f32_packed_bytes(self.shape)
            nw = self.lib.skb_rnn_f32_workspace_bytes(self.shape)
            if nb < 0 or nw < 0 or H > 256 or (F + H) % 4:
                raise LoweringError(f"fp32 recurrent kernel does not support H={H}, F={F} (H <= 256, "
                                    f"(F+H) % 4 == 0)")
        else:
            nb = self.lib.skb_rnn_packed_bytes(self.shape)
            nw = self.lib.skb_rnn_workspace_bytes(self.shape)
        if nb < 0 or nw < 0:
            raise LoweringError(f"recurrent kernel does not support H={H}, F={F} (needs F+H <= 512 "
                                f"after padding and H <= 256)")
        self.packed_bytes = nb
        self.packed = self._get_packed(weights, nb, stream)
        self.ws = torch.empty(int(nw), dtype=torch.uint8, device=self.device)
        self.err = torch.zeros(4, dtype=torch.int32, device=self.device)
        self.max_len = torch.zeros(P, dtype=torch.int32, device=self.device)

    def _get_packed(self, weights, nbytes, stream):
        torch = _torch()
        key = (self.tier, self.prog.cell, self.H, self.F, tuple(id(w) for trip in weights for w in trip))
        packed = _weights.get(key, weights)
        if packed is not None:
            return packed
        dev = [[None if w is None else _to_device(w, torch.float64, self.device) for w in trip]
               for trip in weights]
        ws_ = [t[0] for t in dev] + [dev[0][0]] * (4 - len(dev))
        us_ = [t[1] for t in dev] + [dev[0][1]] * (4 - len(dev))
        bs_ = []
        for t in dev:
            b = t[2]
            if b.dim() == 0:
                b = b.expand(self.H).contiguous()
            bs_.append(b.reshape(-1))
        bs_ += [bs_[0]] * (4 - len(bs_))
        P4 = self.rt._P4
        packed = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        err = torch.zeros(4, dtype=torch.int32, device=self.device)
        st = self.rt.stream_handle(stream)
        if self.tier == "f32":
            self.rt.check(self.lib.skb_rnn_pack_f32(
                self.shape, P4(*[t.data_ptr() if t is not None else None for t in ws_]),
                P4(*[t.data_ptr() if t is not None else None for t in us_]),
                P4(*[t.data_ptr() for t in bs_]), 1, self.rt.ptr(packed), st), "skb_rnn_pack_f32")
            _weights.put(key, weights, packed)
            return packed
        self.rt.check(self.lib.skb_rnn_pack(
            self.shape, P4(*[t.data_ptr() if t is not None else None for t in ws_]),
            P4(*[t.data_ptr() if t is not None else None for t in us_]),
            P4(*[t.data_ptr() for t in bs_]), 1, self.rt.ptr(packed), self.rt.ptr(err), st), "skb_rnn_pack")
        if int(err[0].item()) == E.SKB_ERR_FP16_RANGE:
            raise PrecisionRangeError("a weight exceeds the fp16 range (|w| > 65504) of the tensor-core path")
        _weights.put(key, weights, packed)
        return packed

    def refresh(self, weights, stream=None):
        """Re-validate the packed weights against the weight feeds of this call
        (re-packs when one was modified in place since it was packed)."""
        self.packed = self._get_packed(weights, self.packed_bytes, stream)

    def run(self, x, h0, c0, lens, out, hT=None, cT=None, stream=None):
        """Launch on device buffers (x: [R,T,F] f32/f64, h0/c0: [R,H] f32,
        lens: [R] i64, out: [R,T,H] f32).  Asynchronous; returns nothing."""
        torch = _torch()
        rt = self.rt
        self.err.zero_()
        st = rt.stream_handle(stream)
        fwd = self.lib.skb_rnn_forward_f32 if self.tier == "f32" else self.lib.skb_rnn_forward
        rt.check(fwd(
            self.shape, rt.ptr(self.packed), rt.ptr(x), 1 if x.dtype == torch.float64 else 0,
            rt.ptr(h0), rt.ptr(c0), rt.ptr(lens), rt.ptr(out), rt.ptr(hT), rt.ptr(cT),
            rt.ptr(self.max_len), rt.ptr(self.err), rt.ptr(self.ws), st), "skb_rnn_forward")

    @property
    def precision(self) -> str:
        """What the float outputs carry (DeviceTensor.precision)."""
        return ("fp16 tensor-core operands, fp32 accumulate/state (bound 3e-3)" if self.tier == "f16"
                else "fp32 FFMA, fp32 state (bound 1e-4)")


# ------------------------------------------------------------------ errors
def classify(prog: RnnProgram, max_len: int, T: int):
    """The reference's failure for a problem whose trip count is `max_len`,
    in its evaluation order (Range, While limit, Index, ListStack)."""
    if max_len < 0 and prog.range_node is not None:
        return RuntimeGraphError(f"range of negative length {max_len}", prog.range_node.origin,
                                 E.SHAPE_MISMATCH)
    limit = prog.max_iterations
    if limit is not None and max_len > limit and limit <= T:
        return IterationLimitExceeded(f"loop exceeded max_iterations={limit}", prog.while_node.origin)
    if max_len > T:
        return RuntimeGraphError(f"index {T} out of range for leading dim {T}", prog.index_node.origin,
                                 E.INDEX_OUT_OF_RANGE)
    if max_len <= 0 and prog.stack_node is not None:
        return RuntimeGraphError("stack of an empty list", prog.stack_node.origin, E.EMPTY_POP)
    return None


# ------------------------------------------------------------------ public API
from .runtime import on_stream as _on_stream   # noqa: E402


_vm_plans: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


_stream_plans: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()
STREAM_MIN_ELEMS = 1 << 14   # smaller vectors run on the region VM (one CTA is enough)


def stream_plan(graph):
    """The vector-stream program of `graph` (stream.py), or None if it has none."""
    from . import stream
    with _plans_lock:
        if graph in _stream_plans:
            return _stream_plans[graph]
    try:
        prog = stream.compile_graph(graph)
    except LoweringError:
        prog = None
    with _plans_lock:
        _stream_plans[graph] = prog
    return prog


_decode_plans: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def decode_plan(graph):
    """The staged greedy decoder's operand roles (lowering_decode.py), or None."""
    from .lowering_decode import lower_greedy
    with _plans_lock:
        if graph in _decode_plans:
            return _decode_plans[graph]
    try:
        prog = lower_greedy(graph)
    except (LoweringError, KeyError, IndexError, AttributeError, StopIteration):
        prog = None
    with _plans_lock:
        _decode_plans[graph] = prog
    return prog


def plan_kind(graph, feeds: Optional[dict] = None) -> str:
    """'rnn' when the fused recurrent kernel applies, 'decode' for the staged
    greedy decoder, 'stream' for vector-stream programs whose vectors (static
    shape, else the feeds') have at least STREAM_MIN_ELEMS elements, else 'vm'."""
    try:
        lower(graph)
        return "rnn"
    except LoweringError:
        pass
    if decode_plan(graph) is not None:
        return "decode"
    prog = stream_plan(graph)
    if prog is None:
        return "vm"
    n = int(np.prod(prog.shape)) if all(d is not None for d in prog.shape) else 0
    for name, slot in prog.feeds.items():
        if feeds and name in feeds and slot.kind == 1:
            n = max(n, int(np.prod(shape_of(feeds[name]))))
    return "stream" if n >= STREAM_MIN_ELEMS else "vm"


PRECISIONS = ("fast", "fp32", "f64")


@_on_stream
def execute(graph, feeds: Optional[dict] = None, check: bool = True, *, stream=None,
            precision: Optional[str] = None) -> ExecutionResult:
    """Drop-in for the reference ``execute(graph, feeds, check=True)``.

    Programs with a fused kernel (the dynamic-length recurrent loop) run
    through it; every other graph runs on the device-resident region VM
    (``vm.py`` / ``csrc/vm.cu``).

    ``precision`` (default: env SKB_PRECISION, else "fast") selects the tier of
    the fused recurrent loop: "fast" = fp16 tensor-core operands, fp32
    accumulate / state (stated bound 3e-3; inputs beyond the fp16 range fall
    back to "fp32"); "fp32" = the FFMA kernel with fp32 weights (rtol 1e-4);
    "f64" = every float in float64 like the reference (region VM / vector-stream
    tier), for callers that need the reference's own 1e-9 agreement (its
    differential harness).  Float outputs of the fused loop carry the tier in
    ``DeviceTensor.precision``."""
    from . import runtime as rt
    rt.lib()
    if check:
        validate(graph)
    precision = precision or os.environ.get("SKB_PRECISION", "fast")
    if precision not in PRECISIONS:
        raise ValueError(f"precision {precision!r} (expected one of {PRECISIONS})")
    kind = plan_kind(graph, feeds)
    if kind == "rnn" and precision == "f64":
        kind = "vm"
    if kind == "rnn":
        try:
            return execute_many(graph, [feeds or {}], check=False, stream=stream, precision=precision)[0]
        except LoweringError:   # a shape the fused kernels do not take: the region VM (f64) runs it
            return execute_vm(graph, feeds, stream=stream)
    if kind == "stream":
        try:
            return execute_stream(graph, feeds, stream=stream)
        except LoweringError:   # e.g. a list outgrew the tier's capacity: the region VM runs it
            pass
    if kind == "decode":
        try:
            return execute_decode_many(graph, [feeds or {}], stream=stream)[0]
        except LoweringError:   # feeds outside the fused decoder's contract (e.g. ids != 0..V-1)
            pass
    return execute_vm(graph, feeds, stream=stream)


DECODE_MARGIN = float(os.environ.get("SKB_DECODE_MARGIN", "1e-3"))   # logits gap below which the f64 VM decides


@_on_stream
def execute_decode_many(graph, feeds_list: list, *, stream=None) -> list:
    """The staged greedy decoder for P feed sets sharing one
    weight set, eos and max_len: the P sentences decode together in one
    device-resident loop (csrc/beam.cu, beam 1), each stopping at its own EOS."""
    torch = _torch()
    from .decode import Decoder
    prog = decode_plan(graph)
    if prog is None:
        raise LoweringError("not the staged greedy decoder")
    memo = {}
    bound = [bind_feeds(graph, f or {}, memo) for f in feeds_list]
    f0 = bound[0]
    shared = (prog.emb, prog.w_in, prog.u, prog.w_out, prog.ids, prog.eos, prog.max_len)
    for b in bound[1:]:
        for k in shared:
            if b[k] is not f0[k] and not np.array_equal(as_numpy(b[k]), as_numpy(f0[k])):
                raise LoweringError("batched greedy decoding needs one weight set, eos and max_len")
    emb = as_numpy(f0[prog.emb])
    V = emb.shape[0]
    if not np.array_equal(as_numpy(f0[prog.ids]).reshape(-1), np.arange(V)):
        raise LoweringError("ids must be 0..V-1 for the fused argmax")
    eos = int(as_numpy(f0[prog.eos]).reshape(-1)[0])
    max_len = int(as_numpy(f0[prog.max_len]).reshape(-1)[0])
    P = len(bound)
    if max_len < 0 or not 0 <= eos < V:
        raise LoweringError("max_len / eos outside the fused decoder's contract")
    h0 = np.concatenate([as_numpy(b[prog.h0]).reshape(1, -1) for b in bound], axis=0)
    dec = Decoder("rnn", emb.reshape(V, -1), (as_numpy(f0[prog.w_in]), as_numpy(f0[prog.u]),
                                             as_numpy(f0[prog.w_out])), P, 1, max_len, eos)
    out = dec(h0, stream=stream)
    lengths = out["lengths"][:, 0].to("cpu").numpy()
    margins = dec.margins()[:, 0].to("cpu").numpy()
    toks = out["tokens"][:, 0, :].to(torch.int64)
    results = []
    for p in range(P):
        if not margins[p] > DECODE_MARGIN:
            # an argmax decided by less than the fp32 logits' error bound could differ from the
            # reference's f64 argmax (whose exact ties sum the tied ids): re-run in f64 on the VM
            results.append(execute_vm(graph, feeds_list[p] or {}, stream=stream))
            continue
        n = int(lengths[p])
        vals = [None, None]
        vals[prog.toks_out] = DeviceTensor("i64", toks[p, :n + 1])
        vals[prog.steps_out] = DeviceTensor("i64", torch.tensor(n, dtype=torch.int64, device=toks.device))
        results.append(ExecutionResult(vals, []))
    return results


@_on_stream
def execute_stream(graph, feeds: Optional[dict] = None, *, stream=None) -> ExecutionResult:
    """Run a vector-stream program (stream.py / csrc/stream.cu) at any size;
    raises LoweringError for graphs outside that tier."""
    from . import stream as st
    from . import runtime as rt
    rt.lib()
    bound = bind_feeds(graph, feeds or {})
    prog = stream_plan(graph)
    if prog is None:
        st.compile_graph(graph)   # re-raise the LoweringError with its message
    return ExecutionResult(st.run(prog, bound, stream=stream), [])


@_on_stream
def execute_vm(graph, feeds: Optional[dict] = None, *, stream=None) -> ExecutionResult:
    """Run any staged graph on the region VM (no validation)."""
    from . import vm
    bound = bind_feeds(graph, feeds or {})
    with _plans_lock:
        prog = _vm_plans.get(graph)
    if prog is None:
        prog = vm.compile_graph(graph)
        with _plans_lock:
            _vm_plans[graph] = prog
    outs, log = vm.run(prog, bound, stream=stream)
    return ExecutionResult(outs, log)


@_on_stream
def execute_many(graph, feeds_list: list, check: bool = True, *, stream=None,
                 return_exceptions: bool = False, host_outputs: bool = False, precision: Optional[str] = None) -> list:
    """Run `graph` on P independent feed sets in one device launch.

    Weight feeds must be the same objects (or equal) across the feed sets.
    Raises the first problem's error unless ``return_exceptions`` (then the
    failing entries of the returned list are the exception objects).  With
    ``host_outputs`` the whole output sequence buffer is copied to page-locked
    host memory in one transfer (into ``host_outputs`` itself when it is a
    float32 CPU tensor of R*T*H elements) and results are served from it.
    ``precision``: "fast" (default) or "fp32" (see ``execute``); a fast-tier
    launch whose inputs exceed the fp16 range is re-run on the fp32 tier."""
    precision = precision or os.environ.get("SKB_PRECISION", "fast")
    if precision == "f64":
        raise LoweringError("execute_many runs the fused recurrent kernels; use execute(precision='f64')")
    tier = "f32" if precision == "fp32" else "f16"
    try:
        return _execute_many(graph, feeds_list, check, stream, return_exceptions, host_outputs, tier)
    except PrecisionRangeError:
        if tier == "f32":
            raise
        return _execute_many(graph, feeds_list, False, stream, return_exceptions, host_outputs, "f32")


def _execute_many(graph, feeds_list, check, stream, return_exceptions, host_outputs, tier):
    torch = _torch()
    from . import runtime as rt
    rt.lib()
    if check:
        validate(graph)
    prog = lower(graph)
    memo = {}
    P = len(feeds_list)
    if P == 0:
        return []
    f0 = bind_feeds(graph, feeds_list[0] or {}, memo)
    xshape = shape_of(_source_value(prog.x, f0))
    if len(xshape) != 3:
        raise RuntimeGraphError(f"x must be rank 3, got {list(xshape)}", prog.x.node.origin if prog.x.node else None,
                                E.SHAPE_MISMATCH)
    Bsz, T, F = xshape
    weights = [tuple(_source_value(s, f0) for s in trip) for trip in prog.gates]

    def bind(feeds):
        """bind_feeds plus the execute_many contract: one x shape, one shared weight set"""
        b = bind_feeds(graph, feeds or {}, memo)
        if shape_of(_source_value(prog.x, b)) != xshape:
            raise LoweringError("execute_many needs feed sets of one shape")
        for trip_src, trip in zip(prog.gates, weights):
            for s_, w in zip(trip_src, trip):
                if s_ is None:
                    continue
                v = _source_value(s_, b)
                if v is not w and not np.array_equal(as_numpy(v), as_numpy(w)):
                    raise LoweringError("execute_many needs one weight set shared by all feed sets")
        return b
    H = shape_of(weights[0][1])[0]
    if Bsz == 0:
        err = RuntimeGraphError("reduce_max of empty tensor", prog.reduce_node.origin, E.SHAPE_MISMATCH)
        if return_exceptions:
            return [err] * P
        raise err
    device = torch.device("cuda", torch.cuda.current_device())
    R = Bsz * P

    NPD = {torch.float32: np.float32, torch.float64: np.float64, torch.int64: np.int64}

    def cat(src, dtype):
        """Stack the P feeds of one operand on the device.  CUDA feeds are used
        in place (P == 1) or concatenated on the device; page-locked CPU
        tensors are copied straight into their slice of the device buffer;
        other host feeds go through a reused page-locked staging buffer."""
        vals = [_source_value(src, b) for b in bound]
        if all(isinstance(v, torch.Tensor) and v.is_cuda for v in vals):
            if P == 1:
                return _to_device(vals[0], dtype, device, stream)
            return torch.cat([v.to(dtype) for v in vals]).contiguous()
        if all(isinstance(v, torch.Tensor) and v.is_pinned() and v.dtype == dtype for v in vals):
            n0 = vals[0].shape[0] if vals[0].dim() else 1
            dev = torch.empty((n0 * P,) + tuple(vals[0].shape[1:]), dtype=dtype, device=device)
            for i, v in enumerate(vals):
                dev[i * n0:(i + 1) * n0].copy_(v.reshape((n0,) + tuple(v.shape[1:])), non_blocking=True)
            return dev
        arrs = [as_numpy(v) for v in vals]
        shape = (sum(a.shape[0] if a.ndim else 1 for a in arrs),) + tuple(arrs[0].shape[1:])
        staging = _pinned(src.name or id(src), shape, dtype)
        view = staging.numpy()
        off = 0
        for a in arrs:
            n = a.shape[0] if a.ndim else 1
            view[off:off + n] = a.astype(NPD[dtype], copy=False).reshape((n,) + shape[1:])
            off += n
        return staging.to(device, non_blocking=True)

    x0 = _source_value(prog.x, f0)
    x32 = (isinstance(x0, torch.Tensor) and x0.dtype == torch.float32) or \
          (isinstance(x0, np.ndarray) and x0.dtype == np.float32)
    x_dtype = torch.float32 if x32 else torch.float64
    if host_outputs is not False and host_outputs is not None and T > 0 and P >= 4 and _all_pinned(prog, [f0]):
        # feed sets are bound chunk by chunk inside the pipeline, overlapping the copies
        out_host, hT_h, cT_h, ml_host, status_h, ml_dev, finish = _run_pipelined(
            prog, weights, feeds_list, f0, bind, Bsz, T, F, H, P, device, x_dtype, host_outputs, stream, tier)
        # results are views of the host buffers: built while the last copies are in flight
        results = _assemble(prog, out_host, hT_h, cT_h, ml_host, None, Bsz, T, P, True, tier)
        finish()
        if int(status_h[0]) == E.SKB_ERR_FP16_RANGE:
            raise PrecisionRangeError("an input exceeds the fp16 range (|x| > 65504) of the tensor-core path")
        if not np.array_equal(ml_dev.numpy(), ml_host):   # (host and device trip counts agree by construction)
            results = _assemble(prog, out_host, hT_h, cT_h, ml_dev.numpy(), None, Bsz, T, P, True, tier)
        if not return_exceptions:
            for r in results:
                if isinstance(r, Exception):
                    raise r
        return results
    bound = [f0] + [bind(f) for f in feeds_list[1:]]
    exe = _executable(prog, weights, Bsz, T, F, H, P, device, stream, tier)
    x = cat(prog.x, x_dtype)
    h0 = cat(prog.h0, torch.float32).reshape(R, H)
    c0 = cat(prog.c0, torch.float32).reshape(R, H) if prog.cell == CELL_LSTM else None
    lens = cat(prog.lens, torch.int64).reshape(R)
    out = torch.empty((R, T, H), dtype=torch.float32, device=device)
    want = {o.kind for o in prog.outputs}
    hT = torch.empty((R, H), dtype=torch.float32, device=device) if "h_final" in want else None
    cT = torch.empty((R, H), dtype=torch.float32, device=device) if "c_final" in want else None
    if T > 0:
        exe.run(x, h0, c0, lens, out, hT, cT, stream=stream)
        status = exe.err.to("cpu")
        if int(status[0]) == E.SKB_ERR_HANDOFF:
            # the concurrent auxiliary grid did not get SMs next to the recurrent kernel:
            # stop using it in this process and run the launch sequence instead
            exe.lib.skb_rnn_set_overlap(0)
            exe.run(x, h0, c0, lens, out, hT, cT, stream=stream)
            status = exe.err.to("cpu")
        max_len = exe.max_len.to("cpu").numpy()
    else:
        status = torch.zeros(4, dtype=torch.int32)
        lv = as_numpy(lens.to("cpu")).reshape(P, Bsz)
        max_len = lv.max(axis=1)
    host_out = None
    if host_outputs is not False and host_outputs is not None and int(status[0]) != E.SKB_ERR_FP16_RANGE:
        if isinstance(host_outputs, torch.Tensor):   # caller-owned page-locked buffer
            host_out = host_outputs.view(out.shape)
        else:
            host_out = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        host_out.copy_(out)   # one D2H of the whole [R, T, H] sequence buffer
        host_hT = hT.to("cpu") if hT is not None else None
        host_cT = cT.to("cpu") if cT is not None else None
        out, hT, cT = host_out, host_hT, host_cT
    return _assemble(prog, out, hT, cT, max_len, status, Bsz, T, P, return_exceptions, tier)


PIPELINE_CHUNKS = int(os.environ.get("SKB_PIPELINE_CHUNKS", "12"))   # copy/compute pipeline depth
H2D_ROWS = os.environ.get("SKB_H2D_ROWS", "0") == "1"   # pull only each row's valid timesteps (measured slower: 67.3 vs 62.7 ms)


def _all_pinned(prog, bound) -> bool:
    torch = _torch()
    srcs = [prog.x, prog.h0, prog.lens] + ([prog.c0] if prog.cell == CELL_LSTM else [])
    for b in bound:
        for src in srcs:
            v = _source_value(src, b)
            if not (isinstance(v, torch.Tensor) and not v.is_cuda and v.is_pinned()):
                return False
    return True


def _adjacent_run(vals, shape):
    """If the tensors are back-to-back contiguous views of one host allocation,
    one tensor spanning all of them (so the copy is a single DMA), else None."""
    torch = _torch()
    v0 = vals[0]
    if not all(isinstance(v, torch.Tensor) and v.is_contiguous() and v.dtype == v0.dtype for v in vals):
        return None
    nb = v0.numel() * v0.element_size()
    base = v0.data_ptr()
    if any(v.data_ptr() != base + i * nb or v.numel() != v0.numel() for i, v in enumerate(vals)):
        return None
    try:
        return torch.as_strided(v0, shape, torch.empty(shape, device="meta").stride())
    except RuntimeError:
        return None


def _run_pipelined(prog, weights, feeds_list, f0, bind, Bsz, T, F, H, P, device, x_dtype, host_outputs, stream,
                   tier="f16"):
    """Host-to-host execute_many in PIPELINE_CHUNKS chunks of problems on three
    streams: the H2D copy of chunk k+1, the kernels of chunk k and the D2H of
    chunk k-1 overlap (PCIe full duplex), instead of copy-in, run, copy-out.
    Each chunk's feed sets are bound (checked) just before its copies are
    queued, so host-side checking overlaps the transfers of earlier chunks."""
    torch = _torch()
    R = Bsz * P
    comp = stream or torch.cuda.current_stream()
    lstm = prog.cell == CELL_LSTM
    key = (str(device), R, T, F, H, x_dtype, lstm, threading.get_ident())
    bufs = _pipe_bufs.get(key)
    if bufs is None:   # device buffers and copy streams reused across calls (the call drains them before returning)
        if len(_pipe_bufs) > 4:
            _pipe_bufs.clear()
        bufs = {"x": torch.empty((R, T, F), dtype=x_dtype, device=device),
                "h0": torch.empty((R, H), dtype=torch.float32, device=device),
                "c0": torch.empty((R, H), dtype=torch.float32, device=device) if lstm else None,
                "lens": torch.empty((R,), dtype=torch.int64, device=device),
                "out": torch.empty((R, T, H), dtype=torch.float32, device=device),
                "s_in": torch.cuda.Stream(device=device), "s_out": torch.cuda.Stream(device=device)}
        _pipe_bufs[key] = bufs
    s_in, s_out = bufs["s_in"], bufs["s_out"]
    s_in.wait_stream(comp)   # earlier work on the caller's stream may still read the reused buffers
    if isinstance(host_outputs, torch.Tensor):
        host_out = host_outputs.view(R, T, H)
    else:
        host_out = torch.empty((R, T, H), dtype=torch.float32, pin_memory=True)
    want = {o.kind for o in prog.outputs}
    hT = torch.empty((R, H), dtype=torch.float32, device=device) if "h_final" in want else None
    cT = torch.empty((R, H), dtype=torch.float32, device=device) if "c_final" in want else None
    max_len = torch.zeros(P, dtype=torch.int32, device=device)
    status = torch.zeros(4, dtype=torch.int32, device=device)
    step = -(-P // max(2, min(PIPELINE_CHUNKS, P // 2)))
    lens_vals = []
    try:
        for p0 in range(0, P, step):
            p1 = min(P, p0 + step)
            pc = p1 - p0
            exe = _executable(prog, weights, Bsz, T, F, H, pc, device, comp, tier)
            rows = slice(p0 * Bsz, p1 * Bsz)
            chunk = [f0 if p == 0 else bind(feeds_list[p]) for p in range(p0, p1)]
            lens_vals.extend(_source_value(prog.lens, b) for b in chunk)

            def stack(src, dtype, shape, buf, lens_rows=None):
                dev = buf[rows]
                vals = [_source_value(src, b) for b in chunk]
                run = _adjacent_run(vals, (pc * Bsz,) + shape)
                if run is not None and lens_rows is not None and run.is_pinned() and run.dtype == dtype:
                    # only the timesteps each row reads (t < its length), pulled by a gather
                    # kernel, instead of the padded [rows, T, F] block
                    esz = run.element_size()
                    if exe.lib.skb_h2d_rows(dev.data_ptr(), run.data_ptr(), shape[0] * shape[1] * esz,
                                            lens_rows.data_ptr(), pc * Bsz, shape[1] * esz, shape[0],
                                            torch.cuda.current_stream().cuda_stream) == 0:
                        return dev
                if run is not None:   # the chunk's feeds are one contiguous host range: one DMA
                    dev.copy_(run, non_blocking=True)
                    return dev
                for i, v in enumerate(vals):
                    if not isinstance(v, torch.Tensor):
                        v = torch.as_tensor(as_numpy(v)).to(dtype)
                    dev[i * Bsz:(i + 1) * Bsz].copy_(v.reshape((Bsz,) + shape), non_blocking=True)
                return dev
            with torch.cuda.stream(s_in):
                lens = stack(prog.lens, torch.int64, (), bufs["lens"])
                # the f16 tier's x packers read only rows t < len: copy just those
                x = stack(prog.x, x_dtype, (T, F), bufs["x"], lens if H2D_ROWS and tier == "f16" else None)
                h0 = stack(prog.h0, torch.float32, (H,), bufs["h0"])
                c0 = stack(prog.c0, torch.float32, (H,), bufs["c0"]) if lstm else None
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            out = bufs["out"][rows]
            comp.wait_event(ev_in)
            with torch.cuda.stream(comp):
                exe.run(x, h0, c0, lens, out, hT[rows] if hT is not None else None,
                        cT[rows] if cT is not None else None, stream=comp)
                max_len[p0:p1].copy_(exe.max_len)
                torch.maximum(status, exe.err, out=status)
                ev_out = torch.cuda.Event()
                ev_out.record(comp)
            s_out.wait_event(ev_out)
            with torch.cuda.stream(s_out):
                host_out[rows].copy_(out, non_blocking=True)
    except BaseException:   # a later feed set failed to bind: drain the queued copies before raising
        s_in.synchronize()
        comp.synchronize()
        s_out.synchronize()
        raise
    # final states, trip counts and status follow the last output chunk on the copy-out stream
    s_out.wait_stream(comp)
    hT_h = torch.empty((R, H), dtype=torch.float32, pin_memory=True) if hT is not None else None
    cT_h = torch.empty((R, H), dtype=torch.float32, pin_memory=True) if cT is not None else None
    ml_dev = torch.empty(P, dtype=torch.int32, pin_memory=True)
    status_h = torch.empty(4, dtype=torch.int32, pin_memory=True)
    with torch.cuda.stream(s_out):
        if hT is not None:
            hT_h.copy_(hT, non_blocking=True)
        if cT is not None:
            cT_h.copy_(cT, non_blocking=True)
        ml_dev.copy_(max_len, non_blocking=True)
        status_h.copy_(status, non_blocking=True)
    # the trip counts again on the host (reduce_max of each problem's lengths), for building results early
    run = _adjacent_run(lens_vals, (P * Bsz,))
    if run is not None:
        ml_host = run.view(P, Bsz).max(dim=1).values.numpy().astype(np.int64)
    else:
        ml_host = np.array([int(torch.as_tensor(as_numpy(v)).max()) for v in lens_vals], dtype=np.int64)

    def finish():
        s_out.synchronize()
        comp.synchronize()
    return host_out, hT_h, cT_h, ml_host, status_h, ml_dev, finish


TIER_PRECISION = {"f16": "fp16 tensor-core operands, fp32 accumulate/state (bound 3e-3)",
                  "f32": "fp32 FFMA, fp32 weights/state (bound 1e-4)"}


def _assemble(prog, out, hT, cT, max_len, status, Bsz, T, P, return_exceptions, tier="f16"):
    if status is not None and int(status[0]) == E.SKB_ERR_FP16_RANGE:
        raise PrecisionRangeError("an input exceeds the fp16 range (|x| > 65504) of the tensor-core path")
    if status is not None and int(status[0]) == E.SKB_ERR_HANDOFF:
        raise E.DeviceError("recurrent kernel: the x-image handoff from the concurrent packer timed out")
    results = []
    for p in range(P):
        m = int(max_len[p])
        err = classify(prog, m, T)
        if err is not None:
            if not return_exceptions:
                raise err
            results.append(err)
            continue
        rows = slice(p * Bsz, (p + 1) * Bsz)
        outs = []
        for o in prog.outputs:
            prec = TIER_PRECISION[tier]
            if o.kind == "seq_bm":
                outs.append(DeviceTensor("f64", out[rows, :m, :], precision=prec))
            elif o.kind == "seq_tm":
                outs.append(DeviceTensor("f64", out[rows, :m, :].permute(1, 0, 2), precision=prec))
            elif o.kind == "h_final":
                outs.append(DeviceTensor("f64", hT[rows], precision=prec))
            else:
                outs.append(DeviceTensor("f64", cT[rows], precision=prec))
        results.append(ExecutionResult(outs, []))
    return results


_pinned_pool: dict = {}
_pipe_bufs: dict = {}


def _pinned(tag, shape, dtype):
    """Reused page-locked staging buffers, one per operand (`tag`): execute_many
    synchronises before returning, so a buffer is free again when the next
    call starts, and distinct operands never share one in flight."""
    torch = _torch()
    key = (tag, tuple(shape), dtype, threading.get_ident())
    buf = _pinned_pool.get(key)
    if buf is None:
        if len(_pinned_pool) > 32:
            _pinned_pool.clear()
        buf = torch.empty(shape, dtype=dtype, pin_memory=True)
        _pinned_pool[key] = buf
    return buf


_exes: dict = {}
_exes_lock = threading.Lock()


def _executable(prog, weights, B, T, F, H, P, device, stream, tier="f16") -> RnnExecutable:
    """Cached executable per (program, shape, weight feeds, thread): each owns
    mutable scratch (status word, trip counts, workspace), so concurrent
    callers on different threads never share one."""
    key = (id(prog), B, T, F, H, P, tuple(id(w) for trip in weights for w in trip), threading.get_ident(),
           str(device), tier)
    with _exes_lock:
        hit = _exes.get(key)
    if hit is not None and hit[0] is prog:
        hit[1].refresh(weights, stream)
        return hit[1]
    exe = RnnExecutable(prog, weights, B, T, F, H, P, device, stream, tier)
    with _exes_lock:
        if len(_exes) > 16:
            _exes.clear()
        _exes[key] = (prog, exe, weights)
    return exe
