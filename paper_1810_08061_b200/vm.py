"""Region-VM compiler and runtime: any staged graph on the GPU.

`compile_graph` flattens a (reference or skb) graph into the bytecode the
device interpreter in csrc/vm.cu executes:

* every node output gets a value slot; graph parameters and constants are
  pre-initialised slots in the device arena;
* `While` (reference graph/execute.py:218-238) becomes
      COPY state <- init ; [SET counter 0]
  L:  <test frame> ; JZ test -> END ; [ITER counter, max_iterations]
      <body frame> ; COPY shadow_k <- out_k ; SWAP state_k, shadow_k ; JMP L
  END:
  with the test/body parameters bound to the state slots and the capture
  parameters aliased to the outer values (reference capture routing,
  graph/ir.py:5-7) — the loop predicate is evaluated on the device;
* `Cond` (execute.py:205-216) becomes JZ pred -> ELSE ; then ; VIEW outs ;
  JMP END ; ELSE: else ; VIEW outs ; END — only the taken branch runs, so
  effects (Print/Assert) happen exactly as in the reference;
* `FuncCall` bodies are inlined, except functions on a call-graph cycle
  (recursion, reference graph/execute.py:191-193, e.g. corpus/tree_prod.msl):
  those are compiled once, out of line, over their own slot range [lo, hi),
  and called through a device call stack — CALL saves the range's slot
  descriptors in an arena frame record (one copy per CTA), detaches the
  range from its storage (the callee allocates fresh storage, so the caller's
  values survive), binds the arguments and jumps; RET reads the results,
  restores the caller's descriptors and binds the results to the call
  site's slots;
* static dtype failures (reference tensor.py:252-267, validate rules) compile
  to a RAISE at the failing node, so they fire only if the node executes.

`run` uploads feeds/constants, launches the interpreter (one CTA for small
programs, a cooperative grid for large tensors), and converts results, the
print log and device errors (node uid -> span, reference cause_kind) back.
"""

from __future__ import annotations

import os
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .runtime import on_stream as _on_stream

from . import errors as E
from .errors import LoweringError, RuntimeGraphError
from .values import DeviceTensor, ListValue, Tree, TensorValue, as_numpy, infer_dtype, shape_of

# opcodes / kinds (csrc/vm.cu)
OP = dict(HALT=0, COPY=2, BINOP=3, UNARY=4, MATMUL=5, TRANSPOSE=6, REDUCE=7, WHERE=8, SHAPE=9,
          RANGE=10, INDEX=11, LIST_NEW=12, LIST_APPEND=13, LIST_POP=14, LIST_GET=15, LIST_SET=16,
          LIST_STACK=17, JMP=18, JZ=19, ITER=20, PRINT=21, ASSERT=22, TREE=23, VIEW=24, SET_I64=25,
          RAISE=26, SWAP=27, CALL=28, RET=29)
BIN = {"Add": 0, "Sub": 1, "Mul": 2, "Div": 3, "Mod": 4, "Lt": 5, "Gt": 6, "Le": 7, "Ge": 8, "Eq": 9, "Ne": 10}
BIN_SYMBOL = {"Add": "+", "Sub": "-", "Mul": "*", "Div": "/", "Mod": "%", "Lt": "<", "Gt": ">",
              "Le": "<=", "Ge": ">=", "Eq": "==", "Ne": "!="}
UN = {"Neg": 0, "Not": 1, "Tanh": 2, "Sigmoid": 3}
DT = {"f64": 0, "i64": 1, "bool": 2, "list": 3, "tree": 4}
DT_NAME = {v: k for k, v in DT.items()}
MAX_RANK = 6

# device error code -> reference cause_kind
CAUSE = {10: E.INDEX_OUT_OF_RANGE, 11: E.EMPTY_POP, 12: E.SHAPE_MISMATCH, 13: E.DIVISION_BY_ZERO,
         14: E.ITERATION_LIMIT, 15: E.ASSERTION_FAILED, 16: E.DTYPE_MISMATCH, 17: "MslTypeError"}
E_ARENA = 30
E_STEPS = 31
E_DEPTH = 32
E_OVERFLOW = 33

VAL_DTYPE = np.dtype([("view", "<i8"), ("own", "<i8"), ("own_cap", "<i8"), ("numel", "<i8"),
                      ("dtype", "<i4"), ("rank", "<i4"), ("shape", "<i4", (MAX_RANK,))])
assert VAL_DTYPE.itemsize == 64


@dataclass
class Program:
    code: list = field(default_factory=list)        # [op, uid, a0..a5]
    extra: list = field(default_factory=list)
    nslots: int = 0
    consts: list = field(default_factory=list)      # (slot, TensorValue-like)
    feed_slots: dict = field(default_factory=dict)  # name -> slot
    outputs: list = field(default_factory=list)     # slots of main outputs
    nodes: dict = field(default_factory=dict)       # uid -> node (spans, messages)
    static_elems: int = 0                           # largest statically known tensor


class _Compiler:
    def __init__(self, graph):
        self.g = graph
        self.p = Program()
        self.slot = {}              # (id(node), out) -> slot
        self.call_stack = []
        self.recursive = _recursive_functions(graph)
        self.entries = {}           # recursive function -> (entry pc, lo, hi, param slots)
        self.call_sites = []        # (instruction index, function name) to patch with the entry pc

    # ---------------------------------------------------------------- helpers
    def new_slot(self):
        s = self.p.nslots
        self.p.nslots += 1
        return s

    def emit(self, op, node=None, *args):
        uid = node.uid if node is not None else 0
        if node is not None:
            self.p.nodes[uid] = node
        a = list(args) + [0] * (6 - len(args))
        self.p.code.append([OP[op], uid] + a)
        return len(self.p.code) - 1

    def patch(self, at, k, value):
        self.p.code[at][2 + k] = value

    def here(self):
        return len(self.p.code)

    def extra(self, values):
        off = len(self.p.extra)
        self.p.extra.extend(int(v) for v in values)
        return off

    def of(self, ref):
        return self.slot[(id(ref.node), ref.out)]

    def bind(self, node, out, slot):
        self.slot[(id(node), out)] = slot

    def note_shape(self, spec):
        if spec is not None and spec.shape:
            if all(d is not None for d in spec.shape):
                self.p.static_elems = max(self.p.static_elems, int(np.prod(spec.shape)))

    def raise_at(self, node, cause, outs=1):
        code = {v: k for k, v in CAUSE.items()}[cause]
        self.emit("RAISE", node, code, 0)
        for k in range(outs):
            self.bind(node, k, self.new_slot())

    # ---------------------------------------------------------------- frames
    def frame(self, sg, param_slots):
        for p, s in zip(sg.params, param_slots):
            self.bind(p, 0, s)
        for node in sg.nodes:
            self.node(node)
        return [self.of(r) for r in sg.outputs]

    def node(self, n):
        op = n.op
        for t in n.out_types:
            self.note_shape(t)
        ins = n.inputs
        dts = [r.node.out_types[r.out].dtype for r in ins]
        if op == "Const":
            s = self.new_slot()
            self.p.consts.append((s, n.attrs["value"]))
            self.bind(n, 0, s)
            self.p.static_elems = max(self.p.static_elems, int(np.prod(shape_of(n.attrs["value"]) or (1,))))
        elif op in BIN:
            out_dt = _result_dtype(op, dts[0], dts[1])
            if out_dt is None:
                return self.raise_at(n, E.DTYPE_MISMATCH)
            s = self.new_slot()
            self.emit("BINOP", n, s, self.of(ins[0]), self.of(ins[1]), BIN[op], DT[out_dt])
            self.bind(n, 0, s)
        elif op in UN:
            a = dts[0]
            if (op == "Neg" and a == "bool") or (op == "Not" and a != "bool") or \
                    (op in ("Tanh", "Sigmoid") and a == "bool"):
                return self.raise_at(n, E.DTYPE_MISMATCH)
            out = "f64" if op in ("Tanh", "Sigmoid") else a
            s = self.new_slot()
            self.emit("UNARY", n, s, self.of(ins[0]), UN[op], DT[out])
            self.bind(n, 0, s)
        elif op == "MatMul":
            if "bool" in dts:
                return self.raise_at(n, E.DTYPE_MISMATCH)
            out = "f64" if "f64" in dts else "i64"
            s = self.new_slot()
            self.emit("MATMUL", n, s, self.of(ins[0]), self.of(ins[1]), DT[out])
            self.bind(n, 0, s)
        elif op == "Transpose":
            perm = tuple(int(x) for x in n.attrs["perm"])
            if sorted(perm) != list(range(len(perm))) or len(perm) > MAX_RANK:
                return self.raise_at(n, E.SHAPE_MISMATCH)
            s = self.new_slot()
            self.emit("TRANSPOSE", n, s, self.of(ins[0]), self.extra(perm), len(perm))
            self.bind(n, 0, s)
        elif op in ("ReduceSum", "ReduceMax"):
            if dts[0] == "bool":
                return self.raise_at(n, E.DTYPE_MISMATCH)
            s = self.new_slot()
            self.emit("REDUCE", n, s, self.of(ins[0]), 1 if op == "ReduceMax" else 0)
            self.bind(n, 0, s)
        elif op == "Where":
            if dts[0] != "bool" or dts[1] != dts[2]:
                return self.raise_at(n, E.DTYPE_MISMATCH)
            s = self.new_slot()
            self.emit("WHERE", n, s, self.of(ins[0]), self.of(ins[1]), self.of(ins[2]))
            self.bind(n, 0, s)
        elif op == "Shape":
            s = self.new_slot()
            self.emit("SHAPE", n, s, self.of(ins[0]))
            self.bind(n, 0, s)
        elif op == "Range":
            s = self.new_slot()
            self.emit("RANGE", n, s, self.of(ins[0]))
            self.bind(n, 0, s)
        elif op == "Index":
            s = self.new_slot()
            self.emit("INDEX", n, s, self.of(ins[0]), self.of(ins[1]))
            self.bind(n, 0, s)
        elif op == "ListNew":
            s = self.new_slot()
            self.emit("LIST_NEW", n, s, self.extra([len(ins)] + [self.of(r) for r in ins]))
            self.bind(n, 0, s)
        elif op == "ListAppend":
            s = self.new_slot()
            self.emit("LIST_APPEND", n, s, self.of(ins[0]), self.of(ins[1]))
            self.bind(n, 0, s)
        elif op == "ListPop":
            sl, si = self.new_slot(), self.new_slot()
            self.emit("LIST_POP", n, sl, si, self.of(ins[0]))
            self.bind(n, 0, sl)
            self.bind(n, 1, si)
        elif op == "ListGet":
            s = self.new_slot()
            self.emit("LIST_GET", n, s, self.of(ins[0]), self.of(ins[1]))
            self.bind(n, 0, s)
        elif op == "ListSet":
            s = self.new_slot()
            self.emit("LIST_SET", n, s, self.of(ins[0]), self.of(ins[1]), self.of(ins[2]))
            self.bind(n, 0, s)
        elif op == "ListStack":
            s = self.new_slot()
            self.emit("LIST_STACK", n, s, self.of(ins[0]))
            self.bind(n, 0, s)
        elif op in ("TreeIsEmpty", "TreeLeft", "TreeRight", "TreeValue"):
            s = self.new_slot()
            kind = {"TreeIsEmpty": 0, "TreeLeft": 1, "TreeRight": 2, "TreeValue": 3}[op]
            self.emit("TREE", n, s, self.of(ins[0]), kind)
            self.bind(n, 0, s)
        elif op == "Print":
            self.emit("PRINT", n, self.extra([len(ins)] + [self.of(r) for r in ins]))
        elif op == "Assert":
            self.emit("ASSERT", n, self.of(ins[0]))
        elif op == "Cond":
            self.cond(n)
        elif op == "While":
            self.loop(n)
        elif op == "FuncCall":
            self.call(n)
        else:
            raise LoweringError(f"op {op} has no VM lowering")

    def cond(self, n):
        nt = n.attrs["n_then_caps"]
        pred = self.of(n.inputs[0])
        then_caps = [self.of(r) for r in n.inputs[1:1 + nt]]
        else_caps = [self.of(r) for r in n.inputs[1 + nt:]]
        outs = [self.new_slot() for _ in n.out_types]
        jz = self.emit("JZ", n, pred, 0)
        res = self.frame(n.attrs["then_graph"], then_caps)
        for o, r in zip(outs, res):
            self.emit("VIEW", n, o, r)
        jmp = self.emit("JMP", n, 0)
        self.patch(jz, 1, self.here())
        res = self.frame(n.attrs["else_graph"], else_caps)
        for o, r in zip(outs, res):
            self.emit("VIEW", n, o, r)
        self.patch(jmp, 0, self.here())
        for k, o in enumerate(outs):
            self.bind(n, k, o)

    def loop(self, n):
        ns = n.attrs["n_state"]
        nt = n.attrs["n_test_caps"]
        init = [self.of(r) for r in n.inputs[:ns]]
        test_caps = [self.of(r) for r in n.inputs[ns:ns + nt]]
        body_caps = [self.of(r) for r in n.inputs[ns + nt:]]
        state = [self.new_slot() for _ in range(ns)]
        shadow = [self.new_slot() for _ in range(ns)]
        for s, i in zip(state, init):
            self.emit("COPY", n, s, i)
        limit = n.attrs.get("max_iterations")
        counter = None
        if limit is not None:
            counter = self.new_slot()
            self.emit("SET_I64", n, counter, 0)
        top = self.here()
        t = self.frame(n.attrs["test_graph"], state + test_caps)
        jz = self.emit("JZ", n, t[0], 0)
        if counter is not None:
            self.emit("ITER", n, counter, int(limit))
        outs = self.frame(n.attrs["body_graph"], state + body_caps)
        for z, o in zip(shadow, outs):
            self.emit("COPY", n, z, o)
        for s, z in zip(state, shadow):
            self.emit("SWAP", n, s, z)
        self.emit("JMP", n, top)
        self.patch(jz, 1, self.here())
        for k, s in enumerate(state):
            self.bind(n, k, s)

    def call(self, n):
        name = n.attrs["fn_name"]
        if name in self.recursive:
            return self.call_out_of_line(n, name)
        if name in self.call_stack:
            raise LoweringError(f"recursive FuncCall {name!r} has no VM lowering")
        fn = self.g.functions[name]
        self.call_stack.append(name)
        outs = self.frame(fn.body, [self.of(r) for r in n.inputs])
        self.call_stack.pop()
        for k, s in enumerate(outs):
            # fresh output slots (the body's slots are reused by other calls)
            o = self.new_slot()
            self.emit("VIEW", n, o, s)
            self.bind(n, k, o)


    def call_out_of_line(self, n, name):
        """CALL of a recursive function (compiled once by `function`): extra =
        [nargs, args..., nres, dests...]; the frame range and entry are read
        from the function's header (patched in `finish`)."""
        args = [self.of(r) for r in n.inputs]
        dests = [self.new_slot() for _ in n.out_types]
        ex = self.extra([len(args)] + args + [len(dests)] + dests)
        at = self.emit("CALL", n, 0, ex, 0, 0)
        self.call_sites.append((at, name))
        for k, d in enumerate(dests):
            self.bind(n, k, d)

    def function(self, name):
        """Out-of-line body of a recursive function: params, body, RET."""
        fn = self.g.functions[name]
        entry = self.here()
        lo = self.p.nslots
        params = [self.new_slot() for _ in fn.body.params]
        outs = self.frame(fn.body, params)
        hi = self.p.nslots
        self.emit("RET", None, self.extra([len(outs)] + outs))
        self.entries[name] = (entry, lo, hi, params)

    def finish(self):
        """Compile every recursive function after main's HALT and patch the
        call sites: CALL a = [entry, extra, lo, hi, params extra]."""
        for name in sorted(self.recursive):
            if name in self.g.functions:
                self.function(name)
        for at, name in self.call_sites:
            entry, lo, hi, params = self.entries[name]
            self.patch(at, 0, entry)
            self.patch(at, 2, lo)
            self.patch(at, 3, hi)
            self.patch(at, 4, self.extra([len(params)] + params))


def _recursive_functions(graph) -> set:
    """Functions that can reach themselves through FuncCall (any nesting of
    Cond / While regions in their bodies)."""
    fns = getattr(graph, "functions", {}) or {}
    callees = {}

    def scan(sg, out):
        for node in sg.nodes:
            if node.op == "FuncCall":
                out.add(node.attrs["fn_name"])
            for key in ("then_graph", "else_graph", "test_graph", "body_graph"):
                sub = node.attrs.get(key) if hasattr(node, "attrs") else None
                if sub is not None and hasattr(sub, "nodes"):
                    scan(sub, out)
    for name, fn in fns.items():
        callees[name] = set()
        scan(fn.body, callees[name])
    rec = set()
    for start in fns:
        seen, todo = set(), list(callees.get(start, ()))
        while todo:
            f = todo.pop()
            if f == start:
                rec.add(start)
                break
            if f in seen or f not in callees:
                continue
            seen.add(f)
            todo.extend(callees[f])
    return rec


def _result_dtype(op, a, b):
    """reference tensor.py:252-267 (None = DtypeMismatch)."""
    if op in ("Lt", "Gt", "Le", "Ge", "Eq", "Ne"):
        if op in ("Eq", "Ne"):
            if (a == "bool") != (b == "bool"):
                return None
        elif a == "bool" or b == "bool":
            return None
        return "bool"
    if a == "bool" or b == "bool":
        return None
    if op == "Div":
        return "f64"
    return "f64" if "f64" in (a, b) else "i64"


def compile_graph(graph) -> Program:
    c = _Compiler(graph)
    for p in graph.main.params:
        s = c.new_slot()
        c.p.feed_slots[p.attrs.get("name")] = s
        c.bind(p, 0, s)
        c.note_shape(p.out_types[0])
    for node in graph.main.nodes:
        c.node(node)
    c.p.outputs = [c.of(r) for r in graph.main.outputs]
    c.emit("HALT")
    c.finish()
    return c.p


# ---------------------------------------------------------------- runtime
def _words(arr, dtype):
    """Host value -> int64 words (f64 bit patterns, i64, bool as 0/1)."""
    try:
        a = np.ascontiguousarray(arr)
    except OverflowError:
        raise E.IntegerOverflow("an integer constant or feed exceeds int64 (the reference's ints are unbounded)")
    if a.dtype == object:
        raise E.IntegerOverflow("an integer constant or feed exceeds int64 (the reference's ints are unbounded)")
    if dtype == "f64":
        return a.astype(np.float64).view(np.int64).reshape(-1)
    return a.astype(np.int64).reshape(-1)


class _Trees:
    """Device table of tree nodes: value (NaN = empty), left, right."""

    def __init__(self):
        self.val, self.left, self.right = [], [], []

    def add(self, t) -> int:
        if t is None or getattr(t, "value", None) is None:
            idx = len(self.val)
            self.val.append(float("nan"))
            self.left.append(-1)
            self.right.append(-1)
            return idx
        idx = len(self.val)
        self.val.append(float(t.value))
        self.left.append(-1)
        self.right.append(-1)
        self.left[idx] = self.add(t.left)
        self.right[idx] = self.add(t.right)
        return idx


@_on_stream
def run(prog: Program, feeds: dict, *, stream=None, arena_bytes: Optional[int] = None):
    """Execute a compiled program on the current CUDA device.

    Returns (outputs, print_log)."""
    import torch
    from . import runtime as rt
    lib = rt.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    slots = np.zeros(max(prog.nslots, 1), dtype=VAL_DTYPE)
    slots["own"] = -1
    blobs = []
    off = 0
    trees = _Trees()

    def place(slot, value, dtype):
        nonlocal off
        if dtype == "tree":
            slots[slot]["dtype"] = DT["tree"]
            slots[slot]["numel"] = trees.add(value)
            return
        arr = as_numpy(value)
        shp = tuple(arr.shape)
        if len(shp) > MAX_RANK:
            raise LoweringError(f"rank {len(shp)} exceeds the VM's {MAX_RANK}")
        w = _words(arr, dtype)
        slots[slot]["view"] = off
        slots[slot]["numel"] = w.size
        slots[slot]["dtype"] = DT[dtype]
        slots[slot]["rank"] = len(shp)
        slots[slot]["shape"][:len(shp)] = shp
        blobs.append((off, w))
        off += ((max(w.size, 1) * 8 + 255) // 256) * 256

    for name, s in prog.feed_slots.items():
        v = feeds[name]
        place(s, v, "tree" if isinstance(v, Tree) or (hasattr(v, "is_empty") and not hasattr(v, "dtype"))
              else infer_dtype(v))
    for s, v in prog.consts:
        place(s, v, v.dtype)
    static_bytes = off
    big = max(prog.static_elems, max((w.size for _, w in blobs), default=0))
    if arena_bytes is None:
        arena_bytes = int(min(max(64 << 20, 64 * static_bytes), 8 << 30))
    for attempt in range(4):
        arena = torch.zeros(arena_bytes, dtype=torch.uint8, device=dev)
        host = np.zeros(static_bytes // 8 + 1, dtype=np.int64)
        for o, w in blobs:
            host[o // 8:o // 8 + w.size] = w
        arena[:static_bytes].copy_(torch.from_numpy(host.view(np.uint8)[:static_bytes]))
        code = torch.from_numpy(np.asarray(prog.code, dtype=np.int32).reshape(-1)).to(dev)
        extra = torch.from_numpy(np.asarray(prog.extra + [0], dtype=np.int32)).to(dev)
        ctas = 1
        if big >= int(os.environ.get("SKB_VM_GRID_MIN", 1 << 13)):   # grid of CTAs from 8 K-element tensors
            ctas = max(1, int(lib.skb_vm_max_ctas()))
        # one copy of the slot table per CTA (results are read from copy 0)
        dslots = torch.from_numpy(np.tile(slots.view(np.uint8), ctas)).to(dev)
        scratch = torch.zeros(2 * max(ctas, 1), dtype=torch.float64, device=dev)
        tv = torch.tensor(trees.val + [0.0], dtype=torch.float64, device=dev)
        tl = torch.tensor(trees.left + [0], dtype=torch.int32, device=dev)
        tr = torch.tensor(trees.right + [0], dtype=torch.int32, device=dev)
        log_cap = 1 << 16
        log = torch.zeros(log_cap * 8, dtype=torch.int64, device=dev)
        ctl = torch.zeros(8, dtype=torch.int64, device=dev)
        rt.check(lib.skb_vm_run(rt.ptr(code), rt.ptr(extra), rt.ptr(dslots), rt.ptr(arena), arena_bytes,
                                static_bytes, rt.ptr(scratch), rt.ptr(tv), rt.ptr(tl), rt.ptr(tr), rt.ptr(log),
                                log_cap, rt.ptr(ctl), 1 << 40, ctas, len(slots), rt.stream_handle(stream)), "skb_vm_run")
        c = ctl.cpu().numpy()
        err = int(c[0] & 0xFFFFFFFF)
        if err == E_ARENA and attempt < 3:
            arena_bytes *= 4
            continue
        break
    err_uid = int(c[0] >> 32)
    if err:
        node = prog.nodes.get(err_uid)
        span = getattr(node, "origin", None)
        if err == 14:
            limit = node.attrs.get("max_iterations") if node is not None else None
            raise E.IterationLimitExceeded(f"loop exceeded max_iterations={limit}", span)
        if err in CAUSE:
            raise RuntimeGraphError(_message(err, node, int(c[1])), span, CAUSE[err])
        if err == E_OVERFLOW:
            raise E.IntegerOverflow(f"int64 overflow at node {err_uid} (the reference's ints are unbounded)", span)
        if err == E_DEPTH:
            raise E.DeviceError(f"recursion deeper than {int(c[1])} calls at node {err_uid}")
        raise E.DeviceError(f"VM failure code {err} at node {err_uid}")
    host_slots = np.frombuffer(dslots[:slots.nbytes].cpu().numpy().tobytes(), dtype=VAL_DTYPE)
    outs = [_value(arena, host_slots[s], trees) for s in prog.outputs]
    log_count = int(c[3])
    plog = _print_log(prog, arena, log, log_count, trees) if log_count else []
    return outs, plog


def _message(code, node, detail):
    if code == 15:
        return (node.attrs.get("message") if node is not None else None) or "assertion failed"
    return {10: f"index {detail} out of range", 11: "pop from an empty list", 12: "shape mismatch",
            13: "division by zero", 16: "dtype mismatch", 17: "empty tree has no value"}.get(code, "error")


def _tensor(arena, d):
    import torch
    dt = DT_NAME[int(d["dtype"])]
    rank = int(d["rank"])
    shape = tuple(int(x) for x in d["shape"][:rank])
    n = int(d["numel"])
    start = int(d["view"])
    words = arena[start:start + 8 * n].view(torch.int64)
    if dt == "f64":
        t = words.view(torch.float64).reshape(shape)
    elif dt == "bool":
        t = (words != 0).reshape(shape)
    else:
        t = words.reshape(shape)
    return DeviceTensor(dt, t)


def _value(arena, d, trees):
    dt = int(d["dtype"])
    if dt == DT["list"]:
        n = int(d["numel"])
        raw = arena[int(d["view"]):int(d["view"]) + 64 * n].cpu().numpy()
        items = np.frombuffer(raw.tobytes(), dtype=VAL_DTYPE)
        return ListValue([_value(arena, it, trees) for it in items])
    if dt == DT["tree"]:
        return _tree_from(trees, int(d["numel"]))
    return _tensor(arena, d)


def _tree_from(trees, idx):
    if idx < 0 or math.isnan(trees.val[idx]):
        return Tree()
    return Tree(trees.val[idx], _tree_from(trees, trees.left[idx]), _tree_from(trees, trees.right[idx]))


def _fmt_scalar(v):
    if isinstance(v, (bool, np.bool_)):
        return "True" if v else "False"
    if isinstance(v, (float, np.floating)):
        return repr(float(v))
    return str(int(v))


def _fmt(v):
    """reference execute.py:252-258"""
    if isinstance(v, DeviceTensor):
        a = v.array
        if v.shape == ():
            return _fmt_scalar(a.reshape(-1)[0].item())
        payload = ",".join(_fmt_scalar(x) for x in a.reshape(-1).tolist())
        return f"{v.dtype}[{','.join(str(s) for s in v.shape)}]:{payload}"
    if isinstance(v, Tree):
        return _tree_str(v)
    if isinstance(v, ListValue):
        return "ListValue(items=[" + ", ".join(_fmt(i) for i in v.items) + "])"
    return str(v)


def _tree_str(t):
    if t.value is None:
        return "()"
    return f"({_fmt_scalar(t.value)} {_tree_str(t.left)} {_tree_str(t.right)})"


def _print_log(prog, arena, log, count, trees):
    recs = np.frombuffer(log[:min(count, log.numel() // 8) * 8].cpu().numpy().tobytes(), dtype=VAL_DTYPE)
    out, i = [], 0
    while i < len(recs):
        n = int(recs[i]["numel"])
        vals = [_value(arena, recs[i + 1 + k], trees) for k in range(n)]
        out.append(" ".join(_fmt(v) for v in vals))
        i += 1 + n
    return out
