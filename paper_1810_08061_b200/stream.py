"""Vector-stream tier: staged While/Cond programs over scalars and vectors of
one large shape, executed by the persistent kernel in csrc/stream.cu.

This is the lowering for the BASELINE config C4 class of programs (L-BFGS,
in-graph SGD, element-wise iterative solvers — SURVEY §8(a) A1/A2/A6/A9/A10
with 10^7-element vectors).  `compile_graph` accepts a reference (or skb)
graph when every tensor it carries is either a scalar or has one common
"stream" shape S, and every op is element-wise / a full reduction / list /
control flow.  Anything else raises `LoweringError` and the executor uses the
generic region VM instead (vm.py) — never a CPU path.

Compilation (value classes, reference semantics in parentheses):

* scalars, lists and control flow become scalar-phase instructions that every
  CTA executes redundantly on its private state (no grid barrier);
* element-wise nodes on S-shaped values (tensor.py:227-300, 356-407) are not
  emitted one by one: they are kept as pending expression trees and fused
  into the consumer, so `q - al * y` is one pass over q and y;
* a fused group (VEXEC) collects every expression materialised or reduced
  between two points where the scalar side needs a result; a value the group
  stores and reuses is recomputed from the staged operands (cheap flops, no
  HBM re-read, no temporaries);
* each reduction (tensor.py:335-353) ends in RFIN: the only cross-CTA
  exchange, combined in a fixed order so every CTA holds the same bits.

Vector values are immutable reference-counted buffers; ListGet/ListSet/loop
state moves only move buffer ids (execute.py:148-185 copy semantics hold
because buffers are never written after they are produced).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .runtime import on_stream as _on_stream

from . import errors as E
from .errors import LoweringError, RuntimeGraphError
from .values import DeviceTensor, ListValue, as_numpy, infer_dtype, shape_of

# csrc/stream.cu enums
SOP = dict(HALT=0, BIN=1, UN=2, SEL=3, MOV=4, SELREF=5, LNEW=6, LAPPEND=7, LPOP=8, LGET=9, LSET=10,
           JMP=11, JZ=12, ITER=13, SETI=14, ASSERT=15, RAISE=16, ALLOC=17, VEXEC=18, RFIN=19)
V_PUSH, V_BIN, V_UN, V_SEL, V_STORE, V_RED, V_SAVE, V_POP = 1, 2, 3, 4, 5, 6, 7, 8
SRC_STACK, SRC_VEC, SRC_SCALAR, SRC_TEMP = 0, 1, 2, 3
K_SCALAR, K_VEC, K_LIST_S, K_LIST_V = 0, 1, 2, 3
BIN = {"Add": 0, "Sub": 1, "Mul": 2, "Div": 3, "Mod": 4, "Lt": 5, "Gt": 6, "Le": 7, "Ge": 8, "Eq": 9, "Ne": 10}
UN = {"Neg": 0, "Not": 1, "Tanh": 2, "Sigmoid": 3}
DT = {"f64": 0, "i64": 1, "bool": 2}
DT_NAME = {v: k for k, v in DT.items()}
RMAX = 4
TPB, TILE = 512, 2048
MAX_OPS, MAX_TEMP, MAX_STACK = 5, 4, 3
CAUSE = {10: E.INDEX_OUT_OF_RANGE, 11: E.EMPTY_POP, 12: E.SHAPE_MISMATCH, 13: E.DIVISION_BY_ZERO,
         14: E.ITERATION_LIMIT, 15: E.ASSERTION_FAILED, 16: E.DTYPE_MISMATCH}
E_POOL, E_STEPS, E_CAP = 30, 31, 32
SUPPORTED = set(BIN) | set(UN) | {"Const", "Where", "ReduceSum", "ReduceMax", "ListNew", "ListAppend",
                                  "ListPop", "ListGet", "ListSet", "Cond", "While", "FuncCall", "Assert"}


# ------------------------------------------------------------------ values
@dataclass
class Slot:
    kind: int            # K_*
    word: int
    dtype: str           # element dtype (f64/i64/bool)
    cap: int = 0         # lists


@dataclass
class Leaf:              # expression leaf: a vector or scalar word
    word: int
    dtype: str
    vec: bool


@dataclass
class Expr:              # pending element-wise expression on S-shaped values
    op: str              # 'bin' | 'un' | 'sel'
    code: int
    args: list
    dtype: str
    uses: int = 1        # remaining consumers
    node: object = None
    slot: Optional[Slot] = None   # set once materialised


def _dt_of(x):
    return x.dtype


@dataclass
class Group:
    ops: list = field(default_factory=list)        # vector operand words (staged)
    stores: list = field(default_factory=list)     # store destination words
    reds: list = field(default_factory=list)       # (kind|dt<<4, dst word)
    code: list = field(default_factory=list)       # 4-int vector instructions
    reads: set = field(default_factory=set)        # words read (vector + scalar)
    expr_of: dict = field(default_factory=dict)    # stored word -> its expression (recomputed on reuse)
    uids: dict = field(default_factory=dict)       # vector instruction index -> node uid
    depth: int = 0

    def empty(self):
        return not self.code


@dataclass
class StreamProgram:
    code: list
    extra: list
    nwords: int
    w_init: np.ndarray
    feeds: dict                 # name -> Slot (vector feeds: word holds the feed buffer id)
    outputs: list               # Slot per main output
    shape: tuple                # compile-time stream shape (None dims allowed)
    nodes: dict
    max_ops: int
    max_stack: int
    max_temp: int
    vec_refs: int               # upper bound of simultaneously referenced buffers
    groups: int = 0
    vuids: dict = field(default_factory=dict)

    @property
    def nbuf_bound(self):
        return self.vec_refs


# ------------------------------------------------------------------ analysis
def _subgraphs(node):
    for k in ("then_graph", "else_graph", "test_graph", "body_graph"):
        if k in node.attrs:
            yield node.attrs[k]


def _all_frames(graph):
    seen = []
    stack = [graph.main] + [f.body for f in getattr(graph, "functions", {}).values()]
    while stack:
        sg = stack.pop()
        seen.append(sg)
        for n in sg.nodes:
            stack.extend(_subgraphs(n))
    return seen


def _unify(a, b):
    if a is None:
        return b
    if len(a) != len(b):
        return False
    return tuple(x if x is not None else y for x, y in zip(a, b)) if all(
        x is None or y is None or x == y for x, y in zip(a, b)) else False


def stream_shape(graph):
    """The single non-scalar tensor shape of the graph, or raise LoweringError."""
    shape = None
    lists_append = False
    max_new = 0
    for sg in _all_frames(graph):
        specs = [p.out_types[0] for p in sg.params]
        for n in sg.nodes:
            if n.op not in SUPPORTED:
                raise LoweringError(f"op {n.op} is outside the vector-stream tier")
            if n.op == "Const":
                v = n.attrs["value"]
                if shape_of(v) != () or infer_dtype(v) not in DT:
                    raise LoweringError("non-scalar constant")
            if n.op == "ListAppend":
                lists_append = True
            if n.op == "ListNew":
                max_new = max(max_new, len(n.inputs))
            specs.extend(n.out_types)
        for t in specs:
            if t is None:
                raise LoweringError("untyped value")
            if t.dtype == "list":
                if t.elem is None or t.elem.dtype not in DT or t.elem.shape is None:
                    raise LoweringError("list with unknown element type")
                t = t.elem
            if t.dtype not in DT or t.shape is None:
                raise LoweringError(f"value of type {t.dtype} outside the vector-stream tier")
            if tuple(t.shape) == ():
                continue
            u = _unify(shape, tuple(t.shape))
            if u is False:
                raise LoweringError(f"second tensor shape {t.shape} (stream shape {shape})")
            shape = u
    if shape is None:
        raise LoweringError("no vector values: scalar programs run on the region VM")
    cap = max(max_new, 1) + (64 if lists_append else 0)
    return shape, cap


def _uses(sg):
    u = {}
    for n in sg.nodes:
        for r in n.inputs:
            k = (id(r.node), r.out)
            u[k] = u.get(k, 0) + 1
    for r in sg.outputs:
        k = (id(r.node), r.out)
        u[k] = u.get(k, 0) + 1
    return u


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


# device encoding (csrc/stream.cu DOp): the operand source folded into the opcode
D_PUSH = {SRC_VEC: 1, SRC_SCALAR: 2}
D_BIN = {SRC_VEC: 4, SRC_SCALAR: 5, SRC_STACK: 7}
D_UN, D_SEL, D_STORE, D_RED, D_POP = 8, 9, 10, 11, 13
D_FV, D_FS, D_FK, D_RSUM = 20, 30, 40, 50
F64_ALL = 0 | (0 << 4) | (0 << 8)   # dta | dtb << 4 | dto << 8, all f64


def _device_code(code):
    out = []
    for k in range(0, len(code), 4):
        op, x, y, z = code[k:k + 4]
        if op == V_PUSH:                        # [src, idx, spill]
            out += [D_PUSH[x], y, z, 0]
        elif op == V_BIN:                       # [bop | rev << 8 | src << 12, idx, dts]
            bop, rev, src = x & 255, (x >> 8) & 1, (x >> 12) & 15
            if z == F64_ALL and bop <= 2:       # f64 add/sub/mul: a specialised dispatch case
                if src == SRC_VEC:
                    out += [D_FV + 2 * bop + rev, y, 0, 0]
                    continue
                if src == SRC_SCALAR:
                    out += [D_FS + 2 * bop + rev, y, 0, 0]
                    continue
                if src == SRC_STACK:
                    out += [D_FK + bop, 0, 0, 0]
                    continue
            out += [D_BIN[src], y, x & 0xFFF, z]
        elif op == V_UN:
            out += [D_UN, x, 0, z]
        elif op == V_SEL:
            out += [D_SEL, 0, 0, 0]
        elif op == V_STORE:
            out += [D_STORE, x, 0, 0]
        elif op == V_RED:                       # [r, kind, dt]
            out += [D_RSUM + x, 0, 0, 0] if (y == 0 and z == DT["f64"]) else [D_RED, x, 0, 0]
        else:
            out += [D_POP, 0, 0, 0]
    return out


# ------------------------------------------------------------------ compiler
class _Compiler:
    def __init__(self, graph, shape, cap):
        self.g = graph
        self.shape = shape
        self.cap = cap
        self.code = []
        self.extra = []
        self.nwords = 0
        self.init = {}                  # word -> int64 initial value
        self.val = {}                   # (id(node), out) -> Slot | Expr
        self.uses = {}
        self.nodes = {}
        self.grp = Group()
        self.red_words = set()          # words written by RFIN of the open group
        self.max_ops = 1
        self.max_temp = 1
        self.max_stack = 1
        self.vec_refs = 0
        self.ngroups = 0
        self.call_stack = []
        self.vuids = {}                 # VEXEC pc -> {vector instruction -> node uid}

    # ------------------------------------------------------------ storage
    def new_slot(self, kind, dtype, cap=0):
        w = self.nwords
        if kind in (K_LIST_S, K_LIST_V):
            self.nwords += 1 + cap
            self.init[w] = 0
            for i in range(cap):
                self.init[w + 1 + i] = -1 if kind == K_LIST_V else 0
            if kind == K_LIST_V:
                self.vec_refs += cap
        else:
            self.nwords += 1
            self.init[w] = -1 if kind == K_VEC else 0
            if kind == K_VEC:
                self.vec_refs += 1
        return Slot(kind, w, dtype, cap)

    def slot_for_type(self, t):
        if t.dtype == "list":
            e = t.elem
            return self.new_slot(K_LIST_V if tuple(e.shape) != () else K_LIST_S, e.dtype, self.cap)
        return self.new_slot(K_VEC if tuple(t.shape) != () else K_SCALAR, t.dtype)

    # ------------------------------------------------------------ emission
    def semit(self, op, node, args, reads=(), writes=()):
        """Emit a scalar-phase instruction, flushing the open group first when
        the instruction reads one of its reductions or overwrites a word it reads."""
        if any(w in self.red_words for w in reads) or \
                any(w in self.grp.reads or w in self.grp.stores for w in writes):
            self.flush()
        uid = node.uid if node is not None else 0
        if node is not None:
            self.nodes[uid] = node
        a = list(args) + [0] * (6 - len(args))
        self.code.append([SOP[op], uid] + [int(x) for x in a])
        return len(self.code) - 1

    def here(self):
        return len(self.code)

    def extra_block(self, values):
        off = len(self.extra)
        self.extra.extend(int(v) for v in values)
        return off

    def flush(self):
        g = self.grp
        if g.empty():
            return
        self.grp = Group()
        red_words, self.red_words = self.red_words, set()
        self.max_ops = max(self.max_ops, len(g.ops))
        self.max_stack = max(self.max_stack, g.depth)
        self.ngroups += 1
        blk = [len(g.ops), len(g.stores), len(g.reds), len(g.code) // 4] + g.ops + g.stores + \
            [kd for kd, _ in g.reds] + _device_code(g.code)
        off = self.extra_block(blk)
        self.vuids[len(self.code)] = g.uids
        self.code.append([SOP["VEXEC"], 0, off, 0, 0, 0, 0, 0])
        for r, (kd, w) in enumerate(g.reds):
            self.code.append([SOP["RFIN"], 0, w, r, kd, 1 if r == 0 else 0, 0, 0])
        del red_words

    # ------------------------------------------------------------ values
    def value(self, ref):
        return self.val[(id(ref.node), ref.out)]

    def use(self, ref):
        """Consume one use of a value (pending expressions count down)."""
        v = self.value(ref)
        return v

    def slot_of(self, v, node=None):
        """Materialise `v` (Slot or pending Expr) into a slot."""
        if isinstance(v, Slot):
            return v
        if v.slot is not None:
            return v.slot
        s = self.new_slot(K_VEC, v.dtype)
        self.materialize(v, s, node)
        return s

    def materialize(self, e, s, node=None):
        """Compute pending expression `e` into vector slot `s` in the open group.
        Later readers in the same group recompute it from the staged operands
        (csrc/stream.cu keeps no temporaries)."""
        self._prepare(e)
        self.semit("ALLOC", node or e.node, [s.word], writes=[s.word])
        g = self.grp
        self.gen(e)
        g.code += [V_STORE, len(g.stores), 0, 0]
        g.stores.append(s.word)
        g.expr_of[s.word] = e
        e.slot = s

    def reduce_into(self, e, kind, dst, node):
        self._prepare(e)
        g = self.grp
        if len(g.reds) >= RMAX:
            self.flush()
            self._prepare(e)
            g = self.grp
        self.gen(e)
        kd = kind | (DT[e.dtype] << 4)
        g.code += [V_RED, len(g.reds), kind, DT[e.dtype]]
        g.reds.append((kd, dst.word))
        self.red_words.add(dst.word)

    def _expand(self, e):
        """The expression to generate for `e` in the open group: values the
        group itself stores are recomputed from their expression."""
        g = self.grp
        if isinstance(e, Leaf):
            return g.expr_of.get(e.word, e) if e.vec else e
        if e.slot is not None:
            return g.expr_of.get(e.slot.word, Leaf(e.slot.word, e.dtype, True))
        return e

    def _leaves(self, e, out):
        e = self._expand(e)
        if isinstance(e, Leaf):
            out.append(e)
        else:
            for a in e.args:
                self._leaves(a, out)
        return out

    def _prepare(self, e):
        """Flush first if the open group cannot take `e` (operand budget, or a
        scalar leaf that is one of its own pending reductions)."""
        leaves = self._leaves(e, [])
        if any((not l.vec) and l.word in self.red_words for l in leaves):
            self.flush()
            leaves = self._leaves(e, [])
        g = self.grp
        new_ops = {l.word for l in leaves if l.vec and l.word not in g.ops}
        if len(g.ops) + len(new_ops) > MAX_OPS or len(g.stores) >= 16 or len(g.code) // 4 > 192:
            self.flush()
            if len({l.word for l in self._leaves(e, []) if l.vec}) > MAX_OPS:
                raise LoweringError("element-wise expression reads more vectors than one pass stages")

    def gen(self, e, live=0):
        """Postfix code leaving e's value in the TOS register.  `live` = values
        already on the virtual stack (TOS included)."""
        g = self.grp
        e = self._expand(e)
        if isinstance(e, Leaf):
            src, idx = self.leaf_src(e)
            g.code += [V_PUSH, src, idx, 1 if live > 0 else 0]
            g.depth = max(g.depth, live)
            return
        if e.op == "un":
            self.gen(e.args[0], live)
            g.code += [V_UN, e.code, 0, DT[e.args[0].dtype] | (DT[e.dtype] << 8)]
            return
        if e.op == "sel":
            c, x, y = e.args
            self.gen(c, live)
            self.gen(x, live + 1)
            self.gen(y, live + 2)
            g.code += [V_SEL, 0, 0, 0]
            return
        L, R = e.args
        dts = DT[L.dtype] | (DT[R.dtype] << 4) | (DT[e.dtype] << 8)
        Lx, Rx = self._expand(L), self._expand(R)
        if isinstance(Rx, Leaf):
            self.gen(Lx, live)
            src, idx = self.leaf_src(Rx)
            g.code += [V_BIN, e.code | (src << 12), idx, dts]
        elif isinstance(Lx, Leaf):
            self.gen(Rx, live)
            src, idx = self.leaf_src(Lx)
            g.code += [V_BIN, e.code | (1 << 8) | (src << 12), idx, dts]
        else:
            self.gen(Lx, live)
            self.gen(Rx, live + 1)
            g.code += [V_BIN, e.code | (SRC_STACK << 12), 0, dts]
        if e.node is not None:
            g.uids[len(g.code) // 4 - 1] = e.node.uid
        if g.depth > MAX_STACK:
            raise LoweringError("expression too deep for the vector-stream tier")

    @staticmethod
    def _as_leaf(x):
        return x if isinstance(x, Leaf) else Leaf(x.slot.word, x.dtype, True)

    def leaf_src(self, l):
        g = self.grp
        g.reads.add(l.word)
        if not l.vec:
            return SRC_SCALAR, l.word
        if l.word in g.stores:
            raise LoweringError("internal: group reads a vector it stores")
        if l.word not in g.ops:
            g.ops.append(l.word)
        return SRC_VEC, g.ops.index(l.word)

    def as_operand(self, v):
        """A value as an expression operand (Leaf or pending Expr)."""
        if isinstance(v, Slot):
            return Leaf(v.word, v.dtype, v.kind == K_VEC)
        if v.slot is None and v.uses > 1:   # shared sub-expression: compute once
            self.slot_of(v)
        return v

    # ------------------------------------------------------------ frames
    def frame(self, sg, params):
        """Compile subgraph `sg` with its params bound to `params` (Slot/Expr)."""
        uses = _uses(sg)
        saved = self.uses
        self.uses = uses
        for p, v in zip(sg.params, params):
            n = uses.get((id(p), 0), 0)
            if isinstance(v, Expr) and v.slot is None and n != 1:
                v = self.slot_of(v)
            self.val[(id(p), 0)] = v
        for node in sg.nodes:
            self.node(node)
        outs = [self.value(r) for r in sg.outputs]
        self.uses = saved
        return outs

    def node(self, n):
        op = n.op
        self.nodes[n.uid] = n
        ins = n.inputs
        key = (id(n), 0)
        nuses = self.uses.get(key, 0)
        if op == "Const":
            t = n.out_types[0]
            s = self.new_slot(K_SCALAR, t.dtype)
            v = n.attrs["value"]
            a = as_numpy(v).reshape(-1)
            self.init[s.word] = int(a.astype(np.float64).view(np.int64)[0]) if t.dtype == "f64" else int(a[0])
            self.val[key] = s
            return
        vals = [self.value(r) for r in ins]
        if op in BIN or op in UN or op == "Where":
            out_t = n.out_types[0]
            vec = tuple(out_t.shape) != ()
            if op in BIN:
                out_dt = _result_dtype(op, vals[0].dtype, vals[1].dtype)
            elif op == "Where":
                out_dt = vals[1].dtype if vals[0].dtype == "bool" and vals[1].dtype == vals[2].dtype else None
            else:
                a = vals[0].dtype
                bad = (op == "Neg" and a == "bool") or (op == "Not" and a != "bool") or \
                    (op in ("Tanh", "Sigmoid") and a == "bool")
                out_dt = None if bad else ("f64" if op in ("Tanh", "Sigmoid") else a)
            if out_dt is None:
                raise LoweringError(f"{op}: static dtype failure (left to the region VM)")
            if op == "Where":
                cvec = self._is_vec(vals[0])
                avec, bvec = self._is_vec(vals[1]), self._is_vec(vals[2])
                if avec != bvec or (cvec and not avec):
                    raise LoweringError("Where with mismatched operand shapes")
                if not cvec and avec:       # scalar condition: whole-tensor select (tensor.py:367-368)
                    pred = self.scalar_slot(vals[0], n)
                    a = self.slot_of(vals[1], n)
                    b = self.slot_of(vals[2], n)
                    s = self.new_slot(K_VEC, out_dt)
                    self.semit("SELREF", n, [s.word, pred.word, a.word, b.word],
                               reads=[pred.word, a.word, b.word], writes=[s.word])
                    self.val[key] = s
                    return
                if not cvec:
                    c, a, b = (self.scalar_slot(v, n) for v in vals)
                    s = self.new_slot(K_SCALAR, out_dt)
                    self.semit("SEL", n, [s.word, c.word, a.word, b.word], reads=[c.word, a.word, b.word],
                               writes=[s.word])
                    self.val[key] = s
                    return
                self.val[key] = Expr("sel", 0, [self.as_operand(v) for v in vals], out_dt, nuses, n)
                return
            if not vec:
                if op in BIN:
                    a, b = self.scalar_slot(vals[0], n), self.scalar_slot(vals[1], n)
                    s = self.new_slot(K_SCALAR, out_dt)
                    dts = DT[a.dtype] | (DT[b.dtype] << 4) | (DT[out_dt] << 8)
                    self.semit("BIN", n, [s.word, a.word, b.word, BIN[op], dts], reads=[a.word, b.word],
                               writes=[s.word])
                else:
                    a = self.scalar_slot(vals[0], n)
                    s = self.new_slot(K_SCALAR, out_dt)
                    self.semit("UN", n, [s.word, a.word, UN[op], DT[a.dtype] | (DT[out_dt] << 8)],
                               reads=[a.word], writes=[s.word])
                self.val[key] = s
                return
            code = BIN[op] if op in BIN else UN[op]
            kind = "bin" if op in BIN else "un"
            args = [self.as_operand(v) for v in vals]
            # scalar operands that are pending reductions are fine (flush at emission)
            self.val[key] = Expr(kind, code, args, out_dt, nuses, n)
            if nuses == 0:
                self.val[key] = Expr(kind, code, args, out_dt, 0, n)   # dead: never emitted
            return
        if op in ("ReduceSum", "ReduceMax"):
            v = vals[0]
            if v.dtype == "bool":
                raise LoweringError("reduction of bool (left to the region VM)")
            s = self.new_slot(K_SCALAR, v.dtype)
            if not self._is_vec(v):
                src = self.scalar_slot(v, n)
                self.semit("MOV", n, [s.word, src.word, K_SCALAR], reads=[src.word], writes=[s.word])
            else:
                self.reduce_into(self.as_operand(v), 1 if op == "ReduceMax" else 0, s, n)
            self.val[key] = s
            return
        if op == "ListNew":
            s = self.slot_for_type(n.out_types[0])
            items = [self.item_slot(v, s.kind, n) for v in vals]
            off = self.extra_block([len(items)] + [i.word for i in items])
            self.semit("LNEW", n, [s.word, off, s.kind, s.cap], reads=[i.word for i in items],
                       writes=self._list_words(s))
            self.val[key] = s
            return
        if op == "ListAppend":
            lst = vals[0]
            s = self.slot_for_type(n.out_types[0])
            item = self.item_slot(vals[1], lst.kind, n)
            self.semit("LAPPEND", n, [s.word, lst.word, item.word, lst.kind, s.cap],
                       reads=self._list_words(lst) + [item.word], writes=self._list_words(s))
            self.val[key] = s
            return
        if op == "ListPop":
            lst = vals[0]
            sl = self.slot_for_type(n.out_types[0])
            si = self.new_slot(K_VEC if lst.kind == K_LIST_V else K_SCALAR, lst.dtype)
            self.semit("LPOP", n, [sl.word, si.word, lst.word, lst.kind],
                       reads=self._list_words(lst), writes=self._list_words(sl) + [si.word])
            self.val[key] = sl
            self.val[(id(n), 1)] = si
            return
        if op == "ListGet":
            lst = vals[0]
            idx = self.scalar_slot(vals[1], n)
            s = self.new_slot(K_VEC if lst.kind == K_LIST_V else K_SCALAR, lst.dtype)
            self.semit("LGET", n, [s.word, lst.word, idx.word, lst.kind],
                       reads=self._list_words(lst) + [idx.word], writes=[s.word])
            self.val[key] = s
            return
        if op == "ListSet":
            lst = vals[0]
            idx = self.scalar_slot(vals[1], n)
            item = self.item_slot(vals[2], lst.kind, n)
            s = self.slot_for_type(n.out_types[0])
            self.semit("LSET", n, [s.word, lst.word, idx.word, item.word, lst.kind],
                       reads=self._list_words(lst) + [idx.word, item.word], writes=self._list_words(s))
            self.val[key] = s
            return
        if op == "Assert":
            p = self.scalar_slot(vals[0], n)
            self.semit("ASSERT", n, [p.word], reads=[p.word])
            return
        if op == "Cond":
            return self.cond(n, vals)
        if op == "While":
            return self.loop(n, vals)
        if op == "FuncCall":
            name = n.attrs["fn_name"]
            if name in self.call_stack:
                raise LoweringError(f"recursive FuncCall {name!r}")
            fn = self.g.functions[name]
            self.call_stack.append(name)
            outs = self.frame(fn.body, vals)
            self.call_stack.pop()
            for k, v in enumerate(outs):
                if isinstance(v, Expr) and v.slot is None:
                    v.uses = self.uses.get((id(n), k), 0)
                self.val[(id(n), k)] = v
            return
        raise LoweringError(f"op {op} is outside the vector-stream tier")

    def _is_vec(self, v):
        return (isinstance(v, Slot) and v.kind == K_VEC) or isinstance(v, Expr)

    @staticmethod
    def _list_words(s):
        return [s.word + i for i in range(1 + s.cap)]

    def scalar_slot(self, v, node):
        if not isinstance(v, Slot) or v.kind != K_SCALAR:
            raise LoweringError("expected a scalar value")
        return v

    def item_slot(self, v, list_kind, node):
        if list_kind == K_LIST_V:
            return self.slot_of(v, node)
        return self.scalar_slot(v, node)

    def copy_into(self, dst, v, node):
        """dst <- v for a Cond output / loop state (pending expressions are
        computed straight into dst)."""
        if isinstance(v, Expr) and v.slot is None:
            v.uses = max(v.uses, 1)
            self.materialize(v, dst, node)
            v.slot = None   # the expression may be materialised again elsewhere
            return
        src = self.slot_of(v, node)
        words_w = self._list_words(dst) if dst.kind in (K_LIST_S, K_LIST_V) else [dst.word]
        words_r = self._list_words(src) if src.kind in (K_LIST_S, K_LIST_V) else [src.word]
        self.semit("MOV", node, [dst.word, src.word, dst.kind], reads=words_r, writes=words_w)

    def cond(self, n, vals):
        nt = n.attrs["n_then_caps"]
        pred = self.scalar_slot(vals[0], n)
        # pending captures are computed before the branch: a value first
        # materialised inside one branch would not exist on the other path
        vals = [self.slot_of(v, n) if isinstance(v, Expr) else v for v in vals]
        then_caps, else_caps = vals[1:1 + nt], vals[1 + nt:]
        outs = [self.slot_for_type(t) for t in n.out_types]
        self.flush()
        jz = self.semit("JZ", n, [pred.word, 0], reads=[pred.word])
        res = self.frame(n.attrs["then_graph"], then_caps)
        for o, r in zip(outs, res):
            self.copy_into(o, r, n)
        self.flush()
        jmp = self.semit("JMP", n, [0])
        self.code[jz][3] = self.here()
        res = self.frame(n.attrs["else_graph"], else_caps)
        for o, r in zip(outs, res):
            self.copy_into(o, r, n)
        self.flush()
        self.code[jmp][2] = self.here()
        for k, o in enumerate(outs):
            self.val[(id(n), k)] = o

    def loop(self, n, vals):
        ns = n.attrs["n_state"]
        nt = n.attrs["n_test_caps"]
        init, test_caps, body_caps = vals[:ns], vals[ns:ns + nt], vals[ns + nt:]
        test_caps = [self.slot_of(v, n) if isinstance(v, Expr) else v for v in test_caps]
        body_caps = [self.slot_of(v, n) if isinstance(v, Expr) else v for v in body_caps]
        state = [self.slot_for_type(t) for t in n.out_types]
        shadow = [self.slot_for_type(t) for t in n.out_types]
        for s, v in zip(state, init):
            self.copy_into(s, v, n)
        limit = n.attrs.get("max_iterations")
        counter = None
        if limit is not None:
            counter = self.new_slot(K_SCALAR, "i64")
            self.semit("SETI", n, [counter.word, 0], writes=[counter.word])
        self.flush()
        top = self.here()
        t = self.frame(n.attrs["test_graph"], state + list(test_caps))
        pred = t[0]
        if not isinstance(pred, Slot) or pred.kind != K_SCALAR:
            raise LoweringError("loop test is not a scalar")
        self.flush()
        jz = self.semit("JZ", n, [pred.word, 0], reads=[pred.word])
        if counter is not None:
            self.semit("ITER", n, [counter.word, int(limit)], reads=[counter.word], writes=[counter.word])
        outs = self.frame(n.attrs["body_graph"], state + list(body_caps))
        for z, o in zip(shadow, outs):
            self.copy_into(z, o, n)
        for s, z in zip(state, shadow):
            self.copy_into(s, z, n)
        self.flush()
        self.semit("JMP", n, [top])
        self.code[jz][3] = self.here()
        for k, s in enumerate(state):
            self.val[(id(n), k)] = s


def compile_graph(graph) -> StreamProgram:
    """Compile `graph` for the vector-stream kernel or raise LoweringError."""
    shape, cap = stream_shape(graph)
    c = _Compiler(graph, shape, cap)
    feeds = {}
    c.uses = _uses(graph.main)
    for p in graph.main.params:
        s = c.slot_for_type(p.out_types[0])
        if s.kind in (K_LIST_S, K_LIST_V):
            raise LoweringError("list feeds are outside the vector-stream tier")
        feeds[p.attrs.get("name")] = s
        c.val[(id(p), 0)] = s
    for node in graph.main.nodes:
        c.node(node)
    outs = []
    for r in graph.main.outputs:
        v = c.value(r)
        if isinstance(v, Expr):
            v = c.slot_of(v)
        outs.append(v)
    c.flush()
    c.code.append([SOP["HALT"], 0, 0, 0, 0, 0, 0, 0])
    w = np.zeros(max(c.nwords, 1), dtype=np.int64)
    for k, v in c.init.items():
        w[k] = v
    return StreamProgram(c.code, c.extra, max(c.nwords, 1), w, feeds, outs, shape, c.nodes, c.max_ops,
                         c.max_stack, c.max_temp, c.vec_refs, c.ngroups, c.vuids)


# ------------------------------------------------------------------ runtime
def _feed_tensor(v, dtype, dev):
    import torch
    t = getattr(v, "tensor", None)
    if t is None and isinstance(v, torch.Tensor):
        t = v
    if t is not None and t.is_cuda:
        t = t.reshape(-1)
        want = torch.float64 if dtype == "f64" else torch.int64
        if t.dtype != want:
            t = t.to(want)
        if not t.is_contiguous() or t.data_ptr() % 16 or t.numel() % 2:
            t = _padded(t)
        return t
    a = as_numpy(v).reshape(-1)
    a = a.astype(np.float64) if dtype == "f64" else a.astype(np.int64)
    return _padded(torch.from_numpy(np.ascontiguousarray(a)).to(dev))


def _padded(t):
    """A 16-byte aligned copy whose length is even: the kernel stages whole
    16-byte units, so the last tile of an odd-length vector reads one pad word."""
    import torch
    if t.numel() % 2 == 0 and t.is_contiguous() and t.data_ptr() % 16 == 0:
        return t
    out = torch.zeros(t.numel() + (t.numel() % 2), dtype=t.dtype, device=t.device)
    out[:t.numel()].copy_(t.reshape(-1))
    return out


@_on_stream
def run(prog: StreamProgram, feeds: dict, *, stream=None, pool: Optional[int] = None):
    """Execute on the current CUDA device. Returns the list of outputs."""
    import torch
    from . import runtime as rt
    lib = rt.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    w = prog.w_init.copy()
    vec_feeds = []
    n = None
    for name, s in prog.feeds.items():
        v = feeds[name]
        if s.kind == K_SCALAR:
            a = as_numpy(v).reshape(-1)
            w[s.word] = int(a.astype(np.float64).view(np.int64)[0]) if s.dtype == "f64" else int(a[0])
            continue
        shp = tuple(shape_of(v))
        if n is None:
            n, shape = int(np.prod(shp)), shp
        elif shp != shape:
            raise LoweringError("vector feeds of different shapes")
        w[s.word] = len(vec_feeds)
        vec_feeds.append(_feed_tensor(v, s.dtype, dev))
    if n is None:
        shape = tuple(prog.shape)
        if any(d is None for d in shape):
            raise LoweringError("stream shape is not determined by the feeds")
        n = int(np.prod(shape))
    if n == 0:
        raise LoweringError("empty stream shape")
    nfeed = len(vec_feeds)
    stride = ((n + 31) // 32) * 32
    bound = max(prog.vec_refs, 1)
    npool = pool or min(bound, 64 + prog.max_ops * 4)
    code = torch.from_numpy(np.asarray(prog.code, dtype=np.int32).reshape(-1)).to(dev)
    extra = torch.from_numpy(np.asarray(prog.extra + [0], dtype=np.int32)).to(dev)
    smem = int(lib.skb_stream_smem_bytes(prog.max_ops, prog.max_stack, prog.max_temp, prog.nwords,
                                         nfeed + bound))
    grid = int(lib.skb_stream_grid(smem))
    if grid <= 0:
        raise LoweringError(f"vector-stream program needs {smem} B of shared memory")
    tile = int(lib.skb_stream_tile_elems())
    ntiles = (n + tile - 1) // tile
    for attempt in range(6):
        nbuf = nfeed + npool
        poolbuf = torch.empty(npool * stride, dtype=torch.int64, device=dev)
        ptrs = [t.data_ptr() for t in vec_feeds] + [poolbuf.data_ptr() + 8 * stride * i for i in range(npool)]
        bufptr = torch.tensor(ptrs, dtype=torch.int64, device=dev)
        rc = torch.zeros(nbuf, dtype=torch.int32)
        rc[:nfeed] = 1 << 30
        rc = rc.to(dev)
        w_in = torch.from_numpy(w).to(dev)
        w_out = torch.empty_like(w_in)
        part = torch.empty(2 * RMAX * grid, dtype=torch.int64, device=dev)
        ctl = torch.zeros(16, dtype=torch.int64, device=dev)
        ctl[0] = -1
        g = min(grid, max(1, ntiles))
        cs = torch.cuda.current_stream() if stream is None else stream
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(cs)
        rt.check(lib.skb_stream_run(rt.ptr(code), rt.ptr(extra), rt.ptr(w_in), rt.ptr(w_out), rt.ptr(bufptr),
                                    rt.ptr(rc), rt.ptr(part), rt.ptr(ctl), n, prog.nwords, nbuf, prog.max_ops,
                                    prog.max_stack, prog.max_temp, 1 << 40, len(prog.code), g, smem,
                                    rt.stream_handle(stream)), "skb_stream_run")
        ev1.record(cs)
        c = ctl.cpu().numpy()
        err = int(c[0])
        if err != -1:
            errw = err & 0xFFFFFFFFFFFFFFFF
            code_, pc = errw & 0xFFFF, errw >> 16
            if code_ == E_POOL and npool < bound:
                npool = min(bound, npool * 4)
                continue
            _raise(prog, code_, pc, int(c[1]))
        break
    run.last = {"kernel_ms": ev0.elapsed_time(ev1), "grid": g, "smem": smem, "pool": npool, "barriers": int(c[3]), "steps": int(c[2]),
                "max_live": int(c[5]), "n": n, "cycles_cta0": {"scalar": int(c[6]), "rfin_wait": int(c[7]),
                                                                "vector": int(c[8])}}
    wo = w_out.cpu().numpy()
    outs = [_value(prog, s, wo, w_out, poolbuf, vec_feeds, nfeed, stride, n, shape) for s in prog.outputs]
    return outs


run.last = {}


def _raise(prog, code, pc, detail):
    uid = prog.code[pc][1] if 0 <= pc < len(prog.code) else 0
    if 0 <= pc < len(prog.code) and prog.code[pc][0] == SOP["VEXEC"]:
        uid = prog.vuids.get(pc, {}).get(detail, uid)   # element-wise failure: the fused node
    node = prog.nodes.get(uid)
    span = getattr(node, "origin", None)
    if code == 14:
        limit = node.attrs.get("max_iterations") if node is not None else None
        raise E.IterationLimitExceeded(f"loop exceeded max_iterations={limit}", span)
    if code in CAUSE:
        msg = {10: f"index {detail} out of range", 11: "pop from an empty list", 13: "division by zero",
               15: (node.attrs.get("message") if node is not None else None) or "assertion failed"}.get(code, "error")
        raise RuntimeGraphError(msg, span, CAUSE[code])
    if code == E_CAP:
        raise LoweringError("list grew past the vector-stream tier's capacity")
    raise E.DeviceError(f"vector-stream failure code {code} at instruction {pc} (detail {detail:#x})")


def _vec(buf_id, w_dtype, vec_feeds, nfeed, poolbuf, stride, n, shape):
    import torch
    if buf_id < nfeed:
        t = vec_feeds[buf_id][:n].clone()
    else:
        i = buf_id - nfeed
        t = poolbuf[i * stride:i * stride + n].clone()
    if w_dtype == "f64":
        t = t.view(torch.float64)
    elif w_dtype == "bool":
        t = t != 0
    return DeviceTensor(w_dtype, t.reshape(shape))


def _value(prog, s, wo, w_out, poolbuf, vec_feeds, nfeed, stride, n, shape):
    import torch
    if s.kind == K_SCALAR:
        t = w_out[s.word:s.word + 1].clone()
        if s.dtype == "f64":
            t = t.view(torch.float64)
        elif s.dtype == "bool":
            t = t != 0
        return DeviceTensor(s.dtype, t.reshape(()))
    if s.kind == K_VEC:
        return _vec(int(wo[s.word]), s.dtype, vec_feeds, nfeed, poolbuf, stride, n, shape)
    cnt = int(wo[s.word])
    items = []
    for i in range(cnt):
        x = int(wo[s.word + 1 + i])
        if s.kind == K_LIST_V:
            items.append(_vec(x, s.dtype, vec_feeds, nfeed, poolbuf, stride, n, shape))
        else:
            t = w_out[s.word + 1 + i:s.word + 2 + i].clone()
            t = t.view(torch.float64) if s.dtype == "f64" else (t != 0 if s.dtype == "bool" else t)
            items.append(DeviceTensor(s.dtype, t.reshape(())))
    return ListValue(items)
