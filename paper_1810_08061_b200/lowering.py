"""Lowering of staged graphs onto device kernels.

The reference executes every graph node by node (reference
pkg/src/stagekit/graph/execute.py:98-238).  This module instead recognises
whole staged programs whose hot loop has a device kernel and turns them into
a launch plan; anything else raises ``LoweringError`` (there is no CPU
fallback in the product path).

Recognised today — the dynamic-length recurrent program staged by
``for t in m.range(max_len)`` over a cell (the traced
node list is dumped in SURVEY §8(a) A1):

  main:  Transpose(x, (1,0,2)) ReduceMax(seq_len) Range Const(0) ListNew
         While(state = <idx>, cell states..., outputs-list)
         ListStack(outputs) [Transpose(., (1,0,2))]
  test:  Lt(idx, max_len)                              (dispatch.py:452-453)
  body:  x_t = Index(x_tm, idx)
         gate_k = act_k(MatMul(x_t, W_k) + MatMul(h, U_k) + b_k)   (any + order)
         LSTM: c' = f*c + i*g ; h' = o*tanh(c')     |  RNN: h' = tanh(...)
         GRU (oracle/programs/gru.msl): z, r = sigmoid(x_t Wz + h Uz + bz), ...;
              n = tanh(x_t Wn + bn + r * (h Un + bhn)); h' = (1 - z) * n + z * h
         mask = Lt(idx, seq_len); s = Where(mask, s', s) for each state
         outputs = ListAppend(outputs, h) ; idx' = idx + 1
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from .errors import LoweringError

CELL_LSTM = 1
CELL_RNN_TANH = 2
CELL_GRU = 3


@dataclass
class Source:
    """Where a kernel operand comes from: a graph parameter (feed) or a Const."""
    kind: str                 # "param" | "const"
    name: Optional[str] = None
    value: object = None
    node: object = None

    def key(self):
        return ("param", self.name) if self.kind == "param" else ("const", id(self.value))


@dataclass
class OutputSpec:
    kind: str                 # "seq_bm" | "seq_tm" | "h_final" | "c_final"
    node: object = None


@dataclass
class RnnProgram:
    cell: int
    x: Source                 # batch-major [B, T, F]
    lens: Source              # i64 [B]
    h0: Source
    c0: Optional[Source]
    gates: list               # per gate block (W, U, b) Sources; i, f, g, o (LSTM), (h,) RNN,
                              # z, r, n_x = (Wn, None, bn), n_h = (None, Un, bhn) (GRU)
    outputs: list             # OutputSpec per graph output
    while_node: object = None
    index_node: object = None     # Index(x_tm, idx): IndexOutOfRange span
    range_node: object = None     # Range(max_len):   ShapeMismatch span (negative)
    reduce_node: object = None    # ReduceMax(lens):  ShapeMismatch span (empty)
    stack_node: object = None     # ListStack:        EmptyPop span
    max_iterations: Optional[int] = None
    params: list = field(default_factory=list)   # main Param nodes (feed binding order)


def _t(ref):
    return ref.node.out_types[ref.out]


def _is(ref, op):
    return ref.node.op == op


def _const_value(ref):
    n = ref.node
    return n.attrs.get("value") if n.op == "Const" else None


def _scalar_const(ref):
    v = _const_value(ref)
    if v is None or tuple(v.shape) != ():
        return None
    return v.item() if hasattr(v, "item") else v.data[0]


def _flatten_add(ref, out):
    if _is(ref, "Add"):
        for r in ref.node.inputs:
            _flatten_add(r, out)
    else:
        out.append(ref)
    return out


def _same(a, b) -> bool:
    return a.node is b.node and a.out == b.out


def _fail(msg):
    raise LoweringError(f"no device lowering for this graph: {msg}")


class _Body:
    """Body-frame pattern matching helpers (body param refs -> roles)."""

    def __init__(self, body, n_state, caps_main):
        self.body = body
        self.n_state = n_state
        self.caps_main = caps_main     # capture param index -> main-frame ref

    def param_index(self, ref):
        if ref.node.op != "Param":
            return None
        for i, p in enumerate(self.body.params):
            if p is ref.node:
                return i
        return None

    def is_state(self, ref, k):
        return self.param_index(ref) == k

    def capture(self, ref):
        i = self.param_index(ref)
        if i is None or i < self.n_state:
            return None
        return self.caps_main[i - self.n_state]


def _main_source(ref) -> Source:
    n = ref.node
    if n.op == "Param":
        return Source("param", name=n.attrs.get("name"), node=n)
    if n.op == "Const":
        return Source("const", value=n.attrs["value"], node=n)
    _fail(f"operand produced by main-frame {n.op} (expected a parameter or constant)")


def lower_rnn_program(graph) -> RnnProgram:
    main = graph.main
    for n in main.nodes:
        if n.op in ("Cond", "FuncCall", "Print", "Assert"):
            _fail(f"main frame contains {n.op}")
    whiles = [n for n in main.nodes if n.op == "While"]
    if len(whiles) != 1:
        _fail(f"{len(whiles)} While nodes in the main frame (the recurrent program has one)")
    w = whiles[0]
    allowed = {"Param", "Const", "Transpose", "ReduceMax", "Range", "ListNew", "While", "ListStack"}
    for n in main.nodes:
        if n.op not in allowed:
            _fail(f"main frame op {n.op} outside the recurrent program pattern")
    n_state = w.attrs["n_state"]
    n_test = w.attrs["n_test_caps"]
    init = w.inputs[:n_state]
    test_caps = w.inputs[n_state:n_state + n_test]
    body_caps = w.inputs[n_state + n_test:]
    test_sg, body_sg = w.attrs["test_graph"], w.attrs["body_graph"]
    B = _Body(body_sg, n_state, body_caps)

    # --- loop index: state initialised to Const 0, body output idx + 1
    idx_k = None
    for k in range(n_state):
        if _scalar_const(init[k]) == 0 and _t(init[k]).dtype == "i64":
            out = body_sg.outputs[k]
            if _is(out, "Add"):
                a, b = out.node.inputs
                if (B.is_state(a, k) and _scalar_const(b) == 1) or (B.is_state(b, k) and _scalar_const(a) == 1):
                    idx_k = k
                    break
    if idx_k is None:
        _fail("no loop-index state (Const 0, incremented by 1)")

    # --- test: Lt(idx, max_len) with max_len = ReduceMax(lens)
    tout = test_sg.outputs[0]
    if not _is(tout, "Lt"):
        _fail("loop test is not `idx < bound`")
    ta, tb = tout.node.inputs
    if not (ta.node is test_sg.params[idx_k]):
        _fail("loop test does not compare the loop index")
    tcap_i = next((i for i, p in enumerate(test_sg.params) if p is tb.node), None)
    if tcap_i is None or tcap_i < n_state:
        _fail("loop bound is not a captured value")
    bound = test_caps[tcap_i - n_state]
    if not _is(bound, "ReduceMax") or not _is(bound.node.inputs[0], "Param"):
        _fail("loop bound is not reduce_max(sequence lengths)")
    lens_ref = bound.node.inputs[0]

    # --- per-state body outputs: Where(Lt(idx, lens), new, old) / ListAppend
    list_k, tensor_states = None, []
    mask_node = None
    for k in range(n_state):
        if k == idx_k:
            continue
        out = body_sg.outputs[k]
        spec = _t(init[k])
        if spec.dtype == "list":
            if not _is(out, "ListAppend") or not B.is_state(out.node.inputs[0], k):
                _fail("list state is not appended to once per iteration")
            if not _is(init[k], "ListNew") or init[k].node.inputs:
                _fail("list state does not start empty")
            list_k = k
            continue
        if not _is(out, "Where"):
            _fail(f"state {k} is not updated through a row mask")
        cond, new, old = out.node.inputs
        if not B.is_state(old, k):
            _fail(f"state {k}: masked update does not keep the old state")
        if not _is(cond, "Lt") or not B.is_state(cond.node.inputs[0], idx_k):
            _fail("row mask is not `idx < seq_len`")
        mcap = B.capture(cond.node.inputs[1])
        if mcap is None or mcap.node is not lens_ref.node:
            _fail("row mask compares against a different length vector")
        mask_node = cond.node
        tensor_states.append((k, new, out))
    if list_k is None:
        _fail("no output list")
    appended = body_sg.outputs[list_k].node.inputs[1]

    # --- x_t = Index(x_tm, idx), x_tm = Transpose(x, (1,0,2))
    index_nodes = [n for n in body_sg.nodes if n.op == "Index"]
    if len(index_nodes) != 1:
        _fail("expected exactly one Index (x_tm[t]) in the loop body")
    ix = index_nodes[0]
    if not B.is_state(ix.inputs[1], idx_k):
        _fail("x is not indexed by the loop index")
    xcap = B.capture(ix.inputs[0])
    if xcap is None or not _is(xcap, "Transpose") or tuple(xcap.node.attrs.get("perm", ())) != (1, 0, 2):
        _fail("x_tm is not transpose(x, [1, 0, 2])")
    x_src = _main_source(xcap.node.inputs[0])
    if x_src.kind != "param":
        _fail("x must be a graph parameter")

    def affine(ref, h_k):
        terms = _flatten_add(ref, [])
        xw = hu = bias = None
        for tr in terms:
            if _is(tr, "MatMul"):
                lhs, rhs = tr.node.inputs
                cap = B.capture(rhs)
                if cap is None:
                    _fail("MatMul weight is not a captured value")
                if lhs.node is ix and xw is None:
                    xw = _main_source(cap)
                elif B.is_state(lhs, h_k) and hu is None:
                    hu = _main_source(cap)
                else:
                    _fail("unexpected MatMul operand in a gate")
            else:
                cap = B.capture(tr)
                if cap is None or bias is not None:
                    _fail("gate bias is not a single captured value")
                bias = _main_source(cap)
        if xw is None or hu is None or bias is None:
            _fail("gate is not x_t W + h U + b")
        return (xw, hu, bias)

    def unary(ref, op):
        if not _is(ref, op):
            return None
        return ref.node.inputs[0]

    def gru(new_h, h_k):
        """h' = (1 - z) * n + z * h (either order of every + and *)."""
        if not _is(new_h, "Add"):
            return None
        for a, b in (new_h.node.inputs, new_h.node.inputs[::-1]):
            if not (_is(a, "Mul") and _is(b, "Mul")):
                continue
            for omz, n in (a.node.inputs, a.node.inputs[::-1]):
                if not (_is(omz, "Sub") and _scalar_const(omz.node.inputs[0]) == 1 and _is(n, "Tanh")):
                    continue
                z = omz.node.inputs[1]
                for zz, hh in (b.node.inputs, b.node.inputs[::-1]):
                    if _same(zz, z) and B.is_state(hh, h_k) and _is(z, "Sigmoid"):
                        return z, n
        return None

    def gru_candidate(n, h_k):
        """n = tanh(x_t Wn + bn + r * (h Un + bhn)) -> (r ref, (Wn, None, bn), (None, Un, bhn))."""
        terms = _flatten_add(n.node.inputs[0], [])
        wn = bn = gated = None
        for tr in terms:
            if _is(tr, "MatMul") and tr.node.inputs[0].node is ix and wn is None:
                cap = B.capture(tr.node.inputs[1])
                if cap is None:
                    _fail("GRU n-gate weight is not a captured value")
                wn = _main_source(cap)
            elif _is(tr, "Mul") and gated is None:
                gated = tr
            elif B.capture(tr) is not None and bn is None:
                bn = _main_source(B.capture(tr))
            else:
                _fail("GRU n-gate is not x_t Wn + bn + r * (h Un + bhn)")
        if wn is None or bn is None or gated is None:
            _fail("GRU n-gate is not x_t Wn + bn + r * (h Un + bhn)")
        for r, inner in (gated.node.inputs, gated.node.inputs[::-1]):
            if not _is(r, "Sigmoid"):
                continue
            un = bhn = None
            for tr in _flatten_add(inner, []):
                if _is(tr, "MatMul") and B.is_state(tr.node.inputs[0], h_k) and un is None:
                    cap = B.capture(tr.node.inputs[1])
                    if cap is None:
                        _fail("GRU Un is not a captured value")
                    un = _main_source(cap)
                elif B.capture(tr) is not None and bhn is None:
                    bhn = _main_source(B.capture(tr))
                else:
                    un = None
                    break
            if un is not None and bhn is not None:
                return r, (wn, None, bn), (None, un, bhn)
        _fail("GRU reset gate does not multiply (h Un + bhn)")

    if len(tensor_states) == 1:
        (h_k, new_h, where_h), = tensor_states
        c_k = None
        if not _same(appended, where_h):
            _fail("output list does not collect the masked state")
        pre = unary(new_h, "Tanh")
        zn = gru(new_h, h_k) if pre is None else None
        if pre is not None:
            gates = [affine(pre, h_k)]
            cell = CELL_RNN_TANH
        elif zn is not None:
            z_ref, n_ref = zn
            r_ref, nx, nh = gru_candidate(n_ref, h_k)
            gates = [affine(unary(z_ref, "Sigmoid"), h_k), affine(unary(r_ref, "Sigmoid"), h_k), nx, nh]
            cell = CELL_GRU
        else:
            _fail("single-state cell is neither tanh(x W + h U + b) nor a GRU")
    elif len(tensor_states) == 2:
        # identify c: its new value is f*c + i*g ; h's new value is o*tanh(c')
        cell = CELL_LSTM
        ident = None
        for (ka, na, wa), (kb, nb, wb) in (tensor_states, tensor_states[::-1]):
            if _is(na, "Mul"):
                m0, m1 = na.node.inputs
                for o_ref, t_ref in ((m0, m1), (m1, m0)):
                    if _is(t_ref, "Tanh") and _same(t_ref.node.inputs[0], nb):
                        ident = (ka, na, wa, kb, nb, wb, o_ref)
        if ident is None:
            _fail("two-state cell is not an LSTM (h' = o*tanh(c'))")
        h_k, new_h, where_h, c_k, new_c, where_c, o_ref = ident
        if not _same(appended, where_h):
            _fail("output list does not collect the masked h")
        if not _is(new_c, "Add"):
            _fail("c' is not f*c + i*g")
        p0, p1 = new_c.node.inputs
        f_ref = i_ref = g_ref = None
        for fc, ig in ((p0, p1), (p1, p0)):
            if _is(fc, "Mul") and _is(ig, "Mul"):
                a0, a1 = fc.node.inputs
                for fa, cb in ((a0, a1), (a1, a0)):
                    if B.is_state(cb, c_k):
                        b0, b1 = ig.node.inputs
                        for ia, ga in ((b0, b1), (b1, b0)):
                            if _is(ga, "Tanh") and _is(ia, "Sigmoid"):
                                f_ref, i_ref, g_ref = fa, ia, ga
        if f_ref is None or not _is(f_ref, "Sigmoid") or not _is(o_ref, "Sigmoid"):
            _fail("LSTM gates are not sigmoid/sigmoid/tanh/sigmoid")
        gates = [affine(unary(r, "Sigmoid" if r is not g_ref else "Tanh"), h_k)
                 for r in (i_ref, f_ref, g_ref, o_ref)]
    else:
        _fail(f"{len(tensor_states)} tensor states (RNN / GRU have 1, LSTM 2)")

    h0 = _main_source(init[h_k])
    c0 = _main_source(init[c_k]) if c_k is not None else None
    lens = _main_source(lens_ref)

    # --- graph outputs
    outputs = []
    stack_node = None
    for ref in main.outputs:
        if ref.node is w:
            if ref.out == h_k:
                outputs.append(OutputSpec("h_final", ref.node))
            elif c_k is not None and ref.out == c_k:
                outputs.append(OutputSpec("c_final", ref.node))
            else:
                _fail("graph returns a loop state the kernel does not produce")
        elif _is(ref, "Transpose") and _is(ref.node.inputs[0], "ListStack"):
            if tuple(ref.node.attrs.get("perm", ())) != (1, 0, 2):
                _fail("output transpose is not [1, 0, 2]")
            st = ref.node.inputs[0]
            if st.node.inputs[0].node is not w or st.node.inputs[0].out != list_k:
                _fail("stacked list is not the loop's output list")
            stack_node = st.node
            outputs.append(OutputSpec("seq_bm", ref.node))
        elif _is(ref, "ListStack"):
            if ref.node.inputs[0].node is not w or ref.node.inputs[0].out != list_k:
                _fail("stacked list is not the loop's output list")
            stack_node = ref.node
            outputs.append(OutputSpec("seq_tm", ref.node))
        else:
            _fail(f"graph output produced by {ref.node.op}")
    # a ListStack evaluated but not returned still raises EmptyPop in the reference
    for n in main.nodes:
        if n.op == "ListStack" and stack_node is None:
            stack_node = n
    range_nodes = [n for n in main.nodes if n.op == "Range"]
    return RnnProgram(
        cell=cell, x=x_src, lens=lens, h0=h0, c0=c0, gates=gates, outputs=outputs,
        while_node=w, index_node=ix, range_node=range_nodes[0] if range_nodes else None,
        reduce_node=bound.node, stack_node=stack_node,
        max_iterations=w.attrs.get("max_iterations"), params=list(main.params))
