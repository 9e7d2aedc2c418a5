"""Lowering of the staged greedy decoder (oracle/programs/greedy.msl)
onto the device-resident decode loop (csrc/beam.cu, `decode.Decoder`).

The program, as the reference stages it (runtime/dispatch.py:275-387; the
`break` on EOS lowered into the While test by transforms/lowering.py:95-115):

    While[brk, h, t, tok, toks](test: not brk and t < max_len)
      x      = Index(emb, tok)                         # emb [V, 1, E]
      h'     = Tanh(MatMul(x, w_in) + MatMul(h, u))
      logits = MatMul(h', w_out); row = Index(logits, 0)
      tok'   = ReduceSum(Where(row == ReduceMax(row), ids, ids * 0))   # argmax_row
      toks'  = ListAppend(toks, tok');  t' = t + 1;  brk' = Cond(tok' == eos, True, brk)
    outputs: ListStack(toks), t

`lower_greedy` matches that structure (operand roles are read off the
dataflow, not node order) and returns the feed names of each role; anything
else raises LoweringError and the graph runs on the region VM.  The fused
path computes in fp32 (GEMMs without TF32) and records, per sentence, the
smallest top-1 minus top-2 logit gap of any step; a sentence whose gap is not
above `executor.DECODE_MARGIN` (an argmax fp32 rounding could flip, or an exact
tie, where the reference's `argmax_row` sums the tied ids) is re-run in f64 on
the region VM, so tokens always equal the reference's.  `ids` must be 0..V-1.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import LoweringError


@dataclass
class GreedyProgram:
    h0: str
    emb: str
    w_in: str
    u: str
    w_out: str
    ids: str
    eos: str
    max_len: str
    toks_out: int        # main output index of the token sequence
    steps_out: int       # main output index of the trip count


def _const(ref, value=None):
    n = ref.node
    if n.op != "Const":
        return False
    if value is None:
        return True
    v = n.attrs.get("value")
    data = getattr(v, "data", None)
    if data is None:
        try:
            data = tuple(v.reshape(-1).tolist())
        except AttributeError:
            data = (v,)
    return len(data) == 1 and data[0] == value


def _need(cond, what):
    if not cond:
        raise LoweringError(f"not the staged greedy decoder: {what}")


def lower_greedy(graph) -> GreedyProgram:
    main = graph.main
    params = {id(p): p.attrs.get("name") for p in main.params}
    whiles = [n for n in main.nodes if n.op == "While"]
    _need(len(whiles) == 1 and all(n.op in ("Const", "ListNew", "While", "ListStack") for n in main.nodes),
          "main frame")
    w = whiles[0]
    ns, nt = w.attrs["n_state"], w.attrs["n_test_caps"]
    _need(ns == 5 and nt == 1, "loop state")
    init, tcaps, bcaps = w.inputs[:ns], w.inputs[ns:ns + nt], w.inputs[ns + nt:]
    body, test = w.attrs["body_graph"], w.attrs["test_graph"]
    bp = body.params
    b_state, b_caps = bp[:ns], bp[ns:]
    cap_name = {id(p): params.get(id(r.node)) for p, r in zip(b_caps, bcaps)}
    _need(all(r.node.op == "Param" for r in bcaps), "body captures")
    idx = {id(n): n for n in body.nodes}
    outs = body.outputs
    # --- recognise the body dataflow from its outputs
    tanh = outs[1].node
    _need(tanh.op == "Tanh" and tanh.inputs[0].node.op == "Add", "h' = tanh(x w_in + h u)")
    add = tanh.inputs[0].node
    mms = [r.node for r in add.inputs]
    _need(all(m.op == "MatMul" for m in mms), "gate matmuls")
    mx = next((m for m in mms if m.inputs[0].node.op == "Index"), None)
    mh = next((m for m in mms if m is not mx), None)
    _need(mx is not None and mh is not None, "x / h matmuls")
    emb_ix = mx.inputs[0].node
    h_param, tok_param = mh.inputs[0].node, emb_ix.inputs[1].node
    _need(h_param is b_state[1] and tok_param is b_state[3], "h and tok state")
    emb = cap_name.get(id(emb_ix.inputs[0].node))
    w_in = cap_name.get(id(mx.inputs[1].node))
    u = cap_name.get(id(mh.inputs[1].node))
    tok_new = outs[3].node
    _need(tok_new.op == "ReduceSum" and tok_new.inputs[0].node.op == "Where", "argmax_row")
    where = tok_new.inputs[0].node
    eq, ids_ref, zeros = where.inputs
    _need(eq.node.op == "Eq" and zeros.node.op == "Mul" and _const(zeros.node.inputs[1], 0), "argmax mask")
    ids = cap_name.get(id(ids_ref.node))
    row, red = eq.node.inputs
    _need(red.node.op == "ReduceMax" and red.node.inputs[0].node is row.node and row.node.op == "Index", "row max")
    _need(_const(row.node.inputs[1], 0), "logits[0]")
    lg = row.node.inputs[0].node
    _need(lg.op == "MatMul" and lg.inputs[0].node is tanh, "logits = h' w_out")
    w_out = cap_name.get(id(lg.inputs[1].node))
    app = outs[4].node
    _need(app.op == "ListAppend" and app.inputs[0].node is b_state[4] and app.inputs[1].node is tok_new, "toks")
    inc = outs[2].node
    _need(inc.op == "Add" and inc.inputs[0].node is b_state[2] and _const(inc.inputs[1], 1), "t + 1")
    brk = outs[0].node
    _need(brk.op == "Cond" and brk.inputs[0].node.op == "Eq", "EOS break")
    eos_eq = brk.inputs[0].node
    _need(eos_eq.inputs[0].node is tok_new, "tok' == eos")
    eos = cap_name.get(id(eos_eq.inputs[1].node))
    # --- test: not brk and t < max_len
    tp = test.params
    _need(len(test.nodes) == 2 and test.nodes[0].op == "Not" and test.nodes[1].op == "Cond", "loop test")
    lt_graph = test.nodes[1].attrs["then_graph"]
    _need(len(lt_graph.nodes) == 1 and lt_graph.nodes[0].op == "Lt", "t < max_len")
    _need(test.nodes[0].inputs[0].node is tp[0], "not brk")
    caps = test.nodes[1].inputs[1:1 + test.nodes[1].attrs["n_then_caps"]]
    lt = lt_graph.nodes[0]
    order = {id(p): k for k, p in enumerate(lt_graph.params)}
    t_pos, m_pos = order.get(id(lt.inputs[0].node)), order.get(id(lt.inputs[1].node))
    _need(t_pos is not None and m_pos is not None, "comparison operands")
    _need(caps[t_pos].node is tp[2] and caps[m_pos].node is tp[ns], "t and the max_len capture")
    max_len = params.get(id(tcaps[0].node))
    # --- initial state: brk False, h = h0, t = 0, tok = 0, toks = [0]
    _need(_const(init[0], False) and _const(init[2], 0) and _const(init[3], 0), "initial brk/t/tok")
    _need(init[1].node.op == "Param", "initial h")
    h0 = params.get(id(init[1].node))
    ln = init[4].node
    _need(ln.op == "ListNew" and len(ln.inputs) == 1 and _const(ln.inputs[0], 0), "toks = [0]")
    names = [h0, emb, w_in, u, w_out, ids, eos, max_len]
    _need(all(n is not None for n in names), "operands are graph parameters")
    # --- outputs: ListStack(toks), t
    mo = main.outputs
    stack = next((k for k, r in enumerate(mo) if r.node.op == "ListStack" and r.node.inputs[0].node is w
                  and r.node.inputs[0].out == 4), None)
    steps = next((k for k, r in enumerate(mo) if r.node is w and r.out == 2), None)
    _need(stack is not None and steps is not None and len(mo) == 2, "outputs [stack(toks), t]")
    return GreedyProgram(*names, toks_out=stack, steps_out=steps)
