"""Reverse-mode gradients of staged graphs, While loops included.

The reference's `gradient()` (pkg/src/stagekit/graph/grad.py:35-70)
differentiates Cond and FuncCall structurally but rejects While
(`WhileNotDifferentiable`, grad.py:159-161), so its users hand-write BPTT as
a second staged loop (oracle/programs/lstm_bptt.msl).  `gradient(graph,
output, wrt)` here builds that loop automatically, as an IR-to-IR transform
whose result any backend executes (on the B200: the region VM, vm.py):

* forward: every `While` becomes a taping While that also appends its
  non-list input state to one tape list per state and counts its iterations;
* backward: a reverse While pops the tapes, recomputes the body from the
  popped state (store-state / recompute-body checkpointing), pulls the state
  adjoints back through the recomputed body and accumulates the adjoints of
  the loop's captures; append-only list states (`hs.append(h)`) take their
  item adjoints from the stacked adjoint of the post-loop `ListStack`;
* everything else follows the reference's rules (grad.py:148-290): the same
  per-op adjoints, `_reduce_like` broadcasting limits, ListNew/ListAppend
  stack chains, and a gradient Cond whose branches recompute the primal
  branch; the Index rule is extended from a constant index into a vector to
  any index into a tensor with a static leading dimension (so d loss / d x
  of `x[t]` inside a loop works);
* FuncCalls are inlined rather than turned into `<fn>_grad` functions, and an
  activity analysis skips adjoints of values that do not depend on `wrt`
  (so `x[t]` of a non-differentiated input needs no scatter rule).

Result: a graph whose outputs are the original outputs followed by
d(outputs[output])/d(param) for each name in `wrt` (grad.py:35-70).
"""

from __future__ import annotations

from .errors import LoweringError
from .ir import Graph, Node, Subgraph, TypeSpec, generated_span
from .values import TensorValue

LIST_OPS = {"ListNew", "ListAppend", "ListGet", "ListPop", "ListSet", "ListStack"}
# outputs carry no gradient (the complement of grad.py's _DIFF_OPS): comparisons, integer and tree plumbing
NONDIFF = {"Lt", "Gt", "Le", "Ge", "Eq", "Ne", "Not", "Mod", "Shape", "Range", "ReduceMax",
           "Print", "Assert", "TreeIsEmpty", "TreeLeft", "TreeRight"}


class NotDifferentiable(LoweringError):
    pass


def _key(ref):
    return (id(ref.node), ref.out)


def _f64(t):
    return t is not None and t.dtype == "f64"


def _rev(shape):
    return None if shape is None else tuple(reversed(shape))


def _bcast(a, b):
    if a is None or b is None:
        return None
    n = max(len(a), len(b))
    a, b = (1,) * (n - len(a)) + tuple(a), (1,) * (n - len(b)) + tuple(b)
    return tuple(y if x == 1 else x if (y == 1 or x == y) else None for x, y in zip(a, b))


class _Frame:
    """Node emission into one subgraph (the reference's _FrameBuilder, grad.py:95-123)."""

    def __init__(self, sg: Subgraph):
        self.sg = sg

    def param(self, name, spec):
        return self.sg.add_param(name, spec).ref(0)

    def node(self, op, inputs, attrs=None, out_types=(), origin=None):
        return self.sg.add(Node(op, list(inputs), dict(attrs or {}), origin or generated_span(), list(out_types)))

    def op1(self, op, inputs, t, attrs=None):
        return self.node(op, inputs, attrs, [t]).ref(0)

    def const(self, value, dtype="f64"):
        return self.op1("Const", [], TypeSpec(dtype, ()), {"value": TensorValue(dtype, (), [value])})

    def binary(self, op, a, b):
        dt = "f64" if "f64" in (a.type.dtype, b.type.dtype) else a.type.dtype
        return self.op1(op, [a, b], TypeSpec(dt, _bcast(a.type.shape, b.type.shape)))

    def neg(self, a):
        return self.op1("Neg", [a], a.type)

    def zeros_like(self, ref):
        return self.binary("Mul", ref, self.const(0.0))

    def ones_like(self, ref):
        return self.binary("Add", self.zeros_like(ref), self.const(1.0))

    def add(self, a, b):
        if a is None:
            return b
        if b is None:
            return a
        return self.binary("Add", a, b)


# ------------------------------------------------------------------ activity
def _activity(graph, wrt):
    """Original-graph refs whose value depends on a `wrt` parameter (the union
    over every context a subgraph is entered in)."""
    act = set()

    def frame(sg, live_params):
        for p in sg.params:
            if id(p) in live_params:
                act.add((id(p), 0))
        for n in sg.nodes:
            visit(n)
        return [_key(r) in act for r in sg.outputs]

    def bind(params, flags):
        return {id(p) for p, f in zip(params, flags) if f}

    def visit(n):
        ins = [_key(r) in act for r in n.inputs]
        outs = [False] * len(n.out_types)
        if n.op == "FuncCall":
            body = graph.functions[n.attrs["fn_name"]].body
            outs = frame(body, bind(body.params, ins))
        elif n.op == "Cond":
            nt = n.attrs["n_then_caps"]
            a = frame(n.attrs["then_graph"], bind(n.attrs["then_graph"].params, ins[1:1 + nt]))
            b = frame(n.attrs["else_graph"], bind(n.attrs["else_graph"].params, ins[1 + nt:]))
            outs = [x or y for x, y in zip(a, b)]
        elif n.op == "While":
            ns, nt = n.attrs["n_state"], n.attrs["n_test_caps"]
            body = n.attrs["body_graph"]
            state, caps = ins[:ns], ins[ns + nt:]
            while True:
                got = frame(body, bind(body.params, state + caps))
                new = [s or g for s, g in zip(state, got)]
                if new == state:
                    break
                state = new
            outs = state
        elif n.op in NONDIFF or n.op in ("Const", "Param"):
            pass
        elif n.op == "ListPop":
            outs = [ins[0], ins[0]]
        elif n.op == "ListGet":
            outs = [ins[0]]
        else:
            outs = [any(ins)] * len(n.out_types)
        for k, flag in enumerate(outs):
            if flag and n.out_types[k].dtype in ("f64", "list"):
                act.add((id(n), k))

    main = graph.main
    frame(main, {id(p) for p in main.params if p.attrs.get("name") in set(wrt)})
    return act


# ------------------------------------------------------------------ forward copy
class _Copier:
    """Copies frames into a target frame: FuncCalls inlined (the callee's
    params alias the call's arguments), While nodes of the main frame
    replaced by taping Whiles."""

    def __init__(self, graph):
        self.g = graph
        self.loops = {}

    def frame(self, src, dst, env, allow_while):
        for n in src.nodes:
            self.node(n, dst, env, allow_while)
        return [env[_key(r)] for r in src.outputs]

    def node(self, n, dst, env, allow_while):
        ins = [env[_key(r)] for r in n.inputs]
        if n.op == "FuncCall":
            fn = self.g.functions[n.attrs["fn_name"]]
            sub = {(id(p), 0): v for p, v in zip(fn.body.params, ins)}
            outs = self.frame(fn.body, dst, sub, allow_while)
            env[("call", id(n))] = sub
            for k, r in enumerate(outs):
                env[(id(n), k)] = r
            return
        if n.op == "While":
            if not allow_while:
                raise NotDifferentiable("a While nested inside a loop body or branch")
            self.taped_while(n, ins, dst, env)
            return
        m = dst.node(n.op, ins, n.attrs, n.out_types, n.origin)
        env[("node", id(n))] = m
        for k in range(len(n.out_types)):
            env[(id(n), k)] = m.ref(k)

    def taped_while(self, n, ins, dst, env):
        ns, nt = n.attrs["n_state"], n.attrs["n_test_caps"]
        init, tcaps, bcaps = ins[:ns], ins[ns:ns + nt], ins[ns + nt:]
        test, body = n.attrs["test_graph"], n.attrs["body_graph"]
        st = [p.out_types[0] for p in body.params[:ns]]
        taped = [k for k, t in enumerate(st) if t.dtype != "list"]
        lists = [k for k, t in enumerate(st) if t.dtype == "list"]
        for k in lists:   # append-only: out = ListAppend(param, item); the param is read nowhere else
            r, p = body.outputs[k], body.params[k]
            users = [m for m in body.nodes if any(x.node is p for x in m.inputs)]
            if not (r.node.op == "ListAppend" and r.node.inputs[0].node is p and users == [r.node]) \
                    and not (r.node is p and not users):
                raise NotDifferentiable("loop list states must be append-only")
        tape_t = [TypeSpec("list", None, st[k]) for k in taped]
        tapes0 = [dst.op1("ListNew", [], t) for t in tape_t]
        cnt0 = dst.const(0, "i64")
        i64 = TypeSpec("i64", ())
        # test: the original predicate; the extra state is ignored
        new_test = Subgraph()
        tf = _Frame(new_test)
        tp = [tf.param(f"s{k}", t) for k, t in enumerate(st)]
        for k, t in enumerate(tape_t):
            tf.param(f"tape{k}", t)
        tf.param("iters", i64)
        tcp = [tf.param(f"c{k}", p.out_types[0]) for k, p in enumerate(test.params[ns:])]
        tenv = {(id(p), 0): v for p, v in zip(test.params, tp + tcp)}
        new_test.outputs = self.frame(test, tf, tenv, False)
        # body: the original body, plus the tape appends and the iteration counter
        new_body = Subgraph()
        bf = _Frame(new_body)
        bp = [bf.param(f"s{k}", t) for k, t in enumerate(st)]
        tpp = [bf.param(f"tape{k}", t) for k, t in enumerate(tape_t)]
        cnt = bf.param("iters", i64)
        bcp = [bf.param(f"c{k}", p.out_types[0]) for k, p in enumerate(body.params[ns:])]
        benv = {(id(p), 0): v for p, v in zip(body.params, bp + bcp)}
        outs = self.frame(body, bf, benv, False)
        new_tapes = [bf.op1("ListAppend", [t, bp[k]], t.type) for t, k in zip(tpp, taped)]
        new_body.outputs = outs + new_tapes + [bf.binary("Add", cnt, bf.const(1, "i64"))]
        attrs = dict(n.attrs)
        names = list(n.attrs.get("names") or [f"s{k}" for k in range(ns)])
        attrs.update(test_graph=new_test, body_graph=new_body, n_state=ns + len(taped) + 1,
                     names=names + [f"tape_{names[k]}" for k in taped] + ["iters"])
        w = dst.node("While", init + tapes0 + [cnt0] + tcaps + bcaps, attrs,
                     list(n.out_types) + tape_t + [i64], n.origin)
        env[("node", id(n))] = w
        for k in range(ns):
            env[(id(n), k)] = w.ref(k)
        self.loops[id(n)] = dict(node=w, taped=taped, lists=lists, init=init, bcaps=bcaps, st=st)


# ------------------------------------------------------------------ backward sweep
class _Sweep:
    def __init__(self, copier, act):
        self.cp = copier
        self.act = act

    def frame(self, src, f, env, adj):
        for n in reversed(src.nodes):
            self.visit(n, f, env, adj)

    def acc(self, adj, f, orig, env, g):
        """Accumulate g into the adjoint of this instance of `orig` (grad.py:137-145)."""
        if g is None or _key(orig) not in self.act or not _f64(orig.type):
            return
        k = _key(env[_key(orig)])
        adj[k] = f.add(adj.get(k), g)

    @staticmethod
    def reduce_like(f, g, target):
        """grad.py _reduce_like: equal shapes pass through, scalars reduce fully."""
        ts, zs = target.type.shape, g.type.shape
        if ts == ():
            return g if zs == () else f.op1("ReduceSum", [g], TypeSpec("f64", ()))
        if ts == zs:
            return g
        raise NotDifferentiable(f"gradient of broadcast from {ts} to {zs} is only supported for "
                                "scalars and equal shapes")

    def visit(self, n, f, env, adj):
        op = n.op
        if op in ("Const", "Param", "TreeValue") or op in NONDIFF:
            return
        if op == "FuncCall":
            if any(adj.get(_key(env[(id(n), k)])) is not None for k in range(len(n.out_types))):
                self.frame(self.cp.g.functions[n.attrs["fn_name"]].body, f, env[("call", id(n))], adj)
            return
        if op == "While":
            return self.loop(n, f, env, adj)
        if op == "Cond":
            return self.cond(n, f, env, adj)
        out = env[(id(n), 0)] if n.out_types else None
        dz = adj.get(_key(out)) if out is not None else None
        if op == "ListStack":
            if dz is not None:
                self.stack(n, f, env, adj, dz)
            return
        if dz is None:
            return
        if op in LIST_OPS:
            raise NotDifferentiable(f"adjoint of a list value outside a stack chain ({op})")
        x = [env[_key(r)] for r in n.inputs]
        a = n.inputs
        if op == "Add":
            self.acc(adj, f, a[0], env, self.reduce_like(f, dz, x[0]))
            self.acc(adj, f, a[1], env, self.reduce_like(f, dz, x[1]))
        elif op == "Sub":
            self.acc(adj, f, a[0], env, self.reduce_like(f, dz, x[0]))
            self.acc(adj, f, a[1], env, self.reduce_like(f, f.neg(dz), x[1]))
        elif op == "Mul":
            self.acc(adj, f, a[0], env, self.reduce_like(f, f.binary("Mul", dz, x[1]), x[0]))
            self.acc(adj, f, a[1], env, self.reduce_like(f, f.binary("Mul", dz, x[0]), x[1]))
        elif op == "Div":
            self.acc(adj, f, a[0], env, self.reduce_like(f, f.binary("Div", dz, x[1]), x[0]))
            dy = f.neg(f.binary("Div", f.binary("Mul", dz, out), x[1]))
            self.acc(adj, f, a[1], env, self.reduce_like(f, dy, x[1]))
        elif op == "Neg":
            self.acc(adj, f, a[0], env, f.neg(dz))
        elif op == "MatMul":
            yt = f.op1("Transpose", [x[1]], TypeSpec(x[1].type.dtype, _rev(x[1].type.shape)), {"perm": (1, 0)})
            xt = f.op1("Transpose", [x[0]], TypeSpec(x[0].type.dtype, _rev(x[0].type.shape)), {"perm": (1, 0)})
            self.acc(adj, f, a[0], env, self.matmul(f, dz, yt))
            self.acc(adj, f, a[1], env, self.matmul(f, xt, dz))
        elif op == "Transpose":
            perm = tuple(n.attrs["perm"])
            inv = tuple(perm.index(i) for i in range(len(perm)))
            self.acc(adj, f, a[0], env, f.op1("Transpose", [dz], x[0].type, {"perm": inv}))
        elif op == "ReduceSum":
            if not _f64(x[0].type):
                raise NotDifferentiable("reduce_sum gradient needs f64 input")
            self.acc(adj, f, a[0], env, f.binary("Mul", dz, f.ones_like(x[0])))
        elif op == "Tanh":
            self.acc(adj, f, a[0], env, f.binary("Mul", dz, f.binary("Sub", f.const(1.0), f.binary("Mul", out, out))))
        elif op == "Sigmoid":
            self.acc(adj, f, a[0], env, f.binary("Mul", dz, f.binary("Mul", out, f.binary("Sub", f.const(1.0), out))))
        elif op == "Where":
            zero = f.zeros_like(dz)
            self.acc(adj, f, a[1], env, f.op1("Where", [x[0], dz, zero], dz.type))
            self.acc(adj, f, a[2], env, f.op1("Where", [x[0], zero, dz], dz.type))
        elif op == "Index":
            self.index(n, f, env, adj, dz)
        else:
            raise NotDifferentiable(f"op {op} is not differentiable")

    @staticmethod
    def matmul(f, x, y):
        sx, sy = x.type.shape, y.type.shape
        shape = (sx[0], sy[1]) if sx is not None and sy is not None else None
        return f.op1("MatMul", [x, y], TypeSpec("f64", shape))

    def index(self, n, f, env, adj, dz):
        """grad.py _index_rule (a constant index into a statically sized vector),
        extended to any index into a tensor with a static leading dimension:
        row r of the adjoint is Where(i == r, dz, 0)."""
        xr, ir = n.inputs
        if _key(xr) not in self.act:
            return
        shape = xr.type.shape
        if shape is None or len(shape) == 0 or shape[0] is None:
            raise NotDifferentiable("index gradient needs a statically sized leading dimension")
        if ir.node.op == "Const" and len(shape) == 1:
            i = int(_scalar(ir.node.attrs["value"]))
            elems = [dz if j == i else f.zeros_like(dz) for j in range(shape[0])]
        else:
            iv = env[_key(ir)]
            zero = f.zeros_like(dz)
            elems = []
            for r in range(shape[0]):
                # the reference wraps negative indices (tensor.py:420-430)
                hit = f.op1("Eq", [f.op1("Mod", [iv, f.const(shape[0], "i64")], TypeSpec("i64", ())),
                                   f.const(r, "i64")], TypeSpec("bool", ()))
                elems.append(f.op1("Where", [hit, dz, zero], dz.type))
        lst = f.op1("ListNew", elems, TypeSpec("list", None, dz.type))
        st = f.op1("ListStack", [lst], TypeSpec(xr.type.dtype, (shape[0],) + tuple(dz.type.shape or ())))
        self.acc(adj, f, xr, env, st)

    def stack(self, n, f, env, adj, dz):
        """grad.py _stack_rule over a ListNew/ListAppend chain; a chain rooted at
        a While's list state hands the stacked adjoint to that loop."""
        suffix, ref = [], n.inputs[0]
        while ref.node.op == "ListAppend":
            suffix.append(ref.node.inputs[1])
            ref = ref.node.inputs[0]
        if ref.node.op == "ListNew":
            elems = list(ref.node.inputs) + list(reversed(suffix))
            for pos, e in enumerate(elems):
                part = f.op1("Index", [dz, f.const(pos, "i64")], env[_key(e)].type)
                self.acc(adj, f, e, env, part)
            return
        if ref.node.op == "While" and not suffix:
            k = ("stack",) + _key(env[_key(ref)])
            adj[k] = f.add(adj.get(k), dz)
            return
        raise NotDifferentiable("stack gradient needs a statically traceable list")

    # -- Cond (grad.py _cond_rule / _branch_gradient) -------------------------------
    def cond(self, n, f, env, adj):
        m = env[("node", id(n))]
        dzs = [adj.get(_key(m.ref(k))) for k in range(len(n.out_types))]
        live = [k for k, d in enumerate(dzs) if d is not None]
        if not live:
            return
        nt = n.attrs["n_then_caps"]
        o_then, o_else = n.inputs[1:1 + nt], n.inputs[1 + nt:]
        diff, seen = [], set()
        for r in list(o_then) + list(o_else):
            if _f64(r.type) and _key(r) in self.act and _key(r) not in seen:
                seen.add(_key(r))
                diff.append(r)
        if not diff:
            return
        c_diff = [env[_key(r)] for r in diff]
        c_then, c_else = m.inputs[1:1 + nt], m.inputs[1 + nt:]
        gt = self.branch(n.attrs["then_graph"], o_then, c_diff, diff, live)
        ge = self.branch(n.attrs["else_graph"], o_else, c_diff, diff, live)
        dl = [dzs[k] for k in live]
        g = f.node("Cond", [m.inputs[0]] + c_diff + list(c_then) + dl + c_diff + list(c_else) + dl,
                   {"then_graph": gt, "else_graph": ge,
                    "n_then_caps": len(c_diff) + len(c_then) + len(dl),
                    "n_else_caps": len(c_diff) + len(c_else) + len(dl),
                    "out_symbols": [f"d{i}" for i in range(len(diff))]},
                   [r.type for r in c_diff])
        for k, r in enumerate(diff):
            self.acc(adj, f, r, env, g.ref(k))

    def branch(self, src, o_caps, c_diff, diff, live):
        sg = Subgraph()
        bf = _Frame(sg)
        dparams = [bf.param(f"c{i}", r.type) for i, r in enumerate(c_diff)]
        cparams = [bf.param(f"p{i}", p.out_types[0]) for i, p in enumerate(src.params)]
        zparams = [bf.param(f"dz{i}", src.outputs[k].type) for i, k in enumerate(live)]
        benv = {(id(p), 0): v for p, v in zip(src.params, cparams)}
        for nd in src.nodes:
            self.cp.node(nd, bf, benv, False)
        badj = {}
        for z, k in zip(zparams, live):
            o = src.outputs[k]
            if _key(o) in self.act and _f64(o.type):
                kk = _key(benv[_key(o)])
                badj[kk] = bf.add(badj.get(kk), z)
        self.frame(src, bf, benv, badj)
        outs = []
        for r, dp in zip(diff, dparams):
            got = None
            for oc, p in zip(o_caps, src.params):
                if _key(oc) == _key(r):
                    got = bf.add(got, badj.get(_key(benv[(id(p), 0)])))
            outs.append(got if got is not None else bf.zeros_like(dp))
        sg.outputs = outs
        return sg

    # -- While: taped forward, reverse loop ----------------------------------------
    def loop(self, n, f, env, adj):
        info = self.cp.loops[id(n)]
        w, taped, lists, st = info["node"], info["taped"], info["lists"], info["st"]
        ns = n.attrs["n_state"]
        body = n.attrs["body_graph"]
        act = self.act
        dstates = [k for k in taped if _f64(st[k]) and (id(n), k) in act]
        dlists = [k for k in lists if ("stack",) + _key(w.ref(k)) in adj]
        seeds = {k: adj.get(_key(w.ref(k))) for k in dstates}
        if all(seeds[k] is None for k in dstates) and not dlists:
            return
        bcaps_o = n.inputs[ns + n.attrs["n_test_caps"]:]
        bcaps = info["bcaps"]
        dcaps = [i for i, r in enumerate(bcaps_o) if _f64(r.type) and _key(r) in act]
        tapes = [w.ref(ns + i) for i in range(len(taped))]
        iters = w.ref(ns + len(taped))
        i64 = TypeSpec("i64", ())
        len0 = {}
        for k in dlists:
            root = n.inputs[k].node
            if root.op != "ListNew":
                raise NotDifferentiable("loop list states must start from a list literal")
            len0[k] = len(root.inputs)
        stacked = [adj[("stack",) + _key(w.ref(k))] for k in dlists]
        init = ([f.binary("Sub", iters, f.const(1, "i64"))] +
                [seeds[k] if seeds[k] is not None else f.zeros_like(w.ref(k)) for k in dstates] +
                tapes + stacked + [f.zeros_like(bcaps[i]) for i in dcaps])
        # test: j >= 0
        test = Subgraph()
        tf = _Frame(test)
        tj = tf.param("j", i64)
        for i, r in enumerate(init[1:]):
            tf.param(f"x{i}", r.type)
        test.outputs = [tf.op1("Ge", [tj, tf.const(0, "i64")], TypeSpec("bool", ()))]
        # body: pop the iteration's state, recompute the forward body, sweep it backwards
        sg = Subgraph()
        bf = _Frame(sg)
        j = bf.param("j", i64)
        dps = [bf.param(f"d{k}", init[1 + i].type) for i, k in enumerate(dstates)]
        tps = [bf.param(f"tape{i}", t.type) for i, t in enumerate(tapes)]
        sps = [bf.param(f"stack{k}", r.type) for k, r in zip(dlists, stacked)]
        aps = [bf.param(f"acc{i}", bcaps[i].type) for i in dcaps]
        cps = [bf.param(f"c{i}", r.type) for i, r in enumerate(bcaps)]
        popped, rest = {}, []
        for k, tp in zip(taped, tps):
            pop = bf.node("ListPop", [tp], {}, [tp.type, st[k]])
            rest.append(pop.ref(0))
            popped[k] = pop.ref(1)
        benv = {}
        for k, p in enumerate(body.params[:ns]):
            benv[(id(p), 0)] = popped[k] if k in popped else bf.op1("ListNew", [], st[k])
        for p, c in zip(body.params[ns:], cps):
            benv[(id(p), 0)] = c
        for nd in body.nodes:
            self.cp.node(nd, bf, benv, False)
        badj = {}
        for k, d in zip(dstates, dps):
            o = body.outputs[k]
            if _key(o) in act and _f64(o.type):
                kk = _key(benv[_key(o)])
                badj[kk] = bf.add(badj.get(kk), d)
        for k, s in zip(dlists, sps):
            app = body.outputs[k].node
            item = app.inputs[1] if app.op == "ListAppend" else None
            if item is None or _key(item) not in act:
                continue
            pos = bf.binary("Add", j, bf.const(len0[k], "i64"))
            row = bf.op1("Index", [s, pos], benv[_key(item)].type)
            kk = _key(benv[_key(item)])
            badj[kk] = bf.add(badj.get(kk), row)
        self.frame(body, bf, benv, badj)
        new_d = []
        for k in dstates:
            pr = benv[(id(body.params[k]), 0)]
            g = badj.get(_key(pr))
            new_d.append(g if g is not None else bf.zeros_like(pr))
        new_a = []
        for i, a in zip(dcaps, aps):
            g = badj.get(_key(cps[i]))
            new_a.append(bf.add(a, g) if g is not None else a)
        sg.outputs = [bf.binary("Sub", j, bf.const(1, "i64"))] + new_d + rest + sps + new_a
        names = ["j"] + [f"d_{k}" for k in dstates] + [f"tape{i}" for i in range(len(tapes))] + \
                [f"stack{k}" for k in dlists] + [f"acc{i}" for i in dcaps]
        bw = f.node("While", init + list(bcaps),
                    {"test_graph": test, "body_graph": sg, "n_state": len(init), "n_test_caps": 0,
                     "n_body_caps": len(bcaps), "names": names, "max_iterations": None,
                     "parallel_hint": None},
                    [r.type for r in init], n.origin)
        # adjoints of the loop inputs: initial states, initial list items, captures
        for i, k in enumerate(dstates):
            self.acc(adj, f, n.inputs[k], env, bw.ref(1 + i))
        for k, s in zip(dlists, stacked):
            for pos, e in enumerate(n.inputs[k].node.inputs):
                part = f.op1("Index", [s, f.const(pos, "i64")], env[_key(e)].type)
                self.acc(adj, f, e, env, part)
        base = 1 + len(dstates) + len(tapes) + len(stacked)
        for i, ci in enumerate(dcaps):
            self.acc(adj, f, bcaps_o[ci], env, bw.ref(base + i))


def _scalar(v):
    data = getattr(v, "data", None)
    if data is not None:
        return data[0]
    try:
        return v.item()
    except AttributeError:
        return v


# ------------------------------------------------------------------ entry point
def gradient(graph, output=0, wrt=()) -> Graph:
    """The original outputs followed by d(outputs[output])/d(p) for each
    parameter name p in `wrt` (reference graph/grad.py:35-70), with While
    loops differentiated by a taped reverse loop."""
    out = Graph()
    f = _Frame(out.main)
    cp = _Copier(graph)
    env, pmap = {}, {}
    for p in graph.main.params:
        r = f.param(p.attrs.get("name"), p.out_types[0])
        env[(id(p), 0)] = r
        pmap[p.attrs.get("name")] = (p, r)
    if not isinstance(output, int):
        raise NotDifferentiable("gradient target must be an output index")
    for name in wrt:
        if name not in pmap:
            raise NotDifferentiable(f"no parameter named {name!r}")
        if not _f64(pmap[name][0].out_types[0]):
            raise NotDifferentiable(f"parameter {name!r} has dtype {pmap[name][0].out_types[0].dtype}; "
                                    "gradients need f64")
    outs = cp.frame(graph.main, f, env, True)
    target = outs[output]
    if not (_f64(target.type) and target.type.shape == ()):
        raise NotDifferentiable(f"gradient target must be a scalar f64, got {target.type.render()}")
    act = _activity(graph, wrt)
    adj = {}
    if _key(graph.main.outputs[output]) in act:
        adj[_key(target)] = f.const(1.0)
    _Sweep(cp, act).frame(graph.main, f, env, adj)
    grads = []
    for name in wrt:
        p, r = pmap[name]
        g = adj.get(_key(r))
        grads.append(g if g is not None else f.zeros_like(r))
    out.main.outputs = list(outs) + grads
    return out
