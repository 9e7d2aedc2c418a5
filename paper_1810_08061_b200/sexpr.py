"""S-expression wire format: graphs reach the backend as text.

The reference emits its textual IR with `to_sexpr` (pkg/src/stagekit/graph/
sexpr.py:43-155; grammar at :4-21) for expression-oriented back-ends.  This
module reads that format back into an executable skb `Graph` (`from_sexpr`)
and writes it (`to_sexpr`, the same rendering rules), so a program can be
shipped as text and run by `execute` without Python IR objects.

Reading an expression-shaped program back into a dataflow graph:

* values the emitter inlined once per use site are re-shared by hash-consing
  (identical expressions in one frame are one node), so a `While` whose
  outputs are selected twice with `(out k ...)` runs once;
* a symbol of an enclosing frame becomes a capture parameter of every frame
  in between (the IR's closed-frame rule, reference ir.py:5-7); other
  inlined outer expressions are recomputed in the frame that uses them (pure
  ops; effects only occur at frame level);
* `print` / `assert` forms at the start of a body are the frame's effects,
  the remaining forms its outputs (`_frame_exprs`, sexpr.py:69-74);
* output types are inferred with the reference's dtype rules
  (tensor.py:109-122) and trailing-dimension broadcasting (tensor.py:160-179);
  parameter types come from the `(name type)` declarations.
Assert messages are not part of the format (sexpr.py:145-146).
"""

from __future__ import annotations

from typing import Optional

from .errors import LoweringError
from .ir import Graph, GraphFunction, Node, Subgraph, TypeSpec, generated_span
from .values import TensorValue

_OP_NAMES = {
    "Add": "add", "Sub": "sub", "Mul": "mul", "Div": "div", "Mod": "mod",
    "Neg": "neg", "Lt": "lt", "Gt": "gt", "Le": "le", "Ge": "ge",
    "Eq": "eq", "Ne": "ne", "Not": "not", "MatMul": "matmul",
    "Transpose": "transpose", "ReduceMax": "reduce_max",
    "ReduceSum": "reduce_sum", "Where": "where", "Tanh": "tanh",
    "Sigmoid": "sigmoid", "Shape": "shape", "Range": "range", "Index": "index",
    "ListNew": "list_new", "ListAppend": "list_append", "ListPop": "list_pop",
    "ListGet": "list_get", "ListSet": "list_set", "ListStack": "list_stack",
    "Print": "print", "Assert": "assert",
    "TreeIsEmpty": "tree_is_empty", "TreeLeft": "tree_left",
    "TreeRight": "tree_right", "TreeValue": "tree_value",
}
_OPS = {v: k for k, v in _OP_NAMES.items()}
_ARITH = {"Add", "Sub", "Mul", "Div", "Mod"}
_COMPARE = {"Lt", "Gt", "Le", "Ge", "Eq", "Ne"}


class SexprError(LoweringError):
    pass


# ------------------------------------------------------------------ reader
def parse(text: str) -> list:
    """Text -> nested lists of atoms (strings)."""
    toks = text.replace("(", " ( ").replace(")", " ) ").split()
    out, stack = [], []
    for tok in toks:
        if tok == "(":
            stack.append([])
        elif tok == ")":
            if not stack:
                raise SexprError("unbalanced ')' in s-expression")
            done = stack.pop()
            (stack[-1] if stack else out).append(done)
        else:
            if not stack:
                raise SexprError(f"atom {tok!r} outside a form")
            stack[-1].append(tok)
    if stack:
        raise SexprError("unbalanced '(' in s-expression")
    return out


def _key(e):
    return tuple(_key(x) for x in e) if isinstance(e, list) else e


def _parse_type(text: str) -> TypeSpec:
    """TypeSpec.render() inverse: f64, i64[2,3], f64[?,4], bool, tree, list<f64[3]>."""
    if text == "tree":
        return TypeSpec("tree", None)
    if text.startswith("list<") and text.endswith(">"):
        inner = text[5:-1]
        return TypeSpec("list", None, None if inner == "?" else _parse_type(inner))
    if "[" in text:
        dt, dims = text[:-1].split("[", 1)
        return TypeSpec(dt, tuple(None if d == "?" else int(d) for d in dims.split(",")) if dims else ())
    return TypeSpec(text, ())


def _scalar(dtype, tok):
    if dtype == "bool":
        return tok in ("1", "True", "true")
    if dtype == "i64":
        return int(tok)
    return float(tok)


def _bcast(a, b):
    if a is None or b is None:
        return None
    out = []
    for i in range(max(len(a), len(b))):
        da = a[len(a) - 1 - i] if i < len(a) else 1
        db = b[len(b) - 1 - i] if i < len(b) else 1
        out.append(db if da == 1 else da if (db == 1 or da == db or db is None) else
                   (db if da is None else None))
    return tuple(reversed(out))


class _Scope:
    def __init__(self, sg: Subgraph, parent: Optional["_Scope"]):
        self.sg = sg
        self.parent = parent
        self.symbols = {}
        self.caps = {}        # id-key of the outer ref -> capture param ref
        self.cap_refs = []    # outer refs, in capture-param order
        self.memo = {}

    def param(self, name, spec):
        return self.sg.add_param(name, spec).ref(0)

    def lookup(self, name):
        if name in self.symbols:
            return self.symbols[name]
        if self.parent is None:
            raise SexprError(f"unbound symbol {name!r}")
        outer = self.parent.lookup(name)
        k = (id(outer.node), outer.out)
        if k not in self.caps:
            self.caps[k] = self.param(name, outer.type)
            self.cap_refs.append(outer)
        return self.caps[k]


class _Reader:
    def __init__(self, forms):
        self.forms = forms
        self.graph = Graph()
        self.fn_types = {}    # function name -> output TypeSpec (None while unknown)

    # -- types ------------------------------------------------------------
    def _infer(self, op, ins, attrs):
        t = [r.type for r in ins]
        if op in _ARITH:
            a, b = t[0].dtype, t[1].dtype
            dt = "f64" if op == "Div" or "f64" in (a, b) else "i64"
            return [TypeSpec(dt, _bcast(t[0].shape, t[1].shape))]
        if op in _COMPARE:
            return [TypeSpec("bool", _bcast(t[0].shape, t[1].shape))]
        if op == "Neg":
            return [t[0]]
        if op == "Not":
            return [TypeSpec("bool", t[0].shape)]
        if op == "MatMul":
            dt = "f64" if "f64" in (t[0].dtype, t[1].dtype) else "i64"
            sa, sb = t[0].shape, t[1].shape
            return [TypeSpec(dt, (sa[0], sb[1]) if sa is not None and sb is not None else None)]
        if op == "Transpose":
            s = t[0].shape
            perm = attrs["perm"]
            return [TypeSpec(t[0].dtype, tuple(s[p] for p in perm) if s is not None else None)]
        if op in ("ReduceMax", "ReduceSum"):
            return [TypeSpec(t[0].dtype, ())]
        if op == "Where":
            return [TypeSpec(t[1].dtype, t[1].shape if t[1].shape == t[2].shape else _bcast(t[1].shape, t[2].shape))]
        if op in ("Tanh", "Sigmoid"):
            return [TypeSpec("f64", t[0].shape)]
        if op == "Shape":
            return [TypeSpec("i64", (len(t[0].shape),) if t[0].shape is not None else None)]
        if op == "Range":
            return [TypeSpec("i64", (None,))]
        if op == "Index":
            s = t[0].shape
            return [TypeSpec(t[0].dtype, tuple(s[1:]) if s is not None else None)]
        if op == "ListNew":
            return [TypeSpec("list", None, t[0] if t else None)]
        if op in ("ListAppend", "ListSet"):
            lt = t[0]
            if lt.elem is None:
                lt = TypeSpec("list", None, t[1] if op == "ListAppend" else t[2])
            return [lt]
        if op == "ListPop":
            return [t[0], t[0].elem or TypeSpec("f64", None)]
        if op == "ListGet":
            return [t[0].elem or TypeSpec("f64", None)]
        if op == "ListStack":
            e = t[0].elem
            if e is None:
                return [TypeSpec("f64", None)]
            return [TypeSpec(e.dtype, (None,) + tuple(e.shape) if e.shape is not None else None)]
        if op in ("Print", "Assert"):
            return []
        if op == "TreeIsEmpty":
            return [TypeSpec("bool", ())]
        if op in ("TreeLeft", "TreeRight"):
            return [TypeSpec("tree", None)]
        if op == "TreeValue":
            return [TypeSpec("f64", ())]
        raise SexprError(f"no type rule for {op}")

    # -- expressions -----------------------------------------------------------
    def value(self, e, sc: _Scope):
        """An expression that yields one value -> NodeRef."""
        if isinstance(e, str):
            return sc.lookup(e)
        if e and e[0] == "out":
            k = int(e[1][2])
            node = self.node(e[2], sc)
            return node.ref(k)
        node = self.node(e, sc)
        if len(node.out_types) != 1:
            raise SexprError(f"({e[0]} ...) has {len(node.out_types)} outputs; select one with (out k ...)")
        return node.ref(0)

    def node(self, e, sc: _Scope) -> Node:
        if isinstance(e, str):
            raise SexprError(f"symbol {e!r} where a node was expected")
        k = _key(e)
        hit = sc.memo.get(k)
        if hit is not None:
            return hit
        head = e[0]
        if head == "const":
            n = self.const(e)
        elif head == "cond":
            n = self.cond(e, sc)
        elif head == "while":
            n = self.loop(e, sc)
        elif head == "call":
            n = self.call(e, sc)
        elif head in _OPS:
            op = _OPS[head]
            args = e[1:]
            attrs = {}
            if op == "Transpose":
                rank = len(args) - 1
                perm = tuple(int(a[2]) for a in args[1:])
                attrs["perm"] = perm
                args = args[:1]
                del rank
            ins = [self.value(a, sc) for a in args]
            n = Node(op, ins, attrs, generated_span(), self._infer(op, ins, attrs))
            if op == "Assert":
                n.attrs["message"] = None
        else:
            raise SexprError(f"unknown form ({head} ...)")
        sc.sg.add(n)
        if head not in ("print", "assert"):   # effects are never shared
            sc.memo[k] = n
        return n

    def const(self, e):
        dt = e[1]
        if isinstance(e[2], list) and e[2] and e[2][0] == "dims":
            shape = tuple(int(d) for d in e[2][1:])
            data = [_scalar(dt, t) for t in e[3:]]
        else:
            shape, data = (), [_scalar(dt, e[2])]
        return Node("Const", [], {"value": TensorValue(dt, shape, data)}, generated_span(), [TypeSpec(dt, shape)])

    def frame_body(self, forms, sc: _Scope):
        """Effects first, then outputs (reference _frame_exprs)."""
        outs = []
        for f in forms:
            if isinstance(f, list) and f and f[0] in ("print", "assert"):
                self.node(f, sc)
            else:
                outs.append(self.value(f, sc))
        sc.sg.outputs = outs
        return outs

    def cond(self, e, sc):
        pred = self.value(e[1], sc)
        then_f, else_f = e[2], e[3]
        if then_f[0] != "then" or else_f[0] != "else":
            raise SexprError("(cond p (then ...) (else ...)) expected")
        ts, es = _Scope(Subgraph(), sc), _Scope(Subgraph(), sc)
        t_out = self.frame_body(then_f[1:], ts)
        e_out = self.frame_body(else_f[1:], es)
        out_types = [a.type if a.type.dtype is not None else b.type for a, b in zip(t_out, e_out)]
        return Node("Cond", [pred] + ts.cap_refs + es.cap_refs,
                    {"then_graph": ts.sg, "else_graph": es.sg, "n_then_caps": len(ts.cap_refs),
                     "n_else_caps": len(es.cap_refs), "out_symbols": [f"v{i}" for i in range(len(t_out))]},
                    generated_span(), out_types)

    def loop(self, e, sc):
        vars_f, test_f, body_f = e[1], e[2], e[3]
        names = [v[0] for v in vars_f[1:]]
        inits = [self.value(v[1], sc) for v in vars_f[1:]]
        ts, bs = _Scope(Subgraph(), sc), _Scope(Subgraph(), sc)
        for s in (ts, bs):
            for nm, r in zip(names, inits):
                s.symbols[nm] = s.param(nm, r.type)
        test = self.value(test_f[1], ts)
        ts.sg.outputs = [test]
        outs = self.frame_body(body_f[1:], bs)
        ns = len(names)
        # a list state that starts empty takes its element type from the body's update
        types = [o.type if (r.type.dtype == "list" and r.type.elem is None and o.type.dtype == "list") else r.type
                 for r, o in zip(inits, outs)]
        return Node("While", inits + ts.cap_refs + bs.cap_refs,
                    {"test_graph": ts.sg, "body_graph": bs.sg, "n_state": ns, "n_test_caps": len(ts.cap_refs),
                     "n_body_caps": len(bs.cap_refs), "names": names, "max_iterations": None,
                     "parallel_hint": None},
                    generated_span(), types)

    def call(self, e, sc):
        name = e[1]
        if name not in self.fn_types:
            raise SexprError(f"call of undefined function {name!r}")
        ins = [self.value(a, sc) for a in e[2:]]
        t = self.fn_types[name] or TypeSpec("f64", ())   # recursive call before its type is known
        return Node("FuncCall", ins, {"fn_name": name}, generated_span(), [t])

    # -- program ---------------------------------------------------------------
    def define(self, form):
        if not (isinstance(form, list) and len(form) >= 3 and form[0] == "def"):
            raise SexprError("top-level forms must be (def name (params) body...)")
        name, params = form[1], form[2]
        sc = _Scope(Subgraph(), None)
        for p in params:
            sc.symbols[p[0]] = sc.param(p[0], _parse_type(p[1]))
        outs = self.frame_body(form[3:], sc)
        return name, sc.sg, outs

    def read(self) -> Graph:
        defs = [f for f in self.forms]
        for f in defs:
            if f[1] != "main":
                self.fn_types[f[1]] = None
        for _ in range(2):   # second pass: recursive calls see the function's output type
            self.graph = Graph()
            for f in defs:
                name, sg, outs = self.define(f)
                if name == "main":
                    self.graph.main = sg
                else:
                    if len(outs) != 1:
                        raise SexprError(f"function {name!r} must have exactly one output")
                    self.fn_types[name] = outs[0].type
                    self.graph.functions[name] = GraphFunction(name, sg, ())
        if not self.graph.main.outputs and not self.graph.main.nodes:
            raise SexprError("no (def main ...) form")
        return self.graph


def from_sexpr(text: str) -> Graph:
    """Reference s-expression program (sexpr.py:4-21) -> executable skb Graph."""
    try:
        return _Reader(parse(text)).read()
    except RecursionError:   # the reader recurses once per nesting level, like the emitter
        raise SexprError("s-expression nested deeper than the reader's recursion limit") from None


# ------------------------------------------------------------------ writer
def _number(v, dtype):
    if dtype == "bool":
        return "1" if v else "0"
    if dtype == "f64":
        return repr(float(v))
    return str(int(v))


def _sanitize(name):
    return (name or "v").strip("<>") or "v"


def to_sexpr(graph) -> str:
    """skb or reference Graph -> text, with the reference's rendering rules."""
    forms = [_def(name, fn.body) for name, fn in getattr(graph, "functions", {}).items()]
    forms.append(_def("main", graph.main))
    return "\n".join(forms) + "\n"


def _def(name, sg):
    env = {}
    params = []
    for p in sg.params:
        pn = _sanitize(p.attrs.get("name", "p"))
        env[id(p)] = pn
        params.append(f"({pn} {p.out_types[0].render()})")
    return f"(def {name} ({' '.join(params)}) {' '.join(_frame(sg, env))})"


def _frame(sg, env):
    out = [_node(n, env) for n in sg.nodes if n.op in ("Print", "Assert")]
    return out + [_ref(r, env) for r in sg.outputs]


def _ref(r, env):
    n = r.node
    if n.op == "Param":
        return env[id(n)]
    text = _node(n, env)
    return f"(out (const i64 {r.out}) {text})" if len(n.out_types) > 1 else text


def _sub_env(sg, names, env, caps):
    out = {}
    it = iter(caps)
    for i, p in enumerate(sg.params):
        out[id(p)] = _sanitize(names[i]) if i < len(names) else _ref(next(it), env)
    return out


def _node(n, env):
    op = n.op
    if op == "Const":
        v = n.attrs["value"]
        import numpy as np
        data = np.asarray(v.data).reshape(-1).tolist() if not isinstance(v.data, (list, tuple)) else list(v.data)
        if tuple(v.shape) == ():
            return f"(const {v.dtype} {_number(data[0], v.dtype)})"
        return f"(const {v.dtype} (dims {' '.join(str(d) for d in v.shape)}) " \
               f"{' '.join(_number(x, v.dtype) for x in data)})"
    if op == "Cond":
        nt = n.attrs["n_then_caps"]
        te = _sub_env(n.attrs["then_graph"], [], env, n.inputs[1:1 + nt])
        ee = _sub_env(n.attrs["else_graph"], [], env, n.inputs[1 + nt:])
        return f"(cond {_ref(n.inputs[0], env)} (then {' '.join(_frame(n.attrs['then_graph'], te))}) " \
               f"(else {' '.join(_frame(n.attrs['else_graph'], ee))}))"
    if op == "While":
        ns, nt = n.attrs["n_state"], n.attrs["n_test_caps"]
        names = [_sanitize(x) for x in n.attrs["names"]]
        inits = [_ref(r, env) for r in n.inputs[:ns]]
        te = _sub_env(n.attrs["test_graph"], names, env, n.inputs[ns:ns + nt])
        be = _sub_env(n.attrs["body_graph"], names, env, n.inputs[ns + nt:])
        return f"(while (vars {' '.join(f'({a} {b})' for a, b in zip(names, inits))}) " \
               f"(test {_ref(n.attrs['test_graph'].outputs[0], te)}) " \
               f"(body {' '.join(_frame(n.attrs['body_graph'], be))}))"
    if op == "FuncCall":
        args = " ".join(_ref(r, env) for r in n.inputs)
        return f"(call {n.attrs['fn_name']}{' ' if args else ''}{args})"
    parts = [_ref(r, env) for r in n.inputs]
    if op == "Transpose":
        parts += [f"(const i64 {p})" for p in n.attrs["perm"]]
    joined = " ".join(parts)
    return f"({_OP_NAMES[op]}{' ' if joined else ''}{joined})"
