"""Host-side mirror of the reference dataflow IR plus its JSON wire format.

The executor duck-types graphs, so it accepts both the reference's own
objects (reference pkg/src/stagekit/graph/ir.py:36-163: ``Graph``,
``Subgraph``, ``Node``, ``NodeRef``, ``TypeSpec``) and the classes below,
which carry the same attribute names.  The classes exist so graphs can be
built, stored and replayed without the reference installed (the GPU box has
no copy of it): ``to_json``/``from_json`` serialise a traced graph with every
op, capture route, attribute, output type and origin span.
"""

from __future__ import annotations

import itertools
import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .values import TensorValue

# reference ir.py:19-27
OPS = frozenset({
    "Const", "Param", "Add", "Sub", "Mul", "Div", "Mod", "Neg",
    "Lt", "Gt", "Le", "Ge", "Eq", "Ne", "Not",
    "MatMul", "Transpose", "ReduceMax", "ReduceSum", "Where", "Tanh",
    "Sigmoid", "Shape", "Range", "Index", "Cond", "While",
    "ListNew", "ListAppend", "ListPop", "ListGet", "ListSet", "ListStack",
    "FuncCall", "Print", "Assert",
    "TreeIsEmpty", "TreeLeft", "TreeRight", "TreeValue",
})
SUBGRAPH_KEYS = ("then_graph", "else_graph", "test_graph", "body_graph")

_ids = itertools.count(1)


@dataclass(frozen=True)
class SourceSpan:
    """reference syntax/spans.py:10-37"""
    file: str
    start_line: int
    start_col: int
    end_line: int
    end_col: int

    def __str__(self):
        return f"{self.file}:{self.start_line}:{self.start_col}"


def generated_span() -> SourceSpan:
    return SourceSpan("<generated>", 1, 1, 1, 1)


@dataclass(frozen=True)
class TypeSpec:
    """reference ir.py:36-52"""
    dtype: str
    shape: Optional[tuple] = ()
    elem: Optional["TypeSpec"] = None

    def render(self) -> str:
        if self.dtype == "list":
            return f"list<{self.elem.render() if self.elem else '?'}>"
        if self.dtype == "tree":
            return "tree"
        dims = "" if self.shape == () else \
            "[" + ",".join("?" if d is None else str(d) for d in (self.shape or ())) + "]"
        return f"{self.dtype}{dims}"


@dataclass(eq=False)
class Node:
    """reference ir.py:55-73"""
    op: str
    inputs: list = field(default_factory=list)
    attrs: dict = field(default_factory=dict)
    origin: SourceSpan = field(default_factory=generated_span)
    out_types: list = field(default_factory=list)
    frame: Optional["Subgraph"] = None
    uid: int = field(default_factory=lambda: next(_ids))

    def __post_init__(self):
        if self.op not in OPS:
            raise ValueError(f"unknown graph op {self.op!r}")

    def ref(self, out: int = 0) -> "NodeRef":
        return NodeRef(self, out)

    def __repr__(self):
        return f"<{self.op}#{self.uid}>"


@dataclass(frozen=True)
class NodeRef:
    """reference ir.py:76-83"""
    node: Node
    out: int = 0

    @property
    def type(self) -> TypeSpec:
        return self.node.out_types[self.out]


@dataclass(eq=False)
class Subgraph:
    """reference ir.py:86-109"""
    params: list = field(default_factory=list)
    nodes: list = field(default_factory=list)
    outputs: list = field(default_factory=list)

    def add_param(self, name: str, spec: TypeSpec, origin=None) -> Node:
        node = Node("Param", [], {"name": name}, origin or generated_span(), [spec], frame=self)
        self.params.append(node)
        return node

    def add(self, node: Node) -> Node:
        node.frame = self
        self.nodes.append(node)
        return node

    def all_nodes(self):
        return self.params + self.nodes


@dataclass(eq=False)
class GraphFunction:
    """reference ir.py:112-124"""
    name: str
    body: Subgraph
    specialization_key: tuple = ()

    @property
    def params(self):
        return self.body.params


@dataclass(eq=False)
class Graph:
    """reference ir.py:127-163"""
    main: Subgraph = field(default_factory=Subgraph)
    functions: dict = field(default_factory=dict)

    @property
    def outputs(self):
        return self.main.outputs

    def iter_nodes(self):
        seen = []

        def visit(sg):
            for node in list(sg.params) + list(sg.nodes):
                seen.append(node)
                for key in SUBGRAPH_KEYS:
                    sub = node.attrs.get(key)
                    if sub is not None:
                        visit(sub)

        visit(self.main)
        for fn in self.functions.values():
            visit(fn.body)
        return iter(seen)

    def count_ops(self, op: str) -> int:
        return sum(1 for n in self.iter_nodes() if n.op == op)

    def node_count(self) -> int:
        return sum(1 for _ in self.iter_nodes())


# --------------------------------------------------------------------- JSON
FORMAT = "skb-graph/1"


def _type_to_json(t) -> dict:
    if t is None:
        return None
    shape = None if t.shape is None else [None if d is None else int(d) for d in t.shape]
    return {"dtype": t.dtype, "shape": shape, "elem": _type_to_json(getattr(t, "elem", None))}


def _type_from_json(d) -> Optional[TypeSpec]:
    if d is None:
        return None
    shape = None if d["shape"] is None else tuple(d["shape"])
    return TypeSpec(d["dtype"], shape, _type_from_json(d.get("elem")))


def tensor_to_json(v) -> dict:
    data = list(v.data) if not isinstance(v.data, np.ndarray) else v.data.reshape(-1).tolist()
    if v.dtype == "f64":
        data = [float(x) for x in data]
    return {"dtype": v.dtype, "shape": list(v.shape), "data": data}


def tensor_from_json(d) -> TensorValue:
    dt = {"f64": np.float64, "i64": np.int64, "bool": np.bool_}[d["dtype"]]
    arr = np.asarray(d["data"], dtype=dt).reshape(tuple(d["shape"]))
    return TensorValue(d["dtype"], tuple(d["shape"]), arr)


def _attr_to_json(v):
    if hasattr(v, "params") and hasattr(v, "nodes") and hasattr(v, "outputs"):
        return {"__subgraph__": _sg_to_json(v)}
    if hasattr(v, "dtype") and hasattr(v, "shape") and hasattr(v, "data"):
        return {"__tensor__": tensor_to_json(v)}
    if isinstance(v, tuple):
        return {"__tuple__": [_attr_to_json(x) for x in v]}
    if isinstance(v, list):
        return [_attr_to_json(x) for x in v]
    if isinstance(v, dict):
        return {"__dict__": {k: _attr_to_json(x) for k, x in v.items()}}
    return v


def _attr_from_json(v):
    if isinstance(v, dict):
        if "__subgraph__" in v:
            return _sg_from_json(v["__subgraph__"])
        if "__tensor__" in v:
            return tensor_from_json(v["__tensor__"])
        if "__tuple__" in v:
            return tuple(_attr_from_json(x) for x in v["__tuple__"])
        if "__dict__" in v:
            return {k: _attr_from_json(x) for k, x in v["__dict__"].items()}
    if isinstance(v, list):
        return [_attr_from_json(x) for x in v]
    return v


def _span_to_json(s):
    if s is None:
        return None
    return [s.file, s.start_line, s.start_col, s.end_line, s.end_col]


def _node_to_json(n) -> dict:
    return {
        "uid": n.uid, "op": n.op,
        "inputs": [[r.node.uid, r.out] for r in n.inputs],
        "attrs": {k: _attr_to_json(v) for k, v in n.attrs.items()},
        "out_types": [_type_to_json(t) for t in n.out_types],
        "origin": _span_to_json(n.origin),
    }


def _sg_to_json(sg) -> dict:
    return {"params": [_node_to_json(p) for p in sg.params],
            "nodes": [_node_to_json(n) for n in sg.nodes],
            "outputs": [[r.node.uid, r.out] for r in sg.outputs]}


_LOAD_TABLE: dict = {}


def _sg_from_json(d) -> Subgraph:
    sg = Subgraph()
    for nd in d["params"] + d["nodes"]:
        node = Node(nd["op"], [], {}, SourceSpan(*nd["origin"]) if nd["origin"] else generated_span(),
                    [_type_from_json(t) for t in nd["out_types"]], frame=sg, uid=nd["uid"])
        _LOAD_TABLE[nd["uid"]] = node
        node.inputs = [NodeRef(_LOAD_TABLE[u], o) for u, o in nd["inputs"]]
        node.attrs = {k: _attr_from_json(v) for k, v in nd["attrs"].items()}
        (sg.params if nd["op"] == "Param" else sg.nodes).append(node)
    sg.outputs = [NodeRef(_LOAD_TABLE[u], o) for u, o in d["outputs"]]
    return sg


def to_json(graph) -> str:
    """Serialise a reference or skb graph (duck-typed) to the skb wire format."""
    return json.dumps({
        "format": FORMAT,
        "main": _sg_to_json(graph.main),
        "functions": {name: {"body": _sg_to_json(fn.body),
                             "key": _attr_to_json(getattr(fn, "specialization_key", ()))}
                      for name, fn in getattr(graph, "functions", {}).items()},
    })


def from_json(text: str) -> Graph:
    d = json.loads(text) if isinstance(text, str) else text
    if d.get("format") != FORMAT:
        raise ValueError(f"not an {FORMAT} document")
    _LOAD_TABLE.clear()
    g = Graph()
    g.main = _sg_from_json(d["main"])
    for name, fd in d.get("functions", {}).items():
        g.functions[name] = GraphFunction(name, _sg_from_json(fd["body"]), _attr_from_json(fd["key"]))
    _LOAD_TABLE.clear()
    return g
