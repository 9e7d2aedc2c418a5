"""Text feeds and result formatting at the command-line boundary (SURVEY
§8(f)3), in the reference's literal syntax (reference feeds.py:1-6 grammar):

    NAME=f64[2,3]:1.0,2.0,3.0,4.0,5.0,6.0     row-major tensor
    NAME=i64:7   NAME=bool:true                 scalars
    NAME=tree:(5.0 (3.0 () ()) ())              tree: (value left right), () empty

`parse_feed` returns skb host values (values.TensorValue / values.Tree), which
`execute` binds like any feed; malformed text raises FeedSyntaxError.
`format_value` renders results the way the reference CLI prints them
(runtime/values.py:145-163; scalars via tensor.py format_scalar).
"""

from __future__ import annotations

import re

import numpy as np

from .errors import SkbError
from .values import DTYPES, ListValue, TensorValue, Tree, _format_scalar

_NAME = re.compile(r"[A-Za-z_][A-Za-z0-9_]*\Z")
_HEAD = re.compile(r"(?P<dtype>[a-z0-9]+)(?:\[(?P<dims>[^\]]*)\])?\Z")


class FeedSyntaxError(SkbError):
    """A malformed NAME=SPEC feed (reference feeds.py FeedSyntaxError)."""


def _split(text: str):
    name, eq, spec = text.partition("=")
    if not eq:
        raise FeedSyntaxError(f"expected NAME=SPEC, got {text!r}")
    if not _NAME.match(name):
        raise FeedSyntaxError(f"bad parameter name {name!r}")
    return name, spec


def _head(spec: str):
    """'f64[2,3]:data' -> ('f64', (2, 3), 'data' | None); 'tree:(...)' -> ('tree', None, ...)."""
    head, colon, data = spec.partition(":")
    data = data if colon else None
    if head.startswith("tree"):
        return "tree", None, data
    m = _HEAD.match(head)
    if not m or m.group("dtype") not in DTYPES:
        raise FeedSyntaxError(f"unknown dtype or bad shape in {spec!r}")
    dims = m.group("dims")
    try:
        shape = tuple(int(d) for d in dims.split(",")) if dims else ()
    except ValueError:
        raise FeedSyntaxError(f"bad shape in {spec!r}") from None
    return m.group("dtype"), shape, data


_BOOL = {"true": True, "True": True, "1": True, "false": False, "False": False, "0": False}


def _scalars(dtype: str, items: list):
    try:
        if dtype == "bool":
            return [_BOOL[s] for s in items]
        if dtype == "i64":
            return [int(s) for s in items]
        return [float(s) for s in items]
    except (KeyError, ValueError) as exc:
        raise FeedSyntaxError(f"bad {dtype} literal in {items!r}") from exc


def parse_tree(text: str) -> Tree:
    """(value left right) / () with any whitespace; iterative reader."""
    toks = re.findall(r"\(|\)|[^\s()]+", text)
    pos = 0

    def expect_open():
        nonlocal pos
        if pos >= len(toks) or toks[pos] != "(":
            raise FeedSyntaxError(f"expected '(' in tree literal {text[:24]!r}")
        pos += 1

    # explicit stack of partially built nodes: [value, children]
    expect_open()
    stack = [[None, []]]
    root = None
    while stack:
        if pos >= len(toks):
            raise FeedSyntaxError("unclosed tree node")
        top = stack[-1]
        tok = toks[pos]
        if tok == ")":
            pos += 1
            value, kids = stack.pop()
            if value is None and kids:
                raise FeedSyntaxError("tree node without a value")
            if value is not None and len(kids) != 2:
                raise FeedSyntaxError("a tree node needs exactly two children")
            node = Tree() if value is None else Tree(value, kids[0], kids[1])
            if stack:
                stack[-1][1].append(node)
            else:
                root = node
        elif tok == "(":
            if top[0] is None:
                raise FeedSyntaxError("tree node without a value")
            pos += 1
            stack.append([None, []])
        else:
            if top[0] is not None or top[1]:
                raise FeedSyntaxError(f"unexpected {tok!r} in tree literal")
            try:
                top[0] = float(tok)
            except ValueError:
                raise FeedSyntaxError(f"bad tree value {tok!r}") from None
            pos += 1
    if pos != len(toks):
        raise FeedSyntaxError(f"trailing text after tree literal: {' '.join(toks[pos:])!r}")
    return root


def parse_value(spec: str):
    dtype, shape, data = _head(spec)
    if dtype == "tree":
        if data is None:
            raise FeedSyntaxError("tree feed needs a literal, e.g. tree:(5 () ())")
        return parse_tree(data)
    if data is None:
        raise FeedSyntaxError(f"feed {spec!r} has no data (use NAME=dtype:...)")
    items = [s.strip() for s in data.split(",") if s.strip()]
    want = int(np.prod(shape, dtype=np.int64)) if shape else 1
    if len(items) != want:
        raise FeedSyntaxError(f"feed {spec!r} needs {want} values, got {len(items)}")
    return TensorValue(dtype, shape, _scalars(dtype, items))


def parse_feed(text: str):
    """'NAME=SPEC' -> (name, value)."""
    name, spec = _split(text)
    return name, parse_value(spec)


def parse_param_spec(text: str):
    """'NAME=f64[2,3]' (no data) -> (name, dtype, shape) for graph parameters."""
    name, spec = _split(text)
    dtype, shape, data = _head(spec)
    if data is not None:
        raise FeedSyntaxError(f"unexpected data in parameter spec {text!r}")
    return name, dtype, shape


def _tree_str(t) -> str:
    if t is None or t.is_empty:
        return "()"
    return f"({_format_scalar(float(t.value))} {_tree_str(t.left)} {_tree_str(t.right)})"


def format_value(v) -> str:
    """Display form of one result, as the reference CLI prints it."""
    if v is None:
        return "None"
    if isinstance(v, ListValue):
        return "ListValue"
    if isinstance(v, Tree) or (hasattr(v, "is_empty") and not hasattr(v, "dtype")):
        return _tree_str(v)
    if hasattr(v, "dtype") and hasattr(v, "shape"):
        arr = np.asarray(v.array if hasattr(v, "array") else v)
        flat = arr.reshape(-1)
        conv = {"f64": float, "i64": int, "bool": bool}[v.dtype]
        if tuple(v.shape) == ():
            return _format_scalar(conv(flat[0]))
        payload = ",".join(_format_scalar(conv(x)) for x in flat)
        return f"{v.dtype}[{','.join(str(d) for d in v.shape)}]:{payload}"
    return _format_scalar(v) if isinstance(v, (bool, int, float)) else str(v)
