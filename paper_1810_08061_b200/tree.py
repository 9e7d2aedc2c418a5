"""Batched TreeLSTM over a forest on the GPU (BASELINE config C5; csrc/tree.cu).

The reference evaluates the TreeLSTM program of SURVEY App. D by recursion
over `Tree` values (graph/execute.py:136-146 Tree ops, :191-194 FuncCall).
`Forest` flattens any number of trees (reference `Tree` objects, skb
`values.Tree`, or (value, left, right) arrays in pre-order), computes every
node's height and schedules the forest level by level: all leaves in one
launch, then one GEMM + fused cell per height level across the whole batch.

    forest = Forest(trees)
    h_root, c_root = tree_lstm(forest, weights)      # weights: oracle.fixtures.TREE_WEIGHTS names
"""
from __future__ import annotations

import ctypes

import numpy as np

from .values import DeviceTensor

GATES = (("uil", "uir"), ("ufll", "uflr"), ("ufrl", "ufrr"), ("uol", "uor"), ("uul", "uur"))


def _flatten_tree(t):
    val, left, right = [], [], []
    stack = [(t, -1, 0)]
    while stack:   # iterative pre-order (trees can be deep)
        node, parent, side = stack.pop()
        i = len(val)
        val.append(float(node.value) if node.value is not None else 0.0)
        left.append(-1)
        right.append(-1)
        if parent >= 0:
            (left if side == 0 else right)[parent] = i
        l, r = getattr(node, "left", None), getattr(node, "right", None)
        if l is not None and getattr(l, "value", None) is not None:
            stack.append((r, i, 1))
            stack.append((l, i, 0))
    return np.asarray(val), np.asarray(left, dtype=np.int64), np.asarray(right, dtype=np.int64)


class Forest:
    """Host schedule of a batch of binary trees (leaves: both children empty);
    the O(nodes) scheduling pass is native (skb_forest_schedule in csrc/tree.cu)."""

    def __init__(self, trees):
        flat = [t if isinstance(t, tuple) else _flatten_tree(t) for t in trees]
        vals, lefts, rights = (list(x) for x in zip(*flat)) if flat else ([], [], [])
        sizes = np.fromiter(map(len, vals), dtype=np.int64, count=len(vals))
        bases = np.concatenate([[0], np.cumsum(sizes)[:-1]]) if len(flat) else np.zeros(0, np.int64)
        # (np.concatenate converts array-likes itself; one dtype cast per field)
        self.value = np.concatenate(vals).astype(np.float64, copy=False) if flat else np.zeros(0)
        left = np.ascontiguousarray(np.concatenate(lefts) if flat else np.zeros(0), dtype=np.int64)
        right = np.ascontiguousarray(np.concatenate(rights) if flat else np.zeros(0), dtype=np.int64)
        self.roots = bases.astype(np.int64)
        n = len(self.value)
        from . import runtime as rt
        lib = rt.host_lib()   # the scheduler is host code
        self.left = np.empty(n, dtype=np.int32)    # global child ids (-1: none)
        self.right = np.empty(n, dtype=np.int32)
        self.height = np.empty(n, dtype=np.int32)
        order = np.empty(n, dtype=np.int32)
        level_off = np.empty(n + 1, dtype=np.int32)
        leaves = np.empty(n, dtype=np.int32)
        self.dest = np.empty(n, dtype=np.int32)
        c = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        maxh = lib.skb_forest_schedule(len(flat), c(sizes), c(left), c(right), c(self.left), c(self.right),
                                       c(self.height), c(order), c(level_off), c(leaves), c(self.dest))
        if maxh < 0:
            raise ValueError("TreeLSTM trees must be full binary trees (0 or 2 children, listed in pre-order)")
        self.nlevels = int(maxh)
        self.level_off = level_off[:maxh + 1].copy()
        ninternal = int(self.level_off[-1]) if maxh > 0 else 0
        self.order = order[:ninternal].copy()
        self.leaves = leaves[:n - ninternal].copy()
        self._dev = None

    @property
    def nnodes(self):
        return len(self.value)

    def device(self, dev):
        import torch
        if self._dev is None or self._dev[0] != dev:
            i32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)
            self._dev = (dev, {"leaves": i32(self.leaves), "order": i32(self.order), "left": i32(self.left),
                               "right": i32(self.right), "dest": i32(self.dest),
                               "value": torch.from_numpy(self.value.astype(np.float32)).to(dev),
                               "roots": torch.from_numpy(self.roots).to(dev)})
        return self._dev[1]


def pack_weights(w, dev):
    """U [2H, 5H] (gate blocks i|f_l|f_r|o|u) and bias [5H] on the device."""
    import torch
    H = np.asarray(w["wc"]).shape[-1]
    U = np.zeros((2 * H, 5 * H), dtype=np.float32)
    for k, (a, b) in enumerate(GATES):
        U[:H, k * H:(k + 1) * H] = np.asarray(w[a])
        U[H:, k * H:(k + 1) * H] = np.asarray(w[b])
    bias = np.concatenate([np.asarray(w[k]).reshape(-1) for k in ("bi", "bf", "bf", "bo", "bu")]).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)
    return {"H": H, "wc": t(np.asarray(w["wc"]).reshape(-1)), "U": t(U), "bias": t(bias)}


def tree_lstm(forest, weights, math="fp32", stream=None, packed=None, all_nodes=False):
    """Root (h, c) of every tree, [ntrees, H] float32 DeviceTensors (all nodes'
    states with all_nodes=True)."""
    import torch
    from . import runtime as rt
    lib = rt.lib()
    dev = torch.device("cuda", torch.cuda.current_device())
    pw = packed or pack_weights(weights, dev)
    H = pw["H"]
    d = forest.device(dev)
    n, ni = forest.nnodes, len(forest.order)
    bufs = d.get(("bufs", H))
    if bufs is None:   # reused across evaluations of this forest (stable pointers -> CUDA graph replay)
        bufs = (torch.empty(int(lib.skb_tree_workspace_bytes(n, max(ni, 1), H)), dtype=torch.uint8, device=dev),
                torch.empty((n, H), dtype=torch.float32, device=dev),
                torch.empty((n, H), dtype=torch.float32, device=dev))
        d[("bufs", H)] = bufs
    ws, h, c = bufs
    off = np.ascontiguousarray(forest.level_off, dtype=np.int32)
    p = rt.ptr
    rt.check(lib.skb_tree_lstm(n, len(forest.leaves), ni, H, forest.nlevels, p(d["leaves"]), p(d["order"]),
                               off.ctypes.data_as(ctypes.c_void_p), p(d["left"]), p(d["right"]), p(d["dest"]),
                               p(d["value"]), p(pw["wc"]), p(pw["U"]), p(pw["bias"]), 1 if math == "tf32" else 0,
                               p(h), p(c), p(ws), rt.stream_handle(stream)), "skb_tree_lstm")
    if all_nodes:
        return DeviceTensor("f64", h.clone()), DeviceTensor("f64", c.clone())
    return DeviceTensor("f64", h[d["roots"]]), DeviceTensor("f64", c[d["roots"]])
