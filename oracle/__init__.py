"""oracle — TEST INFRASTRUCTURE ONLY.

A CPU float64 restatement of the reference executor's arithmetic for the
staged recurrent program (``skb_oracle.c``, every function citing the
reference file:line it follows), the deterministic feed generators shared by
the golden-fixture script and the tests, and the loaders for the golden
fixtures under tests/golden/.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
package — as the checker or the timed CPU baseline, never as the thing
measured on the GPU.  The product (paper_1810_08061_b200) never imports it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liboracle.so")

CAUSE = {10: "IndexOutOfRange", 11: "EmptyPop", 12: "ShapeMismatch", 14: "IterationLimitExceeded"}
CELL_LSTM, CELL_RNN, CELL_GRU = 1, 2, 3

_lib = None
_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.POINTER(ctypes.c_int64)
_P4 = ctypes.c_void_p * 4


def build() -> str:
    """Compile skb_oracle.c (gcc, via oracle/Makefile) if needed."""
    srcs = [os.path.join(HERE, f) for f in ("skb_oracle.c", "lbfgs_oracle.c", "Makefile")]
    if not os.path.exists(LIB_PATH) or any(os.path.getmtime(LIB_PATH) < os.path.getmtime(s) for s in srcs):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        h = ctypes.CDLL(LIB_PATH)
        h.oracle_rnn_program.restype = ctypes.c_int
        h.oracle_rnn_program.argtypes = [ctypes.c_int] * 5 + [_D, _D, _D, _I64, _P4, _P4, _P4,
                                                              ctypes.c_longlong, _D, _I64]
        h.oracle_rnn_many.restype = ctypes.c_int
        h.oracle_rnn_many.argtypes = [ctypes.c_int] * 6 + [_D, _D, _D, _I64, _P4, _P4, _P4, _D, _I64,
                                                           ctypes.POINTER(ctypes.c_int), ctypes.c_int]
        h.oracle_matmul.restype = None
        h.oracle_matmul.argtypes = [_D, _D, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        h.oracle_lbfgs.restype = ctypes.c_int64
        h.oracle_lbfgs.argtypes = [ctypes.c_int64, ctypes.c_int, _D, _D, _D, ctypes.c_double, ctypes.c_int64,
                                   _D, _D]
        _lib = h
    return _lib


def _d(a):
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def matmul(a, b):
    a, b = _f64(a), _f64(b)
    out = np.empty((a.shape[0], b.shape[1]))
    lib().oracle_matmul(_d(a), _d(b), _d(out), a.shape[0], a.shape[1], b.shape[1])
    return out


class OracleError(Exception):
    def __init__(self, cause_kind, max_len):
        super().__init__(cause_kind)
        self.cause_kind = cause_kind
        self.max_len = max_len


def rnn_program(cell, x, h0, c0, lens, W, U, b, max_iterations=None):
    """Run the staged recurrent program on the CPU in float64.

    Returns (out [B, max_len, H], max_len); raises OracleError(cause_kind)
    exactly where the reference executor would fail."""
    x, h0 = _f64(x), _f64(h0)
    B, T, F = x.shape
    H = h0.shape[1]
    c0 = _f64(c0) if cell == CELL_LSTM else np.zeros((B, H))
    lens = np.ascontiguousarray(lens, dtype=np.int64)
    W = [_f64(w) for w in W]
    U = [_f64(u) for u in U]
    b = [_f64(np.broadcast_to(v, (H,))) for v in b]
    m_hint = int(max(lens.max(), 0)) if B else 0
    out = np.zeros((B, max(min(m_hint, T), 1), H))
    ml = np.zeros(1, dtype=np.int64)
    rc = lib().oracle_rnn_program(cell, B, T, F, H, _d(x), _d(h0), _d(c0), lens.ctypes.data_as(_I64),
                                  _P4(*[w.ctypes.data for w in W]), _P4(*[u.ctypes.data for u in U]),
                                  _P4(*[v.ctypes.data for v in b]),
                                  -1 if max_iterations is None else int(max_iterations),
                                  _d(out), ml.ctypes.data_as(_I64))
    m = int(ml[0])
    if rc:
        raise OracleError(CAUSE[rc], m)
    return out[:, :m, :] if m > 0 else out[:, :0, :], m


def rnn_many(cell, x, h0, c0, lens, W, U, b, P, threads):
    """P independent problems (x: [P*B, T, F]) over `threads` host threads.
    Returns (out [P*B, T, H] with [:max_len_p] valid per problem, max_len[P])."""
    x, h0 = _f64(x), _f64(h0)
    R, T, F = x.shape
    H = h0.shape[1]
    B = R // P
    c0 = _f64(c0) if cell == CELL_LSTM else np.zeros((R, H))
    lens = np.ascontiguousarray(lens, dtype=np.int64)
    W = [_f64(w) for w in W]
    U = [_f64(u) for u in U]
    b = [_f64(np.broadcast_to(v, (H,))) for v in b]
    out = np.zeros((R, T, H))
    ml = np.zeros(P, dtype=np.int64)
    st = np.zeros(P, dtype=np.int32)
    lib().oracle_rnn_many(cell, B, T, F, H, P, _d(x), _d(h0), _d(c0), lens.ctypes.data_as(_I64),
                          _P4(*[w.ctypes.data for w in W]), _P4(*[u.ctypes.data for u in U]),
                          _P4(*[v.ctypes.data for v in b]), _d(out), ml.ctypes.data_as(_I64),
                          st.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), int(threads))
    return out, ml, st


def lbfgs(x0, a, b, tol, max_iter, m):
    """The staged L-BFGS program (oracle/programs/lbfgs_m*.msl) in float64 on
    one host thread.  Returns (x, k, margin); raises OracleError on the
    reference's DivisionByZero."""
    x0, a, b = _f64(x0).reshape(-1), _f64(a).reshape(-1), _f64(b).reshape(-1)
    x = np.empty_like(x0)
    margin = np.zeros(1)
    k = lib().oracle_lbfgs(x0.size, int(m), _d(x0), _d(a), _d(b), float(tol), int(max_iter), _d(x), _d(margin))
    if k < 0:
        raise OracleError("DivisionByZero", 0)
    return x, int(k), float(margin[0])
