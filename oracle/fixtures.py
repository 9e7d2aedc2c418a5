"""Golden-fixture case table and deterministic feed generation (TEST
INFRASTRUCTURE ONLY).

`gen_golden.py` (run where /root/reference exists) traces each program with
the reference's own `trace_module`, executes it with the reference's own
`execute`, and writes tests/golden/<case>.json holding the traced graph (skb
wire format), the feed specification and the reference's outputs (or its
failure `cause_kind`).  Feeds are regenerated from the spec with numpy's
PCG64 streams, identically on every machine, so fixtures stay small.
"""

from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
GOLDEN = os.path.join(REPO, "tests", "golden")
PROGRAMS = os.path.join(HERE, "programs")

LSTM_PARAMS = ["input_data", "h0", "c0", "sequence_len"] + \
    [f"{k}{g}" for g in "ifgo" for k in ("w", "u", "b")]
RNN_PARAMS = ["input_data", "initial_state", "sequence_len", "w_x", "w_h", "b"]
GRU_PARAMS = ["input_data", "h0", "sequence_len", "wz", "uz", "bz", "wr", "ur", "br", "wn", "un", "bn", "bhn"]


def lstm_case(name, B, T, F, H, lens, seed, program="lstm.msl", entry="dynamic_lstm", wscale=0.1,
              xscale=1.0, note=""):
    return {"name": name, "program": program, "entry": entry, "cell": "lstm",
            "dims": {"B": B, "T": T, "F": F, "H": H}, "lens": lens, "seed": seed,
            "wscale": wscale, "xscale": xscale, "note": note}


def gru_case(name, B, T, F, H, lens, seed, program="gru.msl", entry="dynamic_gru", wscale=0.1,
             xscale=1.0, note=""):
    return {"name": name, "program": program, "entry": entry, "cell": "gru",
            "dims": {"B": B, "T": T, "F": F, "H": H}, "lens": lens, "seed": seed,
            "wscale": wscale, "xscale": xscale, "note": note}


def rnn_case(name, B, T, F, H, lens, seed, program="corpus:dynamic_rnn.msl", entry="dynamic_rnn",
             wscale=1.0, xscale=1.0, note=""):
    return {"name": name, "program": program, "entry": entry, "cell": "rnn",
            "dims": {"B": B, "T": T, "F": F, "H": H}, "lens": lens, "seed": seed,
            "wscale": wscale, "xscale": xscale, "note": note}


# Parity cases: edge cases the reference's own tests and semantics pin
# (SURVEY §8(c)), small enough for the pure-Python reference executor.
CASES = [
    rnn_case("rnn_corpus_2x3x4", 2, 3, 4, 4, [3, 1], 101,
             note="corpus/dynamic_rnn.msl shapes and lengths (manifest.json:45-58)"),
    rnn_case("rnn_accept_2x5x4", 2, 5, 4, 4, [3, 1], 1234,
             note="acceptance criterion 3 shapes (test_acceptance.py:72-110), T longer than max_len"),
    rnn_case("rnn_handwritten_2x3x4", 2, 3, 4, 4, [3, 1], 7, program="handwritten",
             note="graph built by dispatch.while_stmt directly (tests/helpers.py:40-80)"),
    rnn_case("rnn_32x16x64", 32, 16, 64, 64, "random", 11),
    rnn_case("rnn_limit_ok", 3, 6, 4, 4, [4, 2, 1], 5, program="rnn_limited.msl",
             note="max_iterations=4 directive, trip count 4: no failure"),
    rnn_case("rnn_limit_hit", 3, 6, 4, 4, [5, 2, 1], 5, program="rnn_limited.msl",
             note="max_iterations=4 with trip count 5 -> IterationLimitExceeded"),
    lstm_case("lstm_4x8x8", 4, 8, 8, 8, [8, 3, 1, 6], 21, note="SURVEY §8(c) C1 pin shape"),
    lstm_case("lstm_zero_len_rows", 3, 5, 8, 8, [5, 0, 2], 22, note="a row of length 0 keeps h0"),
    lstm_case("lstm_all_full", 4, 4, 8, 8, [4, 4, 4, 4], 23),
    lstm_case("lstm_ragged_12x20", 5, 6, 12, 20, [6, 1, 3, 6, 2], 24, note="F != H, H not a multiple of 16"),
    lstm_case("lstm_32x16x64", 32, 16, 64, 64, "random", 25),
    lstm_case("lstm_4x6x256", 4, 6, 256, 256, [6, 2, 5, 1], 26, note="C1 widths (H=F=256): full 8-CTA cluster"),
    lstm_case("lstm_final_states", 3, 5, 8, 16, [5, 2, 3], 27, program="lstm_final.msl",
              entry="dynamic_lstm_states", note="returns [stacked (time-major), h_T, c_T]"),
    lstm_case("lstm_len_gt_T", 3, 4, 8, 8, [2, 6, 1], 28, note="len > T -> IndexOutOfRange"),
    lstm_case("lstm_all_zero", 3, 4, 8, 8, [0, 0, 0], 29, note="max_len 0 -> EmptyPop"),
    lstm_case("lstm_negative", 3, 4, 8, 8, [-1, -3, -2], 30, note="max_len < 0 -> ShapeMismatch (Range)"),
    lstm_case("lstm_mixed_negative", 3, 4, 8, 8, [-2, 3, 0], 31, note="negative row is frozen at h0"),
    lstm_case("lstm_large_inputs", 3, 5, 8, 8, [5, 4, 2], 32, xscale=100.0, wscale=0.5,
              note="saturating gates"),
    gru_case("gru_4x8x8", 4, 8, 8, 8, [8, 3, 1, 6], 41, note="GRU cell (oracle/programs/gru.msl)"),
    gru_case("gru_zero_len_rows", 3, 5, 8, 8, [5, 0, 2], 42, note="a row of length 0 keeps h0"),
    gru_case("gru_ragged_12x20", 5, 6, 12, 20, [6, 1, 3, 6, 2], 43, note="F != H, H not a multiple of 16"),
    gru_case("gru_32x16x64", 32, 16, 64, 64, "random", 44),
    gru_case("gru_4x6x256", 4, 6, 256, 256, [6, 2, 5, 1], 45, note="C1 widths (H=F=256): dual-lane kernel"),
    gru_case("gru_len_gt_T", 3, 4, 8, 8, [2, 6, 1], 46, note="len > T -> IndexOutOfRange"),
    gru_case("gru_all_zero", 3, 4, 8, 8, [0, 0, 0], 47, note="max_len 0 -> EmptyPop"),
    gru_case("gru_large_inputs", 3, 5, 8, 8, [5, 4, 2], 48, xscale=100.0, wscale=0.5, note="saturating gates"),
]


def case_by_name(name):
    for c in CASES:
        if c["name"] == name:
            return c
    raise KeyError(name)


def param_names(case):
    return {"lstm": LSTM_PARAMS, "gru": GRU_PARAMS}.get(case["cell"], RNN_PARAMS)


def make_feeds(case) -> dict:
    """Deterministic numpy feeds for a case (float64 / int64)."""
    d = case["dims"]
    B, T, F, H = d["B"], d["T"], d["F"], d["H"]
    rng = np.random.default_rng(case["seed"])
    xs, ws = case["xscale"], case["wscale"]
    feeds = {"input_data": rng.uniform(-xs, xs, (B, T, F))}
    if case["lens"] == "random":
        lens = rng.integers(1, T + 1, B)
    else:
        lens = np.asarray(case["lens"])
    if case["cell"] == "lstm":
        feeds["h0"] = rng.uniform(-0.1, 0.1, (B, H))
        feeds["c0"] = rng.uniform(-0.1, 0.1, (B, H))
        feeds["sequence_len"] = lens.astype(np.int64)
        for g in "ifgo":
            feeds["w" + g] = rng.uniform(-ws, ws, (F, H))
            feeds["u" + g] = rng.uniform(-ws, ws, (H, H))
            feeds["b" + g] = rng.uniform(-ws, ws, (H,))
    elif case["cell"] == "gru":
        feeds["h0"] = rng.uniform(-0.1, 0.1, (B, H))
        feeds["sequence_len"] = lens.astype(np.int64)
        for g in "zrn":
            feeds["w" + g] = rng.uniform(-ws, ws, (F, H))
            feeds["u" + g] = rng.uniform(-ws, ws, (H, H))
            feeds["b" + g] = rng.uniform(-ws, ws, (H,))
        feeds["bhn"] = rng.uniform(-ws, ws, (H,))
    else:
        feeds["initial_state"] = rng.uniform(-1, 1, (B, H))
        feeds["sequence_len"] = lens.astype(np.int64)
        feeds["w_x"] = rng.uniform(-ws, ws, (F, H)) / np.sqrt(max(F, 1))
        feeds["w_h"] = rng.uniform(-ws, ws, (H, H)) / np.sqrt(max(H, 1))
        feeds["b"] = rng.uniform(-ws, ws, (H,))
    return feeds


def oracle_args(case, feeds):
    """(cell, x, h0, c0, lens, W, U, b) for oracle.rnn_program."""
    if case["cell"] == "lstm":
        return (1, feeds["input_data"], feeds["h0"], feeds["c0"], feeds["sequence_len"],
                [feeds["w" + g] for g in "ifgo"], [feeds["u" + g] for g in "ifgo"],
                [feeds["b" + g] for g in "ifgo"])
    if case["cell"] == "gru":
        return (3, feeds["input_data"], feeds["h0"], None, feeds["sequence_len"],
                [feeds["w" + g] for g in "zrn"], [feeds["u" + g] for g in "zrn"],
                [feeds["b" + g] for g in "zrn"] + [feeds["bhn"]])
    return (2, feeds["input_data"], feeds["initial_state"], None, feeds["sequence_len"],
            [feeds["w_x"]], [feeds["w_h"]], [feeds["b"]])


def golden_path(name):
    return os.path.join(GOLDEN, f"{name}.json")


def load_golden(name) -> dict:
    with open(golden_path(name)) as f:
        return json.load(f)


def load_graph_fixture(name="graph_lstm_c1"):
    """(graph, case) of a graph-only fixture (traced program at benchmark size)."""
    import sys
    sys.path.insert(0, REPO)
    from paper_1810_08061_b200 import ir
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        doc = json.load(f)
    return ir.from_json(doc["graph"]), doc["case"]


def golden_names():
    return [c["name"] for c in CASES if os.path.exists(golden_path(c["name"]))]


# ---------------------------------------------------------------- vector-stream programs (C4 class)
def stream_case(name, program, entry, feeds, seed, note=""):
    """feeds: name -> {"dtype", "shape", "dist": [lo, hi]} or {"dtype", "value"}."""
    return {"name": name, "program": program, "entry": entry, "feeds": feeds, "seed": seed, "note": note}


def _vecf(n, lo, hi):
    return {"dtype": "f64", "shape": [n], "dist": [lo, hi]}


def lbfgs_feeds(n, tol=1e-18, max_iter=100):
    """Separable quadratic f = 1/2 sum a x^2 - b x."""
    return {"x0": _vecf(n, -1.0, 1.0), "a": _vecf(n, 0.5, 4.0), "b": _vecf(n, -1.0, 1.0),
            "tol": {"dtype": "f64", "value": tol}, "max_iter": {"dtype": "i64", "value": max_iter}}


STREAM_CASES = [
    stream_case("lbfgs_m3_n50", "lbfgs_m3.msl", "lbfgs", lbfgs_feeds(50), 41,
                note="SURVEY App. C L-BFGS, m=3 (converges in ~30 iterations)"),
    stream_case("lbfgs_m10_n2000", "lbfgs_m10.msl", "lbfgs", lbfgs_feeds(2000), 42,
                note="BASELINE C4 program (m=10) at a size the reference finishes in seconds"),
    stream_case("lbfgs_m10_n3000_cap", "lbfgs_m10.msl", "lbfgs", lbfgs_feeds(3001, 1e-30, 7), 43,
                note="iteration cap reached (k == max_iter), ragged length"),
    stream_case("stream_mix_n1500", "stream_mix.msl", "stream_mix",
                {"v": _vecf(1500, -2.0, 2.0), "w": _vecf(1500, -1.0, 1.0),
                 "iv": {"dtype": "i64", "shape": [1500], "dist": [-50, 50]},
                 "c": {"dtype": "f64", "value": 0.25}, "n_iter": {"dtype": "i64", "value": 6}}, 44,
                note="i64/bool vectors, floor-mod, Where, tanh/sigmoid, Cond on a reduction, list append/pop"),
    stream_case("stream_div0", "stream_div0.msl", "stream_div0",
                {"x": _vecf(700, -1.0, 1.0), "y": {"dtype": "f64", "shape": [700], "dist": [3, 3]},
                 "n_iter": {"dtype": "i64", "value": 5}}, 45, note="vector division by zero -> DivisionByZero"),
    stream_case("stream_limit", "stream_limit.msl", "stream_limit",
                {"x": _vecf(900, -1.0, 1.0), "tol": {"dtype": "f64", "value": 1e-6}}, 46,
                note="max_iterations=5 exceeded -> IterationLimitExceeded"),
    stream_case("stream_limit_ok", "stream_limit.msl", "stream_limit",
                {"x": _vecf(900, -1e-3, 1e-3), "tol": {"dtype": "f64", "value": 1e-6}}, 47,
                note="converges within max_iterations"),
    stream_case("stream_index_ok", "stream_index.msl", "stream_index",
                {"x": _vecf(600, -1.0, 1.0), "j": {"dtype": "i64", "value": -1}}, 48, note="negative list index wraps"),
    stream_case("stream_index_oob", "stream_index.msl", "stream_index",
                {"x": _vecf(600, -1.0, 1.0), "j": {"dtype": "i64", "value": 2}}, 49,
                note="list index 2 of 2 -> IndexOutOfRange"),
]


def stream_case_by_name(name):
    for c in STREAM_CASES:
        if c["name"] == name:
            return c
    raise KeyError(name)


def make_stream_feeds(case) -> dict:
    """Deterministic numpy feeds (float64 / int64 arrays, 0-d for scalars)."""
    rng = np.random.default_rng(case["seed"])
    out = {}
    for name in sorted(case["feeds"]):
        f = case["feeds"][name]
        if "value" in f:
            out[name] = np.asarray(f["value"], dtype=np.float64 if f["dtype"] == "f64" else np.int64)
            continue
        lo, hi = f["dist"]
        shape = tuple(f["shape"])
        if f["dtype"] == "f64":
            out[name] = rng.uniform(lo, hi, shape) if lo != hi else np.full(shape, float(lo))
        else:
            out[name] = rng.integers(lo, hi + 1, shape).astype(np.int64)
    return {name: out[name] for name in case["feeds"]}   # the entry's parameter order


# ---------------------------------------------------------------- greedy decode with EOS stop (C3)
def greedy_case(name, V, E, H, max_len, eos, seed, uscale=0.5, note=""):
    """tanh-RNN decoder, logits = h @ w_out, argmax, EOS `break`."""
    return {"name": name, "program": "greedy.msl", "entry": "greedy", "dims": {"V": V, "E": E, "H": H},
            "max_len": max_len, "eos": eos, "seed": seed, "uscale": uscale, "note": note}


GREEDY_CASES = [
    greedy_case("greedy_v64_stop", 64, 8, 16, 30, 46, 3, note="EOS (46) reached at step 9: data-dependent stop"),
    greedy_case("greedy_v64_nostop", 64, 8, 16, 30, 5, 3, note="EOS never produced: runs to max_len"),
    greedy_case("greedy_v300_stop", 300, 12, 24, 40, -1, 4, note="eos picked by the generator (first repeat)"),
    greedy_case("greedy_v64_zero", 64, 8, 16, 0, 46, 3, note="max_len 0: no step, toks = [0]"),
]


def greedy_case_by_name(name):
    for c in GREEDY_CASES:
        if c["name"] == name:
            return c
    raise KeyError(name)


def make_greedy_feeds(case) -> dict:
    d = case["dims"]
    V, E, H = d["V"], d["E"], d["H"]
    rng = np.random.default_rng(case["seed"])
    return {"h0": rng.uniform(-1, 1, (1, H)), "emb": rng.uniform(-1, 1, (V, 1, E)),
            "w_in": rng.uniform(-1, 1, (E, H)), "u": rng.uniform(-1, 1, (H, H)) * case["uscale"],
            "w_out": rng.uniform(-1, 1, (H, V)), "ids": np.arange(V, dtype=np.int64),
            "eos": np.asarray(case["eos"], dtype=np.int64), "max_len": np.asarray(case["max_len"], dtype=np.int64)}


# ---------------------------------------------------------------- TreeLSTM (C5)
TREE_WEIGHTS = ["wc", "uil", "uir", "ufll", "uflr", "ufrl", "ufrr", "uol", "uor", "uul", "uur", "bi", "bf", "bo", "bu"]


def random_tree_arrays(n_leaves, rng):
    """A random binary tree with n_leaves leaves as (value, left, right) arrays
    in pre-order (node 0 = root, -1 = no child); internal values are 0."""
    val, left, right = [], [], []

    def build(n):
        i = len(val)
        val.append(0.0)
        left.append(-1)
        right.append(-1)
        if n == 1:
            val[i] = float(rng.uniform(-1, 1))
            return i
        k = int(rng.integers(1, n))
        left[i] = build(k)
        right[i] = build(n - k)
        return i
    build(n_leaves)
    return np.asarray(val), np.asarray(left, dtype=np.int64), np.asarray(right, dtype=np.int64)


def tree_str(val, left, right, i=0):
    """The reference Tree's text form '(v (l) (r))', '()' for empty."""
    if i < 0:
        return "()"
    return f"({float(val[i])!r} {tree_str(val, left, right, left[i])} {tree_str(val, left, right, right[i])})"


def tree_weights(H, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    w = {"wc": rng.uniform(-1, 1, (1, H))}
    for k in TREE_WEIGHTS[1:11]:
        w[k] = rng.uniform(-1, 1, (H, H)) * scale / np.sqrt(H)
    for k in TREE_WEIGHTS[11:]:
        w[k] = rng.uniform(-0.5, 0.5, (H,))
    return w


TREE_CASES = [
    {"name": "treelstm_h8", "H": 8, "seed": 61, "leaves": [2, 3, 5, 8, 1, 13], "note": "mixed shapes incl. a single leaf"},
    {"name": "treelstm_h16", "H": 16, "seed": 62, "leaves": [32, 7, 20], "note": "C5 leaf count (32)"},
]
