"""Golden fixtures for automatic differentiation through While:
tests/golden/ad_*.json.  Run in the build container, where the reference is
importable:  python oracle/gen_autodiff_golden.py

Test infrastructure only.  Each fixture holds the forward graph as the
reference stages it (skb JSON wire format), the feeds, the `wrt` names and
expected outputs [loss, d loss/d wrt...] from a source independent of
`paper_1810_08061_b200.autodiff`:

* ad_lstm_*: the reference executing the HAND-WRITTEN staged BPTT program
  (oracle/programs/lstm_bptt.msl, goldens lstm_bptt_*.json);
* ad_maml_*: the reference's own gradient() (graph/grad.py:35-70) over the
  While-free MAML task program, executed by the reference;
* ad_rnn_*: central finite differences of the reference executing the
  forward program (a loop with an in-body Cond, a data-dependent break and
  an append-only output list; no reference gradient exists for it).

Each fixture also records the reference executor running the autodiff graph
(`via_reference`), converted to the reference's IR classes by `to_reference`.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import fixtures  # noqa: E402
from oracle.gen_stream_golden import _ref_value, bptt_feeds, BPTT_CASES, MAML_CASES  # noqa: E402
from paper_1810_08061_b200 import autodiff, ir  # noqa: E402

LSTM_W = [f"{k}{g}" for g in "ifgo" for k in "wub"]
RNN_CASES = [
    {"name": "ad_rnn_full", "T": 5, "B": 3, "F": 4, "H": 5, "lens": [5, 3, 0], "limit": 1e9, "seed": 91},
    {"name": "ad_rnn_break", "T": 7, "B": 2, "F": 3, "H": 4, "lens": [7, 6], "limit": None, "seed": 92,
     "note": "limit set between two iterations' sum(h*h): the loop breaks early"},
]
RNN_WRT = ["x", "h0", "w", "u", "b", "scale", "yl"]


def to_reference(g):
    """skb IR graph -> the reference's IR classes (for its validator/executor)."""
    import stagekit.graph.ir as R
    from stagekit.graph import TensorValue as RT
    memo = {}

    def ts(t):
        return None if t is None else R.TypeSpec(t.dtype, t.shape, ts(t.elem))

    def sg(s):
        out = R.Subgraph()
        for n in list(s.params) + list(s.nodes):
            attrs = {}
            for k, v in n.attrs.items():
                if k in ir.SUBGRAPH_KEYS:
                    v = sg(v)
                elif k == "value":
                    v = RT(v.dtype, tuple(v.shape), tuple(np.asarray(v.data).reshape(-1).tolist()))
                attrs[k] = v
            m = R.Node(n.op, [R.NodeRef(memo[id(r.node)], r.out) for r in n.inputs], attrs, n.origin,
                       [ts(t) for t in n.out_types])
            memo[id(n)] = m
            if n.op == "Param":
                m.frame = out
                out.params.append(m)
            else:
                out.add(m)
        out.outputs = [R.NodeRef(memo[id(r.node)], r.out) for r in s.outputs]
        return out

    G = R.Graph()
    G.main = sg(g.main)
    for name, fn in g.functions.items():
        G.functions[name] = R.GraphFunction(name, sg(fn.body), tuple(fn.specialization_key))
    return G


def trace(program, entry, feeds, order):
    from stagekit.runtime import ParamSpec, trace_module
    from stagekit.syntax import parse_module
    module = parse_module(open(os.path.join(fixtures.PROGRAMS, program)).read(), program)
    specs = [ParamSpec(k, "i64" if np.asarray(feeds[k]).dtype == np.int64 else "f64", tuple(np.asarray(feeds[k]).shape))
             for k in order]
    return trace_module(module, entry, specs).graph


def run_ref(graph, feeds):
    from stagekit.graph import execute
    res = execute(graph, {k: _ref_value(v) for k, v in feeds.items()})
    return [np.asarray(o.data, dtype=np.float64) for o in res.outputs]


def via_reference(graph, feeds, wrt, output=0):
    g = autodiff.gradient(ir.from_json(ir.to_json(graph)), output, wrt)
    return run_ref(to_reference(g), feeds)


def feeds_json(feeds, order):
    out = {}
    for k in order:
        a = np.asarray(feeds[k])
        dt = "i64" if a.dtype == np.int64 else "f64"
        out[k] = {"tensor": {"dtype": dt, "shape": list(a.shape), "data": a.reshape(-1).tolist()}}
    return out


def write(name, doc):
    with open(fixtures.golden_path(name), "w") as f:
        json.dump(doc, f, separators=(",", ":"))


def lstm_cases():
    order = ["x", "h0", "c0", "lens", "y"] + LSTM_W + ["inv_b"]
    for case in BPTT_CASES:
        v = bptt_feeds(case)
        g = trace("lstm_loss.msl", "lstm_loss", v, order)
        exp = fixtures.load_golden(case["name"])["outputs"]
        got = via_reference(g, v, LSTM_W)
        err = max(float(np.max(np.abs(a - np.asarray(e["data"])))) for a, e in zip(got, exp))
        name = "ad_lstm_" + case["name"].split("_")[-1]
        write(name, {"case": dict(case, name=name), "generator": "oracle/gen_autodiff_golden.py",
                     "graph": json.loads(ir.to_json(g)), "feeds": feeds_json(v, order), "wrt": LSTM_W, "output": 0,
                     "expected": [list(e["data"]) for e in exp], "expected_source": f"reference executing "
                     f"oracle/programs/lstm_bptt.msl (hand-written BPTT), golden {case['name']}",
                     "via_reference": [a.tolist() for a in got], "via_reference_max_abs_err": err})
        print(name, "autodiff vs hand BPTT max abs err", err)


def maml_cases():
    from oracle import maml as omaml
    case = MAML_CASES[0]
    H, K = case["H"], case["K"]
    th = omaml.init_theta(H, case["seed"])
    xs, ys, xq, yq = omaml.sinusoid_tasks(case["tasks"], K, case["seed"] + 1)
    order = list(omaml.NAMES) + ["xs", "ys", "xq", "yq", "ones", "alpha", "inv_k"]
    v = {k: th[k] for k in omaml.NAMES}
    v.update(xs=xs[0], ys=ys[0], xq=xq[0], yq=yq[0], ones=np.ones((K, 1)), alpha=np.float64(case["alpha"]),
             inv_k=np.float64(1.0 / K))
    g = trace("maml.msl", "maml_task", v, order)
    exp = fixtures.load_golden(case["name"])["outputs"][0]
    got = via_reference(g, v, list(omaml.NAMES))
    err = max(float(np.max(np.abs(a - np.asarray(e)))) for a, e in zip(got, exp))
    write("ad_maml_h8", {"case": {"name": "ad_maml_h8", "from": case["name"]}, "generator": "oracle/gen_autodiff_golden.py",
                         "graph": json.loads(ir.to_json(g)), "feeds": feeds_json(v, order), "wrt": list(omaml.NAMES),
                         "output": 0, "expected": [list(e) for e in exp],
                         "expected_source": f"reference gradient() executed by the reference, golden {case['name']} task 0",
                         "via_reference": [a.tolist() for a in got], "via_reference_max_abs_err": err})
    print("ad_maml_h8 autodiff vs reference gradient() max abs err", err)


def rnn_feeds(case):
    rng = np.random.default_rng(case["seed"])
    T, B, F, H = case["T"], case["B"], case["F"], case["H"]
    return {"x": rng.uniform(-1, 1, (T, B, F)), "h0": rng.uniform(-.5, .5, (B, H)),
            "lens": np.asarray(case["lens"], dtype=np.int64), "yl": rng.uniform(-1, 1, (B, H)),
            "w": rng.uniform(-.8, .8, (F, H)), "u": rng.uniform(-.8, .8, (H, H)), "b": rng.uniform(-.3, .3, (B, H)),
            "scale": np.float64(0.9), "limit": np.float64(1e9)}


def rnn_cases():
    order = ["x", "h0", "lens", "yl", "w", "u", "b", "scale", "limit"]
    for case in RNN_CASES:
        v = rnn_feeds(case)
        g = trace("rnn_seq_loss.msl", "rnn_seq_loss", v, order)
        if case["limit"] is None:   # the middle of the widest limit interval that stops the loop early
            grid = np.linspace(0.0, float(case["B"] * case["H"]), 2000)
            trips = np.asarray([int(run_ref(g, dict(v, limit=np.float64(L)))[1][0]) for L in grid])
            early = [k for k in range(2, case["T"]) if np.any(trips == k)]
            best = max(early, key=lambda k: int(np.sum(trips == k)))
            sel = grid[trips == best]
            v["limit"] = np.float64(0.5 * (sel.min() + sel.max()))
        else:
            v["limit"] = np.float64(case["limit"])
        base = run_ref(g, v)
        fd = [base[0]]
        eps = 1e-6
        for k in RNN_WRT:
            a = np.array(v[k], dtype=np.float64)
            gk = np.zeros(a.size)
            for i in range(a.size):
                hi, lo = a.copy().reshape(-1), a.copy().reshape(-1)
                hi[i] += eps
                lo[i] -= eps
                fp = run_ref(g, dict(v, **{k: hi.reshape(a.shape)}))
                fm = run_ref(g, dict(v, **{k: lo.reshape(a.shape)}))
                assert fp[1][0] == fm[1][0] == base[1][0], "trip count changed under the perturbation"
                gk[i] = (fp[0][0] - fm[0][0]) / (2 * eps)
            fd.append(gk)
        got = via_reference(g, v, RNN_WRT)
        err = max(float(np.max(np.abs(a - b) / (1 + np.abs(b)))) for a, b in zip(got[2:], fd[1:]))
        assert err < 1e-6, err
        write(case["name"], {"case": case, "generator": "oracle/gen_autodiff_golden.py", "graph": json.loads(ir.to_json(g)),
                             "feeds": feeds_json(v, order), "wrt": RNN_WRT, "output": 0,
                             "expected": [base[0].tolist()] + [f.tolist() for f in fd[1:]], "trips": int(base[1][0]),
                             "expected_source": "central finite differences (eps 1e-6) of the reference executing "
                                                "the forward program", "expected_tol": 1e-6,
                             "via_reference": [a.tolist() for a in got], "via_reference_fd_rel_err": err})
        print(case["name"], "trips", int(base[1][0]), "autodiff vs finite differences rel err", err)


if __name__ == "__main__" and not sys.argv[1:]:
    lstm_cases()
    maml_cases()
    rnn_cases()


def bench_graph():
    """tests/golden/graph_lstm_loss_bench.json: the forward LSTM loss program traced
    by the reference at the gradient-bench shape (T=16, B=32, F=H=64)."""
    case = {"name": "bench", "T": 16, "B": 32, "F": 64, "H": 64, "lens": list(range(1, 17)) * 2, "seed": 5}
    v = bptt_feeds(case)
    order = ["x", "h0", "c0", "lens", "y"] + LSTM_W + ["inv_b"]
    g = trace("lstm_loss.msl", "lstm_loss", v, order)
    write("graph_lstm_loss_bench", {"case": case, "generator": "oracle/gen_autodiff_golden.py --bench",
                                    "graph": json.loads(ir.to_json(g)), "order": order})
    print("graph_lstm_loss_bench written")


if __name__ == "__main__" and sys.argv[1:2] == ["--bench"]:
    bench_graph()
