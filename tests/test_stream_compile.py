"""CPU checks of the vector-stream tier: the float64 L-BFGS oracle against the
reference's own outputs (bit-exact), and the compiler's structure (fusion,
grid exchanges per iteration, eligibility) — no GPU needed."""

import numpy as np
import pytest

import oracle
from oracle import fixtures
from paper_1810_08061_b200 import LoweringError, ir
from paper_1810_08061_b200 import stream as st
from paper_1810_08061_b200.executor import plan_kind


@pytest.mark.parametrize("name", ["lbfgs_m3_n50", "lbfgs_m10_n2000", "lbfgs_m10_n3000_cap"])
def test_lbfgs_oracle_bit_exact_with_reference(name):
    doc = fixtures.load_golden(name)
    f = fixtures.make_stream_feeds(doc["case"])
    m = 3 if "_m3_" in name else 10
    x, k, margin = oracle.lbfgs(f["x0"], f["a"], f["b"], float(f["tol"]), int(f["max_iter"]), m)
    exp = doc["expected"]["outputs"]
    assert k == exp[1]["tensor"]["data"][0]
    assert np.array_equal(x, np.asarray(exp[0]["tensor"]["data"]))
    assert margin > 0.01


def _groups(prog):
    out = []
    for c in prog.code:
        if c[0] == st.SOP["VEXEC"]:
            off = c[2]
            nops, nst, nred, nins = prog.extra[off:off + 4]
            out.append((nops, nst, nred, nins))
    return out


@pytest.mark.parametrize("name", [c["name"] for c in fixtures.STREAM_CASES])
def test_stream_fixtures_compile(name):
    prog = st.compile_graph(ir.from_json(fixtures.load_golden(name)["graph"]))
    assert prog.max_ops <= st.MAX_OPS and prog.max_stack <= st.MAX_STACK and prog.max_temp <= st.MAX_TEMP
    assert prog.code[-1][0] == st.SOP["HALT"]


def test_lbfgs_update_is_one_fused_pass():
    prog = st.compile_graph(ir.from_json(fixtures.load_golden("graph_lbfgs_c4")["graph"]))
    groups = _groups(prog)
    # x - r, a*xn - b, xn - x, gn - g stored; s.y, y.y, gn.gn reduced: one pass over x, r, a, b, g
    assert (5, 4, 3) in [(o, s, r) for o, s, r, _ in groups], groups
    # two-loop recursion: every history pair costs one reduce pass + one axpy pass
    assert sum(1 for g in groups if g[2] == 1) >= 2 * 10
    assert prog.shape == (None,)


def test_ineligible_graphs_raise():
    g = ir.from_json(fixtures.load_golden("lstm_4x8x8")["graph"])
    with pytest.raises(LoweringError):
        st.compile_graph(g)


def test_dispatch_by_feed_size():
    g = ir.from_json(fixtures.load_golden("graph_lbfgs_c4")["graph"])
    small = {"x0": np.zeros(100), "a": np.ones(100), "b": np.zeros(100), "tol": np.float64(1e-9),
             "max_iter": np.int64(5)}
    big = dict(small, x0=np.zeros(1 << 15), a=np.ones(1 << 15), b=np.zeros(1 << 15))
    assert plan_kind(g, small) == "vm"
    assert plan_kind(g, big) == "stream"
