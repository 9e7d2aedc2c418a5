"""S-expression wire format (paper_1810_08061_b200/sexpr.py),
CPU side: every program of tests/golden/sexpr_cases.json — the reference's own
`to_sexpr` rendering of the region-VM corpus and fuzz graphs, the corpus
renderings identical to the reference's shipped corpus/golden/*.sexpr files —
reads back into a graph that validates and re-renders to the same text.
Execution on the B200 is tests/test_gpu_sexpr.py."""
import json
import os

import pytest

from paper_1810_08061_b200 import sexpr
from paper_1810_08061_b200.validate import validate

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(GOLDEN, "sexpr_cases.json")) as f:
    CASES = json.load(f)["cases"]


def test_fixture_pinned_to_reference_corpus_files():
    corpus = [c for c in CASES if c["source"] == "corpus"]
    assert len(corpus) == 8 and all(c["matches_reference_corpus_file"] for c in corpus)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_read_validate_and_round_trip(case):
    g = sexpr.from_sexpr(case["sexpr"])
    validate(g)
    assert sexpr.to_sexpr(g).strip() == case["sexpr"].strip()


def test_shared_loop_outputs_are_one_loop():
    """(out 0 W) and (out 1 W) of one rendered While become one While node."""
    case = next(c for c in CASES if c["name"] == "corpus-break_sum")
    g = sexpr.from_sexpr(case["sexpr"])
    assert g.count_ops("While") == 1


@pytest.mark.parametrize("text, msg", [
    ("(def main ((x f64)) (add x y))", "unbound symbol"),
    ("(def main ((x f64)) (frobnicate x))", "unknown form"),
    ("(def main ((x f64)) (add x x)", "unbalanced"),
    ("(def main ((x f64)) (call nope x))", "undefined function"),
])
def test_errors(text, msg):
    with pytest.raises(sexpr.SexprError, match=msg):
        sexpr.from_sexpr(text)
