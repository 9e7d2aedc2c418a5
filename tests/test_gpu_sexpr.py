"""S-expression programs on the B200: the reference's own `to_sexpr` text of
the corpus and differential-fuzz programs (tests/golden/sexpr_cases.json),
read by paper_1810_08061_b200.sexpr.from_sexpr and run by `execute`, against
the reference executor's outputs, print logs and failure kinds
(tests/golden/vm_*.json) — the same bar as tests/test_gpu_vm.py: f64 within
the reference harness's 1e-9, ints/bools exact; the corpus dynamic_rnn lowers
to the fused fp16 tensor-core kernel (3e-3).  Print logs are compared where
the reference's emitter kept every effect (it drops effects inside frames
whose values are unused, e.g. a Cond kept only for its Print)."""
import json
import os

import pytest

from paper_1810_08061_b200 import LoweringError, RuntimeGraphError, execute, sexpr
from paper_1810_08061_b200.executor import plan_kind
from vm_cases import corpus, feed_value, flatten, fuzz_cases, leaf_equal

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
with open(os.path.join(GOLDEN, "sexpr_cases.json")) as f:
    CASES = json.load(f)["cases"]
SOURCES = {"corpus": {p["name"]: p for p in corpus()}, "fuzz": dict(fuzz_cases())}


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_sexpr_program_on_device(case):
    src = SOURCES[case["source"]][case["key"]]
    g = sexpr.from_sexpr(case["sexpr"])
    feeds = {k: feed_value(v) for k, v in src["feeds"].items()}
    exp = src["expected"]
    if "error" in exp:
        with pytest.raises(RuntimeGraphError) as info:
            execute(g, feeds)
        assert info.value.cause_kind == exp["error"]
        return
    res = execute(g, feeds)
    rel = 3e-3 if plan_kind(g) == "rnn" else 1e-9
    got = flatten(res.outputs)
    assert len(got) == len(exp["outputs"])
    for a, b in zip(got, exp["outputs"]):
        assert leaf_equal(a, b, rel)
    if case["effects_preserved"]:   # else the reference's own emitter dropped an effect (see the generator)
        assert res.print_log == exp["print_log"]
