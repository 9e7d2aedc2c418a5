"""The region-VM compiler (host side, no GPU): every reference corpus program
and fuzz graph compiles to bytecode; recursive sexpr functions are refused
explicitly (no CPU fallback)."""

import pytest

from paper_1810_08061_b200 import LoweringError, ir
from paper_1810_08061_b200 import vm
from paper_1810_08061_b200.executor import plan_kind
from vm_cases import corpus, fuzz_cases


@pytest.mark.parametrize("prog", corpus(), ids=lambda p: p["name"])
def test_corpus_compiles(prog):
    g = ir.from_json(prog["graph"])
    if prog["name"] == "tree_prod":
        with pytest.raises(LoweringError):
            vm.compile_graph(g)
        return
    p = vm.compile_graph(g)
    assert p.code[-1][0] == vm.OP["HALT"]
    assert len(p.outputs) == len(g.main.outputs)
    if prog["name"] == "dynamic_rnn":
        assert plan_kind(g) == "rnn"      # the fused kernel takes this one
    else:
        assert plan_kind(g) == "vm"


def test_fuzz_graphs_compile():
    cases = fuzz_cases()
    assert len(cases) > 300
    ops = set()
    for name, c in cases:
        g = ir.from_json(c["graph"])
        p = vm.compile_graph(g)
        ops.update(code[0] for code in p.code)
    # loops and branches are exercised
    assert vm.OP["JZ"] in ops and vm.OP["JMP"] in ops and vm.OP["SWAP"] in ops
