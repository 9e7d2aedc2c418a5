"""The region-VM compiler (host side, no GPU): every reference corpus program
and fuzz graph compiles to bytecode; recursive sexpr functions are refused
out of line and called through the device call stack (CALL / RET)."""

import pytest

from paper_1810_08061_b200 import LoweringError, ir
from paper_1810_08061_b200 import vm
from paper_1810_08061_b200.executor import plan_kind
from vm_cases import corpus, fuzz_cases


@pytest.mark.parametrize("prog", corpus(), ids=lambda p: p["name"])
def test_corpus_compiles(prog):
    g = ir.from_json(prog["graph"])
    p = vm.compile_graph(g)
    if prog["name"] == "tree_prod":   # recursive: main, HALT, then the function body ending in RET
        ops = [c[0] for c in p.code]
        assert vm.OP["CALL"] in ops and ops[-1] == vm.OP["RET"] and vm.OP["HALT"] in ops
        assert vm._recursive_functions(g) == {"tree_prod"}
    else:
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


@pytest.mark.parametrize("prog", __import__("vm_cases").recursion(), ids=lambda p: p["name"])
def test_recursive_programs_compile_to_call_ret(prog):
    """Recursive functions (reference sexpr backend) become out-of-line bodies
    reached by CALL; every call site is patched with its entry and range."""
    g = ir.from_json(prog["graph"])
    p = vm.compile_graph(g)
    rec = vm._recursive_functions(g)
    assert rec
    calls = [c for c in p.code if c[0] == vm.OP["CALL"]]
    assert calls and all(c[2] > 0 and c[4] < c[5] for c in calls)   # entry after HALT, lo < hi
    halt = [i for i, c in enumerate(p.code) if c[0] == vm.OP["HALT"]]
    assert all(c[2] > halt[0] for c in calls)
