"""`skb run` on the GPU: the corpus programs' reference-rendered graphs with
text feeds, printed results equal to the reference CLI's output format;
runtime failures exit 4 with a file:line:col diagnostic."""
import json
import os

import pytest

from paper_1810_08061_b200 import cli

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_run_sexpr_program_with_text_feeds(tmp_path, capsys):
    g = tmp_path / "while_halve.sexpr"
    cases = json.load(open(os.path.join(GOLDEN, "sexpr_cases.json")))
    src = next(c for c in cases["cases"] if c["key"] == "while_halve")
    g.write_text(src["sexpr"])
    assert cli.main(["run", str(g), "--feed", "x=f64:16.0"]) == 0
    assert capsys.readouterr().out.strip() == "1.0"   # the reference executor's result (vm_corpus.json)


def test_run_tree_program(tmp_path, capsys):
    g = tmp_path / "tree_prod.sexpr"
    g.write_text("(def tree_prod ((base f64) (tree tree)) (cond (not (tree_is_empty tree)) (then (mul (mul "
                 "(call tree_prod base (tree_left tree)) (call tree_prod base (tree_right tree))) "
                 "(tree_value tree))) (else base)))\n(def main ((base f64) (tree tree)) (call tree_prod base tree))")
    assert cli.main(["run", str(g), "--feed", "base=f64:2.0", "--feed", "tree=tree:(5.0 (3.0 () ()) (2.0 () ()))"]) == 0
    assert capsys.readouterr().out.strip() == "480.0"   # 5 * (2*2*3) * (2*2*2)


def test_runtime_failure_exit_code(tmp_path, capsys):
    g = tmp_path / "div.sexpr"
    g.write_text("(def main ((x f64)) (div x (const f64 0.0)))")
    assert cli.main(["run", str(g), "--feed", "x=f64:1.0"]) == 4
    assert ": runtime: " in capsys.readouterr().err
