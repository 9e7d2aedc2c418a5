"""Text feeds and the `skb run` CLI on the CPU: the feed
grammar against the reference's own parser on the same strings (when the
reference is importable), result formatting, and the CLI's exit codes for
usage / staging failures (runtime needs the GPU: tests/test_gpu_cli.py)."""
import os
import sys

import numpy as np
import pytest

from paper_1810_08061_b200 import cli
from paper_1810_08061_b200.feeds import FeedSyntaxError, format_value, parse_feed, parse_param_spec
from paper_1810_08061_b200.values import TensorValue, Tree

GOOD = ["x=f64[2,3]:1.0,2,3.5,-4,5e-3,6", "n=i64:7", "b=bool:true", "v=bool[3]:0,1,False", "s=f64:16.0",
        "e=f64[0]:", "t=tree:(5.0 (3.0 () ()) (2.0 () ()))", "u=tree:()", "w=tree:( 1.5 ()(2 () ()) )",
        "m=i64[2,2]:1, 2, 3, 4"]
BAD = ["x", "1x=f64:1", "x=f32:1", "x=f64[2]:1", "x=f64[2,a]:1,2", "x=bool:maybe", "x=i64:1.5", "x=f64",
       "t=tree:(1.0 ())", "t=tree:(1.0 () () ())", "t=tree:(a () ())", "t=tree:(1.0 () ()) x", "t=tree"]


def _ref_feeds():
    for cand in ("/root/reference/pkg/src", os.path.join(os.path.dirname(os.path.dirname(__file__)), "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "stagekit")):
            sys.path.insert(0, cand)
            try:
                import stagekit.feeds as f
                return f
            except ImportError:
                return None
    return None


@pytest.mark.parametrize("text", GOOD)
def test_good_feeds(text):
    name, v = parse_feed(text)
    ref = _ref_feeds()
    if ref is None:
        return
    rname, rv = ref.parse_feed(text)
    assert name == rname
    if isinstance(v, Tree):
        assert format_value(v) == str(rv)
    else:
        assert v.dtype == rv.dtype and tuple(v.shape) == tuple(rv.shape)
        assert tuple(v.array.reshape(-1).tolist()) == tuple(rv.data)
        assert format_value(v) == (str(rv) if rv.shape != () else rv.__class__.__str__(rv).split(":")[1])


@pytest.mark.parametrize("text", BAD)
def test_bad_feeds(text):
    with pytest.raises(FeedSyntaxError):
        parse_feed(text)
    ref = _ref_feeds()
    if ref is not None:   # (the reference lets int()/float() ValueErrors escape for bad numbers)
        with pytest.raises((ref.FeedSyntaxError, ValueError)):
            ref.parse_feed(text)


def test_param_spec_and_formatting():
    assert parse_param_spec("x=f64[2,3]") == ("x", "f64", (2, 3))
    with pytest.raises(FeedSyntaxError):
        parse_param_spec("x=f64[2]:1,2")
    assert format_value(TensorValue("f64", (), [16.0])) == "16.0"
    assert format_value(TensorValue("i64", (2,), [1, -2])) == "i64[2]:1,-2"
    assert format_value(TensorValue("bool", (), [True])) == "True"
    assert format_value(Tree(1.0, Tree(), Tree())) == "(1.0 () ())"


def test_cli_usage_and_staging_exit_codes(tmp_path, capsys):
    g = tmp_path / "p.sexpr"
    g.write_text("(def main ((x f64)) (add x x))")
    with pytest.raises(SystemExit) as e:
        cli.main(["run"])                       # missing file -> usage
    assert e.value.code == 1
    assert cli.main(["run", str(g), "--feed", "x=f64:abc"]) == 3   # feed syntax -> staging
    assert "staging" in capsys.readouterr().err
    assert cli.main(["run", str(tmp_path / "missing.sexpr")]) == 1
