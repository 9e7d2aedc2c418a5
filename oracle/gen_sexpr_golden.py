"""tests/golden/sexpr_cases.json: the reference's own s-expression rendering
(stagekit.graph.sexpr.to_sexpr, graph/sexpr.py:43-155) of every region-VM
golden program (corpus + differential-fuzz graphs traced by the reference),
so the s-expression reader (paper_1810_08061_b200/sexpr.py) is tested on
text the reference produced.  Run in the build container:
    python oracle/gen_sexpr_golden.py
Test infrastructure only."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from oracle.gen_autodiff_golden import to_reference  # noqa: E402
from paper_1810_08061_b200 import ir, sexpr  # noqa: E402

GOLDEN = os.path.join(REPO, "tests", "golden")


def main():
    from stagekit.graph.sexpr import to_sexpr
    cases = []
    with open(os.path.join(GOLDEN, "vm_corpus.json")) as f:
        corpus = json.load(f)["programs"]
    ref_dir = "/root/reference/pkg/corpus/golden"
    for p in corpus:
        text = to_sexpr(to_reference(ir.from_json(p["graph"])))
        shipped = os.path.join(ref_dir, p["name"] + ".sexpr")
        same = open(shipped).read().strip() == text.strip() if os.path.exists(shipped) else None
        cases.append({"name": "corpus-" + p["name"], "source": "corpus", "key": p["name"], "sexpr": text,
                      "matches_reference_corpus_file": same, "effects_preserved": True})
        print(p["name"], "matches corpus/golden file:", same)
    with open(os.path.join(GOLDEN, "vm_fuzz.json")) as f:
        seeds = json.load(f)["seeds"]
    for s in seeds:
        for c in s["cases"]:
            if "graph" not in c:
                continue
            key = f"seed{s['seed']}-v{c['vector']}-{c['mode']}"
            try:
                text = to_sexpr(to_reference(ir.from_json(c["graph"])))
            except Exception as exc:   # a graph the emitter cannot render
                print("skip", key, type(exc).__name__, exc)
                continue
            g = ir.from_json(c["graph"])
            # the reference emitter drops effects inside frames whose values are unused
            # (e.g. a Cond kept only for its Print): record whether every effect survived
            n_eff = sum(1 for n in g.iter_nodes() if n.op in ("Print", "Assert"))
            n_read = sum(1 for n in sexpr.from_sexpr(text).iter_nodes() if n.op in ("Print", "Assert"))
            cases.append({"name": "fuzz-" + key, "source": "fuzz", "key": key, "sexpr": text,
                          "effects_preserved": n_eff == n_read})
    with open(os.path.join(GOLDEN, "sexpr_cases.json"), "w") as f:
        json.dump({"generator": "oracle/gen_sexpr_golden.py", "cases": cases}, f, separators=(",", ":"))
    print(len(cases), "cases;", sum(not c["effects_preserved"] for c in cases), "lose effects in the reference emitter")


if __name__ == "__main__":
    main()
