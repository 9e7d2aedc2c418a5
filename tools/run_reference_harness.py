"""Run the reference's own differential harness against skb on the B200.

The reference binds `execute` at module level in its harness
(pkg/src/stagekit/harness/diff.py:20) and uses it for every staged run
(`_run_staged`, :144-164) and for the golden corpus (`_run_corpus_program`,
:337).  This tool rebinds that name to `paper_1810_08061_b200.stagekit_binding
.execute` and runs

  * `diff_seed(seed)` for seeds [0, N) (default 1000) — each seed is a random
    MSL program, 3 input vectors x {concrete, staged_params}; the verdict
    compares native interpretation with the staged graph executed on the GPU;
  * `run_corpus(corpus_dir)` — the 8 golden corpus programs.

Every seed is also run with the reference's own CPU `execute`, and the two
verdicts are compared report by report: skb must reproduce the reference's
verdict (match, or the same failure class) everywhere.

Needs the reference package importable: the unmodified install under
baseline/_ref (bench.py's reference arm; it travels to the GPU box) or
SKB_REF=/path/to/pkg/src.  Usage:

  python tools/run_reference_harness.py [--seeds 1000] [--out gpurun_out/harness.json]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
REF = os.environ.get("SKB_REF") or os.path.join(REPO, "baseline", "_ref")
sys.path.insert(0, REF)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=1000)
    ap.add_argument("--start", type=int, default=0)
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "harness.json"))
    ap.add_argument("--corpus", default=os.path.join(REF, "corpus"))
    args = ap.parse_args()

    os.environ.setdefault("SKB_PRECISION", "f64")   # the harness compares floats at 1e-9 (diff.py:31)
    import stagekit
    import stagekit.harness.diff as diff
    from paper_1810_08061_b200 import executor, stagekit_binding

    ref_execute = diff.execute
    counts_ref, counts_skb = {}, {}
    disagreements, crashes, overflow = [], [], []
    t_ref = t_skb = 0.0
    for seed in range(args.start, args.start + args.seeds):
        diff.execute = ref_execute
        t0 = time.perf_counter()
        ref_reports = diff.diff_seed(seed)
        t_ref += time.perf_counter() - t0
        diff.execute = stagekit_binding.execute
        t0 = time.perf_counter()
        try:
            skb_reports = diff.diff_seed(seed)
        except executor.E.IntegerOverflow as exc:   # Python ints beyond int64: unrepresentable on the device
            overflow.append({"seed": seed, "error": str(exc)[:200]})
            continue
        except Exception as exc:   # anything that is not a reference error class
            crashes.append({"seed": seed, "error": f"{type(exc).__name__}: {exc}"[:300]})
            continue
        finally:
            t_skb += time.perf_counter() - t0
        for r, s in zip(ref_reports, skb_reports):
            counts_ref[r.verdict] = counts_ref.get(r.verdict, 0) + 1
            counts_skb[s.verdict] = counts_skb.get(s.verdict, 0) + 1
            same_detail = r.detail == s.detail
            if r.verdict != s.verdict or not same_detail:
                disagreements.append({"seed": seed, "reference": [r.verdict, r.detail],
                                      "skb": [s.verdict, s.detail]})
    diff.execute = stagekit_binding.execute
    t0 = time.perf_counter()
    corpus = diff.run_corpus(args.corpus) if os.path.isdir(args.corpus) else None
    t_corpus = time.perf_counter() - t0
    summary = {
        "reference": f"stagekit {getattr(stagekit, '__version__', '?')} from {REF}",
        "seam": "stagekit.harness.diff.execute := paper_1810_08061_b200.stagekit_binding.execute",
        "precision": os.environ.get("SKB_PRECISION"),
        "seeds": [args.start, args.start + args.seeds],
        "reports": sum(counts_skb.values()),
        "verdicts_reference_executor": counts_ref,
        "verdicts_skb": counts_skb,
        "disagreements": len(disagreements),
        "disagreement_samples": disagreements[:20],
        "crashes": crashes[:20],
        "n_crashes": len(crashes),
        "int64_overflow_seeds": overflow,
        "seconds_reference_executor": round(t_ref, 1),
        "seconds_skb": round(t_skb, 1),
        "corpus": None if corpus is None else {"total": corpus.total, "passed": corpus.passed,
                                               "failures": corpus.failures, "seconds": round(t_corpus, 1)},
    }
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k not in ("disagreement_samples", "crashes")}))
    ok = not disagreements and not crashes and (corpus is None or corpus.ok)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
