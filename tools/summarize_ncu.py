"""Summarise gpurun_out/ ncu artefacts into profiles/ (per-config launch shares,
key metrics and top stall sites of each config's own dominant kernel) and
profiles/ncu_summary.json (read by the bench legs for the roofline `traffic`
field: DRAM bytes per launch of the profiled kernel)."""
import csv
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

CONFIGS = [("c1", "C1 dynamic-length LSTM inference (headline)"), ("c2", "C2 LSTM training step"),
           ("c3", "C3 beam-search decoder"), ("c4", "C4 L-BFGS (vector-stream tier)"),
           ("c5", "C5 TreeLSTM"), ("c5m", "C5 MAML")]
CAPTURES = [("rnn_fwd_pair4_kernel", "prof_rnn.ncu-rep", "C1: bench.py --steps 1 --warmup 1 (launch 2)"),
            ("gemm_steps_kernel<EpiBwd>", "prof_c2bwd.ncu-rep", "C2: bench.py --config c2, backward persistent step kernel"),
            ("gemm_steps_kernel<EpiFwd>", "prof_c2fwd.ncu-rep", "C2: bench.py --config c2, forward persistent step kernel"),
            ("stream_kernel", "prof_stream.ncu-rep", "C4 tier: axpy probe n=1e7 x 20 (tools/stream_micro_one.py)"),
            ("beam_rows", "prof_beam_rows.ncu-rep", "C3: bench.py --config c3"),
            ("tree_cell", "prof_tree_cell.ncu-rep", "C5: bench.py --config c5"),
            ("maml_task_kernel", "prof_maml.ncu-rep", "C5 MAML: bench.py --config c5m")]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_max_active",
        "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, defaultdict(lambda: defaultdict(list))
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"]][d.get("Metric Name", "gpu__time_duration.sum")].append(
                float(d["Metric Value"].replace(",", "")))
    return agg


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def stalls(rep, n=8):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    k = next(i for i, r in enumerate(rows) if "Source" in r)
    hdr, data = rows[k], rows[k + 1:]
    iS, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    num = lambda x: float(x) if x.replace(".", "", 1).isdigit() else 0.0
    tot = sum(num(r[iS]) for r in data) or 1
    top = sorted(data, key=lambda r: -num(r[iS]))[:n]
    return [(num(r[iS]) / tot, r[iSrc].strip()) for r in top]


def scaled(r, k):
    u, v = r.get(k, ("", "0"))
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3,
            "msecond": 1.0, "second": 1e3}.get(u, 1)
    return float(v.replace(",", "")) * mult


def main():
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary ({tag})", "",
          "All numbers from `ncu` runs on one B200 via gpurun (`tools/gpu_profiles.sh`); ncu times are",
          "cold-cache and serialised: compare kernel shares, not absolutes (bench lines are the timings).", ""]
    summary = {}
    for cfg, title in CONFIGS:
        p = os.path.join(OUT, f"launches_{cfg}.csv")
        if not os.path.exists(p):
            continue
        shutil.copy(p, os.path.join(PROF, f"{tag}_launches_{cfg}.csv"))
        agg = launches(p)
        t = {k: v["gpu__time_duration.sum"] for k, v in agg.items() if v.get("gpu__time_duration.sum")}
        total = sum(sum(v) for v in t.values()) or 1
        md += [f"## {title}: launch list", "", "| kernel | launches | mean µs | DRAM MB / launch | share of GPU time |",
               "|---|---|---|---|---|"]
        for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1]))[:12]:
            rd = agg[k].get("dram__bytes_read.sum", [0])
            wr = agg[k].get("dram__bytes_write.sum", [0])
            dram = (sum(rd) / len(rd) + sum(wr) / len(wr)) / 1e6
            md.append(f"| `{k[:80]}` | {len(v)} | {sum(v) / len(v) / 1e3:.1f} | {dram:.1f} | {sum(v) / total:.1%} |")
        md.append("")
    for name, rep, what in CAPTURES:
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        r = raw(p)
        md += [f"## `{name}` — `ncu --set full` ({what})", "", "| metric | unit | value |", "|---|---|---|"]
        for k in KEYS:
            if k in r:
                md.append(f"| {k} | {r[k][0]} | {r[k][1]} |")
        dram = scaled(r, "dram__bytes_read.sum") + scaled(r, "dram__bytes_write.sum")
        summary[name] = {"dram_bytes_per_launch": dram, "duration_ms": scaled(r, "gpu__time_duration.sum"),
                         "capture": what}
        try:
            md += ["", "Top stall sites (share of warp-stall samples):", ""]
            for frac, src in stalls(p):
                md.append(f"- {frac:.1%} `{src[:100]}`")
        except Exception:
            pass
        md.append("")
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    path = os.path.join(PROF, "ncu_summary.json")
    old = json.load(open(path)) if os.path.exists(path) else {}
    commit = subprocess.run(["git", "rev-parse", "--short", "HEAD"], capture_output=True, text=True,
                            cwd=REPO).stdout.strip()
    for k, v in summary.items():
        v["commit"] = commit
        if k == "rnn_fwd_pair4_kernel":
            v["problems"] = 1152
        old[k] = v
    with open(path, "w") as f:
        json.dump(old, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
