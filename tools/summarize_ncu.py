"""Summarise gpurun_out/ ncu artefacts into profiles/ (launch shares, key metrics,
top stall sites) and profiles/ncu_summary.json (read by bench.py for the
roofline `traffic` field)."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "gpurun_out")
PROF = os.path.join(REPO, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"


def launches():
    rows = list(csv.reader(open(os.path.join(OUT, "launches.csv"))))
    hdr, agg = None, defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"]].append(float(d["Metric Value"].replace(",", "")))
    return agg


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(txt.splitlines()))
    return {h: (u, v) for h, u, v in zip(r[0], r[1], r[2])}


def stalls(rep, n=12):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, data = rows[1], rows[2:]
    iS, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
    tot = sum(int(r[iS]) for r in data if r[iS].isdigit()) or 1
    top = sorted((r for r in data if r[iS].isdigit()), key=lambda r: -int(r[iS]))[:n]
    return [(int(r[iS]) / tot, r[iSrc].strip()) for r in top]


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__cluster_max_active", "sm__cycles_elapsed.avg.per_second",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_bytes.sum"]


def main():
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary ({tag})", "", "All numbers from `ncu` runs of `bench.py` on one B200 (gpurun);",
          "ncu times are cold-cache and serialised: compare shares, not absolutes.", ""]
    summary = {}
    agg = launches()
    total = sum(sum(v) / len(v) for v in agg.values() if v)
    md += ["## Launch list (gpu__time_duration, mean per launch)", "", "| kernel | launches | mean µs | share of listed |",
           "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        m = sum(v) / len(v)
        md.append(f"| `{k[:90]}` | {len(v)} | {m / 1e3:.1f} | {m / total:.1%} |")
    for name, rep in (("rnn_fwd_kernel", "prof_rnn.ncu-rep"), ("pack_x_kernel", "prof_pack.ncu-rep")):
        p = os.path.join(OUT, rep)
        if not os.path.exists(p):
            continue
        r = raw(p)
        md += ["", f"## {name} (`ncu --set full`)", "", "| metric | unit | value |", "|---|---|---|"]
        for k in KEYS:
            if k in r:
                md.append(f"| {k} | {r[k][0]} | {r[k][1]} |")

        def num(k, scale):
            u, v = r.get(k, ("", "0"))
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return float(v.replace(",", "")) * mult * scale
        dram = num("dram__bytes_read.sum", 1) + num("dram__bytes_write.sum", 1)
        summary[name] = {"dram_bytes_per_launch": dram, "duration_ms": num("gpu__time_duration.sum", 1),
                         "tensor_pipe_active_pct": num("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1)}
        if name == "rnn_fwd_kernel":
            md += ["", "Top stall sites (share of warp-stall samples):", ""]
            for frac, src in stalls(p):
                md.append(f"- {frac:.1%} `{src[:100]}`")
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as f:
        json.dump(summary, f, indent=1)
    if os.path.exists(os.path.join(OUT, "launches.csv")):
        import shutil
        shutil.copy(os.path.join(OUT, "launches.csv"), os.path.join(PROF, f"{tag}_launches.csv"))
    print("\n".join(md))


if __name__ == "__main__":
    main()
