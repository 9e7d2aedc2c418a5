"""Summarise an ncu --csv launch list: per-kernel total/mean time and dram bytes."""
import collections
import csv
import sys


def summarize(path, steps=None):
    hdr, per = None, collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0][-60:]
        v = float(d["Metric Value"].replace(",", ""))
        per[k][d["Metric Name"]] += v
        if d["Metric Name"] == "gpu__time_duration.sum":
            cnt[k] += 1
    tot = sum(m.get("gpu__time_duration.sum", 0) for m in per.values())
    print(f"{'kernel':60s} {'n':>4s} {'mean us':>9s} {'share':>6s} {'MB/launch':>10s}")
    for k, m in sorted(per.items(), key=lambda x: -x[1].get("gpu__time_duration.sum", 0)):
        t = m.get("gpu__time_duration.sum", 0)
        n = max(cnt[k], 1)
        mb = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / n / 1e6
        print(f"{k:60s} {n:4d} {t / n / 1e3:9.1f} {t / tot:6.1%} {mb:10.1f}")


if __name__ == "__main__":
    summarize(sys.argv[1])
