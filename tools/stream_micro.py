"""Bandwidth probes of the vector-stream kernel: one-group loops (dot, axpy,
scale) at n = 1e7, iterations/s -> achieved GB/s of algorithmic traffic."""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import fixtures
from paper_1810_08061_b200 import ir
from paper_1810_08061_b200 import stream as st
from paper_1810_08061_b200.executor import execute_stream

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**7
iters = 200
dev = torch.device("cuda")
x = torch.rand(n, dtype=torch.float64, device=dev)
y = torch.rand(n, dtype=torch.float64, device=dev)
for name, feeds, vecs in (("micro_dot", {"x": x, "y": y}, 2), ("micro_axpy", {"x": x, "y": y}, 3),
                          ("micro_copy", {"x": x}, 2)):
    g = ir.from_json(fixtures.load_golden("graph_" + name)["graph"])
    f = dict(feeds, iters=np.int64(iters))
    execute_stream(g, f)
    ks = []
    for _ in range(3):
        execute_stream(g, f)
        ks.append(st.run.last["kernel_ms"])
    ms = min(ks)
    gbs = vecs * n * 8 * iters / (ms / 1e3) / 1e9
    print(f"{name:11s} n={n:.0e}: {ms / iters * 1e3:8.1f} us/iter  {gbs:7.0f} GB/s  "
          f"(barriers {st.run.last['barriers']}, grid {st.run.last['grid']})")
