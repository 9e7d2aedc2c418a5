"""C4 stream kernel phase split (CTA 0 clock64 totals: scalar interpreter,
reduction waits, vector groups) — needs a SKB_TRACE=1 build via SKB_LIB_PATH."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import fixtures  # noqa: E402
from paper_1810_08061_b200 import execute, ir  # noqa: E402
from paper_1810_08061_b200 import stream as st  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10**7
g = ir.from_json(fixtures.load_golden("graph_lbfgs_c4")["graph"])
rng = np.random.default_rng(100)
dev = torch.device("cuda")
feeds = {"x0": torch.from_numpy(rng.uniform(-1, 1, n)).to(dev), "a": torch.from_numpy(rng.uniform(0.5, 4, n)).to(dev),
         "b": torch.from_numpy(rng.uniform(-1, 1, n)).to(dev), "tol": np.float64(1e-18), "max_iter": np.int64(100)}
for _ in range(2):
    res = execute(g, feeds)
last = st.run.last
cyc = last["cycles_cta0"]
tot = sum(cyc.values())
clk = 1.965e9
print(f"kernel {last['kernel_ms']:.2f} ms, iterations {int(res.outputs[1].item())}, barriers {last['barriers']}")
for k, v in cyc.items():
    print(f"  {k:10s} {v / clk * 1e3:8.2f} ms ({v / max(tot, 1):.1%})")
