"""C1 host-to-host execute_many: wall time per call vs pipeline depth, plus a
cProfile of one call (where the host time goes).  Run on the GPU box."""
import cProfile
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle.fixtures import load_graph_fixture  # noqa: E402
from paper_1810_08061_b200 import executor, execute_many  # noqa: E402

B, T, F, H, P = 32, 64, 256, 256, 576
R = B * P
graph, _ = load_graph_fixture("graph_lstm_c1")
rng = np.random.default_rng(0)
w = {}
for g in "ifgo":
    w["w" + g] = rng.uniform(-0.1, 0.1, (F, H))
    w["u" + g] = rng.uniform(-0.1, 0.1, (H, H))
    w["b" + g] = rng.uniform(-0.1, 0.1, (H,))
hx = (torch.rand((R, T, F)) * 2 - 1).pin_memory()
hh0 = (torch.rand((R, H)) * 0.2 - 0.1).pin_memory()
hc0 = (torch.rand((R, H)) * 0.2 - 0.1).pin_memory()
hl = torch.randint(1, T + 1, (R,)).pin_memory()
feeds = []
for p in range(P):
    rows = slice(p * B, (p + 1) * B)
    f = dict(w)
    f.update(input_data=hx[rows], h0=hh0[rows], c0=hc0[rows], sequence_len=hl[rows])
    feeds.append(f)
host_out = torch.empty(R * T * H, dtype=torch.float32).pin_memory()
for chunks in [int(c) for c in sys.argv[1:]] or [4, 8, 16]:
    executor.PIPELINE_CHUNKS = chunks
    for _ in range(2):
        execute_many(graph, feeds, host_outputs=host_out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        execute_many(graph, feeds, host_outputs=host_out)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print("chunks", chunks, "ms", [round(1e3 * t, 1) for t in ts], flush=True)
pr = cProfile.Profile()
pr.enable()
execute_many(graph, feeds, host_outputs=host_out)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
