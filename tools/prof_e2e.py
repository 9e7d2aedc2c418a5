"""cProfile of one host-to-host execute_many call at the C1 bench size."""
import cProfile
import pstats
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle.fixtures import load_graph_fixture
from paper_1810_08061_b200 import execute_many

B, T, F, H, P = 32, 64, 256, 256, 576
graph, _ = load_graph_fixture("graph_lstm_c1")
rng = np.random.default_rng(0)
w = {}
for g in "ifgo":
    w["w" + g] = rng.uniform(-0.1, 0.1, (F, H))
    w["u" + g] = rng.uniform(-0.1, 0.1, (H, H))
    w["b" + g] = rng.uniform(-0.1, 0.1, (H,))
R = B * P
hx = torch.rand((R, T, F)).pin_memory()
hh = (torch.rand((R, H)) * 0.1).pin_memory()
hc = (torch.rand((R, H)) * 0.1).pin_memory()
hl = torch.randint(1, T + 1, (R,)).pin_memory()
feeds = []
for p in range(P):
    rows = slice(p * B, (p + 1) * B)
    f = dict(w)
    f.update(input_data=hx[rows], h0=hh[rows], c0=hc[rows], sequence_len=hl[rows])
    feeds.append(f)
out = torch.empty(R * T * H).pin_memory()
for _ in range(2):
    execute_many(graph, feeds, host_outputs=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
execute_many(graph, feeds, host_outputs=out)
print("wall", time.perf_counter() - t0)
pr = cProfile.Profile()
pr.enable()
execute_many(graph, feeds, host_outputs=out)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
