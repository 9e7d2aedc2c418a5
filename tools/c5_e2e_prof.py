"""Where the C5 end-to-end step's host time goes (cProfile of Forest + tree_lstm + readback)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from benchmarks import c5  # noqa: E402
from oracle import fixtures  # noqa: E402
from paper_1810_08061_b200.tree import Forest, pack_weights, tree_lstm  # noqa: E402

dev = torch.device("cuda")
trees = c5._forest(1)
pw = pack_weights(fixtures.tree_weights(c5.H, 5), dev)
for _ in range(4):
    hh, cc = tree_lstm(Forest(trees), None, math="tf32", packed=pw)
    hh.tensor.cpu()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    hh, cc = tree_lstm(Forest(trees), None, math="tf32", packed=pw)
    hh.tensor.cpu()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
