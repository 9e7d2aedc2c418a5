"""One micro probe (for ncu): python tools/stream_micro_one.py NAME N ITERS"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from oracle import fixtures
from paper_1810_08061_b200 import ir
from paper_1810_08061_b200.executor import execute_stream

name, n, iters = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
x = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.rand(n, dtype=torch.float64, device="cuda")
g = ir.from_json(fixtures.load_golden("graph_" + name)["graph"])
feeds = {"x": x, "iters": np.int64(iters)}
if name != "micro_copy":
    feeds["y"] = y
execute_stream(g, feeds)
torch.cuda.synchronize()
