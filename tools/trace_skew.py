"""Backward step kernel: when does each CTA of cluster 0 see its accumulator complete, and when
has its partners' partial sums (SKB_TC_TRACE_CTA selects the traced CTA; the globaltimer is
global, so the stamps compare across runs of the same deterministic schedule only loosely --
the per-step offsets relative to the same step's barrier pass are compared instead)."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, ".")
os.environ["SKB_TC_TRACE"] = "1"
import torch  # noqa: E402

from paper_1810_08061_b200.train import LstmTrainer  # noqa: E402

ROWS, T, F, H = 512, 512, 1024, 1024
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
x = torch.rand((ROWS, T, F), device=dev, generator=g) * 2 - 1
y = torch.rand((ROWS, T, H), device=dev, generator=g) * 2 - 1
lens = torch.full((ROWS,), T, dtype=torch.int64, device=dev)
tr = LstmTrainer(F, H, ROWS, T, global_batch=ROWS, lr=0.0, math="bf16", seed=1, device=dev, graph=False)
for _ in range(2):
    tr.forward_backward(x, y, lens)
torch.cuda.synchronize()
buf = np.zeros((T, 8), dtype=np.int64)
n = tr.lib.skb_train_tc_trace(ctypes.c_void_p(buf.ctypes.data), T, 1)
np.save(f"gpurun_out/bwd_trace_cta{os.environ.get('SKB_TC_TRACE_CTA', '0')}.npy", buf)
d = np.diff(buf[16:T - 16], axis=1) / 1e3
print("CTA", os.environ.get("SKB_TC_TRACE_CTA", "0"), "mean phase us:", np.round(d.mean(axis=0), 2))
