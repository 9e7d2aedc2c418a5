"""Per-step timeline of the C2 forward step kernel (CTA 0), SKB_TC_TRACE=1 build-free trace:
where the ~18 us per timestep go."""
import ctypes
import os
import sys

os.environ["SKB_TC_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
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
names = ["start", "barrier passed", "first stage full", "last MMA issued", "TMEM full (epi)",
         "operands ready", "epilogue done", "published"]
for which, title in ((0, "forward"), (1, "backward")):
    buf = np.zeros((T, 8), dtype=np.int64)
    n = tr.lib.skb_train_tc_trace(ctypes.c_void_p(buf.ctypes.data), T, which)
    assert n == T, n
    d = np.diff(buf[16:T - 16], axis=1) / 1e3
    print(f"{title} step kernel: per-step phase durations (us), CTA 0, steps 16..T-16, mean / median:")
    for i in range(7):
        print(f"  {names[i]:>18s} -> {names[i + 1]:<18s} {d[:, i].mean():7.2f} {np.median(d[:, i]):7.2f}")
    step = np.abs(np.diff(buf[16:T - 16, 1])) / 1e3
    print(f"  step period {step.mean():.2f} us")
