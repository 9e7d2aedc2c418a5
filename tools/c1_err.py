"""C1-size accuracy probe: the fused kernel vs the float64 C oracle on P
problems of the bench shape (B=32, T=64, F=H=256, weights U(-0.1,0.1)),
error = max |gpu - ref| / max(1, |gpu|, |ref|) (the parity tests' metric)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from oracle.fixtures import load_graph_fixture  # noqa: E402
from paper_1810_08061_b200 import lower  # noqa: E402
from paper_1810_08061_b200.executor import RnnExecutable  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
H = int(sys.argv[3]) if len(sys.argv) > 3 else 256
B, T, F = 32, 64, H
R = P * B
g, _ = load_graph_fixture("graph_lstm_c1")
prog = lower(g)
rng = np.random.default_rng(7)
W = [rng.uniform(-scale, scale, (F, H)) for _ in range(4)]
U = [rng.uniform(-scale, scale, (H, H)) for _ in range(4)]
b = [rng.uniform(-scale, scale, (H,)) for _ in range(4)]
x = rng.uniform(-1, 1, (R, T, F))
h0 = rng.uniform(-0.1, 0.1, (R, H))
c0 = rng.uniform(-0.1, 0.1, (R, H))
lens = rng.integers(1, T + 1, R).astype(np.int64)
exe = RnnExecutable(prog, [(W[i], U[i], b[i]) for i in range(4)], B, T, F, H, P)
dev = torch.device("cuda")
out = torch.empty((R, T, H), device=dev)
exe.run(torch.tensor(x, dtype=torch.float32, device=dev), torch.tensor(h0, dtype=torch.float32, device=dev),
        torch.tensor(c0, dtype=torch.float32, device=dev), torch.tensor(lens, device=dev), out)
torch.cuda.synchronize()
ref, ml, st = oracle.rnn_many(1, x, h0, c0, lens, W, U, b, P, 16)
got = out.cpu().numpy().astype(np.float64)
errs = []
for p in range(P):
    m = int(ml[p])
    a, r = got[p * B:(p + 1) * B, :m], ref.reshape(P, B * T * H)[p, :B * m * H].reshape(B, m, H)
    errs.append(float(np.max(np.abs(a - r) / np.maximum(1, np.maximum(np.abs(a), np.abs(r))))))
print(f"H={H} act={os.environ.get('SKB_RNN_ACT', '1 (default)')} scale={scale} max rel err {max(errs):.3e} mean {np.mean(errs):.3e}")
