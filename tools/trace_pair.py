"""Per-step clock64 trace of lane 0 of CTA 0 (leader of pair 0, cluster 0) of the
pair kernel at the C1 bench size (build with SKB_TRACE=1 SKB_BUILD_OUT=...)."""
import ctypes, sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.fixtures import load_graph_fixture
from paper_1810_08061_b200 import lower, runtime
from paper_1810_08061_b200.executor import RnnExecutable
B, T, F, H = 32, 64, 256, 256
P = int(sys.argv[1]) if len(sys.argv) > 1 else 1152
R = P * B
g, _ = load_graph_fixture()
prog = lower(g)
rng = np.random.default_rng(0)
w = [tuple(rng.uniform(-0.1, 0.1, s) for s in ((F, H), (H, H), (H,))) for _ in range(4)]
exe = RnnExecutable(prog, w, B, T, F, H, P)
dev = torch.device("cuda")
x = torch.rand((R, T, F), device=dev) * 2 - 1
h0 = torch.rand((R, H), device=dev) * 0.2 - 0.1
c0 = torch.rand((R, H), device=dev) * 0.2 - 0.1
lens = torch.randint(1, T + 1, (R,), device=dev)
out = torch.empty((R, T, H), device=dev)
lib = runtime.lib()
for _ in range(3):
    exe.run(x, h0, c0, lens, out)
tr = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
lib.skb_debug_rnn_trace(ctypes.c_void_p(tr.data_ptr()), 4096)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); exe.run(x, h0, c0, lens, out); e1.record(); torch.cuda.synchronize()
print("kernel", lib.skb_rnn_last_kernel(), "clusters", lib.skb_rnn_last_clusters(), "run ms", e0.elapsed_time(e1))
lib.skb_debug_rnn_trace(None, 0)
a = tr.view(4096, 16).cpu().numpy()
n = int((a[:, 4] != 0).sum())
d = np.diff(a[:n, 4])
print("steps", n, "median step cycles", np.median(d), "mean", d.mean())
names = {0: "mma:xfull", 1: "mma:dfree", 2: "mma:hfull", 3: "mma:commit(h)", 4: "epi:mdone", 5: "epi:ld half0",
         10: "epi:ld half1+dfree", 6: "epi:math done", 7: "epi:sent", 8: "epi:x(t+1) done", 9: "epi:out done",
         11: "odd:epi mdone", 12: "odd:epi ld+dfree", 13: "odd:epi sent", 14: "odd:relay hfull", 15: "odd:relay x"}
for k in sorted(names, key=lambda k: np.median(a[2:n - 1, k] - a[2:n - 1, 4])):
    print(f"{names[k]:22s} median offset from epi:mdone {np.median(a[2:n - 1, k] - a[2:n - 1, 4]):8.0f}")
print("next-step mma:hfull - this-step epi:sent", np.median(a[3:n, 2] - a[2:n - 1, 7]))
