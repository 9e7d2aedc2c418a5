"""Per-step / per-tile clock64 trace of cluster 0 at the full C1 bench size."""
import ctypes, sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.fixtures import load_graph_fixture
from paper_1810_08061_b200 import lower, runtime
from paper_1810_08061_b200.executor import RnnExecutable
B, T, F, H = 32, 64, 256, 256
P = int(sys.argv[1]) if len(sys.argv) > 1 else 576
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
tt = torch.zeros(256 * 8, dtype=torch.int64, device=dev)
lib.skb_debug_rnn_trace(ctypes.c_void_p(tr.data_ptr()), 4096)
lib.skb_debug_rnn_tile_trace(ctypes.c_void_p(tt.data_ptr()), 256)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); exe.run(x, h0, c0, lens, out); e1.record(); torch.cuda.synchronize()
print("run ms", e0.elapsed_time(e1))
lib.skb_debug_rnn_trace(None, 0); lib.skb_debug_rnn_tile_trace(None, 0)
a = tr.view(4096, 16).cpu().numpy(); t = tt.view(256, 8).cpu().numpy()
ntile = int((t[:, 0] != 0).sum())
base = t[0, 0]
tot_setup = tot_loop = tot_tail = 0
for i in range(ntile):
    setup = t[i, 1] - t[i, 0]; loop = t[i, 2] - t[i, 1]
    nxt = t[i + 1, 0] if i + 1 < ntile else None
    tail = (nxt - t[i, 2]) if nxt else 0
    tot_setup += setup; tot_loop += loop; tot_tail += tail
    if i < 6 or i == ntile - 1:
        print(f"tile {i}: trip {t[i,3]} setup {setup} loop {loop} ({loop / max(t[i,3],1):.0f}/step) tail {tail}")
print(f"tiles {ntile}: setup {tot_setup} loop {tot_loop} tail {tot_tail} cycles")
sel = slice(1, ntile - 1)
print("setup parts (median): cluster_sync", np.median(t[sel, 4] - t[sel, 0]), "meta+trip", np.median(t[sel, 5] - t[sel, 4]),
      "h0 image", np.median(t[sel, 6] - t[sel, 5]), "fence+sync", np.median(t[sel, 1] - t[sel, 6]))
nsteps = int(t[:ntile, 3].sum()) if ntile else int((a[:, 4] != 0).sum())
names = {11: "epi:hempty ok", 10: "epi:act", 0: "mma:xfull", 1: "mma:dfree", 2: "mma:hfull", 3: "mma:commit", 4: "epi:mdone", 6: "epi:math", 7: "epi:sent", 8: "ld:start", 9: "ld:done"}
d = np.diff(a[:nsteps, 4])
print("steps", nsteps, "median step cycles", np.median(d))
for k in sorted(names):
    print(names[k], "median offset from epi:mdone", np.median(a[2:nsteps - 1, k] - a[2:nsteps - 1, 4]))
