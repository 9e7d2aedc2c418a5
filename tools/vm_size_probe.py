"""Region-VM gradient-through-While vs the float64 BPTT restatement at growing
shapes (the traced 4x3 LSTM-loss graph with its parameter shapes relaxed)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from autodiff_cases import load  # noqa: E402
from oracle import bptt  # noqa: E402
from paper_1810_08061_b200 import gradient  # noqa: E402
from paper_1810_08061_b200.executor import execute_vm  # noqa: E402
from paper_1810_08061_b200.ir import TypeSpec  # noqa: E402

d = load("ad_lstm_4x3")
g = d["graph_obj"]
def relax(t):
    if t is None:
        return t
    if t.dtype == "list":
        return TypeSpec("list", None, relax(t.elem))
    if t.shape in ((), None):
        return t
    return TypeSpec(t.dtype, tuple(None for _ in t.shape))


for n in g.iter_nodes():
    n.out_types = [relax(t) for t in n.out_types]
wrt = d["wrt"]
gg = gradient(g, 0, wrt)


def feeds_for(T, B, F, H, seed=0):
    rng = np.random.default_rng(seed)
    v = {"x": rng.uniform(-1, 1, (T, B, F)), "h0": rng.uniform(-.5, .5, (B, H)), "c0": rng.uniform(-.5, .5, (B, H)),
         "lens": rng.integers(0, T + 1, B).astype(np.int64), "y": rng.uniform(-1, 1, (T, B, H))}
    v["lens"][0] = T
    for q in "ifgo":
        v["w" + q] = rng.uniform(-1, 1, (F, H))
        v["u" + q] = rng.uniform(-1, 1, (H, H))
        v["b" + q] = np.broadcast_to(rng.uniform(-.5, .5, (1, H)), (B, H)).copy()
    v["inv_b"] = np.float64(1.0 / B)
    return v


SIZES = [(4, 3, 3, 4), (8, 8, 8, 8), (16, 32, 64, 64)] if len(sys.argv) < 2 else \
    [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
for (T, B, F, H) in SIZES:
    v = feeds_for(T, B, F, H)
    fwd = execute_vm(g, v)
    res = execute_vm(gg, v)
    W = np.concatenate([v["w" + q] for q in "ifgo"], axis=1)
    U = np.concatenate([v["u" + q] for q in "ifgo"], axis=1)
    b = np.concatenate([v["b" + q][0] for q in "ifgo"])
    ref = bptt.forward_backward(np.transpose(v["x"], (1, 0, 2)), v["h0"], v["c0"], v["lens"],
                                np.transpose(v["y"], (1, 0, 2)), W, U, b, float(v["inv_b"]))
    outs = [np.asarray(o.array) for o in res.outputs]
    errs = []
    for k, q in enumerate("ifgo"):
        errs.append(float(np.max(np.abs(outs[1 + 3 * k] - ref[1][:, k * H:(k + 1) * H]))))   # dW_q
        errs.append(float(np.max(np.abs(outs[2 + 3 * k] - ref[2][:, k * H:(k + 1) * H]))))   # dU_q
    print((T, B, F, H), "fwd-only loss err", abs(float(np.asarray(fwd.outputs[0].array).reshape(-1)[0]) - ref[0]),
          "grad-graph loss err", abs(float(outs[0].reshape(-1)[0]) - ref[0]), "max dW/dU err", max(errs))
