"""First-contact GPU probe: tcgen05 descriptor convention, DSMEM exchange cost,
and the fused LSTM/RNN kernel against a numpy float64 restatement."""
import ctypes, os, sys, time
import numpy as np
import torch

lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "..", "paper_1810_08061_b200", "libskb.so"))
dev = torch.device("cuda:0")
st = torch.cuda.current_stream().cuda_stream
print("sm count", lib.skb_device_sm_count())

# --- umma gemm
for N in ():
    for K in (64, 512):
        A = torch.randn(128, K, device=dev).half()
        B = torch.randn(N, K, device=dev).half()
        ref = A.float() @ B.float().T
        for swap in (0, 2):
            D = torch.zeros(128, N, device=dev)
            cyc = torch.zeros(1, dtype=torch.int64, device=dev)
            rc = lib.skb_diag_umma_gemm(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                        ctypes.c_void_p(D.data_ptr()), N, K, swap,
                                        ctypes.c_void_p(cyc.data_ptr()), ctypes.c_void_p(st))
            torch.cuda.synchronize()
            err = (D - ref).abs().max().item()
            print(f"umma N={N} K={K} swap={swap} rc={rc} maxerr={err:.3e} cycles={cyc.item()}")

# --- cluster exchange
gs = torch.zeros(1 << 22, dtype=torch.uint8, device=dev)
for C in ():
  for via in (None, gs):
    for sb in (2048, 4096):
        cyc = torch.zeros(1, dtype=torch.int64, device=dev)
        errs = torch.zeros(1, dtype=torch.int32, device=dev)
        rounds = 2000
        rc = lib.skb_diag_cluster_exchange(C, sb, rounds, ctypes.c_void_p(cyc.data_ptr()),
                                           ctypes.c_void_p(errs.data_ptr()), None if via is None else ctypes.c_void_p(via.data_ptr()), ctypes.c_void_p(st))
        torch.cuda.synchronize()
        print(f"exchange via_l2={via is not None} C={C} slice={sb} rc={rc} cycles/round={cyc.item()/rounds:.0f} errors={errs.item()}")

# --- rnn forward
class Shape(ctypes.Structure):
    _fields_ = [("cell", ctypes.c_int32), ("hidden", ctypes.c_int32), ("input", ctypes.c_int32),
                ("time", ctypes.c_int32), ("rows_per_problem", ctypes.c_int32), ("problems", ctypes.c_int32)]
lib.skb_rnn_packed_bytes.restype = ctypes.c_int64
lib.skb_rnn_workspace_bytes.restype = ctypes.c_int64

def sig(x):
    return np.where(x >= 0, 1.0 / (1.0 + np.exp(-np.abs(x))), np.exp(-np.abs(x)) / (1.0 + np.exp(-np.abs(x))))

def ref_lstm(x, h0, c0, lens, W, Uw, b, cell):
    B, T, F = x.shape
    m = int(lens.max())
    h, c = h0.copy(), c0.copy()
    outs = []
    for t in range(m):
        xt = x[:, t, :]
        if cell == 1:
            z = [xt @ W[g] + h @ Uw[g] + b[g] for g in range(4)]
            i, f, gg, o = sig(z[0]), sig(z[1]), np.tanh(z[2]), sig(z[3])
            c2 = f * c + i * gg
            h2 = o * np.tanh(c2)
        else:
            h2 = np.tanh(xt @ W[0] + h @ Uw[0] + b[0]); c2 = c
        mask = (t < lens)[:, None]
        h = np.where(mask, h2, h); c = np.where(mask, c2, c)
        outs.append(h)
    return np.stack(outs, 1)

def run(cell, B, T, F, H, P, seed=0, ctrl=None):
    rng = np.random.default_rng(seed)
    G = 4 if cell == 1 else 1
    R = B * P
    x = rng.uniform(-1, 1, (R, T, F))
    h0 = rng.uniform(-0.1, 0.1, (R, H)); c0 = rng.uniform(-0.1, 0.1, (R, H))
    lens = rng.integers(1, T + 1, R).astype(np.int64) if ctrl is None else ctrl
    W = [rng.uniform(-0.1, 0.1, (F, H)) for _ in range(G)]
    Uw = [rng.uniform(-0.1, 0.1, (H, H)) for _ in range(G)]
    b = [rng.uniform(-0.1, 0.1, (H,)) for _ in range(G)]
    shp = Shape(cell, H, F, T, B, P)
    tw = [torch.tensor(a, device=dev) for a in W]; tu = [torch.tensor(a, device=dev) for a in Uw]; tb = [torch.tensor(a, device=dev) for a in b]
    arr = ctypes.c_void_p * 4
    wp = arr(*[t.data_ptr() for t in tw]); up = arr(*[t.data_ptr() for t in tu]); bp = arr(*[t.data_ptr() for t in tb])
    packed = torch.zeros(lib.skb_rnn_packed_bytes(ctypes.byref(shp)), dtype=torch.uint8, device=dev)
    err = torch.zeros(4, dtype=torch.int32, device=dev)
    rc = lib.skb_rnn_pack(ctypes.byref(shp), wp, up, bp, 1, ctypes.c_void_p(packed.data_ptr()), ctypes.c_void_p(err.data_ptr()), ctypes.c_void_p(st))
    xd = torch.tensor(x, device=dev, dtype=torch.float32)
    h0d = torch.tensor(h0, device=dev, dtype=torch.float32); c0d = torch.tensor(c0, device=dev, dtype=torch.float32)
    ld = torch.tensor(lens, device=dev)
    out = torch.full((R, T, H), float("nan"), device=dev)
    ml = torch.zeros(P, dtype=torch.int32, device=dev)
    ws = torch.zeros(lib.skb_rnn_workspace_bytes(ctypes.byref(shp)), dtype=torch.uint8, device=dev)
    def go():
        return lib.skb_rnn_forward(ctypes.byref(shp), ctypes.c_void_p(packed.data_ptr()), ctypes.c_void_p(xd.data_ptr()), 0,
                             ctypes.c_void_p(h0d.data_ptr()), ctypes.c_void_p(c0d.data_ptr()), ctypes.c_void_p(ld.data_ptr()),
                             ctypes.c_void_p(out.data_ptr()), None, None, ctypes.c_void_p(ml.data_ptr()), ctypes.c_void_p(err.data_ptr()),
                             ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(st))
    rc2 = go()
    torch.cuda.synchronize()
    o = out.cpu().numpy(); mls = ml.cpu().numpy()
    maxerr = 0.0
    nprob = min(P, 4)
    for p in range(nprob):
        sl = slice(p * B, (p + 1) * B)
        ref = ref_lstm(x[sl], h0[sl], c0[sl], lens[sl], W, Uw, b, cell)
        got = o[sl, :mls[p], :]
        assert got.shape == ref.shape, (got.shape, ref.shape)
        maxerr = max(maxerr, float(np.abs(got - ref).max()))
    # timing
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    for _ in range(3): go()
    t0.record()
    n = 10
    for _ in range(n): go()
    t1.record(); torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / n
    print(f"cell={cell} B={B} T={T} F={F} H={H} P={P} rc={rc},{rc2} err={err.cpu().tolist()} max_len={mls[:4]} maxabs={maxerr:.3e} ms={ms:.3f} ex/s={R/ms*1e3:.3e}")

run(2, 2, 3, 4, 4, 1, ctrl=np.array([3, 1]))
run(2, 32, 16, 64, 64, 2)
run(1, 4, 8, 16, 16, 1)
run(1, 32, 64, 256, 256, 1)
run(1, 32, 64, 256, 256, 4)
run(1, 32, 64, 256, 256, 576)
for H in (256,):
    shp = Shape(1, H, 256, 64, 32, 576)
    c = ctypes.c_int32(); cc = ctypes.c_int32(); tr = ctypes.c_int32()
    print("plan", lib.skb_rnn_plan(ctypes.byref(shp), ctypes.byref(c), ctypes.byref(cc), ctypes.byref(tr)), c.value, cc.value, tr.value)
# ---- trace one problem
tr = torch.zeros(64 * 16, dtype=torch.int64, device=dev)
lib.skb_debug_rnn_trace(ctypes.c_void_p(tr.data_ptr()), 64)
run(1, 32, 64, 256, 256, 1)
torch.cuda.synchronize()
a = tr.view(64, 16).cpu().numpy()
base = a[0, 8]
names = {10: "epi:act", 0: "mma:xfull", 1: "mma:dfree", 2: "mma:hfull", 3: "mma:commit", 4: "epi:mdone", 5: "epi:ld", 6: "epi:math", 7: "epi:sent", 8: "ld:start", 9: "ld:done"}
for s in range(0, 64, 8):
    print(s, " ".join(f"{names[k]}={a[s,k]-base}" for k in range(10)))
d = np.diff(a[1:60, 4])
print("per-step cycles (epi mdone->mdone): median", np.median(d))
for k in range(11):
    print(names[k], "median offset from epi:mdone", np.median(a[2:60, k] - a[2:60, 4]))
lib.skb_debug_rnn_trace(None, 0)
