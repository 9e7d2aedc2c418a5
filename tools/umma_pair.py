"""CTA-pair (cta_group::2, A in TMEM) tcgen05.mma: correctness vs torch and cycles
per instruction vs N, next to the single-CTA TS form (skb_diag_umma_gemm)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_08061_b200 import runtime as rt  # noqa: E402

lib = rt.lib()
dev = torch.device("cuda")
torch.manual_seed(0)
for N in (64, 128, 256):
    K = 512 if N <= 128 else 256
    A = (torch.randn(256, K, device=dev) * 0.1).half()
    B = (torch.randn(N, K, device=dev) * 0.1).half()
    D = torch.zeros(256, N, device=dev)
    D2 = torch.zeros(256, N, device=dev)
    cyc = torch.zeros(1, dtype=torch.int64, device=dev)
    ref = A.float() @ B.float().t()
    rt.check(lib.skb_diag_umma_pair(rt.ptr(A), rt.ptr(B), rt.ptr(D), rt.ptr(D2), N, K, 1, rt.ptr(cyc),
                                    rt.stream_handle()), "pair")
    torch.cuda.synchronize()
    e1 = (D - ref).abs().max().item()
    e2 = (D2 - ref).abs().max().item()
    best = None
    for reps in (8,):
        for _ in range(5):
            rt.check(lib.skb_diag_umma_pair(rt.ptr(A), rt.ptr(B), rt.ptr(D), rt.ptr(D2), N, K, reps,
                                            rt.ptr(cyc), rt.stream_handle()), "pair")
            torch.cuda.synchronize()
            c = int(cyc.item())
            best = c if best is None else min(best, c)
        n_mma = reps * K // 16
        per_sm = 2 * 128 * N * 16
        print(f"pair TS N={N:3d} K={K}: err32x32b {e1:.2e} err16x256b {e2:.2e}; {best / n_mma:.1f} cyc/MMA, "
              f"{per_sm * n_mma / best:.0f} flop/cyc/SM", flush=True)
