"""tcgen05.mma cost per instruction vs N (one CTA, K/16 chained MMAs, TS and SS
forms) via skb_diag_umma_gemm's clock64 bracket."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_08061_b200 import runtime as rt  # noqa: E402

lib = rt.lib()
dev = torch.device("cuda")
for mode, name in ((2, "TS (A in TMEM)"), (0, "SS")):
    for N in (32, 64, 128, 256):
        K = 512 if (128 + N) * 512 * 2 <= 200 * 1024 else 256
        A = torch.randn(128, K, device=dev).half()
        B = torch.randn(N, K, device=dev).half()
        D = torch.empty(128, N, device=dev)
        cyc = torch.zeros(1, dtype=torch.int64, device=dev)
        best = None
        for _ in range(5):
            rt.check(lib.skb_diag_umma_gemm(rt.ptr(A), rt.ptr(B), rt.ptr(D), N, K, mode, rt.ptr(cyc),
                                            rt.stream_handle()), "umma")
            torch.cuda.synchronize()
            c = int(cyc.item())
            best = c if best is None else min(best, c)
        n_mma = K // 16
        flop = 2 * 128 * N * 16
        print(f"{name:16s} N={N:3d} K={K}: {best} cycles for {n_mma} MMAs = {best / n_mma:.1f} cyc/MMA, "
              f"{flop * n_mma / best:.0f} flop/cyc/SM")
