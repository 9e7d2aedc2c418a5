"""Per-launch time of small skb_gemm problems (the C2 per-step GEMM shapes) with the
launches captured in a CUDA graph (no host launch overhead in the timing)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_08061_b200 import runtime  # noqa: E402

lib = runtime.lib()


def probe(name, M, N, K, bn, a_rows_stride=None, reps=200):
    A = torch.randn((M, a_rows_stride or K), device="cuda").to(torch.bfloat16)
    B = torch.randn((N, K), device="cuda").to(torch.bfloat16)
    C = torch.empty((M, N), device="cuda")
    s = torch.cuda.Stream()

    def go():
        rc = lib.skb_gemm(0, 0, 0, M, N, K, ctypes.c_void_p(A.data_ptr()), A.shape[1], ctypes.c_void_p(B.data_ptr()),
                          K, ctypes.c_void_p(C.data_ptr()), N, 0, bn, 1, None, ctypes.c_void_p(s.cuda_stream))
        assert rc == 0, rc
    with torch.cuda.stream(s):
        go()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(reps):
            go()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    print(f"{name:34s} M={M:5d} N={N:5d} K={K:5d} bn={bn:3d}: {us:7.2f} us/launch  "
          f"{2.0 * M * N * K / us / 1e6:7.1f} TFLOP/s", flush=True)


probe("empty-ish K=64", 512, 4096, 64, 128)
probe("fwd step K=2064 bn128", 512, 4096, 2064, 128)
probe("fwd step K=2064 bn256", 512, 4096, 2064, 256)
probe("fwd step K=2064 bn64", 512, 4096, 2064, 64)
probe("fwd step strided A", 512, 4096, 2064, 128, a_rows_stride=2064 * 512)
probe("bwd step K=4096 bn32", 512, 1024, 4096, 32)
probe("bwd step K=4096 bn64", 512, 1024, 4096, 64)
probe("bwd step K=4096 bn128", 512, 1024, 4096, 128)
probe("big M=4096 K=2048 bn256", 4096, 4096, 2048, 256, reps=20)
