"""Throughput of skb_gemm (csrc/gemm.cuh) on the C2 shapes vs torch (cuBLAS) for reference."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_1810_08061_b200 import runtime  # noqa: E402

lib = runtime.lib()


def run(name, elem, a_mn, b_mn, M, N, K, bn=0, ksplit=1, reps=5):
    dt = torch.bfloat16 if elem == 0 else torch.float32
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").to(dt)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").to(dt)
    C = torch.empty((M, N), device="cuda")
    nb = lib.skb_gemm_workspace_bytes(M, N, ksplit)
    ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")

    def go():
        rc = lib.skb_gemm(elem, a_mn, b_mn, M, N, K, ctypes.c_void_p(A.data_ptr()), A.shape[1],
                          ctypes.c_void_p(B.data_ptr()), B.shape[1], ctypes.c_void_p(C.data_ptr()), N, 0, bn, ksplit,
                          ctypes.c_void_p(ws.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0, rc
    go()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    Af = A.t() if a_mn else A
    Bf = B if b_mn else B.t()
    for _ in range(2):
        torch.matmul(Af, Bf)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        torch.matmul(Af, Bf)
    e1.record()
    torch.cuda.synchronize()
    ms_t = e0.elapsed_time(e1) / reps
    tf = 2.0 * M * N * K / ms / 1e9
    print(f"{name:28s} M={M} N={N} K={K} bn={bn} ks={ksplit}: skb {ms:.3f} ms {tf:.0f} TFLOP/s | torch {ms_t:.3f} ms "
          f"{2.0 * M * N * K / ms_t / 1e9:.0f} TFLOP/s", flush=True)


run("square bf16", 0, 0, 0, 8192, 8192, 8192)
run("C2 Zx = X W (B mn)", 0, 0, 1, 262144, 4096, 1024)
run("C2 Zx = X W^T (B k)", 0, 0, 0, 262144, 4096, 1024)
run("C2 step h U (B mn)", 0, 0, 1, 512, 4096, 1024, bn=128)
run("C2 step h U bn64", 0, 0, 1, 512, 4096, 1024, bn=64)
run("C2 step dG U^T", 0, 0, 0, 512, 1024, 4096, bn=64)
run("C2 dW = X^T dG", 0, 1, 1, 1024, 4096, 262144, bn=256)
run("C2 dW ks8", 0, 1, 1, 1024, 4096, 262144, bn=256, ksplit=8)
run("tf32 square", 1, 0, 0, 8192, 8192, 4096)
run("C3 logits tf32", 1, 0, 0, 1024, 32000, 512, bn=128)
run("square bf16 pair", 0, 0, 0, 8192, 8192, 8192, bn=-256)
run("C2 dW pair", 0, 1, 1, 1024, 4096, 262144, bn=-256)
run("C3 logits tf32 pair", 1, 0, 0, 1024, 32000, 512, bn=-256)
