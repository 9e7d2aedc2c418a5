"""skb's own tcgen05 + TMA GEMM engine (csrc/gemm.cuh, C ABI skb_gemm) against
torch fp32 matmuls of the same (bf16- / tf32-valued) operands: every operand
layout (K-major / MN-major A and B), tile width, split-K and accumulate mode,
ragged M / N / K (TMA zero fill)."""
import ctypes

import numpy as np
import pytest
import torch

from paper_1810_08061_b200 import runtime

pytestmark = pytest.mark.gpu


def _gemm(elem, a_mn, b_mn, M, N, K, bn=0, ksplit=1, beta=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.bfloat16 if elem == 0 else torch.float32
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda", generator=g).to(dt)
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda", generator=g).to(dt)
    C0 = torch.randn((M, N), device="cuda", generator=g)
    C = C0.clone()
    ws = None
    nb = runtime.lib().skb_gemm_workspace_bytes(M, N, ksplit)
    if nb > 0:
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    rc = runtime.lib().skb_gemm(elem, int(a_mn), int(b_mn), M, N, K, ctypes.c_void_p(A.data_ptr()), A.shape[1],
                                ctypes.c_void_p(B.data_ptr()), B.shape[1], ctypes.c_void_p(C.data_ptr()), N, beta, bn,
                                ksplit, ctypes.c_void_p(ws.data_ptr()) if ws is not None else None, None)
    assert rc == 0, rc
    torch.cuda.synchronize()
    Af = (A.t() if a_mn else A).float().double()
    Bf = (B if b_mn else B.t()).float().double()
    ref = Af @ Bf + (C0.double() if beta else 0)
    return C.double(), ref


@pytest.mark.parametrize("elem", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("bn", [64, 128, 256])
def test_layouts_and_tiles(elem, a_mn, b_mn, bn):
    if elem == 1 and (a_mn or b_mn):
        pytest.skip("kind::tf32 takes K-major operands only (SKB_ERR_UNSUPPORTED)")
    got, ref = _gemm(elem, a_mn, b_mn, 304, 272, 200, bn=bn, seed=bn + 7 * a_mn + 3 * b_mn)
    scale = ref.abs().max().item()
    tol = 1e-5 if elem == 0 else 3e-3   # bf16 products are exact in fp32; tf32 truncates inputs
    assert (got - ref).abs().max().item() <= tol * scale


@pytest.mark.parametrize("elem", [0, 1])
@pytest.mark.parametrize("ksplit,beta", [(1, 1), (3, 0), (4, 1)])
def test_split_k_and_accumulate(elem, ksplit, beta):
    mn = 1 if elem == 0 else 0
    got, ref = _gemm(elem, mn, mn, 512, 256, 1000, bn=128, ksplit=ksplit, beta=beta, seed=ksplit)
    scale = ref.abs().max().item()
    assert (got - ref).abs().max().item() <= (1e-5 if elem == 0 else 3e-3) * scale


def test_split_k_is_deterministic():
    a, _ = _gemm(0, 1, 1, 256, 512, 4096, ksplit=5, seed=3)
    b, _ = _gemm(0, 1, 1, 256, 512, 4096, ksplit=5, seed=3)
    assert torch.equal(a, b)


def test_large_bf16():
    got, ref = _gemm(0, 0, 0, 4096, 4096, 1024, seed=11)
    assert (got - ref).abs().max().item() <= 1e-5 * ref.abs().max().item()


@pytest.mark.parametrize("elem", [0, 1])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("bn", [-128, -256])
def test_cta_pair_tiles(elem, a_mn, b_mn, bn):
    """cta_group::2 tiles (M = 256 across a CTA pair, B split between the two CTAs)."""
    if elem == 1 and (a_mn or b_mn):
        pytest.skip("kind::tf32 takes K-major operands only")
    got, ref = _gemm(elem, a_mn, b_mn, 560, 272 if bn == -128 else 512, 200, bn=bn, beta=1, seed=3 - bn)
    scale = ref.abs().max().item()
    assert (got - ref).abs().max().item() <= (1e-5 if elem == 0 else 3e-3) * scale
