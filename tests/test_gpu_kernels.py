"""GPU self-tests of the hand-written sm_100a building blocks (tcgen05.mma
with shared-memory and tensor-memory operands, TMEM round trips, the
cluster h-exchange) against plain PyTorch fp32 references."""

import ctypes

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_1810_08061_b200 import runtime
    return runtime.lib()


@pytest.mark.parametrize("n,k", [(16, 16), (32, 64), (64, 512), (128, 256), (256, 128), (64, 16)])
@pytest.mark.parametrize("mode", [0, 2], ids=["A_smem", "A_tmem"])
def test_umma_gemm_matches_fp32(lib, n, k, mode):
    import torch
    from paper_1810_08061_b200 import runtime as rt
    torch.manual_seed(n * 1000 + k)
    A = torch.randn(128, k, device="cuda").half()
    B = torch.randn(n, k, device="cuda").half()
    D = torch.full((128, n), float("nan"), device="cuda")
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    rt.check(lib.skb_diag_umma_gemm(rt.ptr(A), rt.ptr(B), rt.ptr(D), n, k, mode, rt.ptr(cyc),
                                    rt.stream_handle()), "umma")
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    assert torch.allclose(D, ref, rtol=1e-5, atol=1e-3 * (k ** 0.5))


@pytest.mark.parametrize("cluster", [2, 4, 8])
@pytest.mark.parametrize("via_l2", [False, True])
def test_cluster_exchange_integrity(lib, cluster, via_l2):
    import torch
    from paper_1810_08061_b200 import runtime as rt
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    errs = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda") if via_l2 else None
    rt.check(lib.skb_diag_cluster_exchange(cluster, 4096, 200, rt.ptr(cyc), rt.ptr(errs), rt.ptr(scratch),
                                           rt.stream_handle()), "exchange")
    torch.cuda.synchronize()
    assert errs.item() == 0
    assert cyc.item() > 0
