"""The NCCL collective behind the libskb C ABI (csrc/comm.cu) on one GPU: a
single-rank communicator runs the same ncclAllReduce path the data-parallel
trainers use at N > 1 (sum and max, f32 / f64 / i64, on a side stream), and
the trainers pick it up through comm.ShardedStep."""
import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _comm():
    from paper_1810_08061_b200.comm import Comm
    return Comm(0, 1, Comm.unique_id())


def test_nccl_loaded_and_versioned():
    from paper_1810_08061_b200 import runtime as rt
    c = _comm()
    assert rt.lib().skb_comm_nccl_version() >= 21800
    c.close()


@pytest.mark.parametrize("dtype,dt", [(torch.float32, 0), (torch.float64, 1), (torch.int64, 3)])
def test_single_rank_allreduce_through_the_abi(dtype, dt):
    from paper_1810_08061_b200 import runtime as rt
    c = _comm()
    lib = rt.lib()
    s = torch.cuda.Stream()
    x = (torch.arange(1 << 20, device="cuda") % 977).to(dtype)
    ref = x.clone()
    with torch.cuda.stream(s):
        for op in (0, 1):   # sum, max over one rank: identity
            assert lib.skb_comm_allreduce(c.handle, rt.ptr(x), x.numel(), dt, op, rt.stream_handle(s)) == 0
    s.synchronize()
    assert torch.equal(x, ref)
    if dtype == torch.float32:
        assert lib.skb_allreduce_f32(c.handle, rt.ptr(x), x.numel(), rt.stream_handle(None)) == 0
    torch.cuda.synchronize()
    assert torch.equal(x, ref)
    assert lib.skb_comm_allreduce(c.handle, rt.ptr(x), x.numel(), 9, 0, None) != 0   # bad dtype
    c.close()


def test_trainer_sync_uses_the_comm():
    from paper_1810_08061_b200.comm import ShardedStep
    c = _comm()
    sync = ShardedStep(c, global_batch=64)
    g = torch.full((1000,), 0.5, device="cuda")
    sync.reduce_(g)
    torch.cuda.synchronize()
    assert torch.all(g == 0.5) and sync.rows() == slice(0, 64) and sync.lr_scale(True) == 1.0
    c.close()
