"""World-size-2 CPU (gloo) checks of the multi-GPU host logic: row sharding of
the global batch and the summed-gradient allreduce used by LstmTrainer.step
(C2).  The sum of per-shard gradients of the float64 BPTT
oracle equals the full-batch gradient when the loss is normalised by the
global batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bptt
from paper_1810_08061_b200.train import allreduce_, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(0)
        B, T, F, H = 6, 5, 4, 3
        x, y = rng.uniform(-1, 1, (B, T, F)), rng.uniform(-1, 1, (B, T, H))
        h0, c0 = rng.uniform(-.5, .5, (B, H)), rng.uniform(-.5, .5, (B, H))
        lens = np.array([5, 3, 0, 4, 1, 5])
        W, U, b = rng.uniform(-1, 1, (F, 4 * H)), rng.uniform(-1, 1, (H, 4 * H)), rng.uniform(-.5, .5, 4 * H)
        sl = shard_rows(B, rank, world)
        loss, dW, dU, db = bptt.forward_backward(x[sl], h0[sl], c0[sl], lens[sl], y[sl], W, U, b, 1.0 / B)
        flat = torch.from_numpy(np.concatenate([[loss], dW.reshape(-1), dU.reshape(-1), db]))
        allreduce_(flat)
        q.put((rank, flat.numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_gradients_allreduce_to_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert np.array_equal(res[0], res[1])   # identical on every rank after the allreduce
    rng = np.random.default_rng(0)
    B, T, F, H = 6, 5, 4, 3
    x, y = rng.uniform(-1, 1, (B, T, F)), rng.uniform(-1, 1, (B, T, H))
    h0, c0 = rng.uniform(-.5, .5, (B, H)), rng.uniform(-.5, .5, (B, H))
    lens = np.array([5, 3, 0, 4, 1, 5])
    W, U, b = rng.uniform(-1, 1, (F, 4 * H)), rng.uniform(-1, 1, (H, 4 * H)), rng.uniform(-.5, .5, 4 * H)
    loss, dW, dU, db = bptt.forward_backward(x, h0, c0, lens, y, W, U, b, 1.0 / B)
    full = np.concatenate([[loss], dW.reshape(-1), dU.reshape(-1), db])
    assert np.allclose(res[0], full, atol=1e-12)


@pytest.mark.parametrize("B,world", [(4096, 8), (10, 3), (1, 2)])
def test_shard_rows_partition(B, world):
    rows = [shard_rows(B, r, world) for r in range(world)]
    assert rows[0].start == 0 and rows[-1].stop == B
    assert all(a.stop == b.start for a, b in zip(rows, rows[1:]))
    sizes = [s.stop - s.start for s in rows]
    assert max(sizes) - min(sizes) <= 1
