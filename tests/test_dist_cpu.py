"""World-size-2 CPU (gloo) checks of the multi-GPU host logic the trainers
run (comm.ShardedStep, used by LstmTrainer.step and MamlTrainer.step; C2 and
C5): row sharding of the global batch, the loss normalisation by
the global batch, the gradient sum across ranks and MAML's mean-of-means
learning-rate scaling.  The per-rank gradients come from the float64 oracles;
after the step every rank holds the full-batch result.  On GPUs the same
ShardedStep reduces through the libskb NCCL communicator (comm.Comm)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bptt
from oracle import maml as maml_oracle
from paper_1810_08061_b200.comm import GlooComm, ShardedStep, default_comm, shard_rows


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _lstm_problem():
    rng = np.random.default_rng(0)
    B, T, F, H = 6, 5, 4, 3
    x, y = rng.uniform(-1, 1, (B, T, F)), rng.uniform(-1, 1, (B, T, H))
    h0, c0 = rng.uniform(-.5, .5, (B, H)), rng.uniform(-.5, .5, (B, H))
    lens = np.array([5, 3, 0, 4, 1, 5])
    W, U, b = rng.uniform(-1, 1, (F, 4 * H)), rng.uniform(-1, 1, (H, 4 * H)), rng.uniform(-.5, .5, 4 * H)
    return B, (x, h0, c0, lens, y), (W, U, b)


def _maml_problem():
    H, K, N = 8, 5, 6
    theta = maml_oracle.init_theta(H, 3)
    xs, ys, xq, yq = maml_oracle.sinusoid_tasks(N, K, 4)
    return N, theta, (xs, ys, xq, yq)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = default_comm()
        assert isinstance(comm, GlooComm) and comm.world == world
        # C2: LstmTrainer's host logic
        B, (x, h0, c0, lens, y), (W, U, b) = _lstm_problem()
        sync = ShardedStep(comm, global_batch=B)
        sl = sync.rows()
        loss, dW, dU, db = bptt.forward_backward(x[sl], h0[sl], c0[sl], lens[sl], y[sl], W, U, b,
                                                 sync.loss_scale(sl.stop - sl.start))
        flat = torch.from_numpy(np.concatenate([[loss], dW.reshape(-1), dU.reshape(-1), db]))
        sync.reduce_(flat)
        # C5: MamlTrainer's host logic (tasks sharded, per-rank task means, lr / world)
        N, theta, (xs, ys, xq, yq) = _maml_problem()
        msync = ShardedStep(comm, global_batch=N)
        ts = msync.rows()
        _, g = maml_oracle.meta_grad(theta, xs[ts], ys[ts], xq[ts], yq[ts], 0.01)
        gmean = torch.from_numpy(np.concatenate([g[k].mean(axis=0).reshape(-1) for k in maml_oracle.NAMES]))
        msync.reduce_(gmean)
        step = gmean.numpy() * msync.lr_scale(mean_of_means=True)
        q.put((rank, flat.numpy(), step))
    finally:
        dist.destroy_process_group()


def test_sharded_steps_reduce_to_full_batch():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (f, s) for r, f, s in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])   # identical ranks
    B, (x, h0, c0, lens, y), (W, U, b) = _lstm_problem()
    loss, dW, dU, db = bptt.forward_backward(x, h0, c0, lens, y, W, U, b, 1.0 / B)
    full = np.concatenate([[loss], dW.reshape(-1), dU.reshape(-1), db])
    assert np.allclose(res[0][0], full, atol=1e-12)
    N, theta, (xs, ys, xq, yq) = _maml_problem()
    _, g = maml_oracle.meta_grad(theta, xs, ys, xq, yq, 0.01)
    full_mean = np.concatenate([g[k].mean(axis=0).reshape(-1) for k in maml_oracle.NAMES])
    assert np.allclose(res[0][1], full_mean, atol=1e-12)   # equal shards: mean of means = mean


def test_single_process_has_no_comm():
    assert default_comm() is None
    s = ShardedStep(None, global_batch=10)
    assert s.rows() == slice(0, 10) and s.loss_scale(10) == 0.1 and s.lr_scale(True) == 1.0
    t = torch.ones(3)
    assert s.reduce_(t) is t and torch.equal(t, torch.ones(3))


@pytest.mark.parametrize("B,world", [(4096, 8), (10, 3), (1, 2)])
def test_shard_rows_partition(B, world):
    rows = [shard_rows(B, r, world) for r in range(world)]
    assert rows[0].start == 0 and rows[-1].stop == B
    assert all(a.stop == b.start for a, b in zip(rows, rows[1:]))
    sizes = [s.stop - s.start for s in rows]
    assert max(sizes) - min(sizes) <= 1
