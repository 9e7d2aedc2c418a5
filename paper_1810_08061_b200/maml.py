"""MAML sinusoid meta-learning on the GPU (BASELINE config C5; csrc/maml.cu).

Replaces executing the reference's `gradient()` of the staged one-task MAML
program (oracle/programs/maml.msl; graph/grad.py:35-70) task by task: one
launch computes every task's second-order meta-gradient (one CTA per task)
and their mean; `step` adds the cross-GPU mean (NCCL allreduce behind the
libskb C ABI, comm.py; tasks sharded by rank) and the meta-SGD update.

    tr = MamlTrainer(hidden=40, shots=10, tasks=4096, alpha=0.01, beta=0.001)
    loss = tr.step(xs, ys, xq, yq)        # [tasks, shots] each
"""
from __future__ import annotations

import numpy as np

NAMES = ("w1", "b1", "w2", "b2", "w3", "b3")


def flatten_theta(th):
    return np.concatenate([np.asarray(th[k], dtype=np.float64).reshape(-1) for k in NAMES])


def unflatten(flat, H):
    sizes = [H, H, H * H, H, H, 1]
    shapes = [(1, H), (1, H), (H, H), (1, H), (H, 1), (1, 1)]
    out, o = {}, 0
    for k, n, s in zip(NAMES, sizes, shapes):
        out[k] = flat[o:o + n].reshape(s)
        o += n
    return out


class MamlTrainer:
    def __init__(self, hidden=40, shots=10, tasks=4096, alpha=0.01, beta=0.001, theta=None, seed=0, device=None,
                 group=None, comm="auto"):
        import torch
        from . import runtime as rt
        self.lib = rt.lib()
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.H, self.K, self.tasks = hidden, shots, tasks
        self.alpha, self.beta, self.group = alpha, beta, group
        from .comm import ShardedStep, default_comm
        self.sync = ShardedStep(default_comm(group) if comm == "auto" else comm)
        self.P = hidden * hidden + 4 * hidden + 1
        if theta is None:
            rng = np.random.default_rng(seed)
            theta = {"w1": rng.normal(0, 1.0, (1, hidden)), "b1": rng.normal(0, 0.1, (1, hidden)),
                     "w2": rng.normal(0, np.sqrt(2.0 / hidden), (hidden, hidden)),
                     "b2": rng.normal(0, 0.1, (1, hidden)),
                     "w3": rng.normal(0, np.sqrt(2.0 / hidden), (hidden, 1)), "b3": rng.normal(0, 0.1, (1, 1))}
        flat = flatten_theta(theta) if isinstance(theta, dict) else np.asarray(theta)
        self.theta = torch.from_numpy(flat.astype(np.float32)).to(self.dev)
        self.grad = torch.zeros_like(self.theta)
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.dev)
        self.ws = torch.empty(int(self.lib.skb_maml_workspace_bytes(hidden, tasks)), dtype=torch.uint8,
                              device=self.dev)

    def meta_grad(self, xs, ys, xq, yq, stream=None):
        """Mean meta-gradient over this rank's tasks (self.grad) and mean query loss."""
        from . import runtime as rt
        p = rt.ptr
        args = [x.reshape(self.tasks, self.K).contiguous() for x in (xs, ys, xq, yq)]
        rt.check(self.lib.skb_maml_meta_grad(self.H, self.K, self.tasks, p(self.theta), *(p(a) for a in args),
                                             self.alpha, p(self.grad), p(self.loss), p(self.ws),
                                             rt.stream_handle(stream)), "skb_maml_meta_grad")
        return self.grad, self.loss

    def step(self, xs, ys, xq, yq, stream=None):
        from . import runtime as rt
        self.meta_grad(xs, ys, xq, yq, stream)
        self.sync.reduce_(self.grad, stream)   # sum of per-rank task means (NCCL, C ABI) -> lr / world
        lr = self.beta * self.sync.lr_scale(mean_of_means=True)
        rt.check(self.lib.skb_sgd_update(rt.ptr(self.theta), rt.ptr(self.grad), self.P, lr,
                                         rt.stream_handle(stream)), "skb_sgd_update")
        return self.loss
