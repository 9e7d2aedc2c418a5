"""Dynamic-length LSTM training on B200s (BASELINE config C2; csrc/train.cu).

One `step` = forward over the staged While (per-row lengths), BPTT, the
gradient allreduce across ranks (NCCL behind the libskb C ABI,
`skb_allreduce_f32` on the trainer's stream — the only data-path collective of
the backend; comm.py) and the SGD update.  It replaces the
reference's hand-derived staged BPTT program (oracle/programs/lstm_bptt.msl;
the reference cannot differentiate a While, graph/grad.py:159-161).

    tr = LstmTrainer(F, H, rows=512, time=512, global_batch=4096, lr=0.1)
    loss = tr.step(x, y, lens)           # x [rows,T,F], y [rows,T,H], lens [rows]

Sharding: the global batch is split by rows; every rank runs
its shard and the summed gradients (loss normalised by the global batch) are
identical on all ranks after the allreduce.
"""
from __future__ import annotations

import ctypes

import numpy as np


from .comm import ShardedStep, default_comm, shard_rows  # noqa: F401  (shard_rows: public)


class LstmTrainer:
    def __init__(self, input_size, hidden, rows, time, global_batch=None, lr=0.1, math="tf32", seed=0,
                 params=None, device=None, group=None, graph=True, comm="auto"):
        import torch
        from . import runtime as rt
        self.lib = rt.lib()
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.F, self.H, self.rows, self.time = input_size, hidden, rows, time
        self.lr = lr
        self.group = group
        self.sync = ShardedStep(default_comm(group) if comm == "auto" else comm, global_batch or rows)
        G = 4 * hidden
        self.n_params = input_size * G + hidden * G + G
        if params is None:
            rng = np.random.default_rng(seed)
            s = 1.0 / np.sqrt(hidden)
            params = rng.uniform(-s, s, self.n_params)
        self.params = torch.as_tensor(np.asarray(params, dtype=np.float32)).to(self.dev).contiguous()
        self.grads = torch.zeros_like(self.params)
        self.loss = torch.zeros(1, dtype=torch.float32, device=self.dev)
        self.shape = rt.TrainShape(rows, time, input_size, hidden, {"fp32": 0, "tf32": 1, "bf16": 2}[math],
                                   1 if graph else 0,
                                   1.0 / float(global_batch or rows))
        self.ws = torch.empty(int(self.lib.skb_train_workspace_bytes(ctypes.byref(self.shape))), dtype=torch.uint8,
                              device=self.dev)

    def views(self, t):
        F, H, G = self.F, self.H, 4 * self.H
        return t[:F * G].view(F, G), t[F * G:F * G + H * G].view(H, G), t[F * G + H * G:]

    def forward_backward(self, x, y, lens, h0=None, c0=None, max_len=None, stream=None):
        """Loss (device scalar) and this shard's gradients in self.grads."""
        from . import runtime as rt
        if max_len is None:   # the While trip count: on the device when the engine runs the step
            if self.lib.skb_train_uses_engine(ctypes.byref(self.shape)):
                max_len = -1
            else:
                max_len = int(lens.max().item()) if lens.numel() else 0
        max_len = -1 if max_len == -1 else max(0, min(int(max_len), self.time))
        p = rt.ptr
        rt.check(self.lib.skb_lstm_train_step(ctypes.byref(self.shape), p(x), p(y), p(lens),
                                              p(h0) if h0 is not None else None, p(c0) if c0 is not None else None,
                                              p(self.params), p(self.grads), p(self.loss), max_len, p(self.ws),
                                              rt.stream_handle(stream)), "skb_lstm_train_step")
        return self.loss

    def step(self, x, y, lens, h0=None, c0=None, max_len=None, stream=None):
        from . import runtime as rt
        loss = self.forward_backward(x, y, lens, h0, c0, max_len, stream)
        self.sync.reduce_(self.grads, stream)   # NCCL sum over ranks, on `stream` (C ABI)
        rt.check(self.lib.skb_sgd_update(rt.ptr(self.params), rt.ptr(self.grads), self.n_params, self.lr,
                                         rt.stream_handle(stream)), "skb_sgd_update")
        return loss
