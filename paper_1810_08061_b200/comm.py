"""Data-parallel plumbing of the training configs.

`Comm` is an NCCL communicator owned by libskb (csrc/comm.cu, include/skb.h
`skb_comm_init` / `skb_allreduce_f32`): the gradient allreduce is enqueued by
the C ABI on the caller's CUDA stream.  torch.distributed is used only to
exchange the 128-byte NCCL unique id (its store / a broadcast: host plumbing).
`GlooComm` is the same interface over torch.distributed's gloo backend, for
the CPU multi-process tests of the host logic.

`ShardedStep` is the host logic the trainers share: which rows of the global
batch a rank owns, the loss normalisation by the global batch, the gradient
sum across ranks, and the learning-rate scaling of a mean-of-means update.
"""

from __future__ import annotations

import ctypes
import os
from typing import Optional


def shard_rows(global_batch: int, rank: int, world: int) -> slice:
    """Rows of the global batch owned by `rank` (contiguous, sizes differ by <= 1)."""
    lo = global_batch * rank // world
    hi = global_batch * (rank + 1) // world
    return slice(lo, hi)


def _nccl_path() -> Optional[str]:
    try:
        import nvidia.nccl
        p = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        return p if os.path.exists(p) else None
    except Exception:
        return None


class Comm:
    """NCCL communicator behind the libskb C ABI (one rank per GPU)."""

    backend = "nccl"

    def __init__(self, rank: int, world: int, uid: bytes):
        from . import runtime as rt
        self.lib = rt.lib()
        self.rank, self.world = rank, world
        rt.check(self.lib.skb_comm_load(_nccl_path().encode() if _nccl_path() else None), "skb_comm_load")
        self.handle = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        rc = self.lib.skb_comm_init(rank, world, buf, ctypes.byref(self.handle))
        if rc:
            raise RuntimeError(f"skb_comm_init: {self.lib.skb_comm_last_error().decode()}")

    @staticmethod
    def unique_id() -> bytes:
        from . import runtime as rt
        lib = rt.lib()
        rt.check(lib.skb_comm_load(_nccl_path().encode() if _nccl_path() else None), "skb_comm_load")
        buf = ctypes.create_string_buffer(128)
        rc = lib.skb_comm_unique_id(buf)
        if rc:
            raise RuntimeError(f"skb_comm_unique_id: {lib.skb_comm_last_error().decode()}")
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """Rank 0 creates the unique id; torch.distributed broadcasts it."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                   group=group)
        return cls(rank, world, obj[0])

    def allreduce_(self, t, op: str = "sum", stream=None):
        """In-place sum (or max) of a contiguous CUDA tensor over all ranks."""
        import torch
        from . import runtime as rt
        if self.world == 1:
            return t
        dt = {torch.float32: 0, torch.float64: 1, torch.int32: 2, torch.int64: 3}[t.dtype]
        rc = self.lib.skb_comm_allreduce(self.handle, rt.ptr(t), t.numel(), dt, {"sum": 0, "max": 1}[op],
                                         rt.stream_handle(stream))
        if rc:
            raise RuntimeError(f"skb_comm_allreduce: {self.lib.skb_comm_last_error().decode()}")
        return t

    def close(self):
        if getattr(self, "handle", None):
            self.lib.skb_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GlooComm:
    """The Comm interface over torch.distributed (gloo, CPU tensors): used by
    the world-size-2 CPU tests of the host logic; never on a GPU data path."""

    backend = "gloo"

    def __init__(self, group=None):
        import torch.distributed as dist
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def allreduce_(self, t, op: str = "sum", stream=None):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX, group=self.group)
        return t


def default_comm(group=None):
    """The communicator a trainer uses: None for a single process, the libskb
    NCCL communicator when torch.distributed runs NCCL (one rank per GPU),
    GlooComm for gloo process groups."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return None
    if dist.get_backend(group) == "gloo":
        return GlooComm(group)
    return Comm.from_process_group(group)


class ShardedStep:
    """Host logic of one data-parallel training step.

    rows(global_batch) -> this rank's slice; loss_scale = 1 / global batch, so
    the per-rank gradient sums add up to the full-batch gradient; reduce_(g)
    sums g over ranks; lr_scale(mean_of_means) is 1/world when every rank
    contributes the mean over its own shard (MAML) and 1 otherwise."""

    def __init__(self, comm=None, global_batch: Optional[int] = None):
        self.comm = comm
        self.rank = comm.rank if comm is not None else 0
        self.world = comm.world if comm is not None else 1
        self.global_batch = global_batch

    def rows(self, global_batch: Optional[int] = None) -> slice:
        return shard_rows(global_batch or self.global_batch, self.rank, self.world)

    def loss_scale(self, local_rows: int) -> float:
        return 1.0 / float(self.global_batch or local_rows * self.world)

    def reduce_(self, grads, stream=None):
        if self.comm is not None:
            self.comm.allreduce_(grads, "sum", stream)
        return grads

    def lr_scale(self, mean_of_means: bool) -> float:
        return 1.0 / self.world if mean_of_means else 1.0
