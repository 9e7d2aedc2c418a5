"""ctypes binding of libskb.so (include/skb.h) and device plumbing.

PyTorch is used only for device allocation, streams and host<->device
copies; every computation on the hot path is a libskb kernel.  The library is
loaded from the package directory (built in-tree by ``build.py``); when it is
missing, or no CUDA device is visible, ``lib()`` raises
``BackendUnavailable`` — the executor never falls back to a CPU path.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import BackendUnavailable, DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKB_LIB_PATH") or os.path.join(HERE, "libskb.so")   # override: A/B builds

SKB_OK = 0
SKB_ERR_INVALID = 1
SKB_ERR_CUDA = 2
SKB_ERR_UNSUPPORTED = 3


class RnnShape(ctypes.Structure):
    """struct skb_rnn_shape (include/skb.h)"""
    _fields_ = [("cell", ctypes.c_int32), ("hidden", ctypes.c_int32), ("input", ctypes.c_int32),
                ("time", ctypes.c_int32), ("rows_per_problem", ctypes.c_int32),
                ("problems", ctypes.c_int32)]


class DecodeShape(ctypes.Structure):
    """include/skb.h skb_decode_shape"""
    _fields_ = [(n, ctypes.c_int32) for n in ("cell", "sentences", "beam", "vocab", "embed", "hidden", "max_len",
                                              "eos", "math", "poll")]


class TrainShape(ctypes.Structure):
    """include/skb.h skb_train_shape"""
    _fields_ = [("rows", ctypes.c_int32), ("time", ctypes.c_int32), ("input", ctypes.c_int32),
                ("hidden", ctypes.c_int32), ("math", ctypes.c_int32), ("graph", ctypes.c_int32),
                ("inv_batch", ctypes.c_float)]


_VP = ctypes.c_void_p
_P4 = ctypes.c_void_p * 4

# name -> (restype, argtypes): the complete exported surface of include/skb.h
SIGNATURES = {
    "skb_version": (ctypes.c_char_p, []),
    "skb_device_sm_count": (ctypes.c_int, []),
    "skb_last_cuda_error": (ctypes.c_int, []),
    "skb_rnn_packed_bytes": (ctypes.c_int64, [ctypes.POINTER(RnnShape)]),
    "skb_rnn_workspace_bytes": (ctypes.c_int64, [ctypes.POINTER(RnnShape)]),
    "skb_rnn_plan": (ctypes.c_int, [ctypes.POINTER(RnnShape), ctypes.POINTER(ctypes.c_int32),
                                     ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32)]),
    "skb_rnn_pack": (ctypes.c_int, [ctypes.POINTER(RnnShape), _P4, _P4, _P4, ctypes.c_int, _VP, _VP, _VP]),
    "skb_rnn_forward": (ctypes.c_int, [ctypes.POINTER(RnnShape), _VP, _VP, ctypes.c_int, _VP, _VP, _VP,
                                        _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "skb_rnn_f32_packed_bytes": (ctypes.c_int64, [ctypes.POINTER(RnnShape)]),
    "skb_rnn_f32_workspace_bytes": (ctypes.c_int64, [ctypes.POINTER(RnnShape)]),
    "skb_rnn_pack_f32": (ctypes.c_int, [ctypes.POINTER(RnnShape), _P4, _P4, _P4, ctypes.c_int, _VP, _VP]),
    "skb_rnn_forward_f32": (ctypes.c_int, [ctypes.POINTER(RnnShape), _VP, _VP, ctypes.c_int, _VP, _VP, _VP,
                                            _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "skb_debug_rnn_trace": (ctypes.c_int, [_VP, ctypes.c_int]),
    "skb_debug_rnn_tile_trace": (ctypes.c_int, [_VP, ctypes.c_int]),
    "skb_profile_begin": (ctypes.c_int, [ctypes.c_int]),
    "skb_profile_read": (ctypes.c_int, [ctypes.POINTER(ctypes.c_float), ctypes.c_int]),
    "skb_profile_end": (ctypes.c_int, []),
    "skb_vm_run": (ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int64, ctypes.c_int64, _VP, _VP, _VP, _VP,
                                   _VP, ctypes.c_int64, _VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _VP]),
    "skb_vm_max_ctas": (ctypes.c_int, []),
    "skb_decode_workspace_bytes": (ctypes.c_int64, [ctypes.POINTER(DecodeShape)]),
    "skb_decode_margin_offset": (ctypes.c_int64, [ctypes.POINTER(DecodeShape)]),
    "skb_decode_profile": (ctypes.c_int, [ctypes.c_int]),
    "skb_decode_last_mode": (ctypes.c_int, []),
    "skb_decode_profile_read": (ctypes.c_int, [ctypes.POINTER(ctypes.c_float)]),
    "skb_decode": (ctypes.c_int, [ctypes.POINTER(DecodeShape)] + [_VP] * 10 + [ctypes.POINTER(ctypes.c_int32), _VP, _VP]),
    "skb_tree_workspace_bytes": (ctypes.c_int64, [ctypes.c_int] * 3),
    "skb_tree_last_mode": (ctypes.c_int, []),
    "skb_tree_schedule": (ctypes.c_int, [ctypes.c_int64] + [_VP] * 7),
    "skb_forest_schedule": (ctypes.c_int, [ctypes.c_int64] + [_VP] * 10),
    "skb_tree_lstm": (ctypes.c_int, [ctypes.c_int] * 5 + [_VP] * 10 + [ctypes.c_int, _VP, _VP, _VP, _VP]),
    "skb_train_workspace_bytes": (ctypes.c_int64, [ctypes.POINTER(TrainShape)]),
    "skb_lstm_train_step": (ctypes.c_int, [ctypes.POINTER(TrainShape)] + [_VP] * 8 + [ctypes.c_int, _VP, _VP]),
    "skb_train_last_mode": (ctypes.c_int, []),
    "skb_train_uses_engine": (ctypes.c_int, [_VP]),
    "skb_train_tc_trace": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int]),
    "skb_sgd_update": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_float, _VP]),
    "skb_maml_workspace_bytes": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int]),
    "skb_maml_meta_grad": (ctypes.c_int, [ctypes.c_int] * 3 + [_VP] * 5 + [ctypes.c_float, _VP, _VP, _VP, _VP]),
    "skb_stream_smem_bytes": (ctypes.c_int64, [ctypes.c_int] * 5),
    "skb_stream_grid": (ctypes.c_int, [ctypes.c_int64]),
    "skb_stream_tile_elems": (ctypes.c_int, []),
    "skb_stream_run": (ctypes.c_int, [_VP] * 8 + [ctypes.c_int64] + [ctypes.c_int] * 5 +
                       [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, _VP]),
    "skb_comm_load": (ctypes.c_int, [ctypes.c_char_p]),
    "skb_comm_last_error": (ctypes.c_char_p, []),
    "skb_comm_nccl_version": (ctypes.c_int, []),
    "skb_comm_unique_id": (ctypes.c_int, [_VP]),
    "skb_comm_init": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _VP, ctypes.POINTER(ctypes.c_void_p)]),
    "skb_comm_allreduce": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _VP]),
    "skb_allreduce_f32": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP]),
    "skb_allreduce_f64": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP]),
    "skb_comm_destroy": (ctypes.c_int, [_VP]),
    "skb_diag_umma_gemm": (ctypes.c_int, [_VP, _VP, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_int, _VP, _VP]),
    "skb_rnn_last_kernel": (ctypes.c_int, []),
    "skb_rnn_last_clusters": (ctypes.c_int, []),
    "skb_rnn_last_overlap": (ctypes.c_int, []),
    "skb_rnn_set_overlap": (ctypes.c_int, [ctypes.c_int]),
    "skb_gemm_workspace_bytes": (ctypes.c_int64, [ctypes.c_int, ctypes.c_int, ctypes.c_int]),
    "skb_h2d_rows": (ctypes.c_int, [_VP, _VP, ctypes.c_int64, _VP, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _VP]),
    "skb_gemm": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                _VP, ctypes.c_int64, _VP, ctypes.c_int64, _VP, ctypes.c_int64, ctypes.c_int,
                                ctypes.c_int, ctypes.c_int, _VP, _VP]),
    "skb_diag_umma_pair": (ctypes.c_int, [_VP, _VP, _VP, _VP, ctypes.c_int, ctypes.c_int, ctypes.c_int, _VP, _VP]),
    "skb_diag_cluster_exchange": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.c_int, _VP, _VP, _VP, _VP]),
}

_lock = threading.Lock()
_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libskb.so and bind every entry point (no CUDA device needed)."""
    if not os.path.exists(path):
        raise BackendUnavailable(
            f"{path} is missing: build it with `python -m paper_1810_08061_b200.build`")
    handle = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    return handle


def lib() -> ctypes.CDLL:
    """The bound library, after checking a CUDA device is present."""
    global _lib
    with _lock:
        if _lib is None:
            import torch
            if not torch.cuda.is_available():
                raise BackendUnavailable("no CUDA device visible: the skb executor runs only on a B200 "
                                         "(there is no CPU fallback)")
            _lib = load_library()
        return _lib


_host_lib = None


def host_lib() -> ctypes.CDLL:
    """The bound library for host-only entry points (e.g. skb_tree_schedule):
    no CUDA device needed, no device work issued."""
    global _host_lib
    with _lock:
        if _host_lib is None:
            _host_lib = _lib if _lib is not None else load_library()
        return _host_lib


def check(status: int, what: str):
    if status == SKB_OK:
        return
    if status == SKB_ERR_CUDA:
        code = lib().skb_last_cuda_error()
        raise DeviceError(f"{what}: CUDA error {code}")
    if status == SKB_ERR_UNSUPPORTED:
        raise DeviceError(f"{what}: configuration not supported by this build of libskb")
    raise DeviceError(f"{what}: invalid argument (status {status})")


def ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def stream_handle(stream=None) -> ctypes.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def on_stream(fn):
    """Decorator: run the whole call (uploads, status resets, launches,
    readbacks) with the caller's `stream` as torch's current stream, so every
    torch copy / fill is ordered with the kernels launched on it and host
    reads wait for it (side streams are not ordered otherwise)."""
    import functools

    @functools.wraps(fn)
    def wrapper(*args, stream=None, **kw):
        if stream is None:
            return fn(*args, stream=None, **kw)
        import torch
        with torch.cuda.stream(stream):
            return fn(*args, stream=stream, **kw)
    return wrapper
