"""Staged decoding with a data-dependent EOS stop on the GPU (BASELINE config C3).

The reference stages greedy decoding (the EOS `break` becomes
part of the While test, transforms/lowering.py:95-115) but cannot express beam
search (no log-softmax/top-k in graph/ir.py:19-27).  `decode` runs either —
beam 1 is the greedy program — as one device-resident loop (csrc/beam.cu):
cell GEMM + fused cell, logits GEMM, and a single-pass log-softmax/top-K/
reindex kernel per step; the stop is decided on the device.

    decode("rnn",  h0, emb, (w_in, u, w_out), beam=1, eos=e, max_len=T)      # App. F
    decode("lstm", h0, emb, (W, bias, w_out, b_out), beam=8, eos=e, max_len=64, c0=c0)

Returns dict(tokens [S,K,T+1] int32 (position 0 = BOS 0), scores [S,K]
float32 (best first), lengths [S,K], steps) with device tensors.
Semantics: oracle/beam.py.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .errors import LoweringError

CELLS = {"lstm": 1, "rnn": 2}
MATH = {"fp32": 0, "tf32": 1}


def _dev(x, dev):
    import torch
    if isinstance(x, torch.Tensor):
        return x.to(device=dev, dtype=torch.float32).contiguous()
    a = getattr(x, "array", None)
    a = np.asarray(a if a is not None else x, dtype=np.float32)
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


class Decoder:
    """A decoder bound to one weight set and problem shape (workspace reused)."""

    def __init__(self, cell, emb, weights, sentences, beam, max_len, eos, math="fp32", poll=4, device=None):
        import torch
        from . import runtime as rt
        if cell not in CELLS:
            raise LoweringError(f"decoder cell {cell!r} (expected one of {sorted(CELLS)})")
        self.lib = rt.lib()
        self.dev = device or torch.device("cuda", torch.cuda.current_device())
        self.cell = cell
        self.emb = _dev(emb, self.dev)
        V, E = self.emb.shape
        if cell == "rnn":
            w_in, u, w_out = weights[:3]
            self.w_gates = _dev(np.vstack([np.asarray(_np(w_in)), np.asarray(_np(u))]), self.dev)
            self.b_gates = None
            self.w_out = _dev(w_out, self.dev)
            self.b_out = None
            H = self.w_out.shape[0]
        else:
            W, bias, w_out, b_out = weights
            self.w_gates = _dev(W, self.dev)
            self.b_gates = _dev(bias, self.dev)
            self.w_out = _dev(w_out, self.dev)
            self.b_out = _dev(b_out, self.dev) if b_out is not None else None
            H = self.w_out.shape[0]
        self.shape = rt.DecodeShape(CELLS[cell], sentences, beam, V, E, H, max_len, int(eos), MATH[math], poll)
        nbytes = int(self.lib.skb_decode_workspace_bytes(ctypes.byref(self.shape)))
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.dev)
        R = sentences * beam
        self.tokens = torch.empty((sentences, beam, max_len + 1), dtype=torch.int32, device=self.dev)
        self.scores = torch.empty((sentences, beam), dtype=torch.float32, device=self.dev)
        self.lengths = torch.empty((sentences, beam), dtype=torch.int32, device=self.dev)
        assert R == self.scores.numel()
        off = int(self.lib.skb_decode_margin_offset(ctypes.byref(self.shape)))
        self.margin = self.ws[off:off + 4 * R].view(torch.float32).view(sentences, beam)

    def margins(self):
        """Greedy (beam 1): per sentence, the smallest top-1 minus top-2 logit
        gap of any step it decoded (device tensor [S, 1]; +inf if none)."""
        return self.margin

    def __call__(self, h0, c0=None, stream=None):
        from . import runtime as rt
        h0 = _dev(h0, self.dev)
        c0 = _dev(c0, self.dev) if c0 is not None else None
        steps = ctypes.c_int32(0)
        p = rt.ptr
        rt.check(self.lib.skb_decode(ctypes.byref(self.shape), p(h0), p(c0) if c0 is not None else None,
                                     p(self.emb), p(self.w_gates), p(self.b_gates) if self.b_gates is not None else None,
                                     p(self.w_out), p(self.b_out) if self.b_out is not None else None,
                                     p(self.tokens), p(self.scores), p(self.lengths), ctypes.byref(steps),
                                     p(self.ws), rt.stream_handle(stream)), "skb_decode")
        return {"tokens": self.tokens, "scores": self.scores, "lengths": self.lengths, "steps": int(steps.value)}


def _np(x):
    a = getattr(x, "array", None)
    if a is not None:
        return a
    try:
        import torch
        if isinstance(x, torch.Tensor):
            return x.detach().cpu().numpy()
    except ImportError:  # pragma: no cover
        pass
    return np.asarray(x)


def decode(cell, h0, emb, weights, beam, eos, max_len, c0=None, math="fp32", poll=4, stream=None):
    """One-shot decode (see module doc)."""
    S = int(np.asarray(_np(h0)).shape[0]) if not hasattr(h0, "shape") else int(h0.shape[0])
    dec = Decoder(cell, emb, weights, S, beam, max_len, eos, math=math, poll=poll)
    out = dec(h0, c0, stream=stream)
    return {k: (v.clone() if hasattr(v, "clone") else v) for k, v in out.items()}
