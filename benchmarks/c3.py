"""C3: seq2seq beam-search decoder (beam 8, vocab 32k, H = E = 512, data-dependent EOS stop).

One step = one complete decode of S sentences (csrc/beam.cu through
paper_1810_08061_b200.decode.Decoder): the whole While over decode steps with
the EOS stop decided on the device.  Metric: decoded sentences/s.
GEMMs on TF32 tensor cores (cuBLAS; stated looser bound: tests compare TF32 to
fp32 and fp32 bit-exact to the float64 oracle at margins > 1e-4).
roofline: the dominant phase by CUDA-event time; beam_select is HBM-bound with
R*V*4 logits bytes read per step (plus R*H*8 state bytes), the logits GEMM is
tensor-bound with 2*R*H*V FLOP per step.
cpu_baseline: the float64 numpy restatement (oracle/beam.py, BLAS-threaded) on
a 2-sentence sample of the same model.
"""
from __future__ import annotations

import ctypes
import json
import time

import numpy as np

from .common import cpu_threads, peaks

METRIC = "sentences/s beam-8 decode (V=32k, H=512, EOS stop)"
V, E, H, K, T, EOS = 32000, 512, 512, 8, 64, 2


def _model(seed):
    rng = np.random.default_rng(seed)
    W = (rng.uniform(-1, 1, (E + H, 4 * H)) / np.sqrt(E + H) * 2).astype(np.float32)
    b_out = rng.uniform(-1, 1, V).astype(np.float32)
    b_out[EOS] += 3.5   # EOS becomes likely after some steps: sentences stop at different steps
    return (rng.uniform(-1, 1, (V, E)).astype(np.float32),
            (W, rng.uniform(-0.1, 0.1, 4 * H).astype(np.float32),
             (rng.uniform(-1, 1, (H, V)) * 8 / np.sqrt(H)).astype(np.float32), b_out))


def _config(S, world):
    return {"workload": f"C3: LSTM decoder, beam {K}, vocab {V}, hidden {H}, embed {E}, max_len {T}, EOS stop, "
                        f"{S} sentences per GPU", "sentences_per_gpu": S, "beam": K, "vocab": V, "hidden": H,
            "max_len": T, "parallelism": f"replicas x{world} (independent sentences, no collective)",
            "l2": "logits 131 MB per step (> L2)"}


def cpu_sample(S=2):
    from oracle import beam as obeam
    emb, w = _model(3)
    rng = np.random.default_rng(4)
    h0, c0 = rng.uniform(-1, 1, (S, H)), rng.uniform(-1, 1, (S, H))
    t0 = time.perf_counter()
    r = obeam.decode("lstm", h0, emb.astype(np.float64), tuple(x.astype(np.float64) for x in w), K, EOS, T, c0=c0)
    dt = time.perf_counter() - t0
    return S / dt, r["steps"], dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample()
    vals = [cpu_sample() for _ in range(args.steps)]
    v = float(np.mean([x[0] for x in vals]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "sentences/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean([x[2] for x in vals])),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(2, 1),
            "cpu_baseline": {"value": v, "unit": "sentences/s", "cores": cpu_threads(), "kind": "port",
                             "sample": "2 sentences per step, float64 numpy restatement (oracle/beam.py)"},
            "e2e": {"value": v, "unit": "sentences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run(args, rank, world, local_rank, clocks_cls):
    import torch
    import torch.distributed as dist
    from paper_1810_08061_b200 import runtime
    from paper_1810_08061_b200.decode import Decoder

    S = args.sentences
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    emb, w = _model(3)
    dec = Decoder("lstm", emb, w, S, K, T, EOS, math="tf32", device=dev)
    rng = np.random.default_rng(100 + rank)
    h0 = torch.from_numpy(rng.uniform(-1, 1, (S, H)).astype(np.float32)).to(dev)
    c0 = torch.from_numpy(rng.uniform(-1, 1, (S, H)).astype(np.float32)).to(dev)
    lib = runtime.lib()
    for _ in range(args.warmup):
        out = dec(h0, c0)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clocks_cls(local_rank)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    steps = []
    for _ in range(args.steps):
        out = dec(h0, c0)
        steps.append(out["steps"])
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * S / (ms_max / 1e3)
    # phase shares (separate profiled run: events between phases)
    lib.skb_decode_profile(1)
    out = dec(h0, c0)
    torch.cuda.synchronize()
    ph = (ctypes.c_float * 4)()
    nst = lib.skb_decode_profile_read(ph)
    lib.skb_decode_profile(0)
    gather, gates, logits_gemm, select = (float(x) for x in ph)
    total = gather + gates + logits_gemm + select
    R = S * K
    sust, burst, hbm, src = peaks()
    tf32_peak = sust / 2
    sel_bytes = nst * (R * V * 4 + R * H * 8 * 2)
    gemm_flops = nst * 2.0 * R * H * V
    phases = {"embedding_gather_ms": gather, "gate_gemm_ms": gates, "cell_and_logits_gemm_ms": logits_gemm,
              "beam_select_ms": select, "steps_profiled": nst}
    if logits_gemm >= select:
        ach = gemm_flops / (logits_gemm / 1e3) / 1e12
        roofline = {"bound": "tensor", "achieved": ach, "peak": tf32_peak, "unit": "TFLOP/s", "frac": ach / tf32_peak,
                    "traffic": None, "kernel": "logits GEMM (cuBLAS TF32) + fused cell", "kernel_ms": logits_gemm / max(nst, 1),
                    "kernel_share_of_step": logits_gemm / total, "flop_basis": "2*R*H*V per step",
                    "peak_source": f"{src} bf16 sustained / 2 (dense TF32)", "phases": phases}
    else:
        ach = sel_bytes / (select / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm, "traffic": None,
                    "kernel": "beam_select (log-softmax + top-K + reindex)", "kernel_ms": select / max(nst, 1),
                    "kernel_share_of_step": select / total, "byte_basis": "R*V*4 + 2*R*H*8 per step",
                    "peak_source": f"{src} HBM copy bandwidth", "phases": phases}
    sel_gbs = sel_bytes / (select / 1e3) / 1e9 if select else None
    # e2e: host h0/c0 -> decode -> tokens and scores back on the host
    hh0, hc0 = h0.cpu().pin_memory(), c0.cpu().pin_memory()
    htok = torch.empty(tuple(out["tokens"].shape), dtype=torch.int32).pin_memory()
    hsc = torch.empty(tuple(out["scores"].shape), dtype=torch.float32).pin_memory()
    ke = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(ke):
        o = dec(hh0.to(dev, non_blocking=True), hc0.to(dev, non_blocking=True))
        htok.copy_(o["tokens"])
        hsc.copy_(o["scores"])
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / ke
    dt_t = torch.tensor([dt], device=dev)
    if world > 1:
        dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
    e2e = {"value": world * S / float(dt_t.item()), "unit": "sentences/s", "h2d_bytes_per_step": 2 * S * H * 4,
           "d2h_bytes_per_step": htok.numel() * 4 + hsc.numel() * 4, "ms_per_step": 1e3 * float(dt_t.item()),
           "steps": ke, "api": "paper_1810_08061_b200.decode.Decoder(...)(h0, c0) from host tensors"}
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "sentences/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 state, TF32 tensor-core GEMMs, f64 beam scores", "data": "synthetic",
            "config": dict(_config(S, world), decode_steps=int(np.mean(steps))), "roofline": roofline,
            "beam_select_gbs": sel_gbs, "e2e": e2e, "gpu_launches": args.steps * (int(np.mean(steps)) * 5 + 2),
            "clocks": clk}
    if world == 1 and not args.no_cpu:
        v, st, dtc = cpu_sample()
        line["cpu_baseline"] = {"value": v, "unit": "sentences/s", "cores": cpu_threads(), "kind": "port",
                                "sample": f"2 sentences ({st} steps, {dtc:.1f} s), float64 numpy restatement "
                                          "(oracle/beam.py, BLAS-threaded)"}
    print(json.dumps(line), flush=True)
