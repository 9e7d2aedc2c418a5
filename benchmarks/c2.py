"""C2: dynamic-length LSTM training step, hidden 1024, input 1024, batch 4096
(512 rows per GPU at 8 GPUs), max_len 512, lengths U{1..512}, gradient
allreduce over NCCL.

One step = forward over the staged While + BPTT + gradients (one CUDA graph of
strided bf16 cuBLAS GEMMs with fp32 accumulation and fused masked cells,
csrc/train.cu; tests bound the gradients at 6e-2 of the largest entry vs the
float64 oracle, fp32 GEMMs at 1e-4) + NCCL
allreduce of the 8,392,704 gradients (33.6 MB) + fused SGD.  Metric:
sequences (examples) trained per second, whole job.
roofline: tensor-bound; padded FLOP per step = 3 * 2*B*n*(F+H)*4H (forward
gate GEMMs + the three backward GEMMs), n = max_len of the batch, against the
dense bf16 sustained peak.
cpu_baseline: the float64 numpy BPTT restatement (oracle/bptt.py, BLAS
threads) at B=16, T=64, F=H=256, scaled to the C2 shape by the MAC ratio.
"""
from __future__ import annotations

import json
import time

import numpy as np

from .common import cpu_threads, peaks

METRIC = "examples/sec dynamic-len LSTM training step (BPTT + allreduce), hidden 1024, max_len 512"
ROWS, T, F, H = 512, 512, 1024, 1024


def _config(world, n):
    return {"workload": f"C2: dynamic-length LSTM training step, hidden {H}, input {F}, {ROWS} rows per GPU "
                        f"(global batch {ROWS * world}), max_len {T}, lengths U{{1..{T}}}, SGD",
            "rows_per_gpu": ROWS, "global_batch": ROWS * world, "seq_len": T, "hidden": H, "input": F,
            "trip_count": n, "parallelism": f"data parallel x{world}, NCCL allreduce of 33.6 MB fp32 grads"}


def cpu_sample():
    from oracle import bptt
    b, t, f, h = 16, 64, 256, 256
    rng = np.random.default_rng(0)
    x, y = rng.uniform(-1, 1, (b, t, f)), rng.uniform(-1, 1, (b, t, h))
    lens = rng.integers(1, t + 1, b)
    s = 1 / np.sqrt(h)
    W, U, bb = rng.uniform(-s, s, (f, 4 * h)), rng.uniform(-s, s, (h, 4 * h)), rng.uniform(-s, s, 4 * h)
    t0 = time.perf_counter()
    bptt.forward_backward(x, np.zeros((b, h)), np.zeros((b, h)), lens, y, W, U, bb, 1 / b)
    dt = time.perf_counter() - t0
    scale = (ROWS * T * (F + H) * H) / (b * t * (f + h) * h)   # MAC ratio of the C2 shard to the sample
    return ROWS / (dt * scale), dt, scale


def run_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample()
    vals = [cpu_sample() for _ in range(args.steps)]
    v = float(np.mean([x[0] for x in vals]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "examples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * ROWS / v,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(1, T),
            "cpu_baseline": {"value": v, "unit": "examples/s", "cores": cpu_threads(), "kind": "port",
                             "sample": "B=16 T=64 F=H=256 float64 numpy BPTT (oracle/bptt.py), extrapolated to the "
                                       "512x512x1024 shard by MAC count"},
            "e2e": {"value": v, "unit": "examples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run(args, rank, world, local_rank, clocks_cls):
    import torch
    import torch.distributed as dist
    from paper_1810_08061_b200.train import LstmTrainer

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.rand((ROWS, T, F), device=dev, generator=gen) * 2 - 1
    y = torch.rand((ROWS, T, H), device=dev, generator=gen) * 2 - 1
    lens = torch.randint(1, T + 1, (ROWS,), device=dev, generator=gen)
    n_local = int(lens.max().item())
    # the While trip count of the global batch is the max over shards (replicas stay in lock step)
    n_t = torch.tensor([n_local], device=dev)
    if world > 1:
        dist.all_reduce(n_t, op=dist.ReduceOp.MAX)
    n = int(n_t.item())
    tr = LstmTrainer(F, H, ROWS, T, global_batch=ROWS * world, lr=0.01, math="bf16", seed=7, device=dev)
    # the While trip count of each step is decided on the device (no host round trip);
    # n (host) only sizes the FLOP count of the roofline below
    for _ in range(args.warmup):
        tr.step(x, y, lens)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clocks_cls(local_rank)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    fb_ms = []
    e0.record(stream)
    for _ in range(args.steps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        tr.forward_backward(x, y, lens)
        b.record(stream)
        tr.sync.reduce_(tr.grads)   # NCCL allreduce behind the libskb C ABI (skb_comm_allreduce)
        from paper_1810_08061_b200 import runtime as rt
        rt.check(tr.lib.skb_sgd_update(rt.ptr(tr.params), rt.ptr(tr.grads), tr.n_params, tr.lr,
                                       rt.stream_handle(None)), "skb_sgd_update")
        fb_ms.append((a, b))
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    kms = float(np.mean([a.elapsed_time(b) for a, b in fb_ms]))
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * ROWS / (ms_max / 1e3)
    sust, _, _, src = peaks()
    flops = 3 * 2.0 * ROWS * n * (F + H) * 4 * H
    ach = flops / (kms / 1e3) / 1e12
    roofline = {"bound": "tensor", "achieved": ach, "peak": sust, "unit": "TFLOP/s", "frac": ach / sust,
                "traffic": None, "kernel": ("forward+BPTT graph: skb's tcgen05 GEMMs (TMA, bf16 operands, fp32 TMEM accumulate) "
                           "with the LSTM cell fused into each step's epilogue, one XH^T dG weight-gradient "
                           "GEMM" if tr.lib.skb_train_last_mode() >= 0 else ""),
                "kernel_ms": kms,
                "kernel_share_of_step": kms / ms, "flops_per_launch": flops,
                "flop_basis": "3 * 2*B*n*(F+H)*4H padded to the trip count n",
                "peak_source": f"{src} dense bf16 sustained"}
    # e2e: host x / y / lens every step, loss back to the host
    # Two device input buffer sets, reused across steps as a training loop does (the captured
    # step graph is keyed by their addresses); the H2D copy of step k+1 runs on a copy stream
    # while step k computes, and every step's loss is read back on the host.
    hx, hy, hl = x.cpu().pin_memory(), y.cpu().pin_memory(), lens.cpu().pin_memory()
    bufs = [(torch.empty_like(x), torch.empty_like(y), torch.empty_like(lens)) for _ in range(2)]
    comp, cp = torch.cuda.current_stream(), torch.cuda.Stream()
    done = [None, None]   # event: the step that last used buffer set j finished
    ke = max(1, min(args.steps, 3))

    def copy_in(j):
        with torch.cuda.stream(cp):
            if done[j] is not None:
                cp.wait_event(done[j])
            for d_, h_ in zip(bufs[j], (hx, hy, hl)):
                d_.copy_(h_, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cp)
        return ev

    def run_steps(count):
        lv = None
        ready = copy_in(0)
        for k in range(count):
            j = k & 1
            comp.wait_event(ready)
            loss = tr.step(*bufs[j])
            done[j] = torch.cuda.Event()
            done[j].record(comp)
            if k + 1 < count:
                ready = copy_in(j ^ 1)
            lv = float(loss.item())
        return lv
    run_steps(4)   # each buffer set seen twice: both step graphs captured before timing
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lv = run_steps(ke)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / ke
    dt_t = torch.tensor([dt], device=dev)
    if world > 1:
        dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
    e2e = {"value": world * ROWS / float(dt_t.item()), "unit": "examples/s",
           "h2d_bytes_per_step": hx.numel() * 4 + hy.numel() * 4 + hl.numel() * 8, "d2h_bytes_per_step": 4,
           "ms_per_step": 1e3 * float(dt_t.item()), "steps": ke, "last_loss": lv,
           "api": "paper_1810_08061_b200.train.LstmTrainer.step(x, y, lens) from pinned host tensors"}
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "examples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 state/grads, bf16 tensor-core GEMM operands with f32 accumulate", "data": "synthetic",
            "config": _config(world, n), "roofline": roofline, "e2e": e2e,
            "gpu_launches": args.steps * (2 * n + 8), "clocks": clk}
    if world == 1 and not args.no_cpu:
        v, dtc, scale = cpu_sample()
        line["cpu_baseline"] = {"value": v, "unit": "examples/s", "cores": cpu_threads(), "kind": "port",
                                "sample": f"B=16 T=64 F=H=256 float64 numpy BPTT (oracle/bptt.py, {dtc:.2f} s), "
                                          f"extrapolated x{scale:.0f} by MAC count to the 512x512x1024 shard"}
    print(json.dumps(line), flush=True)
