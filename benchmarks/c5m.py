"""C5 (MAML half): MAML sinusoid meta-learning, 4096 tasks per GPU, K=10
support + 10 query, MLP 1-40-40-1 ReLU, one inner SGD step (alpha 0.01),
second-order meta-gradient.  One step = meta-gradient over all
tasks (csrc/maml.cu: one CTA per task) + allreduce across GPUs + meta-SGD.
Metric: tasks/s.  FP32 FFMA / latency bound (~0.54 MFLOP per task).
cpu_baseline: the closed-form float64 numpy meta-gradient (oracle/maml.py).
"""
from __future__ import annotations

import json
import time

import numpy as np

from .common import cpu_threads, peaks

METRIC = "MAML meta-gradient tasks/s (sinusoid, 1-40-40-1, 1 inner step, second order)"
TASKS, K, H = 4096, 10, 40
FLOP_PER_TASK = 0.54e6


def _config(world):
    return {"workload": f"C5 MAML: {TASKS} sinusoid tasks per GPU, K={K}+{K}, MLP 1-{H}-{H}-1 ReLU, 1 inner step, "
                        "second-order meta-gradient + meta-SGD", "tasks_per_gpu": TASKS, "shots": K, "hidden": H,
            "parallelism": f"data parallel x{world} (tasks sharded), allreduce of 1,761 meta-gradient floats"}


def cpu_sample():
    from oracle import maml as omaml
    th = omaml.init_theta(H, 3)
    xs, ys, xq, yq = omaml.sinusoid_tasks(TASKS, K, 4)
    t0 = time.perf_counter()
    omaml.meta_grad(th, xs, ys, xq, yq, 0.01)
    dt = time.perf_counter() - t0
    return TASKS / dt, dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample()
    vals = [cpu_sample() for _ in range(args.steps)]
    v = float(np.mean([x[0] for x in vals]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tasks/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean([x[1] for x in vals])),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(1),
            "cpu_baseline": {"value": v, "unit": "tasks/s", "cores": cpu_threads(), "kind": "port",
                             "sample": f"{TASKS} tasks per step, closed-form float64 numpy meta-gradient (oracle/maml.py)"},
            "e2e": {"value": v, "unit": "tasks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run(args, rank, world, local_rank, clocks_cls):
    import torch
    import torch.distributed as dist
    from oracle import maml as omaml
    from paper_1810_08061_b200.maml import MamlTrainer

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    xs, ys, xq, yq = (torch.from_numpy(a[..., 0].astype(np.float32)).to(dev)
                      for a in omaml.sinusoid_tasks(TASKS, K, 10 + rank))
    tr = MamlTrainer(H, K, TASKS, alpha=0.01, beta=0.001, seed=3, device=dev)
    for _ in range(args.warmup):
        tr.step(xs, ys, xq, yq)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clocks_cls(local_rank)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        loss = tr.step(xs, ys, xq, yq)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * TASKS / (ms_max / 1e3)
    fp32_peak = 148 * 128 * 2 * 1.965e9 / 1e12   # FFMA lanes x 2 x clock (B200_PROFILING fallback class)
    ach = TASKS * FLOP_PER_TASK / (ms / 1e3) / 1e12
    roofline = {"bound": "fp32-ffma", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak,
                "traffic": None, "kernel": "maml_task_kernel (one CTA per task) + deterministic task mean",
                "kernel_ms": ms, "flop_basis": "0.54 MFLOP per task (SURVEY 8(d))",
                "peak_source": "derived FP32 FFMA peak 148 SM x 128 lanes x 2 x 1.965 GHz"}
    hx = [t.cpu().pin_memory() for t in (xs, ys, xq, yq)]
    ke = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(ke):
        d = [t.to(dev, non_blocking=True) for t in hx]
        lv = float(tr.step(*d).item())
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / ke
    e2e = {"value": world * TASKS / dt, "unit": "tasks/s", "h2d_bytes_per_step": sum(t.numel() * 4 for t in hx),
           "d2h_bytes_per_step": 4, "ms_per_step": 1e3 * dt, "steps": ke, "last_loss": lv,
           "api": "paper_1810_08061_b200.maml.MamlTrainer.step from pinned host tensors"}
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "tasks/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": _config(world), "roofline": roofline,
            "e2e": e2e, "gpu_launches": args.steps * 3, "clocks": clk}
    if world == 1 and not args.no_cpu:
        v, dtc = cpu_sample()
        line["cpu_baseline"] = {"value": v, "unit": "tasks/s", "cores": cpu_threads(), "kind": "port",
                                "sample": f"{TASKS} tasks, closed-form float64 numpy meta-gradient (oracle/maml.py), "
                                          f"{dtc:.2f} s"}
    print(json.dumps(line), flush=True)
