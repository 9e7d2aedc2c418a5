"""C5 (TreeLSTM half): batched TreeLSTM over 4096 random binary trees, 32
leaves each, H = 128.  One step = one forward evaluation of the
whole forest (csrc/tree.cu: leaves, then one GEMM + fused cell per height
level).  Metric: trees/s.  GEMMs on TF32 tensor cores (tests: 2e-3 vs the
float64 oracle; fp32 path 1e-5).
roofline: tensor-bound, 2*(2H)*(5H) = 327.7 kFLOP per internal node, over the
GEMM time; the cell kernel is HBM-bound (5H gates + 2 child c + h/c writes).
cpu_baseline: the float64 numpy restatement (oracle/tree.py forest, BLAS) on
the same forest.
"""
from __future__ import annotations

import json
import time

import numpy as np

from .common import cpu_threads, peaks

METRIC = "trees/s batched TreeLSTM (4096 trees, 32 leaves, H=128)"
NTREES, LEAVES, H = 4096, 32, 128


def _forest(seed):
    from oracle import fixtures
    rng = np.random.default_rng(seed)
    return [fixtures.random_tree_arrays(LEAVES, rng) for _ in range(NTREES)]


def _config(world):
    return {"workload": f"C5 TreeLSTM: {NTREES} random binary trees per GPU, {LEAVES} leaves, hidden {H}, "
                        "forward over the whole forest", "trees_per_gpu": NTREES, "leaves": LEAVES, "hidden": H,
            "parallelism": f"replicas x{world} (independent trees, no collective)"}


def cpu_sample(trees, w):
    from oracle import tree as otree
    t0 = time.perf_counter()
    otree.forest(trees, w)
    dt = time.perf_counter() - t0
    return len(trees) / dt, dt


def run_reference(args, rank, world):
    from oracle import fixtures
    if rank != 0:
        return
    trees, w = _forest(1), fixtures.tree_weights(H, 5)
    for _ in range(args.warmup):
        cpu_sample(trees, w)
    vals = [cpu_sample(trees, w) for _ in range(args.steps)]
    v = float(np.mean([x[0] for x in vals]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "trees/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean([x[1] for x in vals])),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(1),
            "cpu_baseline": {"value": v, "unit": "trees/s", "cores": cpu_threads(), "kind": "port",
                             "sample": f"{NTREES} trees per step, float64 numpy level-batched restatement (oracle/tree.py)"},
            "e2e": {"value": v, "unit": "trees/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run(args, rank, world, local_rank, clocks_cls):
    import torch
    import torch.distributed as dist
    from oracle import fixtures
    from paper_1810_08061_b200.tree import Forest, pack_weights, tree_lstm

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    trees = _forest(1 + rank)
    w = fixtures.tree_weights(H, 5)
    forest = Forest(trees)
    pw = pack_weights(w, dev)
    for _ in range(args.warmup):
        tree_lstm(forest, w, math="tf32", packed=pw)
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
        h, c = tree_lstm(forest, w, math="tf32", packed=pw)
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * NTREES / (ms_max / 1e3)
    ninternal = len(forest.order)
    flops = ninternal * 2.0 * (2 * H) * (5 * H)
    sust, _, hbm, src = peaks()
    ach = flops / (ms / 1e3) / 1e12
    roofline = {"bound": "tensor", "achieved": ach, "peak": sust / 2, "unit": "TFLOP/s", "frac": ach / (sust / 2),
                "traffic": None, "kernel": "whole forest step (level GEMMs on TF32 + fused cells)",
                "kernel_ms": ms, "flops_per_launch": flops, "flop_basis": "2*(2H)*(5H) per internal node",
                "levels": forest.nlevels, "peak_source": f"{src} bf16 sustained / 2 (dense TF32)"}
    # e2e: tree structure + leaf values from the host every step (schedule built on the host)
    ke = max(1, min(args.steps, 5))
    for _ in range(3):   # warm-up: the repeated forest shape is captured as a CUDA graph on its second sighting
        f2 = Forest(trees)
        hh, cc = tree_lstm(f2, w, math="tf32", packed=pw)
        hh.tensor.cpu()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(ke):
        f2 = Forest(trees)
        hh, cc = tree_lstm(f2, w, math="tf32", packed=pw)
        hh.tensor.cpu()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / ke
    e2e = {"value": world * NTREES / dt, "unit": "trees/s",
           "h2d_bytes_per_step": forest.nnodes * (4 * 5) + 8 * NTREES, "d2h_bytes_per_step": NTREES * H * 4,
           "ms_per_step": 1e3 * dt, "steps": ke,
           "api": "paper_1810_08061_b200.tree.tree_lstm(Forest(trees), weights) incl. host scheduling"}
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "trees/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32 state, TF32 tensor-core GEMMs", "data": "synthetic",
            "config": _config(world), "roofline": roofline, "e2e": e2e,
            "gpu_launches": args.steps * (1 + 2 * forest.nlevels), "clocks": clk}
    if world == 1 and not args.no_cpu:
        v, dtc = cpu_sample(trees, w)
        line["cpu_baseline"] = {"value": v, "unit": "trees/s", "cores": cpu_threads(), "kind": "port",
                                "sample": f"the same {NTREES}-tree forest, float64 numpy level-batched restatement "
                                          f"(oracle/tree.py, BLAS-threaded), {dtc:.2f} s"}
    print(json.dumps(line), flush=True)
