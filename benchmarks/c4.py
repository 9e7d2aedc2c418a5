"""C4: L-BFGS (converted while_stmt, 10^7-dim separable quadratic, history m=10).

One step = one complete staged solve: `execute` of the traced program
(tests/golden/graph_lbfgs_c4.json, oracle/programs/lbfgs_m10.msl) runs the
whole While — two-loop recursion, update, convergence test — in ONE launch of
the vector-stream kernel (csrc/stream.cu).  Metric: L-BFGS iterations/s
(trip count of the solve / its time), float64 like the reference.

roofline: HBM-bound; algorithmic bytes per iteration =
(8m + 12) * n * 8 = 7.36 GB at n = 1e7, m = 10, over the kernel's CUDA-event
time per iteration.  N > 1: replicas (one independent problem per GPU).
cpu_baseline: the float64 C restatement (oracle/lbfgs_oracle.c, bit-exact with
the reference executor) on one host thread at n = 1e6, scaled to n = 1e7
(linear in n: every iteration is n-element streams).
"""
from __future__ import annotations

import json
import time

import numpy as np

from .common import cpu_threads, ncu_traffic, peaks

METRIC = "L-BFGS iterations/s (staged while_stmt, n=1e7, m=10, f64)"
M = 10


def _problem(n, seed):
    rng = np.random.default_rng(seed)
    return (rng.uniform(-1, 1, n), rng.uniform(0.5, 4.0, n), rng.uniform(-1, 1, n))


def _config(n, world):
    return {"workload": f"C4: L-BFGS m={M} on a separable quadratic, n={n:.0e}, unit step, tol 1e-18 on |g|^2, "
                        "max 100 iterations, whole solve in one launch",
            "n": n, "m": M, "parallelism": f"replicas x{world} (independent problems, no collective)",
            "l2": "vectors larger than L2 (80 MB each, 10+ live)"}


def cpu_sample(n=1_000_000, target=10**7):
    import oracle
    x0, a, b = _problem(n, 5)
    t0 = time.perf_counter()
    _, k, _ = oracle.lbfgs(x0, a, b, 1e-18, 100, M)
    dt = time.perf_counter() - t0
    return k / dt * (n / target), k, dt


def run_reference(args, rank, world):
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_sample()
    vals = [cpu_sample() for _ in range(args.steps)]
    v = float(np.mean([x[0] for x in vals]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iterations/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * float(np.mean([x[2] for x in vals])),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(10**7, 1),
            "cpu_baseline": {"value": v, "unit": "iterations/s", "cores": 1, "kind": "port",
                             "sample": "one solve at n=1e6 on the float64 C restatement (oracle/lbfgs_oracle.c), "
                                       "iterations/s scaled by 1e6/1e7"},
            "e2e": {"value": v, "unit": "iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run(args, rank, world, local_rank, clocks_cls):
    import torch
    import torch.distributed as dist
    from oracle import fixtures
    from paper_1810_08061_b200 import execute, ir
    from paper_1810_08061_b200 import stream as st
    from paper_1810_08061_b200.executor import plan_kind

    n = args.n or 10**7
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    graph = ir.from_json(fixtures.load_golden("graph_lbfgs_c4")["graph"])
    x0, a, b = _problem(n, 100 + rank)
    tol, max_iter = np.float64(1e-18), np.int64(100)
    dfeeds = {"x0": torch.from_numpy(x0).to(dev), "a": torch.from_numpy(a).to(dev),
              "b": torch.from_numpy(b).to(dev), "tol": tol, "max_iter": max_iter}
    assert plan_kind(graph, dfeeds) == "stream"
    for _ in range(max(1, args.warmup)):   # at least one solve: its trip count sizes the metric
        res = execute(graph, dfeeds)
    k = int(res.outputs[1].item())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clocks_cls(local_rank)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream()
    kms = []
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        res = execute(graph, dfeeds)
        kms.append(st.run.last["kernel_ms"])
    e1.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * k / (ms_max / 1e3)
    kernel_ms = float(np.mean(kms))
    info = dict(st.run.last)
    _, _, hbm, src = peaks()
    alg = (8 * M + 12) * n * 8 * k
    achieved = alg / (kernel_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": ncu_traffic("stream_kernel"), "kernel": "stream_kernel (persistent vector-stream region)",
                "kernel_ms": kernel_ms, "kernel_share_of_step": kernel_ms / ms, "bytes_per_launch": alg,
                "byte_basis": "(8m+12)*n*8 per L-BFGS iteration x trip count (SURVEY 8(d))",
                "grid_exchanges_per_launch": info.get("barriers"), "peak_source": f"{src} HBM copy bandwidth"}
    # e2e: host feeds -> execute -> x and k back on the host
    hx0, ha, hb = (torch.from_numpy(v).pin_memory() for v in (x0, a, b))
    hfeeds = {"x0": hx0, "a": ha, "b": hb, "tol": tol, "max_iter": max_iter}
    hout = torch.empty(n, dtype=torch.float64).pin_memory()
    ke = max(1, min(args.steps, 5))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(ke):
        feeds = {kk: (v.to(dev, non_blocking=True) if isinstance(v, torch.Tensor) else v) for kk, v in hfeeds.items()}
        r = execute(graph, feeds)
        hout.copy_(r.outputs[0].tensor)
        kk_ = int(r.outputs[1].item())
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / ke
    dt_t = torch.tensor([dt], device=dev)
    if world > 1:
        dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
    e2e = {"value": world * kk_ / float(dt_t.item()), "unit": "iterations/s", "h2d_bytes_per_step": 3 * n * 8 + 16,
           "d2h_bytes_per_step": n * 8 + 8, "ms_per_step": 1e3 * float(dt_t.item()), "steps": ke,
           "api": "paper_1810_08061_b200.execute(graph, feeds) with host feeds, x copied back"}
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "iterations/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": dict(_config(n, world), trip_count=k),
            "roofline": roofline, "e2e": e2e, "gpu_launches": args.steps, "clocks": clk,
            "stream_tier": {kk: info[kk] for kk in ("grid", "smem", "pool", "max_live", "barriers")}}
    if world == 1 and not args.no_cpu:
        v, kc, dtc = cpu_sample()
        line["cpu_baseline"] = {"value": v, "unit": "iterations/s", "cores": 1, "kind": "port",
                                "sample": f"one solve at n=1e6 ({kc} iterations, {dtc:.1f} s) on the float64 C "
                                          "restatement (oracle/lbfgs_oracle.c, bit-exact with the reference), "
                                          "scaled by 1e6/1e7"}
    print(json.dumps(line), flush=True)
