#!/usr/bin/env python
"""bench.py — examples/sec of the staged dynamic-length LSTM on B200.

Workload (BASELINE.json configs[0], "C1"): the LSTM program staged by the
reference's to_graph (tests/golden/graph_lstm_c1.json, traced by
oracle/gen_golden.py) — hidden 256, input 256, batch 32, max_len 64, lengths
U{1..64} — executed as P independent batch-32 problems per GPU per step
(throughput mode: one launch sequence per step).  Synthetic inputs
(x ~ U(-1,1), weights ~ U(-0.1,0.1)); x is 1.2 GB per step per GPU, larger
than the 126 MB L2.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl skb|reference]

N > 1 runs under torchrun, one process per GPU: replicas (the problems are
independent), no data-path collective; time = max over ranks.

value      device-resident throughput (inputs already in HBM), CUDA events.
e2e        the same metric through the public API execute_many() from pinned
           host tensors: H2D of the inputs and D2H of the output sequence are
           inside the timed region.
roofline   dominant kernel (the persistent recurrent kernel): useful FLOPs
           2*(F+H)*4H per (row, step < len) over its CUDA-event duration,
           against the measured dense fp16/bf16 tensor peak.
cpu_baseline  the float64 C port of the reference executor's arithmetic
           (oracle/, bit-exact with the reference) on all host threads.
--impl reference  times that CPU port alone (the reference arm).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "examples/sec dynamic-len LSTM (staged while_loop) at 1/2/4/8 B200 vs CPU ref"
B, T, F, H = 32, 64, 256, 256
FLOP_PER_ROW_STEP = 2 * (F + H) * 4 * H          # 1.049 MFLOP


KERNELS = {4: "rnn_fwd_pair4_kernel (persistent 8-CTA clusters of 4 CTA pairs, M=256 cta_group::2 tcgen05 f16 "
                "MMAs, four independent 64-row recurrences per pair)",
           5: "rnn_fwd_pair_kernel (persistent 8-CTA clusters of 4 CTA pairs, M=256 cta_group::2 tcgen05 f16 "
                "MMAs, two 128-row recurrences per pair)",
           3: "rnn_fwd_dl_kernel (persistent 8-CTA clusters, two 64-row recurrences per CTA, tcgen05 f16)"}


KERNEL_KEYS = {4: "rnn_fwd_pair4_kernel", 5: "rnn_fwd_pair_kernel", 3: "rnn_fwd_dl_kernel"}   # ncu_summary.json


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d["bf16_tflops_sustained"], d["bf16_tflops"], d["hbm_gbs"], "measured"
    except Exception:
        return 1400.0, 1590.0, 6650.0, "fallback"


def config(P, N):
    return {"workload": "C1: dynamic-length LSTM staged While (to_graph), hidden 256, input 256, "
                        "batch 32 per problem, max_len 64, lengths U{1..64}",
            "model": "LSTM cell (4 gates) in a staged while_loop", "global_batch": B * P * N,
            "problems_per_gpu": P, "batch_per_problem": B, "seq_len": T, "hidden": H, "input": F,
            "parallelism": f"replicas x{N} (independent problems, no collective)",
            "l2": "inputs larger than L2 (x is %.2f GB per GPU per step)" % (B * P * T * F * 4 / 1e9)}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader",
                                          "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9 or parts[0] != str(self.index):
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                mx = max(mx, float(parts[2].split()[0]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        os.unlink(self.path)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


# ----------------------------------------------------------------------------- CPU legs
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_problems(rng, P):
    W = [rng.uniform(-0.1, 0.1, (F, H)) for _ in range(4)]
    U = [rng.uniform(-0.1, 0.1, (H, H)) for _ in range(4)]
    b = [rng.uniform(-0.1, 0.1, (H,)) for _ in range(4)]
    x = rng.uniform(-1, 1, (P * B, T, F))
    h0 = rng.uniform(-0.1, 0.1, (P * B, H))
    c0 = rng.uniform(-0.1, 0.1, (P * B, H))
    lens = rng.integers(1, T + 1, P * B)
    return x, h0, c0, lens, W, U, b


def cpu_run(P, threads, seed=0):
    """One bounded sample of the C1 workload on the float64 C port (oracle/)."""
    import oracle
    x, h0, c0, lens, W, U, b = cpu_problems(np.random.default_rng(seed), P)
    t0 = time.perf_counter()
    oracle.rnn_many(1, x, h0, c0, lens, W, U, b, P, threads)
    return time.perf_counter() - t0


def cpu_baseline(threads, target_s=10.0):
    """A bounded sample of ~target_s seconds of CPU work: batches of P problems
    until the budget is spent."""
    P = max(threads, 32)
    done, dt, k = 0, 0.0, 0
    while dt < target_s and k < 64:
        dt += cpu_run(P, threads, seed=123 + k)
        done += P
        k += 1
    return {"value": done * B / dt, "unit": "examples/s", "cores": threads, "kind": "port",
            "sample": f"{done} C1 problems ({done * B} examples) of the float64 C port of the reference "
                      f"executor's arithmetic (oracle/skb_oracle.c, bit-exact with the reference) "
                      f"on {threads} host threads, {dt:.1f} s wall"}


def run_reference(args, rank, world):
    """--impl reference: the CPU port on all host threads, same metric/config."""
    if rank != 0:
        return
    threads = cpu_threads()
    P = max(threads, 8)
    for _ in range(args.warmup):
        cpu_run(P, threads, seed=7)
    times = [cpu_run(P, threads, seed=11 + k) for k in range(args.steps)]
    ms = 1e3 * float(np.mean(times))
    value = P * B / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "examples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config(P, 1),
            "cpu_baseline": {"value": value, "unit": "examples/s", "cores": threads, "kind": "port",
                             "sample": f"{P} C1 problems per step on {threads} host threads "
                                       f"(float64 C port of the reference executor, oracle/)"},
            "e2e": {"value": value, "unit": "examples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def run_skb(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from oracle.fixtures import load_graph_fixture
    from paper_1810_08061_b200 import execute_many, lower, runtime
    from paper_1810_08061_b200.executor import RnnExecutable

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    P = args.problems
    R = P * B
    graph, _ = load_graph_fixture("graph_lstm_c1")
    prog = lower(graph)
    rng = np.random.default_rng(1000 + rank)
    weights_np = {}
    for g in "ifgo":
        weights_np["w" + g] = rng.uniform(-0.1, 0.1, (F, H))
        weights_np["u" + g] = rng.uniform(-0.1, 0.1, (H, H))
        weights_np["b" + g] = rng.uniform(-0.1, 0.1, (H,))
    weights = [tuple(weights_np[k + g] for k in "wub") for g in "ifgo"]
    exe = RnnExecutable(prog, weights, B, T, F, H, P, device=dev)
    lib = runtime.lib()

    gen = torch.Generator(device=dev).manual_seed(rank)
    x = torch.rand((R, T, F), device=dev, generator=gen) * 2 - 1
    h0 = (torch.rand((R, H), device=dev, generator=gen) * 2 - 1) * 0.1
    c0 = (torch.rand((R, H), device=dev, generator=gen) * 2 - 1) * 0.1
    lens = torch.randint(1, T + 1, (R,), device=dev, generator=gen)
    out = torch.empty((R, T, H), device=dev)
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        exe.run(x, h0, c0, lens, out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    rt_prof = lib.skb_profile_begin(args.steps)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        exe.run(x, h0, c0, lens, out)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    status = int(exe.err[0].item())
    if status != 0:
        raise RuntimeError(f"C1 launch reported status {status}")
    kernel_id, nclus = int(lib.skb_rnn_last_kernel()), int(lib.skb_rnn_last_clusters())
    ms = e0.elapsed_time(e1) / args.steps
    import ctypes
    kms = (ctypes.c_float * args.steps)()
    nk = lib.skb_profile_read(kms, args.steps) if rt_prof == 0 else 0
    lib.skb_profile_end()
    kernel_ms = float(np.mean(kms[:nk])) if nk > 0 else None
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * R / (ms_max / 1e3)

    # roofline of the dominant kernel
    lens_np = lens.cpu().numpy()
    useful = float(np.minimum(lens_np, T).sum()) * FLOP_PER_ROW_STEP
    sust, burst, hbm, src = peaks()
    roofline = None
    if kernel_ms:
        achieved = useful / (kernel_ms / 1e3) / 1e12
        traffic, traffic_src = None, None
        try:   # dram bytes of one launch from `ncu --set full` of this kernel at this shape (profiles/)
            with open(os.path.join(REPO, "profiles", "ncu_summary.json")) as f:
                ent = json.load(f).get(KERNEL_KEYS.get(kernel_id, ""), {})
            if ent.get("problems") == P:
                traffic = ent.get("dram_bytes_per_launch")
                traffic_src = f"ncu --set full, {ent.get('capture')}, commit {ent.get('commit')}"
        except Exception:
            pass
        # a ~1.4 ms kernel at the 1965 MHz max clock (no power cap): the burst peak applies
        roofline = {"bound": "tensor", "achieved": achieved, "peak": burst, "unit": "TFLOP/s",
                    "frac": achieved / burst, "traffic": traffic, "traffic_source": traffic_src,
                    "kernel": KERNELS.get(kernel_id, str(kernel_id)), "clusters": nclus,
                    "kernel_ms": kernel_ms, "kernel_share_of_step": kernel_ms / ms,
                    "flops_per_launch": useful,
                    "flop_basis": "useful 2*(F+H)*4H per (row, t < len), SURVEY 8(d)",
                    "peak_source": f"{src} dense bf16/fp16 burst (MEASURED_PEAKS.json bf16_tflops)"}

    # e2e through the public API: pinned host feeds -> execute_many -> host outputs
    e2e = None
    if not args.no_e2e:
        hx = x.to("cpu").pin_memory()
        hh0 = h0.to("cpu").pin_memory()
        hc0 = c0.to("cpu").pin_memory()
        hl = lens.to("cpu").pin_memory()
        feeds = []
        for p in range(P):
            rows = slice(p * B, (p + 1) * B)
            f = dict(weights_np)
            f.update(input_data=hx[rows], h0=hh0[rows], c0=hc0[rows], sequence_len=hl[rows])
            feeds.append(f)
        host_out = torch.empty(R * T * H, dtype=torch.float32).pin_memory()
        for _ in range(max(1, min(args.warmup, 2))):
            execute_many(graph, feeds, host_outputs=host_out)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ke = max(1, min(args.steps, args.e2e_steps))
        for _ in range(ke):
            res = execute_many(graph, feeds, host_outputs=host_out)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / ke
        dt_t = torch.tensor([dt], device=dev)
        if world > 1:
            dist.all_reduce(dt_t, op=dist.ReduceOp.MAX)
        h2d = hx.numel() * 4 + hh0.numel() * 4 + hc0.numel() * 4 + hl.numel() * 8
        d2h = R * T * H * 4 + 4 * P + 16
        e2e = {"value": world * R / float(dt_t.item()), "unit": "examples/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * float(dt_t.item()), "steps": ke,
               "api": "paper_1810_08061_b200.execute_many(graph, feeds, host_outputs=...)"}
        del res

    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "examples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f16 tensor-core MMA, f32 accumulate/state", "data": "synthetic",
            "config": config(P, world), "roofline": roofline, "e2e": e2e,
            "gpu_launches": 7 * args.steps, "clocks": clk}
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(cpu_threads())
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="skb", choices=["skb", "reference"])
    ap.add_argument("--problems", type=int, default=1152, help="batch-32 problems per GPU per step")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--config", default="c1", choices=["c1", "c2", "c3", "c4", "c5", "c5m"],
                    help="c1 = the headline metric (default); c3 = beam-search decoder; c4 = L-BFGS "
                         "(benchmarks/c*.py)")
    ap.add_argument("--sentences", type=int, default=128, help="c3: sentences per GPU")
    ap.add_argument("--n", type=int, default=0, help="c4: vector length (default 1e7)")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    leg = None
    if args.config != "c1":
        import importlib
        leg = importlib.import_module(f"benchmarks.{args.config}")
    if args.impl == "reference":
        (leg.run_reference if leg else run_reference)(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if leg:
            leg.run(args, rank, world, local_rank, ClockSampler)
        else:
            run_skb(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
