"""Cycles per round of the cluster all-to-all h exchange (skb_diag_cluster_exchange):
bulk DSMEM pushes vs L2 + multicast, cluster of 8, slice sizes of the C1 kernels."""
import sys
import torch
sys.path.insert(0, ".")
from paper_1810_08061_b200 import runtime as rt  # noqa: E402
lib = rt.lib()
dev = torch.device("cuda")
for slice_bytes in (4096, 8192):
    for mode in ("dsmem", "l2"):
        cyc = torch.zeros(1, dtype=torch.int64, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        g = torch.zeros(16 * slice_bytes * 8, dtype=torch.uint8, device=dev) if mode == "l2" else None
        rounds = 200
        rt.check(lib.skb_diag_cluster_exchange(8, slice_bytes, rounds, rt.ptr(cyc), rt.ptr(err),
                                               rt.ptr(g) if g is not None else None, rt.stream_handle()), "x")
        torch.cuda.synchronize()
        print(f"{mode:5s} slice {slice_bytes}: {int(cyc.item()) / rounds:.0f} cycles/round, errors {int(err.item())}")
