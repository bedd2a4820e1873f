"""Dequantize throughput per (bits, group) on 16M x 128 fp32 (A/B probe for
K2: the warp-per-group kernel at G >= 128 and the 4-threads-per-group kernel
at G = 64).  Usage: python tools/dq_wide_probe.py [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_04540_b200 as kgq  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
x = torch.randn(16 << 20, 128, device="cuda")
res = []
for bits, group in ((2, 64), (2, 64), (8, 128), (4, 128), (2, 128), (8, 256), (4, 256), (2, 256), (8, 64)):
    q = kgq.quantize_tensor(x, kgq.QuantConfig(bits=bits, group=group, rng="fast"), kgq.RandomStream(1), tensor_id=0)
    out = kgq.dequantize_tensor(q)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        out = kgq.dequantize_tensor(q)
    b.record()
    torch.cuda.synchronize()
    n = x.numel()
    bpe = 4 + bits / 8 + 8 / group
    res.append(f"b{bits}g{group} {n * bpe / (a.elapsed_time(b) / reps) / 1e6:.0f}")
    del q, out
print(" ".join(res))
