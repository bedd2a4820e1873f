"""Timing probe for the host-buffer entry points (not a benchmark)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_04540_b200 as kgq

rows = 8 << 20
x = torch.randn(rows, 128).pin_memory()
cfg = kgq.QuantConfig(bits=2, group=64, rng="fast")
st = kgq.RandomStream(1)
def t(f, n=3):
    f(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n): r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3, r
ctx = kgq.empty_context(rows, 128, cfg)
ob0 = torch.empty(rows, 128).pin_memory()
ms, q = t(lambda: kgq.quantize_tensor(x, cfg, st, tensor_id=1, out=ctx))
print("quantize host pinned ms", ms, "GB/s h2d", x.numel() * 4 / ms / 1e6)
ms, o = t(lambda: kgq.dequantize_tensor(q, out=ob0))
print("dequantize host ms", ms, "pinned out", o.is_pinned(), "GB/s d2h", x.numel() * 4 / ms / 1e6)
ms, _ = t(lambda: torch.empty(rows, 128, pin_memory=True))
print("pinned alloc 4GB ms", ms)
ms, _ = t(lambda: x.cuda())
print("plain h2d ms", ms)
xd = x.cuda()
ms, _ = t(lambda: xd.cpu())
print("plain d2h (pageable) ms", ms)
ob = torch.empty(rows, 128).pin_memory()
ms, _ = t(lambda: ob.copy_(xd))
print("plain d2h (pinned) ms", ms)
xp = torch.randn(rows, 128)
ms, q2 = t(lambda: kgq.quantize_tensor(xp, cfg, st, tensor_id=1))
print("quantize host pageable ms", ms)
