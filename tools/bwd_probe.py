"""Time the fused layer backward (K7) on the Amazon shape in isolation:
159,251 rows x d, INT2 codes, both gradient terms (run under ncu for the
per-kernel split).  Usage: python tools/bwd_probe.py [d] [bits] [iters]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_04540_b200 as kgq
from paper_2212_04540_b200 import functional as F

d = int(sys.argv[1]) if len(sys.argv) > 1 else 64
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 2
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 20
rows = 159251
torch.manual_seed(0)
x = torch.randn(rows, d, device="cuda")
q = kgq.quantize_tensor(x, kgq.QuantConfig(bits=bits, rng="fast"), kgq.RandomStream(1), tensor_id=2)
_, mask = kgq.relu(torch.randn(rows, d, device="cuda"))
gr, ge = torch.randn(rows, d, device="cuda"), torch.randn(rows, d, device="cuda")
th = torch.randn(d, d, device="cuda") / d ** 0.5
for _ in range(3):
    F.layer_backward(gr, ge, mask, q, th)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(iters):
    F.layer_backward(gr, ge, mask, q, th)
b.record()
torch.cuda.synchronize()
print(f"layer_backward d={d} bits={bits}: {a.elapsed_time(b) / iters * 1e3:.1f} us per call (incl. partial reduce)")
