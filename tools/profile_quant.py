"""Short driver for ncu captures of the hot kernels (not a benchmark)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2212_04540_b200 as kgq

rows = int(sys.argv[1]) if len(sys.argv) > 1 else (16 << 20)
bits = int(sys.argv[2]) if len(sys.argv) > 2 else 2
rng = sys.argv[3] if len(sys.argv) > 3 else "fast"
x = torch.randn((rows, 128), device="cuda")
cfg = kgq.QuantConfig(bits=bits, group=64, rng=rng)
st = kgq.RandomStream(1)
for i in range(3):
    q = kgq.quantize_tensor(x, cfg, st, tensor_id=i)
    out = kgq.dequantize_tensor(q)
torch.cuda.synchronize()
