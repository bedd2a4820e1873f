import sys; sys.path.insert(0, "/root/repo")
import torch, paper_2212_04540_b200 as kgq
x = torch.randn(16 << 20, 128, device="cuda")
for G in (64, 256):
    cfg = kgq.QuantConfig(bits=2, group=G, rng="fast")
    q = kgq.quantize_tensor(x, cfg, kgq.RandomStream(1), tensor_id=1)
    for _ in range(2): out = kgq.dequantize_tensor(q)
torch.cuda.synchronize()
