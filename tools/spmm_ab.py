"""A/B timing of the K4 SpMM (and the split layer epilogue) on the Amazon
dataset as the reference generates it, d = 64 and 128 (not a benchmark).
Usage: python tools/spmm_ab.py LABEL  (libkgq.so variant chosen by the caller)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2212_04540_b200 as kgq
from paper_2212_04540_b200 import data, tensorops
from paper_2212_04540_b200 import functional as F

ds = data.reference_dataset("amazon")
A = data.build_adjacency(ds)
N = A.shape[0]
res = {"label": sys.argv[1] if len(sys.argv) > 1 else ""}


def timeit(f, n=50):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n * 1e3, 1)


for d in (64, 128):
    x = torch.randn(N, d, device="cuda")
    res[f"spmm_d{d}_us"] = timeit(lambda: tensorops.spmm(A, x))
    th = torch.randn(d, d, device="cuda") / d ** 0.5
    cfg = kgq.QuantConfig(bits=2, rng="fast")
    st = kgq.RandomStream(0)
    for split in (False, True):
        res[f"layer_d{d}_{'split' if split else 'fused'}_us"] = timeit(
            lambda: F.graph_conv_forward(A, x, th, cfg, st, 1, split=split))
    # fused layer backward on the same rows
    e_next, mask, q, _ = F.graph_conv_forward(A, x, th, cfg, st, 1)
    gr, ge = torch.randn_like(x), torch.randn_like(x)
    res[f"layer_bwd_d{d}_us"] = timeit(lambda: F.layer_backward(gr, ge, mask, q, th))
print(json.dumps(res))
