"""Small driver that launches every libkgq kernel family once at sizes
compute-sanitizer finishes quickly (memcheck / racecheck / synccheck /
initcheck runs, summaries in profiles/).  Not a test: results are checked by
the GPU suite; this only exercises the launch paths.

    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import torch  # noqa: E402

import paper_2212_04540_b200 as kgq  # noqa: E402
from paper_2212_04540_b200 import functional as F  # noqa: E402
from paper_2212_04540_b200 import train as T  # noqa: E402
from paper_2212_04540_b200.model import ModelConfig, init_params  # noqa: E402
from paper_2212_04540_b200.tape import Tape  # noqa: E402

torch.manual_seed(0)
dev = "cuda"
rng = np.random.default_rng(0)

# K1 / K2: fast (aligned, G in 32..256) and generic (misaligned) paths, every width and mode
for g in (32, 64, 128, 256):
    x = torch.randn(3000, g, device=dev)
    for bits in (1, 2, 4, 8):
        for rounding, rng_mode in (("nearest", "fast"), ("stochastic", "fast"), ("stochastic", "compat")):
            cfg = kgq.QuantConfig(bits=bits, rounding=rounding, rng=rng_mode)
            q = kgq.quantize_tensor(x, cfg, kgq.RandomStream(1), tensor_id=2)
            kgq.dequantize_tensor(q)
    buf = torch.empty(3000 * g + 1, device=dev)
    xm = buf[1:].view(3000, g)
    xm.copy_(x)
    q = kgq.quantize_tensor(xm, kgq.QuantConfig(bits=2, rng="fast"), kgq.RandomStream(1), tensor_id=3)
    kgq.dequantize_tensor(q)
# a partial last tile (rows not a multiple of the warp tile), 4 and 8 lanes per group
for g in (64, 256):
    for bits in (2, 8):
        xt = torch.randn(1001, g, device=dev)
        xt[5] = 1.5                                        # a zero-range group (K2's R == 0 path)
        kgq.dequantize_tensor(kgq.quantize_tensor(xt, kgq.QuantConfig(bits=bits, rng="fast"),
                                                  kgq.RandomStream(1), tensor_id=4))

# K4 SpMM with hub rows (CTA-per-row path) + K5 relu/mask
n = 3000
a = sp.random(n, n, density=0.004, random_state=1, format="lil", dtype=np.float32)
a[5, rng.choice(n, 2000, replace=False)] = 0.5
a = a.tocsr()
a = (a + a.T + sp.eye(n, dtype=np.float32)).tocsr()
a.sum_duplicates()
a.sort_indices()
A = kgq.CSR.from_scipy(a)
for d in (32, 64, 128):
    e = torch.randn(n, d, device=dev)
    kgq.spmm(A, e)
    kgq.relu(e)

# K6 fused layer forward and the split epilogues (K6t tcgen05 d=32/64/128), K7 backward (tcgen05 d=64/128, FFMA d=32),
# BPR, scatter/gather, Adam + health check: a few training steps of a toy model
from paper_2212_04540_b200 import data as D  # noqa: E402
ds = D.reference_dataset("default")
adj = D.build_adjacency(ds, dev)
for d in (64, 32, 128):
    for split in (False, True):
        F.SPLIT_LAYER_DEFAULT = split
        q = kgq.QuantConfig(bits=2, rng="fast")
        mcfg, cfg = ModelConfig(layers=2, dim=d, quant=q), T.TrainConfig(batch_size=256, quant=q)
        params = init_params(ds.num_nodes, mcfg, 0, dev)
        state = T.AdamState(params.as_dict())
        T.train_epoch(ds, adj, params, mcfg, cfg, state, kgq.RandomStream(0), np.random.default_rng(0),
                      max_steps=2)
F.SPLIT_LAYER_DEFAULT = None

# pass-through (b = 32) training steps through the same fused kernels
for d in (64, 128):
    q = kgq.QuantConfig(bits=32)
    mcfg, cfg = ModelConfig(layers=2, dim=d, quant=q), T.TrainConfig(batch_size=256, quant=q)
    params = init_params(ds.num_nodes, mcfg, 0, dev)
    state = T.AdamState(params.as_dict())
    T.train_epoch(ds, adj, params, mcfg, cfg, state, kgq.RandomStream(0), np.random.default_rng(0), max_steps=1)

# source-block phases of the SpMM (the partitioned step's exchange overlap)
from paper_2212_04540_b200.parallel import GpuOps, RowPartition  # noqa: E402
from paper_2212_04540_b200.tensorops import spmm_phased_into  # noqa: E402
ip, ix, vv = D.adjacency_arrays(ds)
for world in (3,):
    part = RowPartition.build(ip, world, 1)
    al = GpuOps.local_adjacency(ip, ix, vv, part.lo, part.hi, ds.num_nodes, dev)
    for d in (32, 64, 128):
        xx = torch.randn(ds.num_nodes, d, device=dev)
        spmm_phased_into(al, xx, torch.empty(al.shape[0], d, device=dev), al.block_phases(part.cuts), lambda p: None)

# K11 top-k and K12 fused scoring + top-k (evaluation)
s = torch.randn(300, 5000, device=dev)
F.topk_rows(s, 20)
F.topk_rows(s, 64)
for d in (32, 64):
    ro = torch.randn(ds.num_nodes, d, device=dev)
    T.evaluate(ds, ro, 20, fused=True)
# the tcgen05 rowmm
from paper_2212_04540_b200.tensorops import mm_theta  # noqa: E402
for d in (32, 64):
    mm_theta(torch.randn(1000, d, device=dev), torch.randn(d, d, device=dev))
torch.cuda.synchronize()
print("sanitize driver done")
