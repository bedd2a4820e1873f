"""SpMM (K4) time on the Amazon graph vs a uniform random graph of the same
n / nnz (L2-gather ceiling shape), and vs the heavy-row threshold (not a
benchmark).  Usage: python tools/spmm_shape_probe.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import scipy.sparse as sp
import torch
from paper_2212_04540_b200 import data, tensorops


def timeit(f, n=50):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n * 1e3, 1)


ds = data.reference_dataset("amazon")
ip, ix, vv = data.adjacency_arrays(ds)
n, nnz = len(ip) - 1, int(ip[-1])
res = {}
x = torch.randn(n, 64, device="cuda")
for thr in (128, 256, 512, 1024, 1 << 30):
    tensorops.CSR.HEAVY_NNZ = thr
    A = tensorops.CSR.from_scipy(sp.csr_matrix((vv, ix, ip), shape=(n, n)))
    res[f"amazon_heavy{thr}"] = timeit(lambda: tensorops.spmm(A, x))
tensorops.CSR.HEAVY_NNZ = 256
rng = np.random.default_rng(1)
uip = (np.arange(n + 1, dtype=np.int64) * nnz // n).astype(np.int32)
uix = np.sort(rng.integers(0, n, nnz).astype(np.int32).reshape(-1), kind="stable")
uix = np.concatenate([np.sort(uix[uip[r]:uip[r + 1]]) for r in range(0)]) if False else rng.integers(0, n, nnz).astype(np.int32)
U = tensorops.CSR.from_scipy(sp.csr_matrix((np.ones(nnz, np.float32), uix, uip), shape=(n, n)))
res["uniform"] = timeit(lambda: tensorops.spmm(U, x))
# Amazon rows with their columns randomly relabelled (same degrees, no locality)
perm = rng.permutation(n).astype(np.int32)
P = tensorops.CSR.from_scipy(sp.csr_matrix((vv, perm[ix], ip), shape=(n, n)))
res["amazon_relabelled"] = timeit(lambda: tensorops.spmm(P, x))
print(json.dumps(res))
