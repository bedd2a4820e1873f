"""SpMM schedule probe on the Amazon-shaped graph (not a benchmark): time the
K4 kernel for several heavy-row thresholds and the hub row alone."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_04540_b200 import data, tensorops

shape = sys.argv[1] if len(sys.argv) > 1 else "amazon"
ds = data.reference_dataset(shape) if shape in data.REFERENCE_DATASETS else data.synth_kg(data.SHAPES[shape], seed=0)
A = data.build_adjacency(ds)
N = A.shape[0]
x = torch.randn(N, 64, device="cuda")


def timeit(f, n=20):
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


ref = tensorops.spmm(A, x)
for th in (128, 256, 512, 1024, 2048, 4096, 1 << 30):
    A._row_order = None
    A.HEAVY_NNZ = th
    A.schedule()
    out = tensorops.spmm(A, x)
    assert torch.equal(out, ref)
    print(f"heavy>{th}: n_heavy={A._n_heavy} {timeit(lambda: tensorops.spmm(A, x)):.1f} us")
deg = torch.diff(A.indptr.long())
hub = int(torch.argmax(deg))
ip = A.indptr.cpu().numpy()
sl = slice(ip[hub], ip[hub + 1])
one = tensorops.CSR(torch.tensor([0, sl.stop - sl.start], dtype=torch.int32, device="cuda"),
                    A.indices[sl].clone(), A.data[sl].clone(), (1, N))
for th in (256, 1 << 30):
    one._row_order = None
    one.HEAVY_NNZ = th
    print(f"hub row alone ({sl.stop - sl.start} nnz), heavy>{th}: {timeit(lambda: tensorops.spmm(one, x)):.1f} us")
