"""Row-partitioned multi-GPU training step.

Nodes are split into contiguous equal-nnz row ranges (``data.partition_rows``);
rank r owns rows [lo, hi) of the adjacency (global column ids), of E0 and of
every layer's activations.  Per layer and direction there is one exchange:

    forward : E^(l)  all-gather  -> local fused layer (spmm -> quantize -> mm -> relu)
    backward: dH     all-gather  -> local spmm (A_hat symmetric: dE = A_local . dH)
    params  : dtheta all-reduce (L*d*d floats), E0 rows stay local

plus one all-gather of the readout so every rank evaluates the (tiny) BPR
head on the same batch.  The quantization noise is keyed by GLOBAL row
(``row_offset``), so the forward pass -- activations, codes, ranges, masks --
is bit-identical to the single-GPU run at any world size; only the dtheta
all-reduce reorders a sum (tolerance).

Compute goes through an ``ops`` object so the same exchange logic runs on
libkgq (``GpuOps``, the product) and, in the CPU tests, on the oracle.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import functional as F
from .data import partition_rows, row_block
from .quantize import QuantConfig, RandomStream, dequantize_tensor, quantize_tensor
from .tensorops import CSR, mask_apply, spmm


class Comm:
    """Collectives over a torch.distributed group (nccl on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

        self.gloo = dist.get_backend(group) == "gloo"

    def all_gather_rows(self, local: torch.Tensor, counts) -> torch.Tensor:
        """Concatenate every rank's row block (uneven blocks padded to the max)."""
        m = max(counts)
        dev = local.device
        if self.gloo:
            local = local.cpu()
        buf = local.new_zeros((m,) + tuple(local.shape[1:]))
        buf[:local.shape[0]] = local
        if self.gloo:
            parts = [torch.empty_like(buf) for _ in range(self.world)]
            self.dist.all_gather(parts, buf, group=self.group)
        else:
            out = local.new_empty((self.world * m,) + tuple(local.shape[1:]))
            self.dist.all_gather_into_tensor(out, buf.contiguous(), group=self.group)
            parts = [out[r * m:(r + 1) * m] for r in range(self.world)]
        return torch.cat([parts[r][:counts[r]] for r in range(self.world)], 0).to(dev)

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.gloo and t.is_cuda:
            c = t.cpu()
            self.dist.all_reduce(c, group=self.group)
            t.copy_(c)
        else:
            self.dist.all_reduce(t, group=self.group)
        return t


class SoloComm:
    """World size 1 (no communication)."""
    world, rank = 1, 0

    def all_gather_rows(self, local, counts):
        return local

    def all_reduce_sum(self, t):
        return t


class GpuOps:
    """The product path: libkgq kernels."""

    @staticmethod
    def local_adjacency(indptr, indices, vals, lo, hi, n, device):
        ip, ix, vv = row_block(indptr, indices, vals, lo, hi)
        return CSR.from_arrays(ip, ix, vv, (hi - lo, n), device=device, symmetric=False)

    graph_conv = staticmethod(F.layer_forward)
    dequant_gemm = staticmethod(F.dequant_gemm_tn)
    mask_apply = staticmethod(mask_apply)
    spmm = staticmethod(spmm)
    quantize = staticmethod(quantize_tensor)
    dequantize = staticmethod(dequantize_tensor)
    scatter_rows = staticmethod(F.scatter_rows)

    layer_backward = staticmethod(F.layer_backward)


@dataclass
class RowPartition:
    world: int
    rank: int
    cuts: np.ndarray            # world + 1 row boundaries
    n: int

    @property
    def lo(self) -> int:
        return int(self.cuts[self.rank])

    @property
    def hi(self) -> int:
        return int(self.cuts[self.rank + 1])

    @property
    def counts(self) -> list:
        return [int(self.cuts[r + 1] - self.cuts[r]) for r in range(self.world)]

    @classmethod
    def build(cls, indptr, world: int, rank: int) -> "RowPartition":
        return cls(world, rank, partition_rows(indptr, world), len(indptr) - 1)


def partitioned_step(part: RowPartition, a_local, e0_local: torch.Tensor, thetas, users, pos, neg,
                     l2: float, cfg: QuantConfig, stream: RandomStream, comm, ops=GpuOps):
    """One forward+backward of the KGNN backbone + BPR head on this rank's
    rows.  Returns (loss tensor, dE0 for the local rows, [dtheta_i] summed
    over ranks).  Mirrors tape.py:193-253's routing order."""
    lo, counts = part.lo, part.counts
    saved = []
    e_local = e0_local
    readout_local = None
    for theta in thetas:
        e_full = comm.all_gather_rows(e_local, counts)
        e_next, mask, q, _ = ops.graph_conv(a_local, e_full, theta, cfg, stream, row_offset=lo)
        saved.append((mask, q))
        readout_local = e_next if readout_local is None else readout_local + e_next
        e_local = e_next
    readout = comm.all_gather_rows(readout_local, counts)
    u, p, n = readout[users], readout[pos], readout[neg]
    loss, margins = F.bpr_forward(u, p, n, l2)
    qu, qp, qn = (ops.quantize(t, cfg, stream) for t in (u, p, n))
    one = torch.ones((), dtype=u.dtype, device=u.device)
    gu, gp, gn = F.bpr_backward(one, margins, ops.dequantize(qu), ops.dequantize(qp),
                                ops.dequantize(qn), l2, u.shape[0])
    # readout gradient rows owned here: (scat_n + scat_p) + scat_u (reference.py:59-67)
    hi = lo + counts[part.rank]

    def local_scatter(idx, g):
        sel = (idx >= lo) & (idx < hi)
        return ops.scatter_rows(hi - lo, (idx[sel] - lo).to(torch.int32), g[sel])

    g_read = (local_scatter(neg, gn) + local_scatter(pos, gp)) + local_scatter(users, gu)
    g_e = None
    dthetas = [None] * len(thetas)
    for i in range(len(thetas) - 1, -1, -1):
        mask, q = saved[i]
        dthetas[i], dh_local = ops.layer_backward(g_read, g_e, mask, q, thetas[i])
        dh_full = comm.all_gather_rows(dh_local, counts)
        g_e = ops.spmm(a_local, dh_full)
    dth = comm.all_reduce_sum(torch.stack(dthetas))
    return loss, g_e, list(dth.unbind(0))
