"""PyTorch plugin surface: quantized autograd Functions and nn.Modules.

Each Function saves exactly the context the corresponding reference Tape
record keeps (kgact.tape, /root/reference/pkg/src/kgact/tape.py), so a torch
user gets TinyKG's activation compression by swapping modules:

    SpMM            ~ Tape.record_spmm   (adjacency reference, tape.py:101-110)
    QuantLinear     ~ Tape.record_mm     (Quant(H), tape.py:112-120, backward :219-223)
    MaskedReLU      ~ Tape.record_relu   (1-bit mask, tape.py:122-126)
    QuantGraphConv  ~ one forward_all layer (spmm -> mm -> relu) in ONE fused kernel
    Gather          ~ Tape.record_gather (int32 indices, tape.py:143-152)
    BPRLoss         ~ Tape.record_bpr_loss (Quant(u,p,n) + margins, tape.py:154-183)

A ``ContextLedger`` (optional argument) reproduces the Tape's byte
accounting: bytes are added when a context is saved and released when its
backward has run.
"""

import torch

from . import functional as F
from .quantize import (row_group_offset, QuantConfig, RandomStream, dequantize_tensor, fp32_equivalent_bytes,
                       quantize_tensor, stored_bytes)
from .tensorops import CSR, mask_apply, mm_theta, relu, spmm, spmm_t


class ContextLedger:
    """Peak / current context bytes (tape.py:68-71, :86-93, :187-191)."""

    def __init__(self):
        self.current = self.peak = 0
        self.current_eq = self.peak_eq = 0
        self._adj = set()

    def push(self, nbytes: int, eq: int) -> None:
        self.current += nbytes
        self.current_eq += eq
        self.peak = max(self.peak, self.current)
        self.peak_eq = max(self.peak_eq, self.current_eq)

    def free(self, nbytes: int, eq: int) -> None:
        self.current -= nbytes
        self.current_eq -= eq

    def adjacency(self, adj: CSR) -> int:
        if id(adj) in self._adj:
            return 0
        self._adj.add(id(adj))
        b = adj.nbytes()
        self.push(b, b)
        return b

    @property
    def compression_ratio(self) -> float:
        return self.peak_eq / self.peak if self.peak else 1.0


def _ledger_push(ledger, nbytes, eq):
    if ledger is not None:
        ledger.push(nbytes, eq)


def _ledger_free(ledger, nbytes, eq):
    if ledger is not None:
        ledger.free(nbytes, eq)


class SpMMFn(torch.autograd.Function):
    """Context: the shared adjacency, counted once per ledger and released by
    the node that first registered it (tape.py:101-110, :187-191)."""

    @staticmethod
    def forward(ctx, x, adj: CSR, ledger=None):
        ctx.adj, ctx.ledger = adj, ledger
        ctx.adj_bytes = ledger.adjacency(adj) if ledger is not None else 0
        return spmm(adj, x)

    @staticmethod
    def backward(ctx, g):
        _ledger_free(ctx.ledger, ctx.adj_bytes, ctx.adj_bytes)
        return spmm_t(ctx.adj, g.contiguous()), None, None


class QuantLinearFn(torch.autograd.Function):
    """J = H @ theta; saves Quant(H) only (theta is never quantized)."""

    @staticmethod
    def forward(ctx, h, theta, cfg: QuantConfig, stream: RandomStream, ledger=None, row_offset=0):
        q = quantize_tensor(h, cfg, stream, group_offset=row_group_offset(row_offset, h.shape[1], cfg.group))
        ctx.q = q
        ctx.ledger = ledger
        ctx.bytes = (stored_bytes(q), fp32_equivalent_bytes(q))
        _ledger_push(ledger, *ctx.bytes)
        ctx.save_for_backward(theta)
        return h @ theta

    @staticmethod
    def backward(ctx, g):
        (theta,) = ctx.saved_tensors
        g = g.contiguous()
        dtheta = F.dequant_gemm_tn(ctx.q, g)
        dh = mm_theta(g, theta, transpose=True)
        ctx.q = None
        _ledger_free(ctx.ledger, *ctx.bytes)
        return dh, dtheta, None, None, None, None


class MaskedReLUFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, j, ledger=None):
        out, mask = relu(j)
        ctx.mask = mask
        ctx.ledger = ledger
        _ledger_push(ledger, mask.nbytes, mask.nbytes)
        return out

    @staticmethod
    def backward(ctx, g):
        out = mask_apply(g.contiguous(), ctx.mask)
        _ledger_free(ctx.ledger, ctx.mask.nbytes, ctx.mask.nbytes)
        ctx.mask = None
        return out, None


class QuantGraphConvFn(torch.autograd.Function):
    """E' = relu(spmm(A, E) @ theta) in one fused sm_100a kernel; saves
    Quant(H) + 1-bit mask + the adjacency reference (model.py:81-85)."""

    @staticmethod
    def forward(ctx, e, theta, adj: CSR, cfg: QuantConfig, stream: RandomStream, ledger=None,
                row_offset=0):
        e_next, mask, q, _ = F.graph_conv_forward(adj, e, theta, cfg, stream, row_offset=row_offset)
        ctx.adj, ctx.q, ctx.mask, ctx.ledger = adj, q, mask, ledger
        adj_b = ledger.adjacency(adj) if ledger is not None else 0
        ctx.bytes = (stored_bytes(q) + mask.nbytes, fp32_equivalent_bytes(q) + mask.nbytes)
        _ledger_push(ledger, *ctx.bytes)
        ctx.bytes = (ctx.bytes[0] + adj_b, ctx.bytes[1] + adj_b)
        ctx.save_for_backward(theta)
        return e_next

    @staticmethod
    def backward(ctx, g):
        (theta,) = ctx.saved_tensors
        dtheta, dh = F.layer_backward(g.contiguous(), None, ctx.mask, ctx.q, theta)
        de = spmm_t(ctx.adj, dh)
        _ledger_free(ctx.ledger, *ctx.bytes)
        ctx.q = ctx.mask = None
        return de, dtheta, None, None, None, None, None


class GatherFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, src, idx, ledger=None):
        idx32 = idx.to(torch.int32)
        ctx.idx, ctx.rows, ctx.ledger = idx32, src.shape[0], ledger
        _ledger_push(ledger, idx32.numel() * 4, idx32.numel() * 4)
        return src.index_select(0, idx32.to(torch.int64))

    @staticmethod
    def backward(ctx, g):
        out = F.scatter_rows(ctx.rows, ctx.idx, g.contiguous())
        _ledger_free(ctx.ledger, ctx.idx.numel() * 4, ctx.idx.numel() * 4)
        return out, None, None


class BPRLossFn(torch.autograd.Function):
    """BPR + L2 (tape.py:154-183); saves Quant(u), Quant(p), Quant(n) + margins."""

    @staticmethod
    def forward(ctx, u, p, n, l2: float, cfg: QuantConfig, stream: RandomStream, ledger=None):
        loss, margins = F.bpr_forward(u, p, n, l2)
        ctx.qs = [quantize_tensor(t, cfg, stream) for t in (u, p, n)]
        ctx.margins, ctx.l2, ctx.batch, ctx.ledger = margins, l2, u.shape[0], ledger
        nb = sum(stored_bytes(q) for q in ctx.qs) + margins.numel() * 4
        eq = sum(fp32_equivalent_bytes(q) for q in ctx.qs) + margins.numel() * 4
        ctx.bytes = (nb, eq)
        _ledger_push(ledger, nb, eq)
        return loss

    @staticmethod
    def backward(ctx, g):
        uh, ph, nh = (dequantize_tensor(q) for q in ctx.qs)
        gu, gp, gn = F.bpr_backward(g, ctx.margins, uh, ph, nh, ctx.l2, ctx.batch)
        _ledger_free(ctx.ledger, *ctx.bytes)
        ctx.qs = None
        return gu, gp, gn, None, None, None, None


class QuantGraphConv(torch.nn.Module):
    """One KGNN layer with a compressed context (drop-in nn.Module)."""

    def __init__(self, dim: int, cfg: QuantConfig, stream: RandomStream, weight=None):
        super().__init__()
        self.cfg, self.stream = cfg, stream
        w = torch.empty(dim, dim) if weight is None else weight
        if weight is None:
            torch.nn.init.xavier_uniform_(w)
        self.weight = torch.nn.Parameter(w)

    def forward(self, e, adj: CSR, ledger=None, row_offset=0):
        if F.can_fuse(self.cfg, e.shape[1]):
            return QuantGraphConvFn.apply(e, self.weight, adj, self.cfg, self.stream, ledger, row_offset)
        h = SpMMFn.apply(e, adj, ledger)
        j = QuantLinearFn.apply(h, self.weight, self.cfg, self.stream, ledger, row_offset)
        return MaskedReLUFn.apply(j, ledger)


class KGNN(torch.nn.Module):
    """The reference backbone (model.py:66-88) as an nn.Module: E0 and
    theta_i are Parameters; forward(adj) returns the readout."""

    def __init__(self, e0: torch.Tensor, thetas, cfg: QuantConfig, stream: RandomStream,
                 aggregation: str = "sum"):
        super().__init__()
        self.e0 = torch.nn.Parameter(e0)
        self.layers = torch.nn.ModuleList(
            [QuantGraphConv(e0.shape[1], cfg, stream, weight=t) for t in thetas])
        self.aggregation = aggregation

    def forward(self, adj: CSR, ledger=None):
        e = self.e0
        out = None
        for layer in self.layers:
            e = layer(e, adj, ledger)
            out = e if (out is None or self.aggregation == "last") else out + e
        return out
