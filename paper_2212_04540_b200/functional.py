"""Stateless hot-path ops shared by the Tape and the autograd Functions.

Each op is one (or two) libkgq launches on the current CUDA stream:

* ``graph_conv_forward``: fused KGNN layer forward -- H = A_hat.E (bit-exact
  SpMM), quantize H on chip, J = H.theta, E' = relu(J), 1-bit mask -- the
  three nodes ``record_spmm -> record_mm -> record_relu`` of model.py:81-85 in
  one kernel.  H and J never reach HBM.
* ``dequant_gemm_tn``: fused decompressor -> dtheta = Hhat^T g (tape.py:220-222).
* ``bpr_forward`` / ``bpr_backward``: the BPR + L2 head (tape.py:154-183,
  :233-244) on torch ops in the reference's op order.
"""

import ctypes
import os

import numpy as np
import torch

from . import _lib
from .quantize import (row_group_offset, PASSTHROUGH_BITS, QuantConfig, QuantizedTensor, RandomStream,
                       dequantize_tensor, packed_group_bytes, quantize_tensor)
from .tensorops import CSR, BitMask, mm, relu, spmm, spmm_phased_into

FUSED_DIMS = (32, 64, 128)


def can_fuse(cfg: QuantConfig, d: int) -> bool:
    return d in FUSED_DIMS and (cfg.passthrough or cfg.group is None or cfg.group == d)


# None = by the size of the gathered table (split at or below SPLIT_L2_BYTES).
# Round 1 chose fused beyond L2 (industry shard, 28 GB table: fused 41 vs
# split ~48 ms per layer); with the round-2 SpMM (one neighbour per batch,
# 5 CTAs/SM) and epilogues the split path wins at every measured size:
# Amazon d=64 223 vs 149 us per layer, d=128 715 vs 411 us, industry rank 7
# step 267 vs 251 ms (peak memory 90 -> 124 GB: the H buffer), so the limit
# is now unbounded.  KGQ_SPLIT_LAYER=0/1 forces one path.
SPLIT_L2_BYTES = 1 << 62
_env_split = os.environ.get("KGQ_SPLIT_LAYER")
SPLIT_LAYER_DEFAULT = None if _env_split is None else _env_split == "1"


# The split layer's epilogue (kgq_layer_epilogue_f32) may write E' over H:
# every epilogue variant is row-local and reads a tile's H rows before it
# stores that tile's E' rows (TMA or plain loads, then the J tile, then the
# stores), so the quantized layer needs one N x d buffer instead of two.  Not
# for b = 32, where H itself is the context.
EPILOGUE_IN_PLACE = True


def graph_conv_forward(adj: CSR, e: torch.Tensor, theta: torch.Tensor, cfg: QuantConfig,
                       stream: RandomStream | None, tensor_id: int | None = None,
                       row_offset: int = 0, want_h: bool = False, split: bool | None = None):
    """One fused layer.  Returns (e_next, mask, q, h) where q is the quantized
    H context (per-row groups) and h is H only if ``want_h``.

    ``split``: run it as spmm_kernel (H to a scratch buffer) + the epilogue
    kernel instead of the single fused kernel; bit-identical results.  None
    = ``SPLIT_LAYER_DEFAULT`` (by table size: split while the gathered E is
    L2-resident, where the gather kernel alone keeps full occupancy).

    ``adj`` may be a row block of the global adjacency (rows ``row_offset``..)
    with global column ids; ``e`` then holds all the rows it references.
    """
    n_rows, d = adj.shape[0], e.shape[1]
    if not can_fuse(cfg, d):
        raise ValueError("graph_conv_forward needs d in (32, 64, 128) and group == d")
    if cfg.passthrough:
        # b = 32 (quantize.py:182-183): the context is H itself, no tensor id is
        # drawn; H comes from the SpMM kernel, the epilogue does J, relu, mask
        return _graph_conv_passthrough(adj, e, theta, row_offset, want_h)
    if cfg.rounding == "stochastic":
        if stream is None:
            raise ValueError("stochastic rounding needs a RandomStream")
        if tensor_id is None:
            tensor_id = stream.next_tensor_id()
        seed = stream.seed
    else:
        seed, tensor_id = 0, 0
    dev = e.device
    e = e.contiguous()
    theta = theta.contiguous()
    codes = torch.empty((n_rows, packed_group_bytes(d, cfg.bits)), dtype=torch.uint8, device=dev)
    ranges = torch.empty(n_rows, dtype=torch.float32, device=dev)
    offsets = torch.empty(n_rows, dtype=torch.float32, device=dev)
    mask = torch.empty(((n_rows * d + 7) // 8 + 3) // 4 * 4, dtype=torch.uint8, device=dev)
    if split is None:
        split = (SPLIT_LAYER_DEFAULT if SPLIT_LAYER_DEFAULT is not None
                 else e.numel() * e.element_size() <= SPLIT_L2_BYTES)
    h = torch.empty((n_rows, d), dtype=torch.float32, device=dev) if (want_h or split) else None
    # split: E' is written over H (row-local epilogue: every tile reads its H
    # rows before it stores E'; H is scratch once quantized) unless H is wanted
    e_next = h if (split and not want_h and EPILOGUE_IN_PLACE) else \
        torch.empty((n_rows, d), dtype=torch.float32, device=dev)
    if split:
        L = _lib.load()
        st = L.kgq_spmm_csr_f32(adj.indptr.data_ptr(), adj.indices.data_ptr(), adj.data.data_ptr(), n_rows,
                                *adj.schedule(), e.data_ptr(), d, h.data_ptr(), _lib.stream_ptr(dev))
        _lib.check(st, "kgq_spmm_csr_f32")
        st = L.kgq_layer_epilogue_f32(
            h.data_ptr(), n_rows, d, theta.data_ptr(), cfg.bits, cfg.mode, seed,
            int(tensor_id) & 0xFFFFFFFFFFFFFFFF, stream.tid_base_ptr() if stream is not None else None,
            row_offset, codes.data_ptr(), ranges.data_ptr(), offsets.data_ptr(), e_next.data_ptr(),
            mask.data_ptr(), _lib.stream_ptr(dev))
        _lib.check(st, "kgq_layer_epilogue_f32")
        q = QuantizedTensor(n_rows, d, cfg.bits, codes, ranges, offsets)
        return e_next, BitMask(mask[:(n_rows * d + 7) // 8], (n_rows, d)), q, (h if want_h else None)
    st = _lib.load().kgq_layer_forward_f32(
        adj.indptr.data_ptr(), adj.indices.data_ptr(), adj.data.data_ptr(), n_rows,
        *adj.schedule(), e.data_ptr(), d,
        theta.data_ptr(), cfg.bits, cfg.mode, seed, int(tensor_id) & 0xFFFFFFFFFFFFFFFF,
        stream.tid_base_ptr() if stream is not None else None, row_offset,
        codes.data_ptr(), ranges.data_ptr(), offsets.data_ptr(), e_next.data_ptr(), mask.data_ptr(),
        _lib.ptr(h), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_layer_forward_f32")
    q = QuantizedTensor(n_rows, d, cfg.bits, codes, ranges, offsets)
    return e_next, BitMask(mask[:(n_rows * d + 7) // 8], (n_rows, d)), q, h


def layer_forward(adj: CSR, e: torch.Tensor, theta: torch.Tensor, cfg: QuantConfig,
                  stream: RandomStream | None, tensor_id: int | None = None, row_offset: int = 0):
    """One KGNN layer: the fused kernel when it applies, else the separate ops."""
    if can_fuse(cfg, e.shape[1]):
        return graph_conv_forward(adj, e, theta, cfg, stream, tensor_id, row_offset)
    return layer_forward_unfused(adj, e, theta, cfg, stream, tensor_id, row_offset)


def layer_forward_unfused(adj: CSR, e: torch.Tensor, theta: torch.Tensor, cfg: QuantConfig,
                          stream: RandomStream | None, tensor_id: int | None = None,
                          row_offset: int = 0):
    """spmm -> quantize -> mm -> relu as separate launches (any d / bits)."""
    h = spmm(adj, e)
    q = quantize_tensor(h, cfg, stream, tensor_id,
                        group_offset=row_group_offset(row_offset, h.shape[1], cfg.group))
    j = mm(h, theta)
    e_next, mask = relu(j)
    return e_next, mask, q, h


def _graph_conv_passthrough(adj: CSR, e: torch.Tensor, theta: torch.Tensor, row_offset: int, want_h: bool):
    n_rows, d = adj.shape[0], e.shape[1]
    dev = e.device
    e = e.contiguous()
    theta = theta.contiguous()
    h = torch.empty((n_rows, d), dtype=torch.float32, device=dev)
    e_next = torch.empty((n_rows, d), dtype=torch.float32, device=dev)
    mask = torch.empty(((n_rows * d + 7) // 8 + 3) // 4 * 4, dtype=torch.uint8, device=dev)
    L = _lib.load()
    st = L.kgq_spmm_csr_f32(adj.indptr.data_ptr(), adj.indices.data_ptr(), adj.data.data_ptr(), n_rows,
                            *adj.schedule(), e.data_ptr(), d, h.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_spmm_csr_f32")
    st = L.kgq_layer_epilogue_f32(h.data_ptr(), n_rows, d, theta.data_ptr(), PASSTHROUGH_BITS, 0, 0, 0, None,
                                  row_offset, None, None, None, e_next.data_ptr(), mask.data_ptr(),
                                  _lib.stream_ptr(dev))
    _lib.check(st, "kgq_layer_epilogue_f32")
    q = QuantizedTensor(n_rows, d, PASSTHROUGH_BITS, None, None, None, raw=h)
    return e_next, BitMask(mask[:(n_rows * d + 7) // 8], (n_rows, d)), q, (h if want_h else None)


def graph_conv_forward_overlap(adj: CSR, e: torch.Tensor, phases, wait_block, theta: torch.Tensor,
                               cfg: QuantConfig, stream: RandomStream | None, tensor_id: int | None = None,
                               row_offset: int = 0):
    """graph_conv_forward (split form) with a pipelined SpMM: column block p
    of ``e`` is used as soon as ``wait_block(p)`` returns (CSR.block_phases),
    then the epilogue over all rows.  Same per-row chains, same noise keys:
    bit-identical to graph_conv_forward."""
    n_rows, d = adj.shape[0], e.shape[1]
    if not can_fuse(cfg, d):
        raise ValueError("graph_conv_forward_overlap needs d in (32, 64, 128) and group == d")
    h = torch.empty((n_rows, d), dtype=torch.float32, device=e.device)
    spmm_phased_into(adj, e, h, phases, wait_block)
    return _split_epilogue(h, theta.contiguous(), cfg, stream, tensor_id, row_offset)


def _split_epilogue(h: torch.Tensor, theta: torch.Tensor, cfg: QuantConfig, stream: RandomStream | None,
                    tensor_id: int | None, row_offset: int):
    """The split layer's part 2 on a given H (kgq_layer_epilogue_f32)."""
    n_rows, d = h.shape
    dev = h.device
    mask = torch.empty(((n_rows * d + 7) // 8 + 3) // 4 * 4, dtype=torch.uint8, device=dev)
    L = _lib.load()
    if cfg.passthrough:
        e_next = torch.empty((n_rows, d), dtype=torch.float32, device=dev)
        st = L.kgq_layer_epilogue_f32(h.data_ptr(), n_rows, d, theta.data_ptr(), PASSTHROUGH_BITS, 0, 0, 0, None,
                                      row_offset, None, None, None, e_next.data_ptr(), mask.data_ptr(),
                                      _lib.stream_ptr(dev))
        _lib.check(st, "kgq_layer_epilogue_f32")
        q = QuantizedTensor(n_rows, d, PASSTHROUGH_BITS, None, None, None, raw=h)
        return e_next, BitMask(mask[:(n_rows * d + 7) // 8], (n_rows, d)), q, None
    if cfg.rounding == "stochastic":
        if stream is None:
            raise ValueError("stochastic rounding needs a RandomStream")
        if tensor_id is None:
            tensor_id = stream.next_tensor_id()
        seed = stream.seed
    else:
        seed, tensor_id = 0, 0
    codes = torch.empty((n_rows, packed_group_bytes(d, cfg.bits)), dtype=torch.uint8, device=dev)
    ranges = torch.empty(n_rows, dtype=torch.float32, device=dev)
    offsets = torch.empty(n_rows, dtype=torch.float32, device=dev)
    # H is this function's scratch: E' over it
    e_next = h if EPILOGUE_IN_PLACE else torch.empty((n_rows, d), dtype=torch.float32, device=dev)
    st = L.kgq_layer_epilogue_f32(
        h.data_ptr(), n_rows, d, theta.data_ptr(), cfg.bits, cfg.mode, seed,
        int(tensor_id) & 0xFFFFFFFFFFFFFFFF, stream.tid_base_ptr() if stream is not None else None,
        row_offset, codes.data_ptr(), ranges.data_ptr(), offsets.data_ptr(), e_next.data_ptr(),
        mask.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_layer_epilogue_f32")
    q = QuantizedTensor(n_rows, d, cfg.bits, codes, ranges, offsets)
    return e_next, BitMask(mask[:(n_rows * d + 7) // 8], (n_rows, d)), q, None


def spmm_overlap(adj: CSR, x: torch.Tensor, phases, wait_block) -> torch.Tensor:
    """adj @ x, pipelined over the column blocks of x (see graph_conv_forward_overlap)."""
    out = torch.empty((adj.shape[0], x.shape[1]), dtype=torch.float32, device=x.device)
    return spmm_phased_into(adj, x, out, phases, wait_block)


def dequant_gemm_tn(q: QuantizedTensor, g: torch.Tensor, out: torch.Tensor | None = None,
                    accumulate: bool = False) -> torch.Tensor:
    """dtheta (+)= dequantize(q)^T @ g without materializing the dequantized H."""
    if q.bits == PASSTHROUGH_BITS:
        r = q.raw.t() @ g
        if out is None:
            return r
        if accumulate:
            out.add_(r)
        else:
            out.copy_(r)
        return out
    d = q.cols
    if q.group_size != d:
        # per-group contexts: dequantize then GEMM (rare path)
        r = dequantize_tensor(q).t() @ g
        if out is None:
            return r
        return out.add_(r) if accumulate else out.copy_(r)
    g = g.contiguous()
    dev = g.device
    if out is None:
        out = torch.empty((d, d), dtype=torch.float32, device=dev)
        accumulate = False
    L = _lib.load()
    ws_bytes = int(L.kgq_dequant_gemm_workspace_bytes(q.rows, d))
    ws = torch.empty(max(ws_bytes, 4) // 4, dtype=torch.float32, device=dev)
    st = L.kgq_dequant_gemm_tn_f32(q.codes.data_ptr(), q.ranges.data_ptr(), q.offsets.data_ptr(),
                                   q.rows, d, q.bits, g.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                   ws_bytes, 1 if accumulate else 0, _lib.stream_ptr(dev))
    _lib.check(st, "kgq_dequant_gemm_tn_f32")
    return out


class SparseRows:
    """A row-sparse gradient: row r is ``rows[rowmap[r]]`` when rowmap[r] >= 0,
    else +0 -- the readout gradient of a training batch (the scatter of the
    B-row gathers, ~3B of N rows) as kgq_scatter_rows_multi_sparse_f32 leaves
    it.  ``dense()`` materializes the N x d tensor (once, cached) for the
    consumers that need it; the tensor-core layer backward reads it as is."""

    def __init__(self, rowmap: torch.Tensor, rows: torch.Tensor, n_rows: int):
        self.rowmap, self.rows, self.n_rows = rowmap, rows, int(n_rows)
        self._dense = None

    @property
    def shape(self):
        return (self.n_rows, self.rows.shape[1])

    @property
    def device(self):
        return self.rows.device

    def dense(self) -> torch.Tensor:
        if self._dense is None:           # gather with a zero row in front: no host sync
            ext = torch.cat([self.rows.new_zeros((1, self.rows.shape[1])), self.rows])
            self._dense = ext.index_select(0, (self.rowmap + 1).to(torch.int64))
        return self._dense


def _rows_concat(parts, d: int) -> torch.Tensor:
    """torch.cat of fp32 row blocks, or a view when they already lie back to
    back in one buffer in this order (the BPR gradients, bpr_backward)."""
    parts = [x.reshape(-1, d) for x in parts]
    p0 = parts[0]
    if all(x.dtype == torch.float32 and x.is_contiguous() for x in parts):
        base, off, ok = p0.untyped_storage().data_ptr(), p0.data_ptr(), True
        for x in parts:
            if x.untyped_storage().data_ptr() != base or x.data_ptr() != off:
                ok = False
                break
            off += x.numel() * 4
        if ok:
            n = sum(x.shape[0] for x in parts)
            return p0.as_strided((n, d), (d, 1))
    return torch.cat([x.to(torch.float32) for x in parts]).contiguous()


def scatter_rows_multi_sparse(src_rows: int, idxs, gs):
    """scatter_rows_multi in compact form (SparseRows); None when the
    sort-free kernel does not apply (the caller takes the dense path)."""
    d = gs[0].shape[1]
    m = sum(int(i.numel()) for i in idxs)
    if m == 0 or m > 16384 or d > 128 or len(idxs) > 8 or not gs[0].is_cuda:
        return None
    dev = gs[0].device
    idx = torch.cat([i.reshape(-1).to(torch.int32) for i in idxs])
    g = _rows_concat(gs, d)
    ends = np.ascontiguousarray(np.cumsum([i.numel() for i in idxs]), dtype=np.int64)
    rows = torch.empty((m, d), dtype=torch.float32, device=dev)
    rowmap = torch.full((src_rows,), -1, dtype=torch.int32, device=dev)
    st = _lib.load().kgq_scatter_rows_multi_sparse_f32(idx.data_ptr(), m, ends.ctypes.data, len(idxs), g.data_ptr(),
                                                       d, rows.data_ptr(), rowmap.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_scatter_rows_multi_sparse_f32")
    return SparseRows(rowmap, rows, src_rows)


def layer_backward(g_read, g_e, mask: BitMask, q: QuantizedTensor, theta: torch.Tensor):
    """Fused layer backward (tape.py:217-225): returns (dtheta, dh) for
    g_j = (g_read + g_e) * mask, dh = g_j theta^T, dtheta = Hhat^T g_j, with
    the dequantized H never materialized.  Falls back to the separate ops for
    d not in (32, 64, 128) or pass-through contexts.  ``g_read`` may be a
    SparseRows (read compactly by the d = 64 tensor-core kernel)."""
    from .tensorops import mask_apply, mm_theta
    if isinstance(g_read, SparseRows):
        d = g_read.shape[1]
        if d == 64 and (q.bits == PASSTHROUGH_BITS or q.group_size == d) and \
                not (q.bits == PASSTHROUGH_BITS and q.raw is None):
            passthrough = q.bits == PASSTHROUGH_BITS
            dev = g_read.device
            rows = g_read.n_rows
            dh = torch.empty((rows, d), dtype=torch.float32, device=dev)
            dth = torch.empty((d, d), dtype=torch.float32, device=dev)
            L = _lib.load()
            ws_bytes = int(L.kgq_layer_backward_workspace_bytes(rows, d))
            ws = torch.empty(max(ws_bytes, 4) // 4, dtype=torch.float32, device=dev)
            ge = None if g_e is None else g_e.contiguous()
            codes_ptr = q.raw.contiguous().data_ptr() if passthrough else q.codes.data_ptr()
            st = L.kgq_layer_backward_rows_f32(g_read.rowmap.data_ptr(), g_read.rows.data_ptr(), _lib.ptr(ge),
                                               mask.packed.data_ptr(), codes_ptr, _lib.ptr(q.ranges),
                                               _lib.ptr(q.offsets), rows, d, q.bits, theta.contiguous().data_ptr(),
                                               dh.data_ptr(), dth.data_ptr(), ws.data_ptr(), ws_bytes, 0,
                                               _lib.stream_ptr(dev))
            if st == _lib.KGQ_OK:
                return dth, dh
            if st != _lib.KGQ_ERR_INVALID_ARG:
                _lib.check(st, "kgq_layer_backward_rows_f32")
        g_read = g_read.dense()
    src = g_read if g_read is not None else g_e
    d = src.shape[1]
    passthrough = q.bits == PASSTHROUGH_BITS
    if d not in (32, 64, 128) or (not passthrough and q.group_size != d) or (passthrough and q.raw is None):
        g = g_read if g_e is None else (g_e if g_read is None else g_read + g_e)
        g_j = mask_apply(g, mask)
        return dequant_gemm_tn(q, g_j), mm_theta(g_j, theta, transpose=True)
    dev = src.device
    rows = src.shape[0]
    dh = torch.empty((rows, d), dtype=torch.float32, device=dev)
    dth = torch.empty((d, d), dtype=torch.float32, device=dev)
    L = _lib.load()
    ws_bytes = int(L.kgq_layer_backward_workspace_bytes(rows, d))
    ws = torch.empty(max(ws_bytes, 4) // 4, dtype=torch.float32, device=dev)
    gr = None if g_read is None else g_read.contiguous()
    ge = None if g_e is None else g_e.contiguous()
    codes_ptr = q.raw.contiguous().data_ptr() if passthrough else q.codes.data_ptr()   # b=32: fp32 H
    st = L.kgq_layer_backward_f32(_lib.ptr(gr), _lib.ptr(ge), mask.packed.data_ptr(),
                                  codes_ptr, _lib.ptr(q.ranges), _lib.ptr(q.offsets), rows,
                                  d, q.bits, theta.contiguous().data_ptr(), dh.data_ptr(),
                                  dth.data_ptr(), ws.data_ptr(), ws_bytes, 0, _lib.stream_ptr(dev))
    _lib.check(st, "kgq_layer_backward_f32")
    return dth, dh


def bpr_forward(u: torch.Tensor, p: torch.Tensor, n: torch.Tensor, l2: float):
    """tape.py:162-166: margins = sum(u*(p-n)); loss = mean softplus(-m) +
    l2*(|u|^2+|p|^2+|n|^2)/B, one kernel (kgq_bpr_forward_f32).  Returns
    (loss 0-d tensor, margins)."""
    batch, d = u.shape
    dev = u.device
    u, p, n = u.contiguous(), p.contiguous(), n.contiguous()
    margins = torch.empty(batch, dtype=torch.float32, device=dev)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    L = _lib.load()
    ws_bytes = int(L.kgq_bpr_forward_workspace_bytes(batch))
    ws = torch.empty(max(ws_bytes, 4) // 4, dtype=torch.float32, device=dev)
    st = L.kgq_bpr_forward_f32(u.data_ptr(), p.data_ptr(), n.data_ptr(), batch, d, float(l2),
                               margins.data_ptr(), loss.data_ptr(), ws.data_ptr(), ws_bytes, _lib.stream_ptr(dev))
    _lib.check(st, "kgq_bpr_forward_f32")
    return loss, margins


def bpr_backward(g, margins, uh, ph, nh, l2: float, batch: int):
    """tape.py:233-244 (against the dequantized blocks, exact margins), one
    elementwise kernel (kgq_bpr_backward_f32); g is a 0-d device tensor."""
    d = uh.shape[1]
    dev = uh.device
    # one buffer, negatives first: the backward scatters the gathers' gradients
    # in reverse record order (n, p, u), which then need no concatenation
    buf = torch.empty((3,) + tuple(uh.shape), dtype=torch.float32, device=dev)
    gn, gp, gu = buf[0], buf[1], buf[2]
    g = g.reshape(()).to(device=dev, dtype=torch.float32).contiguous()
    reg = float(np.float32(2.0 * l2 / batch))
    st = _lib.load().kgq_bpr_backward_f32(g.data_ptr(), margins.contiguous().data_ptr(), uh.contiguous().data_ptr(),
                                          ph.contiguous().data_ptr(), nh.contiguous().data_ptr(), batch, d, reg,
                                          gu.data_ptr(), gp.data_ptr(), gn.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_bpr_backward_f32")
    return gu, gp, gn


def scatter_rows(src_rows: int, idx: torch.Tensor, g: torch.Tensor) -> torch.Tensor:
    """np.add.at(zeros, idx, g) (tape.py:229-231), deterministic."""
    return scatter_rows_multi(src_rows, [idx], [g])


def scatter_rows_multi(src_rows: int, idxs, gs) -> torch.Tensor:
    """((s_0 + s_1) + ...) with s_i = np.add.at(zeros, idxs[i], gs[i]): the
    reference's dense sum of several gathers' scatters (tape.py:204-209,
    229-232), bit-deterministic (kgq_scatter_rows_multi_f32; positions
    sorted by (row, position), one warp per row)."""
    dev = gs[0].device
    d = gs[0].shape[1]
    idx = torch.cat([i.reshape(-1).to(torch.int32) for i in idxs])
    g = torch.cat([x.reshape(-1, d).to(torch.float32) for x in gs]).contiguous()
    m = idx.numel()
    out = torch.zeros((src_rows, d), dtype=torch.float32, device=dev)
    if m == 0:
        return out
    ends = np.ascontiguousarray(np.cumsum([i.numel() for i in idxs]), dtype=np.int64)   # host, by value
    order = None
    if m > 16384 or d > 128:     # the sort-free kernel is quadratic in m, <= 128 features
        key = idx.to(torch.int64) * m + torch.arange(m, device=dev, dtype=torch.int64)
        order = torch.sort(key).indices
    if len(idxs) > 8:
        raise ValueError("at most 8 gathers per scatter")
    st = _lib.load().kgq_scatter_rows_multi_f32(_lib.ptr(order), idx.data_ptr(), m, ends.ctypes.data, len(idxs),
                                                g.data_ptr(), d, out.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_scatter_rows_multi_f32")
    return out

def gather_rows_sum(terms, idx64: torch.Tensor) -> torch.Tensor:
    """((terms[0][idx] + terms[1][idx]) + ...) in one kernel
    (kgq_gather_rows_sum_f32): the rows of the sum readout, bit-identical to
    gathering the materialized sum."""
    t0 = terms[0]
    d = t0.shape[1]
    out = torch.empty((idx64.shape[0], d), dtype=torch.float32, device=t0.device)
    ptrs = (ctypes.c_void_p * len(terms))(*[t.data_ptr() for t in terms])
    st = _lib.load().kgq_gather_rows_sum_f32(ctypes.cast(ptrs, ctypes.c_void_p), len(terms),
                                             idx64.contiguous().data_ptr(), idx64.shape[0], d, out.data_ptr(),
                                             _lib.stream_ptr(t0.device))
    _lib.check(st, "kgq_gather_rows_sum_f32")
    return out


def gather_rows_acc(base: torch.Tensor, terms, idx64: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """((base + terms[0][idx]) + terms[1][idx]) + ... into ``out`` (default:
    in place on ``base``) with kgq_gather_rows_acc_f32: a gathered sum readout
    accumulated term by term, bit-identical to gather_rows_sum over all the
    terms."""
    d = base.shape[1]
    out = base if out is None else out
    ptrs = (ctypes.c_void_p * len(terms))(*[t.data_ptr() for t in terms])
    st = _lib.load().kgq_gather_rows_acc_f32(base.data_ptr(), ctypes.cast(ptrs, ctypes.c_void_p), len(terms),
                                             idx64.contiguous().data_ptr(), idx64.shape[0], d, out.data_ptr(),
                                             _lib.stream_ptr(base.device))
    _lib.check(st, "kgq_gather_rows_acc_f32")
    return out


def topk_rows(scores: torch.Tensor, k: int) -> torch.Tensor:
    """Indices of the k best entries of every row of a fp32 score block, best
    first, ties by ascending column (kgq_topk_rows_f32; the stable
    ``np.argsort(-s, kind="stable")[:k]`` of train.py:141-143); int32, -1
    past the row length.  1 <= k <= 64 runs the K11 kernel; the reference
    accepts any K, so k > 64 ranks with a stable device sort of -s (NaN last,
    as numpy's argsort)."""
    if scores.dtype != torch.float32 or scores.dim() != 2 or not scores.is_cuda:
        raise TypeError("topk_rows: expected a 2-D fp32 CUDA tensor")
    if k < 1:
        raise ValueError("topk_rows: k must be >= 1")
    if scores.stride(1) != 1:
        scores = scores.contiguous()
    n, m = scores.shape
    if k > 64:
        order = torch.sort(-scores, dim=1, stable=True).indices[:, :k].to(torch.int32)
        if k > m:
            order = torch.cat([order, order.new_full((n, k - m), -1)], 1)
        return order
    out = torch.empty((n, k), dtype=torch.int32, device=scores.device)
    st = _lib.load().kgq_topk_rows_f32(scores.data_ptr(), n, m, scores.stride(0), k, out.data_ptr(),
                                       _lib.stream_ptr(scores.device))
    _lib.check(st, "kgq_topk_rows_f32")
    return out


def score_topk(readout: torch.Tensor, users: torch.Tensor, item_emb: torch.Tensor, train_items: torch.Tensor,
               train_start: torch.Tensor, train_end: torch.Tensor, k: int) -> torch.Tensor:
    """K12 (kgq_score_topk_f32): for each user row readout[users[i]], the k
    best items of its dot products with item_emb after its train positives
    train_items[train_start[i]:train_end[i]] (sorted) are set to -inf -- the
    score block + ``np.argsort(-s, kind="stable")[:k]`` of train.py:121-160
    with no score block in memory (3xTF32 tensor-core scores, fp32-level).
    d in {32, 64}, 1 <= k <= 32; int32 (n_users, k), -1 past the item count."""
    n, d = readout.shape
    I = item_emb.shape[0]
    if not (readout.is_cuda and readout.dtype == torch.float32 and item_emb.dtype == torch.float32):
        raise TypeError("score_topk: fp32 CUDA tensors expected")
    if d not in (32, 64) or not 1 <= k <= 32:
        raise ValueError("score_topk: d must be 32 or 64 and 1 <= k <= 32")
    readout, item_emb = readout.contiguous(), item_emb.contiguous()
    users = users.to(torch.int64).contiguous()
    out = torch.empty((users.numel(), k), dtype=torch.int32, device=readout.device)
    lib = _lib.load()
    ws = torch.empty(lib.kgq_score_topk_workspace_bytes(I, d), dtype=torch.uint8, device=readout.device)
    st = lib.kgq_score_topk_f32(readout.data_ptr(), users.data_ptr(), users.numel(), item_emb.data_ptr(), I, d,
                                train_items.to(torch.int32).contiguous().data_ptr(),
                                train_start.to(torch.int64).contiguous().data_ptr(),
                                train_end.to(torch.int64).contiguous().data_ptr(), k, out.data_ptr(),
                                ws.data_ptr(), ws.numel(), _lib.stream_ptr(readout.device))
    _lib.check(st, "kgq_score_topk_f32")
    return out
