"""Row-partitioned multi-GPU training step.

Nodes are split into contiguous equal-nnz row ranges (``data.partition_rows``);
rank r owns rows [lo, hi) of the adjacency (global column ids), of E0 and of
every layer's activations.  Per layer and direction there is one exchange:

    forward : E^(l)  all-gather  -> local fused layer (spmm -> quantize -> mm -> relu)
    backward: dH     all-gather  -> local spmm (A_hat symmetric: dE = A_local . dH)
    params  : dtheta all-reduce (L*d*d floats), E0 rows stay local

plus one exchange of the 3*B readout rows of the batch (all-reduce of an
owner-filled 3B x d block, the readout summed over layers at those rows only)
so every rank evaluates the (tiny) BPR head on the same batch.  The gathers can target a padded [world*max_count] layout whose
row ids the local CSR is remapped to once, so the collective writes the
SpMM's input directly (no concatenation copy of a full N x d tensor).  The quantization noise is keyed by GLOBAL row
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

    def all_gather_padded(self, local: torch.Tensor, m: int, out: torch.Tensor | None = None) -> torch.Tensor:
        """Every rank's block in a [world*m, ...] buffer, block r at rows
        [r*m, r*m + count_r) (the padded layout ``RowPartition.padded_cols``
        indexes), so no concatenation copy follows the collective."""
        if out is None:
            out = local.new_empty((self.world * m,) + tuple(local.shape[1:]))
        if local.shape[0] == m:
            buf = local.contiguous()
        else:
            buf = local.new_zeros((m,) + tuple(local.shape[1:]))
            buf[:local.shape[0]] = local
        if self.gloo:
            parts = [torch.empty_like(buf, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, buf.cpu(), group=self.group)
            out.copy_(torch.cat(parts, 0))
        else:
            self.dist.all_gather_into_tensor(out, buf, group=self.group)
        return out

    def all_gather_global(self, local: torch.Tensor, cuts, out: torch.Tensor | None = None) -> torch.Tensor:
        """All-gather-v into the GLOBAL row layout: rank r's block lands at
        rows [cuts[r], cuts[r+1]) of one [n, ...] buffer (one broadcast per
        source rank, issued together), so uneven equal-nnz blocks move
        exactly n - count rows per rank and the local CSR keeps its global
        column ids (no padding, no concatenation copy)."""
        out, pending = self.all_gather_global_start(local, cuts, out)
        pending.wait()
        return out

    def all_gather_global_start(self, local: torch.Tensor, cuts, out: torch.Tensor | None = None):
        """all_gather_global, returned before the remote blocks have landed:
        (out, pending).  The local block is in ``out`` at once (rows [lo, hi),
        copied on the caller's stream before the collectives are issued), so
        work that reads only those rows can run while the broadcasts of the
        others are in flight; ``pending.wait()`` orders the caller's stream
        after them (NCCL) or completes them (gloo)."""
        n = int(cuts[-1])
        lo, hi = int(cuts[self.rank]), int(cuts[self.rank + 1])
        if out is None:
            out = local.new_empty((n,) + tuple(local.shape[1:]))
        out[lo:hi].copy_(local)
        stage = out.cpu() if (self.gloo and out.is_cuda) else out
        works = {r: self.dist.broadcast(stage[int(cuts[r]):int(cuts[r + 1])], src=r, group=self.group,
                                        async_op=True) for r in range(self.world) if cuts[r + 1] > cuts[r]}
        return out, _Pending(works, stage, out, cuts=cuts)

    def all_gather_padded_start(self, local: torch.Tensor, m: int, out: torch.Tensor | None = None):
        """all_gather_padded, returned before the remote blocks have landed:
        (out, pending); the local block is copied into its slot first and the
        collective runs in place (NCCL skips the own slot), so the slot can be
        read meanwhile."""
        if out is None:
            out = local.new_empty((self.world * m,) + tuple(local.shape[1:]))
        mine = out[self.rank * m:(self.rank + 1) * m]
        mine[:local.shape[0]].copy_(local)
        if local.shape[0] < m:
            mine[local.shape[0]:].zero_()
        if self.gloo:
            parts = [torch.empty_like(mine, device="cpu") for _ in range(self.world)]
            w = self.dist.all_gather(parts, mine.cpu(), group=self.group, async_op=True)
            return out, _Pending({None: w}, None, out, parts=parts)
        w = self.dist.all_gather_into_tensor(out, mine, group=self.group, async_op=True)
        return out, _Pending({None: w}, None, out)

    def gather_index_rows(self, local: torch.Tensor, lo: int, idx: torch.Tensor) -> torch.Tensor:
        """rows ``idx`` (global ids) of the row-partitioned tensor whose block
        [lo, lo+len(local)) lives here: each rank fills the rows it owns and
        the others contribute +0, so the all-reduce sum is exact."""
        sel = (idx >= lo) & (idx < lo + local.shape[0])
        out = local.new_zeros((idx.shape[0],) + tuple(local.shape[1:]))
        out[sel] = local[idx[sel] - lo]
        return self.all_reduce_sum(out)

    def all_to_all_v(self, send: torch.Tensor, send_counts, recv_counts, out: torch.Tensor | None = None):
        """Rows send[sum(send_counts[:r]) : +send_counts[r]] go to rank r; the
        rows from rank r land at out[sum(recv_counts[:r]) : ...] (NCCL
        all_to_all_single with split sizes; gloo on CPU tensors)."""
        n_out = int(sum(recv_counts))
        if out is None:
            out = send.new_empty((n_out,) + tuple(send.shape[1:]))
        if self.gloo and send.is_cuda:
            o = torch.empty((n_out,) + tuple(send.shape[1:]), dtype=send.dtype)
            self.dist.all_to_all_single(o, send.cpu(), output_split_sizes=[int(c) for c in recv_counts],
                                        input_split_sizes=[int(c) for c in send_counts], group=self.group)
            out.copy_(o)
        else:
            self.dist.all_to_all_single(out, send.contiguous(), output_split_sizes=[int(c) for c in recv_counts],
                                        input_split_sizes=[int(c) for c in send_counts], group=self.group)
        return out

    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        if self.gloo and t.is_cuda:
            c = t.cpu()
            self.dist.all_reduce(c, group=self.group)
            t.copy_(c)
        else:
            self.dist.all_reduce(t, group=self.group)
        return t


class _Pending:
    """In-flight exchange.  ``wait()`` completes it; ``wait_source(r)`` only
    the block of source rank r (per-source broadcasts; a single collective
    waits whole).  gloo stages through host memory and copies back."""

    def __init__(self, works: dict, stage, out, parts=None, cuts=None):
        self.works, self.stage, self.out, self.parts, self.cuts = works, stage, out, parts, cuts

    def wait_source(self, r: int):
        if None in self.works or self.cuts is None:
            return self.wait()
        w = self.works.pop(r, None)
        if w is not None:
            w.wait()
            if self.stage is not None and self.stage is not self.out:
                a, b = int(self.cuts[r]), int(self.cuts[r + 1])
                self.out[a:b].copy_(self.stage[a:b])

    def wait(self):
        for w in self.works.values():
            w.wait()
        self.works = {}
        if self.parts is not None:
            self.out.copy_(torch.cat(self.parts, 0))
            self.parts = None
        if self.stage is not None and self.stage is not self.out:
            self.out.copy_(self.stage)
            self.stage = None


class _Done:
    def wait(self):
        pass

    def wait_source(self, r):
        pass


class SoloComm:
    """World size 1 (no communication)."""
    world, rank = 1, 0

    def all_gather_global_start(self, local, cuts, out=None):
        return local, _Done()

    def all_gather_padded_start(self, local, m, out=None):
        return local, _Done()

    def all_gather_rows(self, local, counts):
        return local

    def all_gather_padded(self, local, m, out=None):
        return local

    def all_gather_global(self, local, cuts, out=None):
        return local

    def gather_index_rows(self, local, lo, idx):
        return local[idx - lo]

    def all_to_all_v(self, send, send_counts, recv_counts, out=None):
        return send if out is None else out.copy_(send)

    def all_reduce_sum(self, t):
        return t


class SimulatedRankComm:
    """One rank of a ``world``-way partition run alone on one GPU (the 8-GPU
    configurations measured on a 1-GPU box): collectives keep their shapes
    and buffers, but the other ranks' blocks are whatever the persistent
    gather buffers hold (initialised once, standing in for remote rows) and
    reductions see only this rank's contribution.  Compute per rank is
    exactly the real one; communication is not timed (bytes are reported
    analytically by the caller).  Not for correctness runs."""

    def __init__(self, world: int, rank: int, fill_std: float = 0.1, seed: int = 0):
        self.world, self.rank = world, rank
        self.fill_std, self.seed = fill_std, seed
        self._bufs = {}

    def _buf(self, key, shape, like):
        b = self._bufs.get(key)
        if b is None or tuple(b.shape) != tuple(shape):
            g = torch.Generator(device=like.device).manual_seed(self.seed + len(self._bufs))
            b = torch.empty(shape, dtype=like.dtype, device=like.device)
            b.normal_(0.0, self.fill_std, generator=g).abs_()
            self._bufs[key] = b
        return b

    def all_gather_padded(self, local, m, out=None):
        buf = self._buf("gather", (self.world * m,) + tuple(local.shape[1:]), local) if out is None else out
        buf[self.rank * m:self.rank * m + local.shape[0]].copy_(local)
        return buf

    def all_gather_global(self, local, cuts, out=None):
        n = int(cuts[-1])
        buf = self._buf("gather", (n,) + tuple(local.shape[1:]), local) if out is None else out
        lo = int(cuts[self.rank])
        buf[lo:lo + local.shape[0]].copy_(local)
        return buf

    def all_gather_global_start(self, local, cuts, out=None):
        return self.all_gather_global(local, cuts, out), _Done()

    def all_gather_padded_start(self, local, m, out=None):
        return self.all_gather_padded(local, m, out), _Done()

    def gather_index_rows(self, local, lo, idx):
        out = self._buf(("rows", idx.shape[0]), (idx.shape[0],) + tuple(local.shape[1:]), local)
        sel = (idx >= lo) & (idx < lo + local.shape[0])
        out[sel] = local[idx[sel] - lo]
        return out

    def all_to_all_v(self, send, send_counts, recv_counts, out=None):
        """The received halo rows keep their stand-in values (filled once)."""
        n_out = int(sum(recv_counts))
        if out is not None:
            if "halo_fill" not in self._bufs:
                self._bufs["halo_fill"] = True
                g = torch.Generator(device=out.device).manual_seed(self.seed + 17)
                out.normal_(0.0, self.fill_std, generator=g).abs_()
            return out
        return self._buf(("a2a", n_out), (n_out,) + tuple(send.shape[1:]), send)

    def all_reduce_sum(self, t):
        return t


class HaloPlan:
    """Boundary ("halo") exchange of one rank of a row partition: instead of
    all-gathering every row, the rank receives only the remote rows its CSR
    block references and sends the local rows the other ranks reference
    (one all_to_all_v per exchange).  Local CSR columns are remapped once to
    a compact space: [0, n_local) the rank's own rows, [n_local, n_local +
    n_halo) the halo rows in (owner, global id) order.  Same values in the
    same per-row column order -> the SpMM is bit-identical to the full
    all-gather."""

    def __init__(self, part, remote_ids: torch.Tensor, recv_counts, send_counts, send_idx: torch.Tensor):
        self.part = part
        self.n_local = part.hi - part.lo
        self.remote_ids = remote_ids            # int64, sorted, device
        self.n_halo = int(remote_ids.numel())
        self.recv_counts = [int(c) for c in recv_counts]
        self.send_counts = [int(c) for c in send_counts]
        self.send_idx = send_idx                # int64 local row ids, grouped by destination rank

    @classmethod
    def build(cls, part, cols: torch.Tensor, comm) -> "HaloPlan":
        """cols: the block's global column ids (any order).  Collective: every
        rank of the partition calls it (counts, then the requested ids, are
        exchanged with all_to_all_v)."""
        dev = cols.device
        lo, hi = part.lo, part.hi
        u = torch.unique(cols.to(torch.int64))
        remote = u[(u < lo) | (u >= hi)]
        cuts = torch.as_tensor(np.asarray(part.cuts, dtype=np.int64), device=dev)
        owner = torch.searchsorted(cuts, remote, right=True) - 1
        recv_counts = torch.bincount(owner, minlength=part.world).to(torch.int64)
        ones = [1] * part.world
        send_counts = comm.all_to_all_v(recv_counts.reshape(-1, 1), ones, ones).reshape(-1)
        rc, sc = recv_counts.cpu().tolist(), send_counts.cpu().tolist()
        requested = comm.all_to_all_v(remote.reshape(-1, 1), rc, sc).reshape(-1)
        return cls(part, remote, rc, sc, (requested - lo).to(torch.int64))

    def remap(self, cols: torch.Tensor) -> torch.Tensor:
        """Global column ids -> compact ids (int32)."""
        c = cols.to(torch.int64)
        lo, hi = self.part.lo, self.part.hi
        local = (c >= lo) & (c < hi)
        pos = torch.searchsorted(self.remote_ids, c)
        return torch.where(local, c - lo, self.n_local + pos).to(torch.int32)

    def exchange(self, x_local: torch.Tensor, comm, out: torch.Tensor | None = None) -> torch.Tensor:
        """[own rows | halo rows] for the SpMM: one all_to_all_v of the rows
        the other ranks reference."""
        if self.n_halo == 0 and sum(self.send_counts) == 0:
            return x_local
        d = x_local.shape[1]
        if out is None:
            out = x_local.new_empty((self.n_local + self.n_halo, d))
        out[:self.n_local].copy_(x_local)
        send = x_local.index_select(0, self.send_idx)
        comm.all_to_all_v(send, self.send_counts, self.recv_counts, out=out[self.n_local:])
        return out

    def recv_bytes(self, d: int) -> int:
        return self.n_halo * d * 4

    def send_bytes(self, d: int) -> int:
        return int(sum(self.send_counts)) * d * 4


class GpuOps:
    """The product path: libkgq kernels."""

    @staticmethod
    def local_adjacency(indptr, indices, vals, lo, hi, n, device, part: "RowPartition | None" = None):
        """CSR rows [lo, hi); with ``part`` the column ids index the padded
        gather buffer (``all_gather_padded``) instead of the global rows."""
        ip, ix, vv = row_block(indptr, indices, vals, lo, hi)
        if part is not None:
            ix = part.padded_cols(ix)
            if part.world * part.block >= 1 << 31:
                raise ValueError("padded gather layout exceeds int32 column ids")
            ix = ix.astype(np.int32)
            n = part.world * part.block
        return CSR.from_arrays(ip, ix, vv, (hi - lo, n), device=device, symmetric=False)

    graph_conv = staticmethod(F.layer_forward)
    dequant_gemm = staticmethod(F.dequant_gemm_tn)
    mask_apply = staticmethod(mask_apply)
    spmm = staticmethod(spmm)
    quantize = staticmethod(quantize_tensor)
    dequantize = staticmethod(dequantize_tensor)
    scatter_rows = staticmethod(F.scatter_rows)
    scatter_rows_multi = staticmethod(F.scatter_rows_multi)
    bpr_forward = staticmethod(F.bpr_forward)
    bpr_backward = staticmethod(F.bpr_backward)

    layer_backward = staticmethod(F.layer_backward)

    @staticmethod
    def overlap_plan(a_local, col_cuts):
        """Per source block: row ranges + schedules of the local block (CSR.block_phases)."""
        return a_local.block_phases(col_cuts)

    @staticmethod
    def graph_conv_overlap(a_local, plan, e_full, wait_block, theta, cfg, stream, row_offset=0):
        return F.graph_conv_forward_overlap(a_local, e_full, plan, wait_block, theta, cfg, stream,
                                            row_offset=row_offset)

    @staticmethod
    def spmm_overlap(a_local, plan, x, wait_block):
        return F.spmm_overlap(a_local, x, plan, wait_block)


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

    @property
    def block(self) -> int:
        """Rows per block of the padded gather layout (max count)."""
        return max(self.counts)

    def padded_cols(self, cols: np.ndarray) -> np.ndarray:
        """Global row id -> row of the padded [world*block] gather buffer."""
        cols = np.asarray(cols, dtype=np.int64)
        r = np.searchsorted(self.cuts, cols, side="right") - 1
        return (r * self.block + (cols - self.cuts[r])).astype(np.int64)

    def preferred_layout(self, max_imbalance: float = 1.05) -> str:
        """The E / dH exchange layout for this partition: one
        all_gather_into_tensor into the padded [world*block] buffer when the
        row blocks are near-equal (max/min <= ``max_imbalance``: the padding
        moves almost nothing extra), else the exact all-gather-v ("global").
        Equal-nnz cuts of the reference KGs are far from equal in rows
        (Amazon max/min 1.31 / 5.4 / 13.4 at W = 2 / 4 / 8), so they take
        "global"; equal-row partitions take "padded"."""
        c = self.counts
        return "padded" if min(c) > 0 and max(c) / min(c) <= max_imbalance else "global"

    @classmethod
    def build(cls, indptr, world: int, rank: int) -> "RowPartition":
        return cls(world, rank, partition_rows(indptr, world), len(indptr) - 1)


def partitioned_step(part: RowPartition, a_local, e0_local: torch.Tensor, thetas, users, pos, neg,
                     l2: float, cfg: QuantConfig, stream: RandomStream, comm, ops=GpuOps,
                     padded: bool = False, layout: str | None = None, halo: "HaloPlan | None" = None,
                     overlap: bool = False, plan=None):
    """One forward+backward of the KGNN backbone + BPR head on this rank's
    rows.  Returns (loss tensor, dE0 for the local rows, [dtheta_i] summed
    over ranks).  Mirrors tape.py:193-253's routing order.

    ``layout`` of the E / dH exchanges: "concat" (all_gather of padded
    blocks, then concatenated), "padded" (``a_local`` indexes the padded
    layout, ``GpuOps.local_adjacency(..., part=part)``: one
    all_gather_into_tensor, no copy; best for equal-row blocks) or "global"
    (all-gather-v by per-source broadcasts into the global layout: exact
    bytes for uneven equal-nnz blocks, global column ids, no copy) or "halo"
    (only the rows the block references, ``HaloPlan``; ``a_local`` columns
    remapped by ``HaloPlan.remap``).  ``padded=True`` is shorthand for
    layout="padded".  The BPR head only
    needs the 3*B batch rows of the readout: they are exchanged by index
    (``gather_index_rows``), never the whole readout."""
    lo, counts = part.lo, part.counts
    m = part.block

    layout = layout or ("halo" if halo is not None else "padded" if padded else "concat")
    if layout not in ("concat", "padded", "global", "halo"):
        raise ValueError(f"unknown exchange layout {layout!r}")
    if layout == "halo" and halo is None:
        raise ValueError("layout='halo' needs a HaloPlan (a_local remapped with HaloPlan.remap)")

    if overlap:
        if layout != "global":
            raise ValueError("overlap needs layout 'global' (one broadcast per source block)")
        if plan is None:
            plan = ops.overlap_plan(a_local, part.cuts)

    def gather_start(x):
        return comm.all_gather_global_start(x, part.cuts)

    def gather(x):
        if layout == "halo":
            return halo.exchange(x, comm)
        if layout == "padded":
            return comm.all_gather_padded(x, m)
        if layout == "global":
            return comm.all_gather_global(x, part.cuts)
        return comm.all_gather_rows(x, counts)

    saved = []
    e_local = e0_local
    # the sum readout is only read at the batch rows: accumulate those rows
    # layer by layer ((E1 + E2) + E3, the reference's order, on 3B x d
    # instead of N x d), owner-filled, then one exact all-reduce
    # (no boolean indexing: fixed shapes, no host synchronisation)
    idx = torch.cat([users, pos, neg])
    n_loc = e0_local.shape[0]
    own = (idx >= lo) & (idx < lo + n_loc)
    li = torch.clamp(idx - lo, 0, max(n_loc - 1, 0)).to(torch.int64)
    acc_rows = None
    for theta in thetas:
        if overlap:
            e_full, pending = gather_start(e_local)
            e_next, mask, q, _ = ops.graph_conv_overlap(a_local, plan, e_full, pending.wait_source, theta, cfg,
                                                        stream, row_offset=lo)
        else:
            e_full = gather(e_local)
            e_next, mask, q, _ = ops.graph_conv(a_local, e_full, theta, cfg, stream, row_offset=lo)
        saved.append((mask, q))
        r_l = e_next.index_select(0, li)
        acc_rows = r_l if acc_rows is None else acc_rows + r_l
        e_local = e_next
    b = users.shape[0]
    block = torch.where(own[:, None], acc_rows, torch.zeros((), dtype=acc_rows.dtype, device=acc_rows.device))
    rows = comm.all_reduce_sum(block)
    u, p, n = rows[:b], rows[b:2 * b], rows[2 * b:]
    loss, margins = ops.bpr_forward(u, p, n, l2)
    qu, qp, qn = (ops.quantize(t, cfg, stream) for t in (u, p, n))
    one = torch.ones((), dtype=u.dtype, device=u.device)
    gu, gp, gn = ops.bpr_backward(one, margins, ops.dequantize(qu), ops.dequantize(qp),
                                ops.dequantize(qn), l2, u.shape[0])
    # readout gradient rows owned here: (scat_n + scat_p) + scat_u (reference.py:59-67),
    # one deterministic scatter; rows owned by other ranks carry index -1 (skipped)
    hi = lo + counts[part.rank]

    def local_idx(ix):
        return torch.where((ix >= lo) & (ix < hi), ix - lo, torch.full_like(ix, -1)).to(torch.int32)

    g_read = ops.scatter_rows_multi(hi - lo, [local_idx(neg), local_idx(pos), local_idx(users)], [gn, gp, gu])
    g_e = None
    dthetas = [None] * len(thetas)
    for i in range(len(thetas) - 1, -1, -1):
        mask, q = saved[i]
        dthetas[i], dh_local = ops.layer_backward(g_read, g_e, mask, q, thetas[i])
        if overlap:
            dh_full, pending = gather_start(dh_local)
            g_e = ops.spmm_overlap(a_local, plan, dh_full, pending.wait_source)
        else:
            g_e = ops.spmm(a_local, gather(dh_local))
    dth = comm.all_reduce_sum(torch.stack(dthetas))
    return loss, g_e, list(dth.unbind(0))


class PartitionedStepGraph:
    """One rank's partitioned training step (``partitioned_step`` + Adam on the
    rank's E0 rows and the thetas) captured once as a CUDA graph and replayed
    per batch, with the same device-side counters as the single-GPU
    ``train._StepGraph``: tensor ids advance on the device (``base``), Adam's
    step and bias corrections come from ``step_rel`` / ``c12``.  The step has
    fixed shapes and no host synchronisation, so the collectives (NCCL) are
    captured with it; a replay equals the eager step bit for bit."""

    def __init__(self, part: RowPartition, a_local, params: dict, state, cfg, stream: RandomStream, comm,
                 n_layers: int, batch: int, capacity: int, layout: str = "global", halo=None, ops=GpuOps,
                 overlap: bool = False, plan=None):
        from .train import AdamState  # noqa: F401  (state is a train.AdamState)
        dev = params["E0"].device
        self.B, self.capacity, self.n_layers = batch, capacity, n_layers
        sr = cfg.quant.rounding == "stochastic" and not cfg.quant.passthrough
        self.n_tids = (n_layers + 3) if sr else 0
        self.idx = torch.zeros((3, batch), dtype=torch.int64, device=dev)     # users, pos, neg node ids
        self.base = torch.zeros(1, dtype=torch.int64, device=dev)
        self.step_rel = torch.zeros(1, dtype=torch.int64, device=dev)
        self.c12 = torch.ones(2 * (capacity + 1), dtype=torch.float32, device=dev)
        host_tid = stream._next_tensor_id
        stream.bind_device_base(self.base)
        stream._next_tensor_id = 0
        from . import _lib
        if overlap and plan is None:        # built outside the capture (it syncs with the host)
            plan = ops.overlap_plan(a_local, part.cuts)
        self.graph = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(self.graph):
                self.step_rel.add_(1)
                thetas = [params[f"theta{i}"] for i in range(n_layers)]
                loss, de0, dth = partitioned_step(part, a_local, params["E0"], thetas, self.idx[0], self.idx[1],
                                                  self.idx[2], cfg.l2, cfg.quant, stream, comm, ops=ops,
                                                  layout=layout, halo=halo, overlap=overlap, plan=plan)
                grads = {"E0": de0}
                grads.update({f"theta{i}": t for i, t in enumerate(dth)})
                L = _lib.load()
                for name, g in grads.items():
                    p = params[name]
                    st = L.kgq_adam_step_dev_f32(p.data_ptr(), g.contiguous().data_ptr(), state.m[name].data_ptr(),
                                                 state.v[name].data_ptr(), p.numel(), cfg.lr, state.beta1,
                                                 state.beta2, state.eps, self.c12.data_ptr(),
                                                 self.step_rel.data_ptr(), _lib.ptr(getattr(state, "status", None)),
                                                 _lib.stream_ptr(dev))
                    _lib.check(st, "kgq_adam_step_dev_f32")
                self.base.add_(self.n_tids)
                self.loss = loss
        finally:
            stream.bind_device_base(None)
            stream._next_tensor_id = host_tid

    def run(self, batches, stream: RandomStream, state):
        """Replay once per (users, pos, neg) node-id batch; returns the losses."""
        from .train import _bias_rows
        n = len(batches)
        if n > self.capacity:
            raise ValueError("graph capacity exceeded")
        self.base.fill_(stream._next_tensor_id)
        self.step_rel.zero_()
        self.c12.copy_(torch.from_numpy(_bias_rows(state, state.step, self.capacity)))
        losses = []
        for u, p, ng in batches:
            self.idx[0].copy_(u)
            self.idx[1].copy_(p)
            self.idx[2].copy_(ng)
            self.graph.replay()
            losses.append(self.loss.clone())
        stream._next_tensor_id += n * self.n_tids
        state.step += n
        return losses
