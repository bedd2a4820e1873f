"""Dense/sparse kernels of the engine on B200 (mirror of kgact.tensorops,
/root/reference/pkg/src/kgact/tensorops.py).

* ``CSR``: device-resident canonical CSR (int32 indptr/indices, fp32 data) --
  the format ``build_adjacency`` produces (data.py:230-266).
* ``spmm`` / ``spmm_t``: libkgq warp-per-row SpMM, accumulation in ascending
  column order, bit-identical to scipy (tensorops.py:37-50).  ``spmm_t`` of a
  bitwise-symmetric matrix is ``spmm`` (test_tape.py:45-50); otherwise the
  transpose CSR is built once and cached.
* ``relu`` -> (out, BitMask): one pass, mask LSB-first flat (tensorops.py:57-92).
* ``mm``: dense GEMM (cuBLAS via torch; fp32, TF32 disabled).
"""

import numpy as np
import torch

from . import _lib


class ShapeMismatchError(ValueError):
    """tensorops.py:19."""


def _require_2d(name, x):
    if not isinstance(x, torch.Tensor) or x.dim() != 2:
        raise TypeError(f"{name} must be a 2-D torch.Tensor, got {type(x).__name__}")


class CSR:
    """Canonical CSR matrix on a CUDA device."""

    def __init__(self, indptr: torch.Tensor, indices: torch.Tensor, data: torch.Tensor, shape,
                 symmetric: bool | None = None):
        _lib.require_cuda(indptr, indices, data)
        if indptr.dtype != torch.int32 or indices.dtype != torch.int32:
            raise TypeError("CSR indptr/indices must be int32")
        if data.dtype != torch.float32:
            raise TypeError("CSR data must be float32")
        self.indptr = indptr.contiguous()
        self.indices = indices.contiguous()
        self.data = data.contiguous()
        self.shape = (int(shape[0]), int(shape[1]))
        self._symmetric = symmetric
        self._transpose = None
        self._row_order = None
        self._n_heavy = 0

    @classmethod
    def from_scipy(cls, m, device="cuda", symmetric: bool | None = None) -> "CSR":
        m = m.tocsr()
        return cls(torch.from_numpy(np.ascontiguousarray(m.indptr, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(m.indices, dtype=np.int32)).to(device),
                   torch.from_numpy(np.ascontiguousarray(m.data, dtype=np.float32)).to(device),
                   m.shape, symmetric)

    @classmethod
    def from_arrays(cls, indptr, indices, data, shape, device="cuda", symmetric=None) -> "CSR":
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a, dtype=dt)).to(device)
        return cls(t(indptr, np.int32), t(indices, np.int32), t(data, np.float32), shape, symmetric)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.data.cpu().numpy(), self.indices.cpu().numpy(),
                              self.indptr.cpu().numpy()), shape=self.shape)

    HEAVY_NNZ = 256     # rows above this many nonzeros get a whole CTA in the kernels

    def schedule(self):
        """(row_order pointer, n_heavy): rows by decreasing degree (stable),
        built once.  The kernels give each of the first n_heavy (long) rows a
        CTA and pack the rest d/8 lanes per row, so the rows sharing a warp
        have similar lengths.  The schedule never changes results."""
        if self._row_order is None:
            deg = torch.diff(self.indptr.to(torch.int64))
            self._row_order = torch.sort(deg, descending=True, stable=True).indices.to(torch.int32)
            self._n_heavy = int((deg > self.HEAVY_NNZ).sum())
        return self._row_order.data_ptr(), self._n_heavy

    def block_phases(self, col_cuts) -> "BlockPhases":
        """The pipelined-SpMM plan for column blocks [col_cuts[p], col_cuts[p+1])
        (the source blocks of a partitioned exchange, ascending): per block,
        each row's nonzero range inside it and a row schedule of the rows that
        have any (by decreasing count).  Running the blocks in order with
        ``spmm_phased_into`` continues every row's ascending-column chain, so
        the result is bit-identical to spmm while block p+1.. may still be in
        flight when block p is computed."""
        cuts = torch.as_tensor(np.asarray(col_cuts, dtype=np.int64), device=self.device)
        W, n = int(cuts.numel()) - 1, self.shape[0]
        ip = self.indptr.to(torch.int64)
        rows = torch.repeat_interleave(torch.arange(n, device=self.device), ip[1:] - ip[:-1])
        blk = torch.searchsorted(cuts, self.indices.to(torch.int64), right=True) - 1
        cnt = torch.bincount(rows * W + blk, minlength=n * W).view(n, W)
        off = torch.cat([ip[:-1, None], ip[:-1, None] + torch.cumsum(cnt, 1)], 1)      # [n][W+1]
        bounds = off.t().to(torch.int32).contiguous()                                   # [W+1][n]
        ids = torch.arange(n, device=self.device)
        scheds = []
        for p in range(W):
            c = cnt[:, p]
            sel = c > 0
            scheds.append(RowSchedule.build(ids[sel], c[sel], self.HEAVY_NNZ))
        return BlockPhases(bounds, scheds)

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    @property
    def device(self):
        return self.data.device

    def nbytes(self) -> int:
        """csr_nbytes, tensorops.py:121-123: indptr + indices + values."""
        return (self.indptr.numel() + self.indices.numel()) * 4 + self.data.numel() * 4

    @property
    def symmetric(self) -> bool:
        """Bitwise symmetry (A == A^T including values)."""
        if self._symmetric is None:
            if self.shape[0] != self.shape[1]:
                self._symmetric = False
            else:
                t = self.transpose()
                self._symmetric = bool(torch.equal(t.indptr, self.indptr) and
                                       torch.equal(t.indices, self.indices) and
                                       torch.equal(t.data.view(torch.int32), self.data.view(torch.int32)))
        return self._symmetric

    def transpose(self) -> "CSR":
        """A^T in canonical CSR (built once; stable sort keeps column order)."""
        if self._transpose is None:
            n_rows, n_cols = self.shape
            counts = torch.diff(self.indptr.to(torch.int64))
            rows = torch.repeat_interleave(torch.arange(n_rows, device=self.device), counts)
            cols = self.indices.to(torch.int64)
            key = cols * max(n_rows, 1) + rows
            order = torch.argsort(key, stable=True)
            t_indices = rows[order].to(torch.int32)
            t_data = self.data[order]
            t_counts = torch.bincount(cols, minlength=n_cols)
            t_indptr = torch.zeros(n_cols + 1, dtype=torch.int64, device=self.device)
            t_indptr[1:] = torch.cumsum(t_counts, 0)
            self._transpose = CSR(t_indptr.to(torch.int32), t_indices, t_data, (n_cols, n_rows))
        return self._transpose


def mm(a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """tensorops.py:28-34 (dense product; cuBLAS SGEMM, no TF32)."""
    _require_2d("a", a)
    _require_2d("b", b)
    if a.shape[1] != b.shape[0]:
        raise ShapeMismatchError(f"mm: inner dims differ, a is {tuple(a.shape)}, b is {tuple(b.shape)}")
    return a @ b


def mm_theta(a: torch.Tensor, theta: torch.Tensor, transpose: bool = False) -> torch.Tensor:
    """a @ theta (or a @ theta.T) for the d x d layer weights: tcgen05 tensor
    cores (3xTF32, kgq_rowmm_f32) for d in (32, 64), cuBLAS otherwise."""
    _require_2d("a", a)
    d = theta.shape[0]
    if a.shape[1] != d or theta.shape[1] != d:
        raise ShapeMismatchError(f"mm: a is {tuple(a.shape)}, theta is {tuple(theta.shape)}")
    if d not in (32, 64) or a.dtype != torch.float32 or not a.is_cuda:
        return a @ (theta.t() if transpose else theta)
    a = a.contiguous()
    out = torch.empty_like(a)
    st = _lib.load().kgq_rowmm_f32(a.data_ptr(), a.shape[0], d, theta.contiguous().data_ptr(),
                                   1 if transpose else 0, out.data_ptr(), _lib.stream_ptr(a.device))
    _lib.check(st, "kgq_rowmm_f32")
    return out


class RowSchedule:
    """A subset of a CSR's rows as a kernel row schedule: ``order`` (int32,
    decreasing degree, stable), ``n_heavy`` rows above CSR.HEAVY_NNZ first."""

    __slots__ = ("order", "n_heavy")

    def __init__(self, order: torch.Tensor, n_heavy: int):
        self.order, self.n_heavy = order, int(n_heavy)

    @classmethod
    def build(cls, rows: torch.Tensor, deg: torch.Tensor, heavy: int) -> "RowSchedule":
        p = torch.sort(deg, descending=True, stable=True).indices
        return cls(rows[p].to(torch.int32).contiguous(), int((deg > heavy).sum()))

    def __len__(self) -> int:
        return int(self.order.numel())


class BlockPhases:
    """CSR.block_phases: ``bounds`` [W+1][n] int32 (row r's nonzeros of block
    p are [bounds[p][r], bounds[p+1][r])), ``scheds[p]`` its rows."""

    __slots__ = ("bounds", "scheds")

    def __init__(self, bounds: torch.Tensor, scheds):
        self.bounds, self.scheds = bounds, scheds

    def __len__(self) -> int:
        return len(self.scheds)


def spmm_phased_into(s: CSR, d: torch.Tensor, out: torch.Tensor, phases: BlockPhases, wait_block) -> torch.Tensor:
    """out = s @ d, one column block at a time (``wait_block(p)`` before block
    p: e.g. the exchange of that block of ``d`` has landed); each phase
    continues the rows' running chains in out (kgq_spmm_csr_seg_f32), so the
    result equals spmm bit for bit."""
    out.zero_()
    L = _lib.load()
    n = s.shape[0]
    for p, sch in enumerate(phases.scheds):
        wait_block(p)
        if len(sch) == 0:
            continue
        b = phases.bounds
        st = L.kgq_spmm_csr_seg_f32(s.indptr.data_ptr(), s.indices.data_ptr(), s.data.data_ptr(), len(sch),
                                    sch.order.data_ptr(), sch.n_heavy, b[p].data_ptr(), b[p + 1].data_ptr(),
                                    d.data_ptr(), d.shape[1], out.data_ptr(), _lib.stream_ptr(d.device))
        _lib.check(st, "kgq_spmm_csr_seg_f32")
    return out


def spmm_into(s: CSR, d: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    st = _lib.load().kgq_spmm_csr_f32(s.indptr.data_ptr(), s.indices.data_ptr(), s.data.data_ptr(),
                                      s.shape[0], *s.schedule(), d.data_ptr(), d.shape[1],
                                      out.data_ptr(), _lib.stream_ptr(d.device))
    _lib.check(st, "kgq_spmm_csr_f32")
    return out


def spmm(s: CSR, d: torch.Tensor) -> torch.Tensor:
    """tensorops.py:37-43: s @ d, ascending-column accumulation (bit-exact)."""
    _require_2d("d", d)
    if s.shape[1] != d.shape[0]:
        raise ShapeMismatchError(f"spmm: inner dims differ, s is {s.shape}, d is {tuple(d.shape)}")
    if d.dtype != torch.float32:
        raise TypeError("spmm: d must be float32")
    _lib.require_cuda(d)
    d = d.contiguous()
    out = torch.empty((s.shape[0], d.shape[1]), dtype=torch.float32, device=d.device)
    return spmm_into(s, d, out)


def spmm_t(s: CSR, d: torch.Tensor) -> torch.Tensor:
    """tensorops.py:46-50: transpose(s) @ d without materializing it per call."""
    _require_2d("d", d)
    if s.shape[0] != d.shape[0]:
        raise ShapeMismatchError(f"spmm_t: s is {s.shape} so d needs {s.shape[0]} rows, got {tuple(d.shape)}")
    return spmm(s if s.symmetric else s.transpose(), d)


class BitMask:
    """Boolean matrix packed one bit per element, LSB-first flat (tensorops.py:57-82)."""

    __slots__ = ("packed", "shape")

    def __init__(self, packed: torch.Tensor, shape):
        self.packed = packed
        self.shape = tuple(int(v) for v in shape)

    @classmethod
    def from_bool(cls, mask: torch.Tensor) -> "BitMask":
        flat = mask.reshape(-1).to(torch.uint8)
        n = flat.numel()
        pad = (-n) % 8
        if pad:
            flat = torch.cat([flat, flat.new_zeros(pad)])
        weights = (1 << torch.arange(8, device=flat.device, dtype=torch.int32))
        packed = (flat.view(-1, 8).to(torch.int32) * weights).sum(1).to(torch.uint8)
        return cls(packed, mask.shape)

    def to_bool(self) -> torch.Tensor:
        n = int(np.prod(self.shape))
        bits = (self.packed.to(torch.int32).unsqueeze(1) >> torch.arange(8, device=self.packed.device)) & 1
        return bits.reshape(-1)[:n].to(torch.bool).reshape(self.shape)

    @property
    def nbytes(self) -> int:
        return self.packed.numel()

    def count(self) -> int:
        return int(self.to_bool().sum())


def relu(x: torch.Tensor):
    """tensorops.py:84-92: (max(x, 0), BitMask(x > 0)) in one kernel."""
    _require_2d("x", x)
    if x.dtype != torch.float32:
        raise TypeError("relu: x must be float32")
    _lib.require_cuda(x)
    x = x.contiguous()
    out = torch.empty_like(x)
    mask = torch.empty((x.numel() + 7) // 8 + 3 & ~3, dtype=torch.uint8, device=x.device)
    st = _lib.load().kgq_relu_mask_f32(x.data_ptr(), x.numel(), out.data_ptr(), mask.data_ptr(),
                                       _lib.stream_ptr(x.device))
    _lib.check(st, "kgq_relu_mask_f32")
    return out, BitMask(mask[:(x.numel() + 7) // 8], x.shape)


def mask_apply(g: torch.Tensor, mask: BitMask) -> torch.Tensor:
    """ReLU backward, tape.py:224-225: g * mask.to_bool() (exact signed zeros)."""
    _lib.require_cuda(g)
    if tuple(g.shape) != mask.shape:
        raise ShapeMismatchError(f"mask {mask.shape} vs grad {tuple(g.shape)}")
    g = g.contiguous()
    out = torch.empty_like(g)
    st = _lib.load().kgq_mask_apply_f32(g.data_ptr(), mask.packed.data_ptr(), g.numel(),
                                        out.data_ptr(), _lib.stream_ptr(g.device))
    _lib.check(st, "kgq_mask_apply_f32")
    return out


def densify(s: CSR) -> torch.Tensor:
    out = torch.zeros(s.shape, dtype=torch.float32, device=s.device)
    counts = torch.diff(s.indptr.to(torch.int64))
    rows = torch.repeat_interleave(torch.arange(s.shape[0], device=s.device), counts)
    out[rows, s.indices.to(torch.int64)] = s.data
    return out


def make_csr(dense, device="cuda") -> CSR:
    """Canonical CSR from a dense array (test/demo convenience, tensorops.py:95-100)."""
    import scipy.sparse as sp
    a = dense.cpu().numpy() if isinstance(dense, torch.Tensor) else np.asarray(dense)
    m = sp.csr_matrix(a.astype(np.float32))
    m.sum_duplicates()
    m.sort_indices()
    return CSR.from_scipy(m, device)


def validate_csr(s: CSR) -> None:
    """tensorops.py:103-118 structural invariants (vectorized on device)."""
    if not isinstance(s, CSR):
        raise TypeError("expected a CSR")
    rows, cols = s.shape
    ip = s.indptr.to(torch.int64)
    if ip.numel() != rows + 1 or int(ip[0]) != 0 or int(ip[-1]) != s.nnz:
        raise ValueError("csr: indptr is not a valid offset array")
    if bool((torch.diff(ip) < 0).any()):
        raise ValueError("csr: indptr must be nondecreasing")
    if s.nnz:
        idx = s.indices.to(torch.int64)
        if int(idx.min()) < 0 or int(idx.max()) >= cols:
            raise ValueError("csr: column index out of range")
        rowid = torch.repeat_interleave(torch.arange(rows, device=s.device), torch.diff(ip))
        same_row = rowid[1:] == rowid[:-1]
        bad = same_row & (idx[1:] <= idx[:-1])
        if bool(bad.any()):
            r = int(rowid[1:][bad][0])
            raise ValueError(f"csr: row {r} has unsorted or duplicate column indices")


def csr_nbytes(s: CSR) -> int:
    return s.nbytes()
