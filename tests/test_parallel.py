"""Row-partitioned training at world size 2 over gloo on CPU.

The exchange logic of ``parallel.partitioned_step`` runs with the CPU oracle
as its compute ops; the forward pass must be bit-identical to world size 1
(noise keyed by global row), and so must the local E0 gradient rows; the
theta gradients differ only by the all-reduce summation order."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_2212_04540_b200 import data as D
from paper_2212_04540_b200.parallel import RowPartition, SoloComm, partitioned_step
from paper_2212_04540_b200.quantize import QuantConfig, RandomStream
from tests import golden_io


class _Q:
    def __init__(self, codes, ranges, offsets, rows, cols, bits):
        self.codes, self.ranges, self.offsets = codes, ranges, offsets
        self.rows, self.cols, self.bits = rows, cols, bits


class _Mask:
    def __init__(self, bits):
        self.bits = bits


class OracleOps:
    """CPU stand-ins for the libkgq ops (the oracle is the checker)."""

    @staticmethod
    def local_adjacency(indptr, indices, vals, lo, hi, n, device=None):
        return D.row_block(indptr, indices, vals, lo, hi)

    @staticmethod
    def _quant(x, cfg, stream, row_offset=0, tensor_id=None):
        tid = stream.next_tensor_id() if tensor_id is None else tensor_id
        x = np.ascontiguousarray(x.numpy(), dtype=np.float32)
        mode = orc.MODE_SR_FAST if cfg.rng == "fast" else orc.MODE_SR_COMPAT
        c, r, o = orc.quantize(x, x.shape[1], cfg.bits, mode, stream.seed, tid, group_offset=row_offset)
        return _Q(c, r, o, x.shape[0], x.shape[1], cfg.bits)

    @staticmethod
    def graph_conv(a_local, e_full, theta, cfg, stream, row_offset=0):
        ip, ix, vv = a_local
        h = orc.spmm_csr(ip, ix, vv, e_full.numpy())
        q = OracleOps._quant(torch.from_numpy(h), cfg, stream, row_offset)
        j = h @ theta.numpy()
        out, mask = orc.relu_mask(j)
        return torch.from_numpy(out), _Mask(j > 0), q, None

    @staticmethod
    def quantize(t, cfg, stream):
        return OracleOps._quant(t, cfg, stream)

    @staticmethod
    def overlap_plan(a_local, col_cuts):
        return np.asarray(col_cuts, dtype=np.int64)

    @staticmethod
    def _spmm_overlap(a_local, cuts, x, wait_block):
        """block p of the chain from a copy of x whose blocks > p are NaN (read
        before their exchange would show), after wait_block(p); fp32 chain
        continued across blocks (ascending columns), as the kernel does."""
        ip, ix, vv = a_local
        xn = x.numpy()
        h = np.zeros((len(ip) - 1, x.shape[1]), dtype=np.float32)
        for p in range(len(cuts) - 1):
            wait_block(p)
            buf = np.full(xn.shape, np.nan, dtype=np.float32)
            buf[:cuts[p + 1]] = xn[:cuts[p + 1]]
            for r in range(len(ip) - 1):
                for j in range(ip[r], ip[r + 1]):
                    if cuts[p] <= ix[j] < cuts[p + 1]:
                        h[r] = h[r] + np.float32(vv[j]) * buf[ix[j]]
        return h

    @staticmethod
    def graph_conv_overlap(a_local, plan, e_full, wait, theta, cfg, stream, row_offset=0):
        h = OracleOps._spmm_overlap(a_local, plan, e_full, wait)
        q = OracleOps._quant(torch.from_numpy(h), cfg, stream, row_offset)
        j = h @ theta.numpy()
        out, mask = orc.relu_mask(j)
        return torch.from_numpy(out), _Mask(j > 0), q, None

    @staticmethod
    def spmm_overlap(a_local, plan, x, wait):
        return torch.from_numpy(OracleOps._spmm_overlap(a_local, plan, x, wait))

    @staticmethod
    def dequantize(q):
        return torch.from_numpy(orc.dequantize(q.codes, q.ranges, q.offsets, q.cols, q.bits))

    @staticmethod
    def dequant_gemm(q, g):
        return OracleOps.dequantize(q).t() @ g

    @staticmethod
    def mask_apply(g, mask):
        return g * torch.from_numpy(mask.bits.astype(np.float32))

    @staticmethod
    def spmm(a_local, x):
        ip, ix, vv = a_local
        return torch.from_numpy(orc.spmm_csr(ip, ix, vv, x.numpy()))

    @staticmethod
    def layer_backward(g_read, g_e, mask, q, theta):
        g = g_read if g_e is None else g_read + g_e
        g_j = OracleOps.mask_apply(g, mask)
        return OracleOps.dequant_gemm(q, g_j), g_j @ theta.t()

    @staticmethod
    def bpr_forward(u, p, n, l2):
        """tape.py:162-166 in numpy-order torch ops (CPU checker)."""
        batch = u.shape[0]
        margins = (u * (p - n)).sum(dim=1)
        data = torch.logaddexp(torch.zeros_like(margins), -margins).mean()
        reg = l2 * ((u * u).sum() + (p * p).sum() + (n * n).sum()) / batch
        return data + reg, margins

    @staticmethod
    def bpr_backward(g, margins, uh, ph, nh, l2, batch):
        coef = (torch.sigmoid(-margins) / batch)[:, None]
        reg = 2.0 * l2 / batch
        return (g * (-coef * (ph - nh) + reg * uh), g * (-coef * uh + reg * ph),
                g * (coef * uh + reg * nh))

    @staticmethod
    def scatter_rows_multi(rows, idxs, gs):
        """(s_0 + s_1) + ... with s_i = np.add.at over list i; index -1 skipped."""
        total = None
        for idx, g in zip(idxs, gs):
            ix = idx.numpy().astype(np.int64)
            keep = ix >= 0
            s = np.zeros((rows, g.shape[1]), dtype=np.float32)
            np.add.at(s, ix[keep], g.numpy()[keep])
            total = s if total is None else total + s
        return torch.from_numpy(total)

    @staticmethod
    def scatter_rows(rows, idx, g):
        out = np.zeros((rows, g.shape[1]), dtype=np.float32)
        np.add.at(out, idx.numpy().astype(np.int64), g.numpy())
        return torch.from_numpy(out)


def _problem():
    z = golden_io.load("tape")
    n = int(z["n"])
    thetas = [torch.from_numpy(z[f"d64_theta{i}"]) for i in range(3)]
    e0 = torch.from_numpy(z["d64_E0"])
    idx = [torch.from_numpy(z[k].astype(np.int64)) for k in ("users", "pos", "neg")]
    return z, n, e0, thetas, idx


def _run(world, rank, comm, layout="concat", overlap=False):
    z, n, e0, thetas, (users, pos, neg) = _problem()
    part = RowPartition.build(z["indptr"], world, rank)
    ip, ix, vv = OracleOps.local_adjacency(z["indptr"], z["indices"], z["data"], part.lo, part.hi, n)
    halo = None
    if layout == "padded":           # columns index the padded gather buffer
        ix = part.padded_cols(ix).astype(np.int32)
    elif layout == "halo":           # columns index [own rows | halo rows]
        from paper_2212_04540_b200.parallel import HaloPlan
        halo = HaloPlan.build(part, torch.from_numpy(ix.astype(np.int64)), comm)
        ix = halo.remap(torch.from_numpy(ix.astype(np.int64))).numpy()
    cfg = QuantConfig(bits=2, rng="fast")
    loss, de0, dth = partitioned_step(part, (ip, ix, vv), e0[part.lo:part.hi], thetas, users, pos, neg,
                                      1e-5, cfg, RandomStream(21), comm, ops=OracleOps, layout=layout,
                                      halo=halo, overlap=overlap)
    return part, loss, de0, dth


def _worker(rank, world, port, out_q, layout="concat", overlap=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2212_04540_b200.parallel import Comm
        part, loss, de0, dth = _run(world, rank, Comm(), layout, overlap)
        out_q.put((rank, part.lo, part.hi, float(loss), de0.numpy(), [t.numpy() for t in dth]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("layout,overlap", [("concat", False), ("padded", False), ("global", False),
                                            ("halo", False), ("global", True)])
def test_partitioned_step_world2_gloo_matches_world1(layout, overlap):
    """overlap=True: every exchange is started asynchronously (one broadcast
    per source) and the SpMM runs block by block as each lands (from a buffer
    whose later blocks are NaN, so reading one too early would show)."""
    part1, loss1, de1, dth1 = _run(1, 0, SoloComm())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + 7 * (["concat", "padded", "global", "halo"].index(layout) + 4 * overlap)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, layout, overlap)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    de_full = np.zeros_like(de1.numpy())
    for rank, lo, hi, loss, de, dth in res:
        assert loss == float(loss1)                       # forward bit-identical
        de_full[lo:hi] = de
        for a, b in zip(dth, dth1):
            np.testing.assert_allclose(a, b.numpy(), rtol=1e-5, atol=1e-8)
    assert np.array_equal(de_full, de1.numpy())           # local E0 rows bit-identical


def test_partitioned_world1_matches_reference_tape():
    """W=1 partitioned step vs the reference Tape fed the same (fast) noise
    (golden tape.npz, b=2): same loss, gradients equal (0 difference observed;
    bound 1e-6 of max|grad| for BLAS summation-order differences across hosts)."""
    z, n, e0, thetas, (users, pos, neg) = _problem()
    part, loss, de0, dth = _run(1, 0, SoloComm())
    assert float(loss) == pytest.approx(float(z["d64_b2_loss"]), rel=1e-5)
    for name, g in [("E0", de0)] + [(f"theta{i}", t) for i, t in enumerate(dth)]:
        ref = z["d64_b2_grad_" + name]
        assert np.abs(g.numpy() - ref).max() <= 1e-6 * np.abs(ref).max(), name


def test_padded_cols_layout():
    indptr = np.array([0, 5, 9, 20, 22, 30, 31, 40], dtype=np.int64)   # 7 rows
    for world in (1, 2, 3):
        parts = [RowPartition.build(indptr, world, r) for r in range(world)]
        p = parts[0]
        cols = np.arange(7)
        pc = p.padded_cols(cols)
        for r in range(world):
            lo, hi = int(p.cuts[r]), int(p.cuts[r + 1])
            assert np.array_equal(pc[lo:hi], r * p.block + np.arange(hi - lo))
        assert pc.max() < world * p.block


def test_simulated_rank_comm_shapes_and_local_rows():
    """SimulatedRankComm (1-GPU measurement of one rank of a W-way partition)
    keeps the collective shapes, writes this rank's block where the real
    collective would, and fills remote rows once (stable across calls)."""
    from paper_2212_04540_b200.parallel import SimulatedRankComm
    cuts = np.array([0, 3, 10, 12])
    comm = SimulatedRankComm(world=3, rank=1)
    local = torch.arange(14, dtype=torch.float32).reshape(7, 2)
    full = comm.all_gather_global(local, cuts)
    assert full.shape == (12, 2) and torch.equal(full[3:10], local)
    remote = full[:3].clone()
    full2 = comm.all_gather_global(local + 1, cuts)
    assert full2.data_ptr() == full.data_ptr() and torch.equal(full2[:3], remote)
    idx = torch.tensor([4, 0, 9])
    rows = comm.gather_index_rows(local, 3, idx)
    assert torch.equal(rows[0], local[1]) and torch.equal(rows[2], local[6])
    padded = comm.all_gather_padded(local, 7)
    assert padded.shape == (21, 2) and torch.equal(padded[7:14], local)
    t = torch.ones(3)
    assert comm.all_reduce_sum(t) is t


def test_halo_plan_world1_is_identity():
    from paper_2212_04540_b200.parallel import HaloPlan
    z, n, e0, thetas, idx = _problem()
    part = RowPartition.build(z["indptr"], 1, 0)
    plan = HaloPlan.build(part, torch.from_numpy(z["indices"].astype(np.int64)), SoloComm())
    assert plan.n_halo == 0 and plan.send_counts == [0]
    assert torch.equal(plan.remap(torch.from_numpy(z["indices"].astype(np.int64))),
                       torch.from_numpy(z["indices"].astype(np.int32)))
