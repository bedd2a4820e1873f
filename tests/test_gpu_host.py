"""Host-buffer entry points (kgq_quantize_host_f32 / kgq_dequantize_host_f32):
numpy-style host tensors in and out, streamed through the device in chunks.
Bytes must equal the device call for every chunking, and the reference's own
golden outputs in compat mode."""
import ctypes

import numpy as np
import pytest
import torch

from tests import golden_io

pytestmark = pytest.mark.gpu


def _kgq():
    import paper_2212_04540_b200 as kgq
    return kgq


def _dev_q(kgq, x, cfg, seed, tid, goff=0):
    return kgq.quantize_tensor(x.cuda(), cfg, kgq.RandomStream(seed), tensor_id=tid, group_offset=goff)


def _same(a, b):
    return torch.equal(a.cpu().view(torch.uint8) if a.dtype != torch.uint8 else a.cpu(),
                       b.cpu().view(torch.uint8) if b.dtype != torch.uint8 else b.cpu())


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("bits,group,rng", [(2, 64, "fast"), (4, 128, "compat"), (8, None, "fast"),
                                            (1, 32, "fast")])
def test_host_quantize_equals_device(pinned, bits, group, rng):
    kgq = _kgq()
    g = torch.Generator().manual_seed(bits)
    x = torch.randn(20000, 128, generator=g)
    x[::97] = 0.5
    if pinned:
        x = x.pin_memory()
    cfg = kgq.QuantConfig(bits=bits, group=group, rng=rng)
    qh = kgq.quantize_tensor(x, cfg, kgq.RandomStream(5), tensor_id=3)
    qd = _dev_q(kgq, x, cfg, 5, 3)
    assert qh.codes.device.type == "cpu"
    assert _same(qh.codes, qd.codes) and _same(qh.ranges, qd.ranges) and _same(qh.offsets, qd.offsets)
    oh = kgq.dequantize_tensor(qh)
    od = kgq.dequantize_tensor(qd)
    assert oh.device.type == "cpu" and _same(oh, od)


@pytest.mark.parametrize("n_streams", [1, 2, 3])
def test_host_chunking_is_byte_identical(n_streams):
    """Explicit small workspace -> many chunks (incl. a ragged last one)."""
    kgq = _kgq()
    from paper_2212_04540_b200 import _lib
    L = _lib.load()
    rows, cols, group, bits = 10007, 64, 64, 2
    x = torch.randn(rows, cols, generator=torch.Generator().manual_seed(0)).pin_memory()
    n_groups = rows * cols // group
    ws_bytes = L.kgq_host_workspace_bytes(1000, group, bits, n_streams)
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(n_streams)]
    arr = (ctypes.c_void_p * n_streams)(*[s.cuda_stream for s in streams])
    codes = torch.empty(n_groups, group * bits // 8, dtype=torch.uint8).pin_memory()
    r = torch.empty(n_groups).pin_memory()
    z = torch.empty(n_groups).pin_memory()
    goff = 12345
    st = L.kgq_quantize_host_f32(x.data_ptr(), n_groups, group, bits, _lib.ROUND_SR_FAST, 9, 4, goff,
                                 codes.data_ptr(), r.data_ptr(), z.data_ptr(), ws.data_ptr(), ws_bytes,
                                 ctypes.cast(arr, ctypes.c_void_p), n_streams,
                                 torch.cuda.current_stream().cuda_stream)
    assert st == 0
    cfg = kgq.QuantConfig(bits=bits, group=group, rng="fast")
    qd = _dev_q(kgq, x, cfg, 9, 4, goff)
    assert _same(codes, qd.codes) and _same(r, qd.ranges) and _same(z, qd.offsets)
    out = torch.empty(rows, cols).pin_memory()
    st = L.kgq_dequantize_host_f32(codes.data_ptr(), r.data_ptr(), z.data_ptr(), n_groups, group, bits,
                                   out.data_ptr(), ws.data_ptr(), ws_bytes,
                                   ctypes.cast(arr, ctypes.c_void_p), n_streams,
                                   torch.cuda.current_stream().cuda_stream)
    assert st == 0
    assert _same(out, kgq.dequantize_tensor(qd))


def test_host_path_matches_reference_golden():
    """compat mode, per-row: the host call reproduces the reference's bytes."""
    kgq = _kgq()
    n = 0
    for case in golden_io.quant_cases():
        if case["mode"] != 2 or case["group"] != case["x"].shape[1]:
            continue
        x = torch.from_numpy(np.ascontiguousarray(case["x"], dtype=np.float32))
        cfg = kgq.QuantConfig(bits=case["bits"], rng="compat")
        q = kgq.quantize_tensor(x, cfg, kgq.RandomStream(case["seed"]), tensor_id=case["tid"])
        assert np.array_equal(q.codes.numpy(), case["codes"])
        assert np.array_equal(q.ranges.numpy().view(np.uint32), np.asarray(case["ranges"]).view(np.uint32))
        deq = kgq.dequantize_tensor(q)
        assert np.array_equal(deq.numpy().view(np.uint32), case["deq"].reshape(deq.shape).view(np.uint32))
        n += 1
    assert n > 0


def test_host_errors():
    kgq = _kgq()
    from paper_2212_04540_b200 import _lib
    L = _lib.load()
    x = torch.randn(8, 64)
    with pytest.raises(ValueError):
        kgq.quantize_tensor(x, kgq.QuantConfig(bits=2, rng="fast"), kgq.RandomStream(1), tensor_id=0,
                            noise=torch.zeros(8 * 64, dtype=torch.float64, device="cuda"))
    assert L.kgq_quantize_host_f32(x.data_ptr(), 8, 64, 2, _lib.ROUND_SR_NOISE, 0, 0, 0, None, None, None,
                                   None, 0, None, 0, None) == _lib.KGQ_ERR_INVALID_ARG
    # workspace too small for one 8-group chunk per stream
    assert L.kgq_quantize_host_f32(x.data_ptr(), 8, 64, 2, 0, 0, 0, 0, x.data_ptr(), x.data_ptr(),
                                   x.data_ptr(), x.data_ptr(), 16, None, 0, None) \
        == _lib.KGQ_ERR_INVALID_ARG
    # empty input is a no-op
    e = torch.empty(0, 64)
    q = kgq.quantize_tensor(e, kgq.QuantConfig(bits=2, rng="fast"), kgq.RandomStream(1), tensor_id=0)
    assert q.codes.shape[0] == 0 and kgq.dequantize_tensor(q).shape == (0, 64)


def test_numpy_ctypes_binding_from_integration_md():
    """The maintainer-side stub of INTEGRATION.md §2 (numpy + ctypes only,
    NULL workspace/streams) reproduces the reference's golden bytes."""
    from paper_2212_04540_b200 import _lib
    L = ctypes.CDLL(_lib.LIB_PATH)
    P, I64, U64, I32, SZ = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_size_t
    L.kgq_quantize_host_f32.argtypes = [P, I64, I32, I32, I32, U64, U64, I64, P, P, P, P, SZ, P, I32, P]
    L.kgq_dequantize_host_f32.argtypes = [P, P, P, I64, I32, I32, P, P, SZ, P, I32, P]
    ptr = lambda a: a.ctypes.data_as(ctypes.c_void_p)
    n = 0
    for case in golden_io.quant_cases():
        if case["group"] != case["x"].shape[1] or case["mode"] == 1:
            continue
        x = np.ascontiguousarray(case["x"], np.float32)
        rows, cols = x.shape
        bits = case["bits"]
        codes = np.empty((rows, (cols * bits + 7) // 8), np.uint8)
        r, z = np.empty(rows, np.float32), np.empty(rows, np.float32)
        st = L.kgq_quantize_host_f32(ptr(x), rows, cols, bits, case["mode"], case["seed"], case["tid"], 0,
                                     ptr(codes), ptr(r), ptr(z), None, 0, None, 0, None)
        assert st == 0
        assert np.array_equal(codes, case["codes"])
        assert np.array_equal(r.view(np.uint32), np.asarray(case["ranges"]).view(np.uint32))
        assert np.array_equal(z.view(np.uint32), np.asarray(case["offsets"]).view(np.uint32))
        out = np.empty((rows, cols), np.float32)
        st = L.kgq_dequantize_host_f32(ptr(codes), ptr(r), ptr(z), rows, cols, bits, ptr(out),
                                       None, 0, None, 0, None)
        assert st == 0
        assert np.array_equal(out.view(np.uint32), case["deq"].reshape(out.shape).view(np.uint32))
        n += 1
    assert n > 0
