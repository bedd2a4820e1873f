"""Per-row / per-group uniform quantization with stochastic rounding, on B200.

Drop-in mirror of the reference quantizer API (kgact.quantize,
/root/reference/pkg/src/kgact/quantize.py) over CUDA tensors:

    QuantConfig, RandomStream, QuantizedTensor, quantize_tensor,
    dequantize_tensor, quantize_row, dequantize_row, pack_codes, unpack_codes,
    pack_bits, unpack_bits, stored_bytes, fp32_equivalent_bytes,
    stochastic_round, nearest_round, EncodingError

Compute runs in libkgq (sm_100a) through the C ABI in include/kgq.h; there is
no CPU path.  Additions over the reference, both defaulting to the
reference's behaviour where it is defined:

* ``QuantConfig.group``: quantization group size G.  ``None`` means one group
  per row (the reference, quantize.py:184-186); otherwise groups are the rows
  of the ``(-1, G)`` view of the row-major tensor.
* ``QuantConfig.rng``: ``"compat"`` (default) draws the reference's numpy
  Philox4x64-10 stream bit-for-bit (quantize.py:61-102), so the same
  ``RandomStream(seed)`` gives the same codes as kgact; ``"fast"`` (opt-in,
  the throughput configuration) draws Philox4x32-7 16-bit uniforms
   and is checked bit-exact against the reference through the
  exported-noise route.
"""

import math
from dataclasses import dataclass

import torch

from . import _lib

ROUND_STOCHASTIC = "stochastic"
ROUND_NEAREST = "nearest"
RNG_FAST = "fast"
RNG_COMPAT = "compat"

PASSTHROUGH_BITS = 32
SUPPORTED_BITS = (1, 2, 4, 8, 32)


class EncodingError(ValueError):
    """A code does not fit in the requested bit width (quantize.py:36)."""


@dataclass(frozen=True)
class QuantConfig:
    """quantize.py:40-58 plus ``group`` and ``rng`` (module docstring)."""
    bits: int = PASSTHROUGH_BITS
    rounding: str = ROUND_STOCHASTIC
    group: int | None = None
    rng: str = RNG_COMPAT

    def __post_init__(self):
        if self.bits not in SUPPORTED_BITS:
            raise ValueError(f"bits must be one of {SUPPORTED_BITS}, got {self.bits}")
        if self.rounding not in (ROUND_STOCHASTIC, ROUND_NEAREST):
            raise ValueError(f"unknown rounding mode {self.rounding!r}")
        if self.rng not in (RNG_FAST, RNG_COMPAT):
            raise ValueError(f"unknown rng {self.rng!r}, expected 'fast' or 'compat'")
        if self.group is not None and int(self.group) < 1:
            raise ValueError("group must be >= 1")

    @property
    def bins(self) -> int:
        return (1 << self.bits) - 1

    @property
    def passthrough(self) -> bool:
        return self.bits == PASSTHROUGH_BITS

    @property
    def mode(self) -> int:
        """kgq_rounding enum value for the kernels."""
        if self.rounding == ROUND_NEAREST:
            return _lib.ROUND_NEAREST
        return _lib.ROUND_SR_FAST if self.rng == RNG_FAST else _lib.ROUND_SR_COMPAT


class RandomStream:
    """Keyed uniform draws, quantize.py:61-102.

    Holds only ``seed`` and the monotone tensor-id counter; the draws
    themselves are generated inside the quantize kernels from
    (seed, tensor id, global group index), so nothing here touches the GPU
    except the explicit export helpers used by the parity tests.
    """

    def __init__(self, seed: int):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self._next_tensor_id = 0
        self._device_base = None    # uint64 device counter while capturing CUDA graphs

    def next_tensor_id(self) -> int:
        tid = self._next_tensor_id
        self._next_tensor_id += 1
        return tid

    def tid_base_ptr(self):
        """Device pointer the kernels add to tensor ids (None = host ids only)."""
        return None if self._device_base is None else self._device_base.data_ptr()

    def bind_device_base(self, base: "torch.Tensor | None") -> None:
        """Key subsequent draws by (host id + *base): a captured CUDA graph
        increments ``base`` between replays so each replay gets fresh tensor
        ids -- the same ids the eager path would have used."""
        self._device_base = base

    def matrix_uniforms(self, tensor_id: int, rows: int, cols: int, dtype=torch.float64,
                        rng: str = RNG_COMPAT, device=None) -> torch.Tensor:
        """Uniform draws for a whole (rows, cols) tensor as a CUDA tensor.

        ``rng="compat"`` equals the reference's ``matrix_uniforms`` exactly.
        """
        dev = torch.device("cuda") if device is None else torch.device(device)
        if rng == RNG_COMPAT:
            raw = compat_noise_raw53(self.seed, tensor_id, rows, cols, device=dev)
            return (raw.to(torch.float64) * 2.0 ** -53).to(dtype)
        u16 = fast_noise_u16(self.seed, tensor_id, rows, cols, device=dev)
        return (u16.to(torch.float64) / 65536.0).to(dtype)

    def row_uniforms(self, tensor_id: int, row: int, cols: int, rng: str = RNG_COMPAT,
                     device=None) -> torch.Tensor:
        dev = torch.device("cuda") if device is None else torch.device(device)
        if rng == RNG_COMPAT:
            raw = compat_noise_raw53(self.seed, tensor_id, 1, cols, group_offset=row, device=dev)
            return raw.to(torch.float64)[0] * 2.0 ** -53
        u16 = fast_noise_u16(self.seed, tensor_id, 1, cols, group_offset=row, device=dev)
        return u16.to(torch.float64)[0] / 65536.0


def stochastic_round(x: float, u: float) -> int:
    """quantize.py:105-108."""
    f = math.floor(x)
    return f + 1 if u < (x - f) else f


def nearest_round(x: float) -> int:
    """quantize.py:111-113 (round half to even)."""
    return round(float(x))


@dataclass
class QuantizedTensor:
    """Packed codes + per-group fp32 (range, offset), quantize.py:135-148.

    ``codes`` is uint8 (n_groups, ceil(group*bits/8)); with the default
    per-row group this is (rows, row_bytes) exactly as in the reference.
    """
    rows: int
    cols: int
    bits: int
    codes: torch.Tensor | None
    ranges: torch.Tensor | None
    offsets: torch.Tensor | None
    raw: torch.Tensor | None = None
    group: int | None = None

    @property
    def n_groups(self) -> int:
        return 0 if self.ranges is None else self.ranges.shape[0]

    @property
    def group_size(self) -> int:
        return self.group if self.group is not None else self.cols


def _require_fp32_2d(x, name="x", allow_host=False):
    if not isinstance(x, torch.Tensor) or x.dim() != 2:
        raise TypeError(f"{name} must be a 2-D torch.Tensor")
    if x.dtype != torch.float32:
        raise TypeError(f"{name} must be float32 (the B200 engine is fp32), got {x.dtype}")
    if not (allow_host and x.device.type == "cpu"):
        _lib.require_cuda(x)


class _HostPipe:
    """Streams + device workspace for the host-buffer calls.  Three streams
    per device are created once; the workspace comes from torch's caching
    allocator on the current stream (the library orders its streams after
    it), 64 MB of fp32 per chunk slot."""
    _streams: dict = {}
    CHUNK_ELEMS = 16 << 20

    @classmethod
    def args(cls, n_groups: int, group: int, bits: int):
        """(workspace tensor, streams ctypes array, n_streams, order stream)
        -- or Nones without CUDA (the library then reports the missing
        device; there is no CPU path)."""
        import ctypes
        if not torch.cuda.is_available():
            return None, None, 0, 0
        dev = torch.cuda.current_device()
        if dev not in cls._streams:
            ss = [torch.cuda.Stream(dev) for _ in range(3)]
            cls._streams[dev] = (ss, (ctypes.c_void_p * 3)(*[x.cuda_stream for x in ss]))
        ss, arr = cls._streams[dev]
        chunk = max(8, min(cls.CHUNK_ELEMS // max(group, 1), -(-n_groups // 8) * 8))
        nbytes = _lib.load().kgq_host_workspace_bytes(chunk, group, bits, len(ss))
        ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        return ws, ctypes.cast(arr, ctypes.c_void_p), len(ss), torch.cuda.current_stream().cuda_stream


def empty_context(rows: int, cols: int, cfg: "QuantConfig", pin_memory: bool = True) -> "QuantizedTensor":
    """Host buffers for ``quantize_tensor(host_x, ..., out=ctx)``: reusing
    pinned buffers keeps the host-buffer path at PCIe speed (allocating
    page-locked memory per call costs more than the transfer)."""
    group = cols if cfg.group is None else int(cfg.group)
    n_groups = rows * cols // group
    return QuantizedTensor(rows, cols, cfg.bits,
                           torch.empty((n_groups, packed_group_bytes(group, cfg.bits)), dtype=torch.uint8,
                                       pin_memory=pin_memory),
                           torch.empty(n_groups, dtype=torch.float32, pin_memory=pin_memory),
                           torch.empty(n_groups, dtype=torch.float32, pin_memory=pin_memory),
                           group=None if cfg.group is None else group)


def packed_group_bytes(group: int, bits: int) -> int:
    return (group * bits + 7) // 8


def row_group_offset(row_offset: int, cols: int, group: int | None) -> int:
    """Global index of the first quantization group of a row block that starts
    at global row ``row_offset`` (row-partitioned runs): groups are the rows
    of the ``(-1, G)`` view of the whole tensor, so the block must start on a
    group boundary.  Keying the noise by this global group index is what makes
    the codes byte-identical at any world size."""
    G = cols if group is None else int(group)
    if (row_offset * cols) % G:
        raise ValueError(f"row block at row {row_offset} does not start on a group boundary "
                         f"(cols {cols}, group {G})")
    return row_offset * cols // G


def quantize_tensor(x: torch.Tensor, cfg: QuantConfig, stream: RandomStream | None = None,
                    tensor_id: int | None = None, *, noise: torch.Tensor | None = None,
                    group_offset: int = 0, out: QuantizedTensor | None = None) -> QuantizedTensor:
    """quantize.py:177-196 on an fp32 tensor.

    A CUDA tensor is quantized in place on its device.  A host (CPU) tensor
    takes the reference's own numpy-in/numpy-out convention: it streams
    through the GPU (``kgq_quantize_host_f32``, chunked and pipelined) and
    the returned context lives in host memory -- computed on the GPU, not a
    CPU fallback (without a GPU the call raises).

    ``noise`` (float64 uniforms, one per element) replaces the stream's
    draws -- the exported-noise parity seam (device tensors only).
    ``group_offset`` is the global index of this tensor's first group
    (row-partitioned tensors).  ``out`` (host path only): preallocated host
    context from ``empty_context`` to write into.
    """
    _require_fp32_2d(x, allow_host=True)
    host = x.device.type == "cpu"
    if host and noise is not None:
        raise ValueError("the exported-noise seam takes device tensors")
    rows, cols = x.shape
    if cfg.passthrough:
        return QuantizedTensor(rows, cols, cfg.bits, None, None, None, raw=x)
    group = cols if cfg.group is None else int(cfg.group)
    if group == 0 or x.numel() % max(group, 1):
        raise ValueError(f"tensor of {x.numel()} elements is not divisible by group {group}")
    n_groups = x.numel() // group if group else 0
    mode = cfg.mode
    seed = tid = 0
    if cfg.rounding == ROUND_STOCHASTIC:
        if noise is not None:
            mode = _lib.ROUND_SR_NOISE
            _lib.require_cuda(noise)
            if noise.dtype != torch.float64 or noise.numel() != x.numel():
                raise ValueError("noise must be float64 with one draw per element")
            noise = noise.contiguous()
        else:
            if stream is None:
                raise ValueError("stochastic rounding needs a RandomStream")
            if tensor_id is None:
                tensor_id = stream.next_tensor_id()
            seed, tid = stream.seed, int(tensor_id) & 0xFFFFFFFFFFFFFFFF
    x = x.contiguous()
    dev = x.device
    if host:
        gb = packed_group_bytes(group, cfg.bits)
        if out is None:
            out = empty_context(rows, cols, cfg, pin_memory=x.is_pinned())
        elif (out.codes.device.type != "cpu" or tuple(out.codes.shape) != (n_groups, gb)
              or out.ranges.numel() != n_groups or out.offsets.numel() != n_groups
              or not (out.codes.is_contiguous() and out.ranges.is_contiguous()
                      and out.offsets.is_contiguous())):
            raise ValueError("out must be a contiguous host context of this shape (empty_context)")
        ws, sarr, ns, order = _HostPipe.args(n_groups, group, cfg.bits)
        st = _lib.load().kgq_quantize_host_f32(x.data_ptr(), n_groups, group, cfg.bits, mode, seed, tid,
                                               int(group_offset), out.codes.data_ptr(), out.ranges.data_ptr(),
                                               out.offsets.data_ptr(), _lib.ptr(ws),
                                               0 if ws is None else ws.numel(), sarr, ns, order)
        _lib.check(st, "kgq_quantize_host_f32")
        return QuantizedTensor(rows, cols, cfg.bits, out.codes, out.ranges, out.offsets,
                               group=None if cfg.group is None else group)
    if out is not None:
        raise ValueError("out= is for host tensors")
    codes = torch.empty((n_groups, packed_group_bytes(group, cfg.bits)), dtype=torch.uint8, device=dev)
    ranges = torch.empty(n_groups, dtype=torch.float32, device=dev)
    offsets = torch.empty(n_groups, dtype=torch.float32, device=dev)
    tb = stream.tid_base_ptr() if (stream is not None and mode != _lib.ROUND_SR_NOISE) else None
    st = _lib.load().kgq_quantize_f32(x.data_ptr(), n_groups, group, cfg.bits, mode, seed, tid, tb,
                                      int(group_offset), _lib.ptr(noise), codes.data_ptr(),
                                      ranges.data_ptr(), offsets.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_quantize_f32")
    return QuantizedTensor(rows, cols, cfg.bits, codes, ranges, offsets,
                           group=None if cfg.group is None else group)


def dequantize_tensor(q: QuantizedTensor, dtype=None, *, out: torch.Tensor | None = None) -> torch.Tensor:
    """quantize.py:199-210: (R*c)/B + Z in fp32, R == 0 -> Z.

    A host context (from the host path of ``quantize_tensor``) is streamed
    through the GPU and returns a host tensor (``out``: preallocated,
    ideally pinned, host fp32 tensor of shape (rows, cols))."""
    if q.bits == PASSTHROUGH_BITS:
        return q.raw
    if dtype not in (None, torch.float32):
        raise ValueError("the B200 engine dequantizes to float32 only")
    dev = q.codes.device
    if dev.type == "cpu":      # host context: streamed through the GPU (see quantize_tensor)
        codes, ranges, offsets = q.codes.contiguous(), q.ranges.contiguous(), q.offsets.contiguous()
        if out is None:
            out = torch.empty((q.rows, q.cols), dtype=torch.float32, pin_memory=codes.is_pinned())
        elif (out.device.type != "cpu" or out.dtype != torch.float32 or tuple(out.shape) != (q.rows, q.cols)
              or not out.is_contiguous()):
            raise ValueError("out must be a contiguous host float32 tensor of shape (rows, cols)")
        ws, sarr, ns, order = _HostPipe.args(q.n_groups, q.group_size, q.bits)
        st = _lib.load().kgq_dequantize_host_f32(codes.data_ptr(), ranges.data_ptr(), offsets.data_ptr(),
                                                 q.n_groups, q.group_size, q.bits, out.data_ptr(),
                                                 _lib.ptr(ws), 0 if ws is None else ws.numel(), sarr, ns,
                                                 order)
        _lib.check(st, "kgq_dequantize_host_f32")
        return out
    if out is not None:
        raise ValueError("out= is for host contexts")
    out = torch.empty((q.rows, q.cols), dtype=torch.float32, device=dev)
    st = _lib.load().kgq_dequantize_f32(q.codes.data_ptr(), q.ranges.data_ptr(), q.offsets.data_ptr(),
                                        q.n_groups, q.group_size, q.bits, out.data_ptr(),
                                        _lib.stream_ptr(dev))
    _lib.check(st, "kgq_dequantize_f32")
    return out


def quantize_row(e: torch.Tensor, cfg: QuantConfig, stream: RandomStream | None = None,
                 tensor_id: int = 0, row: int = 0):
    """quantize.py:151-166: one row with the noise of row ``row``.
    Returns (codes uint8 per element, range, offset)."""
    if e.dim() != 1:
        raise TypeError("row must be 1-D")
    q = quantize_tensor(e.reshape(1, -1), QuantConfig(cfg.bits, cfg.rounding, None, cfg.rng),
                        stream, tensor_id, group_offset=row)
    if q.raw is not None:
        raise ValueError("quantize_row needs bits < 32")
    codes = unpack_codes(q.codes, cfg.bits, e.shape[0])[0]
    return codes, q.ranges[0], q.offsets[0]


def dequantize_row(codes: torch.Tensor, r, z, bins: int) -> torch.Tensor:
    """quantize.py:169-174 in fp32: (R*c)/B + Z, exact Z when R == 0."""
    r = torch.as_tensor(r, dtype=torch.float32, device=codes.device)
    z = torch.as_tensor(z, dtype=torch.float32, device=codes.device)
    if float(r) == 0.0:
        return torch.full((codes.shape[0],), float(z), dtype=torch.float32, device=codes.device)
    return (r * codes.to(torch.float32)) / torch.tensor(float(bins), dtype=torch.float32,
                                                       device=codes.device) + z


def pack_codes(codes: torch.Tensor, bits: int) -> torch.Tensor:
    """quantize.py:213-233: LSB-first, rows padded to a byte boundary."""
    if bits not in (1, 2, 4, 8):
        raise EncodingError(f"packing supports 1/2/4/8 bits, got {bits}")
    if codes.dim() != 2 or codes.dtype != torch.uint8:
        raise TypeError("codes must be a 2-D uint8 tensor")
    _lib.require_cuda(codes)
    rows, cols = codes.shape
    codes = codes.contiguous()
    out = torch.empty((rows, packed_group_bytes(cols, bits)), dtype=torch.uint8, device=codes.device)
    overflow = torch.zeros(1, dtype=torch.int32, device=codes.device)
    st = _lib.load().kgq_pack_codes(codes.data_ptr(), rows, cols, bits, out.data_ptr(),
                                    overflow.data_ptr(), _lib.stream_ptr(codes.device))
    _lib.check(st, "kgq_pack_codes", {_lib.KGQ_ERR_UNSUPPORTED_BITS: EncodingError})
    if int(overflow.item()):
        raise EncodingError(f"code {int(codes.max())} does not fit in {bits} bits")
    return out


def unpack_codes(packed: torch.Tensor, bits: int, cols: int) -> torch.Tensor:
    """quantize.py:236-247."""
    if packed.dim() != 2 or packed.dtype != torch.uint8:
        raise TypeError("packed must be a 2-D uint8 tensor")
    _lib.require_cuda(packed)
    rows = packed.shape[0]
    if packed.shape[1] != packed_group_bytes(cols, bits):
        raise ValueError("packed width does not match cols/bits")
    packed = packed.contiguous()
    out = torch.empty((rows, cols), dtype=torch.uint8, device=packed.device)
    st = _lib.load().kgq_unpack_codes(packed.data_ptr(), rows, cols, bits, out.data_ptr(),
                                      _lib.stream_ptr(packed.device))
    _lib.check(st, "kgq_unpack_codes", {_lib.KGQ_ERR_UNSUPPORTED_BITS: EncodingError})
    return out


def pack_bits(codes, bits: int, device=None) -> torch.Tensor:
    """quantize.py:250-253."""
    c = torch.as_tensor(codes, dtype=torch.uint8, device=device or "cuda")
    return pack_codes(c.reshape(1, -1), bits)[0]


def unpack_bits(packed, bits: int, count: int, device=None) -> torch.Tensor:
    """quantize.py:256-258."""
    p = torch.as_tensor(packed, dtype=torch.uint8, device=device or "cuda")
    return unpack_codes(p.reshape(1, -1), bits, count)[0]


def stored_bytes(q: QuantizedTensor) -> int:
    """quantize.py:261-272 ledger: per group ceil(G*b/8) + 8 bytes; b=32: 4/elem."""
    if q.bits == PASSTHROUGH_BITS:
        return q.rows * q.cols * 4
    return q.n_groups * (packed_group_bytes(q.group_size, q.bits) + 8)


def fp32_equivalent_bytes(q: QuantizedTensor) -> int:
    """quantize.py:275-277."""
    return q.rows * q.cols * 4


def fast_noise_u16(seed: int, tensor_id: int, n_groups: int, group: int, group_offset: int = 0,
                   device=None) -> torch.Tensor:
    """The fast-mode draws a quantize call consumes (u = value / 65536)."""
    dev = torch.device("cuda") if device is None else torch.device(device)
    out = torch.empty((n_groups, group), dtype=torch.int16, device=dev)
    st = _lib.load().kgq_fast_noise_u16(int(seed) & 0xFFFFFFFFFFFFFFFF,
                                        int(tensor_id) & 0xFFFFFFFFFFFFFFFF, group_offset,
                                        n_groups, group, out.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_fast_noise_u16")
    return out.to(torch.int32) & 0xFFFF


def compat_noise_raw53(seed: int, tensor_id: int, n_groups: int, group: int, group_offset: int = 0,
                       device=None) -> torch.Tensor:
    """The compat-mode draws (u = value * 2^-53), equal to numpy's stream."""
    dev = torch.device("cuda") if device is None else torch.device(device)
    out = torch.empty((n_groups, group), dtype=torch.int64, device=dev)
    st = _lib.load().kgq_compat_noise_raw53(int(seed) & 0xFFFFFFFFFFFFFFFF,
                                            int(tensor_id) & 0xFFFFFFFFFFFFFFFF, group_offset,
                                            n_groups, group, out.data_ptr(), _lib.stream_ptr(dev))
    _lib.check(st, "kgq_compat_noise_raw53")
    return out
