"""paper_2212_04540_b200: B200-native (sm_100a) activation-compression hot path
of TinyKG (arXiv 2212.04540), a drop-in for the reference package ``kgact``.

Public names mirror kgact (/root/reference/pkg/src/kgact/__init__.py:9-25) for
the hot path: the quantizer API, the dense/sparse kernels, the compressed-
context Tape, the KGNN layer wrapper and the quantized autograd Functions.
Everything computes on CUDA through libkgq.so (include/kgq.h); there is no
CPU fallback.
"""

from . import _lib
from .quantize import (EncodingError, QuantConfig, QuantizedTensor, RandomStream,
                       compat_noise_raw53, dequantize_row, dequantize_tensor, empty_context, fast_noise_u16,
                       fp32_equivalent_bytes, nearest_round, pack_bits, pack_codes, quantize_row,
                       quantize_tensor, stochastic_round, stored_bytes, unpack_bits, unpack_codes)
from .tensorops import (CSR, BitMask, ShapeMismatchError, csr_nbytes, densify, make_csr, mm,
                        relu, spmm, spmm_t, validate_csr)
from .formats import (CheckpointError, ParseError, load_checkpoint, load_dataset, save_checkpoint,
                      save_dataset)

__version__ = "0.1.0"
