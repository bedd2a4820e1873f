"""ctypes binding of libkgq.so (include/kgq.h), the sm_100a kernels.

The library is built in-tree (``paper_2212_04540_b200/libkgq.so``, by
``__graft_entry__.build()`` or ``make -C paper_2212_04540_b200/csrc``).
There is no CPU fallback: if the library is missing or no CUDA device is
present, every op raises instead of silently computing something else.
"""

import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkgq.so")

KGQ_OK = 0
KGQ_ERR_INVALID_ARG = 1
KGQ_ERR_UNSUPPORTED_BITS = 2
KGQ_ERR_CUDA = 3
KGQ_ERR_MISALIGNED = 4
KGQ_ERR_SHAPE = 5

ROUND_NEAREST = 0
ROUND_SR_FAST = 1
ROUND_SR_COMPAT = 2
ROUND_SR_NOISE = 3

# (name, restype, argtypes) -- must match include/kgq.h
_P = ctypes.c_void_p
_I64, _U64, _I32, _SZ = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int32, ctypes.c_size_t
SIGNATURES = {
    "kgq_version": (ctypes.c_int, []),
    "kgq_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "kgq_last_cuda_error": (ctypes.c_int, []),
    "kgq_quantize_f32": (ctypes.c_int, [_P, _I64, _I32, _I32, _I32, _U64, _U64, _P, _I64, _P, _P, _P, _P, _P]),
    "kgq_dequantize_f32": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _P, _P]),
    "kgq_host_workspace_bytes": (ctypes.c_size_t, [_I64, _I32, _I32, _I32]),
    "kgq_quantize_host_f32": (ctypes.c_int, [_P, _I64, _I32, _I32, _I32, _U64, _U64, _I64, _P, _P, _P,
                                              _P, ctypes.c_size_t, _P, _I32, _P]),
    "kgq_dequantize_host_f32": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _P, _P, ctypes.c_size_t,
                                                _P, _I32, _P]),
    "kgq_fast_noise_u16": (ctypes.c_int, [_U64, _U64, _I64, _I64, _I32, _P, _P]),
    "kgq_compat_noise_raw53": (ctypes.c_int, [_U64, _U64, _I64, _I64, _I32, _P, _P]),
    "kgq_pack_codes": (ctypes.c_int, [_P, _I64, _I32, _I32, _P, _P, _P]),
    "kgq_unpack_codes": (ctypes.c_int, [_P, _I64, _I32, _I32, _P, _P]),
    "kgq_spmm_csr_f32": (ctypes.c_int, [_P, _P, _P, _I64, _P, _I64, _P, _I32, _P, _P]),
    "kgq_relu_mask_f32": (ctypes.c_int, [_P, _I64, _P, _P, _P]),
    "kgq_mask_apply_f32": (ctypes.c_int, [_P, _P, _I64, _P, _P]),
    "kgq_dequant_gemm_workspace_bytes": (_SZ, [_I64, _I32]),
    "kgq_dequant_gemm_tn_f32": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _I32, _P, _P, _P, _SZ, _I32, _P]),
    "kgq_adam_step_f32": (ctypes.c_int, [_P, _P, _P, _P, _I64, ctypes.c_double, ctypes.c_double,
                                         ctypes.c_double, ctypes.c_double, _I64, _P, _P]),
    "kgq_adam_step_dev_f32": (ctypes.c_int, [_P, _P, _P, _P, _I64, ctypes.c_double, ctypes.c_double,
                                             ctypes.c_double, ctypes.c_double, _P, _P, _P, _P]),
    "kgq_check_finite_f32": (ctypes.c_int, [_P, _P, _I32, _I32, _P, _I64, _P, _P]),
    "kgq_rowmm_f32": (ctypes.c_int, [_P, _I64, _I32, _P, _I32, _P, _P]),
    "kgq_layer_backward_workspace_bytes": (_SZ, [_I64, _I32]),
    "kgq_layer_backward_f32": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P, _P,
                                              _SZ, _I32, _P]),
    "kgq_layer_forward_f32": (ctypes.c_int, [_P, _P, _P, _I64, _P, _I64, _P, _I32, _P, _I32, _I32, _U64, _U64,
                                             _P, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "kgq_layer_epilogue_f32": (ctypes.c_int, [_P, _I64, _I32, _P, _I32, _I32, _U64, _U64, _P, _I64, _P, _P,
                                              _P, _P, _P, _P]),
    "kgq_bpr_forward_workspace_bytes": (_SZ, [_I64]),
    "kgq_bpr_forward_f32": (ctypes.c_int, [_P, _P, _P, _I64, _I32, ctypes.c_float, _P, _P, _P, _SZ, _P]),
    "kgq_bpr_backward_f32": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I32, ctypes.c_float, _P, _P, _P, _P]),
    "kgq_scatter_rows_multi_f32": (ctypes.c_int, [_P, _P, _I64, _P, _I32, _P, _I32, _P, _P]),
    "kgq_gather_rows_sum_f32": (ctypes.c_int, [_P, _I32, _P, _I64, _I32, _P, _P]),
    "kgq_gather_rows_acc_f32": (ctypes.c_int, [_P, _P, _I32, _P, _I64, _I32, _P, _P]),
    "kgq_topk_rows_f32": (ctypes.c_int, [_P, _I64, _I64, _I64, _I32, _P, _P]),
    "kgq_spmm_csr_seg_f32": (ctypes.c_int, [_P, _P, _P, _I64, _P, _I64, _P, _P, _P, _I32, _P, _P]),
    "kgq_batch_indices": (ctypes.c_int, [_P, _I64, _I64, _P, _P, _P]),
    "kgq_scatter_rows_multi_sparse_f32": (ctypes.c_int, [_P, _I64, _P, _I32, _P, _I32, _P, _P, _P]),
    "kgq_layer_backward_rows_f32": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _P, _P, _P, _P,
                                                    _SZ, _I32, _P]),
    "kgq_counters_add": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _I64, _P]),
    "kgq_score_topk_workspace_bytes": (_SZ, [_I64, _I32]),
    "kgq_score_topk_f32": (ctypes.c_int, [_P, _P, _I64, _P, _I64, _I32, _P, _P, _P, _I32, _P, _P, _SZ, _P]),
}

_lib = None


class KgqError(RuntimeError):
    pass


def load():
    """Load libkgq.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libkgq.so not built at {LIB_PATH}; run __graft_entry__.build() "
                              f"or make -C {os.path.join(HERE, 'csrc')}")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    L = load()
    return [n for n in SIGNATURES if hasattr(L, n)]


def check(status: int, what: str, exc_map=None) -> None:
    if status == KGQ_OK:
        return
    msg = load().kgq_status_string(status).decode()
    if exc_map and status in exc_map:
        raise exc_map[status](f"{what}: {msg}")
    if status in (KGQ_ERR_INVALID_ARG, KGQ_ERR_UNSUPPORTED_BITS, KGQ_ERR_MISALIGNED):
        raise ValueError(f"{what}: {msg}")
    raise KgqError(f"{what}: {msg}")


def require_cuda(*tensors) -> None:
    for t in tensors:
        if t is not None and not t.is_cuda:
            raise ValueError("libkgq ops take CUDA tensors (no CPU fallback); got a "
                             f"{t.device} tensor")


def ptr(t):
    return None if t is None else t.data_ptr()


def stream_ptr(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream
