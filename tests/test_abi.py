"""The C ABI boundary on CPU: libkgq.so loads, exports every entry point
include/kgq.h declares, and the ctypes signatures the host layer binds have
the header's arity.  No compute calls (no GPU here) beyond the ones that must
fail loudly without a device."""
import ctypes
import re
from pathlib import Path

import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "kgq.h"


def _declarations():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)           # strip comments
    decls = {}
    for m in re.finditer(r"KGQ_API\s+[\w\s\*]+?\b(kgq_\w+)\s*\(([^)]*)\)\s*;", text, flags=re.S):
        name, params = m.group(1), m.group(2).strip()
        n = 0 if params in ("", "void") else len([p for p in params.split(",") if p.strip()])
        decls[name] = n
    return decls


def test_header_declares_the_entry_points():
    decls = _declarations()
    for name in ("kgq_quantize_f32", "kgq_dequantize_f32", "kgq_spmm_csr_f32", "kgq_layer_forward_f32",
                 "kgq_layer_backward_f32", "kgq_quantize_host_f32", "kgq_dequantize_host_f32"):
        assert name in decls, name


def test_library_exports_every_declared_symbol():
    from paper_2212_04540_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declarations() if not hasattr(lib, n)]
    assert not missing, f"declared in kgq.h but not exported: {missing}"


def test_ctypes_signatures_match_header_arity():
    from paper_2212_04540_b200 import _lib
    decls = _declarations()
    for name, (_, args) in _lib.SIGNATURES.items():
        assert name in decls, f"{name} bound but not declared in kgq.h"
        assert len(args) == decls[name], f"{name}: ctypes {len(args)} args, header {decls[name]}"
    unbound = sorted(set(decls) - set(_lib.SIGNATURES))
    assert not unbound, f"declared but not bound by the host layer: {unbound}"


def test_status_strings_and_version():
    from paper_2212_04540_b200 import _lib
    L = _lib.load()
    assert L.kgq_version() > 0
    for st in range(0, 6):
        assert L.kgq_status_string(st)
    # argument validation happens before any device work
    assert L.kgq_quantize_f32(None, 1, 64, 3, 0, 0, 0, None, 0, None, None, None, None, None) \
        == _lib.KGQ_ERR_UNSUPPORTED_BITS
    assert L.kgq_host_workspace_bytes(0, 64, 2, 3) == 0
    assert L.kgq_host_workspace_bytes(1000, 64, 2, 3) >= 3 * 1000 * (64 * 4 + 16 + 8)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-device behaviour")
def test_host_path_without_gpu_raises_not_falls_back():
    import paper_2212_04540_b200 as kgq
    x = torch.randn(64, 64)
    cfg = kgq.QuantConfig(bits=2, rng="fast")
    with pytest.raises(Exception):
        kgq.quantize_tensor(x, cfg, kgq.RandomStream(1), tensor_id=0)
