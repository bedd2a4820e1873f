"""Loaders for the committed golden fixtures (generated from the reference
by tests/golden/make_golden.py)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
MODE_NAMES = {0: "nearest", 1: "fast", 2: "compat"}


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def quant_cases():
    z = load("quant")
    for i in range(int(z["n_cases"])):
        p = f"c{i}_"
        g, bits, mode = (int(v) for v in z[p + "meta"])
        seed, tid = (int(v) for v in z[p + "seed_tid"])
        yield dict(idx=i, x=z[p + "x"], group=g, bits=bits, mode=mode, seed=seed, tid=tid,
                   codes=z[p + "codes"], ranges=z[p + "ranges"], offsets=z[p + "offsets"],
                   deq=z[p + "deq"], stored_bytes=int(z[p + "stored_bytes"]))


def special_cases():
    """IEEE special-value cases (quant_special.npz): +-0, subnormals, +-inf, NaN."""
    z = load("quant_special")
    for i in range(int(z["n_cases"])):
        p = f"c{i}_"
        g, bits, mode = (int(v) for v in z[p + "meta"])
        seed, tid = (int(v) for v in z[p + "seed_tid"])
        yield dict(idx=i, x=z[p + "x"], group=g, bits=bits, mode=mode, seed=seed, tid=tid,
                   codes=z[p + "codes"], ranges=z[p + "ranges"], offsets=z[p + "offsets"],
                   deq=z[p + "deq"], stored_bytes=int(z[p + "stored_bytes"]))


def mixed_zero_groups(x, group):
    """Groups whose min or max is a zero while holding both +0.0 and -0.0: numpy's
    SIMD min/max reduction order (not the data) picks the sign of that zero, so
    only there the sign of R/Z (and of the R == 0 dequantized value) is free."""
    v = np.asarray(x, dtype=np.float32).reshape(-1, group)
    zero = v == 0
    mixed = (zero & np.signbit(v)).any(1) & (zero & ~np.signbit(v)).any(1)
    with np.errstate(invalid="ignore"):
        ext0 = (np.nanmin(v, 1) == 0) | (np.nanmax(v, 1) == 0)
    return mixed & ext0


def same_bits(a, b, free_zero_sign=None):
    """Bitwise fp32 equality with NaN == NaN (payloads are platform-defined:
    x86 numpy keeps the input's, the GPU's min.NaN returns the canonical one)
    and, on rows flagged in ``free_zero_sign``, +0.0 == -0.0."""
    a = np.array(a, dtype=np.float32, copy=True)
    b = np.array(b, dtype=np.float32, copy=True)
    if a.shape != b.shape:
        return False
    both_nan = np.isnan(a) & np.isnan(b)
    a[both_nan] = 0
    b[both_nan] = 0
    if free_zero_sign is not None:
        rows = np.asarray(free_zero_sign).reshape(a.shape[0], *([1] * (a.ndim - 1)))
        rows = np.broadcast_to(rows, a.shape)
        zz = rows & (a == 0) & (b == 0)
        a[zz] = 0
        b[zz] = 0
    return bool(np.array_equal(a.view(np.uint32), b.view(np.uint32)))
