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
