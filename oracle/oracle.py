"""CPU oracle for the activation-compression hot path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference`` arm) may import this module, and
only as the checker / CPU baseline.  The product package
(``paper_2212_04540_b200``) never imports it and has no CPU fallback.

Two layers:

* ``kgq_oracle.c`` (ctypes, built by ``oracle/Makefile``): bit-exact fp32
  restatement of the reference quantizer (quantize.py:177-247), numpy's
  Philox4x64-10 stream (quantize.py:61-102), our fast Philox4x32-7 noise,
  the ordered CSR SpMM (tensorops.py:37-50) and ReLU + bit mask
  (tensorops.py:57-92).
* numpy restatements of the dense engine (tape.py:193-253 accumulation order,
  mirrored from the reference's own tests/reference.py:16-86) used as the
  gradient oracle.

Parity of this oracle with the reference is pinned by tests/golden/*.npz,
which tests/golden/make_golden.py generates by running the reference itself.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libkgq_oracle.so")

MODE_NEAREST = 0
MODE_SR_FAST = 1
MODE_SR_COMPAT = 2
MODE_SR_NOISE = 3

_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with its Makefile (gcc, -ffp-contract=off)."""
    src = os.path.join(HERE, "kgq_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE])
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64, u64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        L.oracle_philox4x64_10.argtypes = [P, P, P]
        L.oracle_philox4x32_10.argtypes = [P, P, P]
        L.oracle_philox4x32_r.argtypes = [P, P, P, i32]
        L.oracle_fast_noise_u16.argtypes = [u64, u64, i64, i64, P]
        L.oracle_compat_noise_raw53.argtypes = [u64, u64, i64, i64, P]
        L.oracle_quantize.argtypes = [P, i64, i64, i32, i32, u64, u64, i64, P, P, P, P, i32]
        L.oracle_quantize.restype = i32
        L.oracle_dequantize.argtypes = [P, P, P, i64, i64, i32, P, i32]
        L.oracle_dequantize.restype = i32
        L.oracle_spmm_csr.argtypes = [P, P, P, i64, P, i64, P]
        L.oracle_relu_mask.argtypes = [P, i64, P, P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def philox4x64_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint64)
    k = np.ascontiguousarray(key, dtype=np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().oracle_philox4x64_10(_p(c), _p(k), _p(out))
    return out


def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def philox4x32(ctr, key, rounds: int):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_r(_p(c), _p(k), _p(out), rounds)
    return out


FAST_ROUNDS = 7     # the fast SR stream: Philox4x32-7


def fast_noise_u16(seed: int, tid: int, n_groups: int, group: int) -> np.ndarray:
    out = np.empty((n_groups, group), dtype=np.uint16)
    lib().oracle_fast_noise_u16(seed & (2**64 - 1), tid & (2**64 - 1), n_groups, group, _p(out))
    return out


def fast_uniforms(seed: int, tid: int, n_groups: int, group: int) -> np.ndarray:
    """The fast-mode noise as the float64 uniforms the reference compares."""
    return fast_noise_u16(seed, tid, n_groups, group).astype(np.float64) / 65536.0


def compat_noise_raw53(seed: int, tid: int, n_groups: int, group: int) -> np.ndarray:
    out = np.empty((n_groups, group), dtype=np.uint64)
    lib().oracle_compat_noise_raw53(seed & (2**64 - 1), tid & (2**64 - 1), n_groups, group, _p(out))
    return out


def packed_group_bytes(group: int, bits: int) -> int:
    return (group * bits + 7) // 8


def quantize(x: np.ndarray, group: int, bits: int, mode: int, seed: int = 0, tid: int = 0,
             noise: np.ndarray | None = None, threads: int = 1, group_offset: int = 0):
    """Oracle quantize over the (-1, group) view.  Returns (codes, ranges, offsets)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.size % group:
        raise ValueError("size not divisible by group")
    n_groups = x.size // group
    codes = np.empty((n_groups, packed_group_bytes(group, bits)), dtype=np.uint8)
    ranges = np.empty(n_groups, dtype=np.float32)
    offsets = np.empty(n_groups, dtype=np.float32)
    nz = None
    if noise is not None:
        nz = np.ascontiguousarray(noise, dtype=np.float64).reshape(n_groups, group)
    st = lib().oracle_quantize(_p(x), n_groups, group, bits, mode, seed & (2**64 - 1),
                               tid & (2**64 - 1), group_offset, _p(nz), _p(codes), _p(ranges), _p(offsets),
                               threads)
    if st:
        raise ValueError(f"oracle_quantize status {st}")
    return codes, ranges, offsets


def dequantize(codes, ranges, offsets, group: int, bits: int, threads: int = 1) -> np.ndarray:
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    ranges = np.ascontiguousarray(ranges, dtype=np.float32)
    offsets = np.ascontiguousarray(offsets, dtype=np.float32)
    n_groups = ranges.shape[0]
    out = np.empty((n_groups, group), dtype=np.float32)
    st = lib().oracle_dequantize(_p(codes), _p(ranges), _p(offsets), n_groups, group, bits,
                                 _p(out), threads)
    if st:
        raise ValueError(f"oracle_dequantize status {st}")
    return out


def spmm_csr(indptr, indices, vals, x) -> np.ndarray:
    indptr = np.ascontiguousarray(indptr, dtype=np.int32)
    indices = np.ascontiguousarray(indices, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = indptr.shape[0] - 1
    out = np.empty((n, x.shape[1]), dtype=np.float32)
    lib().oracle_spmm_csr(_p(indptr), _p(indices), _p(vals), n, _p(x), x.shape[1], _p(out))
    return out


def relu_mask(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty_like(x)
    mask = np.empty((x.size + 7) // 8, dtype=np.uint8)
    lib().oracle_relu_mask(_p(x), x.size, _p(out), _p(mask))
    return out, mask


# ---------------------------------------------------------------------------
# numpy dense engine (gradient oracle).  Restates the reference's reverse
# sweep (tape.py:193-253) with its accumulation order (tests/reference.py:
# 59-85): readout grad = (scat_n + scat_p) + scat_u, layer grad = g_read + g_e.
# ``deq`` optionally supplies the dequantized contexts that the compressed
# engine would use (H per layer, u/p/n blocks) so quantized runs can be
# checked with the same noise.
# ---------------------------------------------------------------------------

def _softplus(x):
    return np.logaddexp(0, x)


def _expit(x):
    return 1.0 / (1.0 + np.exp(-x))


def dense_step(e0, thetas, indptr, indices, vals, users, pos, neg, l2, aggregation="sum",
               h_hat=None, uph_hat=None, dtype=np.float64):
    """One forward+backward of the KGNN backbone (model.py:66-88) + BPR head
    (tape.py:154-183, backward :233-244).  Returns (loss, grads dict)."""
    import scipy.sparse as sp
    n = e0.shape[0]
    A = sp.csr_matrix((np.asarray(vals, dtype=dtype), indices, indptr), shape=(n, n))
    e = e0.astype(dtype)
    hs, js = [], []
    per_layer = []
    for i, th in enumerate(thetas):
        h = A @ e
        j = h @ th.astype(dtype)
        e = np.maximum(j, 0)
        hs.append(h)
        js.append(j)
        per_layer.append(e)
    if aggregation == "last":
        readout = per_layer[-1]
    else:
        readout = per_layer[0]
        for x in per_layer[1:]:
            readout = readout + x
    u, p, ng = readout[users], readout[pos], readout[neg]
    batch = u.shape[0]
    margins = (u * (p - ng)).sum(axis=1)
    loss = float(_softplus(-margins).mean() + l2 * ((u * u).sum() + (p * p).sum() + (ng * ng).sum()) / batch)
    if uph_hat is not None:
        uh, ph, nh = (b.astype(dtype) for b in uph_hat)
    else:
        uh, ph, nh = u, p, ng
    coef = (_expit(-margins) / batch)[:, None]
    reg = 2.0 * l2 / batch
    gu = -coef * (ph - nh) + reg * uh
    gp = -coef * uh + reg * ph
    gn = coef * uh + reg * nh
    scat_n = np.zeros_like(readout)
    np.add.at(scat_n, neg, gn)
    scat_p = np.zeros_like(readout)
    np.add.at(scat_p, pos, gp)
    scat_u = np.zeros_like(readout)
    np.add.at(scat_u, users, gu)
    g_read = (scat_n + scat_p) + scat_u
    L = len(thetas)
    layer_grads = [g_read] * L if aggregation != "last" else [None] * (L - 1) + [g_read]
    grads = {}
    g_e = None
    for i in range(L - 1, -1, -1):
        g = layer_grads[i]
        if g is None:
            g = g_e
        elif g_e is not None:
            g = g + g_e
        g_j = g * (js[i] > 0)
        hh = hs[i] if h_hat is None else h_hat[i].astype(dtype)
        grads[f"theta{i}"] = hh.T @ g_j
        g_h = g_j @ thetas[i].astype(dtype).T
        g_e = A.T @ g_h
    grads["E0"] = g_e
    return loss, grads


def adam_step(params: dict, grads: dict, m: dict, v: dict, t: int, lr: float,
              b1: float = 0.9, b2: float = 0.999, eps: float = 1e-8) -> None:
    """The reference's numpy Adam update (train.py:42-59), in place, float32."""
    for name, g in grads.items():
        mm, vv = m[name], v[name]
        mm *= b1
        mm += (1 - b1) * g
        vv *= b2
        vv += (1 - b2) * (g * g)
        m_hat = mm / (1 - b1 ** t)
        v_hat = vv / (1 - b2 ** t)
        params[name] -= lr * m_hat / (np.sqrt(v_hat) + eps)


# ---------------------------------------------------------------------------
# Evaluation (kgact/train.py:108-160), restated in numpy
# ---------------------------------------------------------------------------

def topk_stable(scores: np.ndarray, k: int) -> np.ndarray:
    """train.py:143: ``np.argsort(-s, kind="stable")[:k]`` per row (float64)."""
    s = np.asarray(scores, dtype=np.float64)
    return np.argsort(-s, axis=1, kind="stable")[:, :k]


def evaluate(num_users: int, num_items: int, train: np.ndarray, test: np.ndarray,
             readout: np.ndarray, k: int):
    """train.py:119-160: mean Recall@k / NDCG@k over the users with test
    pairs; train positives set to -inf before the stable ranking; readout
    scores in float32 (readout[u] @ item_emb.T), ranked in float64."""
    test_pos: dict[int, list[int]] = {}
    for u, i in np.asarray(test):
        test_pos.setdefault(int(u), []).append(int(i))
    train_pos: dict[int, set] = {}
    for u, i in np.asarray(train):
        train_pos.setdefault(int(u), set()).add(int(i))
    users = sorted(test_pos)
    if not users:
        raise ValueError("test split is empty")
    item_emb = readout[num_users:num_users + num_items]
    recalls, ndcgs = [], []
    for u in users:
        s = np.asarray(readout[u] @ item_emb.T, dtype=np.float64)
        held = sorted(train_pos.get(u, ()))
        if held:
            s[held] = -np.inf
        top = topk_stable(s[None, :], k)[0]
        pos = set(test_pos[u])
        hits = [r for r, item in enumerate(top, start=1) if int(item) in pos]
        recalls.append(len(hits) / len(pos))
        idcg = sum(1.0 / np.log2(r + 1) for r in range(1, min(len(pos), k) + 1))
        ndcgs.append(sum(1.0 / np.log2(r + 1) for r in hits) / idcg)
    return float(np.mean(recalls)), float(np.mean(ndcgs))
