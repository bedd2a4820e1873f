"""GPU parity of the Top-K evaluation (K11 kgq_topk_rows_f32 + train.evaluate)
against the stable argsort of the reference (train.py:141-143, restated in
oracle.topk_stable) and against kgact.train.evaluate's own numbers
(tests/golden/make_eval_golden.py)."""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from tests import golden_io

pytestmark = pytest.mark.gpu


def _topk(s: np.ndarray, k: int) -> np.ndarray:
    from paper_2212_04540_b200 import functional as F
    return F.topk_rows(torch.from_numpy(np.ascontiguousarray(s, dtype=np.float32)).cuda(), k).cpu().numpy()


def _expect(s: np.ndarray, k: int) -> np.ndarray:
    want = orc.topk_stable(s.astype(np.float64), k)
    if want.shape[1] < k:     # rows shorter than k: -1 past the end
        want = np.concatenate([want, -np.ones((s.shape[0], k - want.shape[1]), np.int64)], 1)
    return want


@pytest.mark.parametrize("k", [1, 5, 16, 20, 32, 33, 64])
@pytest.mark.parametrize("cols", [1, 31, 128, 129, 1000, 24915])
def test_topk_rows_matches_stable_argsort(k, cols):
    rng = np.random.default_rng(k * 100003 + cols)
    rows = 37
    s = rng.standard_normal((rows, cols)).astype(np.float32)
    s[::3] = np.round(s[::3] * 2) / 2                      # heavy ties
    s[1::5] = 0.0
    s[1::5, ::2] = -0.0                                    # -0.0 == +0.0: index order
    s[2::7, rng.integers(0, cols, size=max(1, cols // 3))] = -np.inf   # masked positives
    s[4::9, rng.integers(0, cols, size=max(1, cols // 5))] = np.nan
    got = _topk(s, k)
    np.testing.assert_array_equal(got, _expect(s, k))


def test_topk_rows_all_masked_and_strided():
    from paper_2212_04540_b200 import functional as F
    rng = np.random.default_rng(5)
    base = rng.standard_normal((40, 700)).astype(np.float32)
    base[3] = -np.inf                                      # every item masked: index order
    base[4] = 1.0                                          # all tied
    t = torch.from_numpy(base).cuda()
    view = t[:, 50:650]                                    # row stride 700 > 600 columns
    got = F.topk_rows(view, 20).cpu().numpy()
    np.testing.assert_array_equal(got, _expect(base[:, 50:650], 20))
    assert got[3].tolist() == list(range(20)) and got[4].tolist() == list(range(20))


def test_topk_rows_rejects_bad_k():
    from paper_2212_04540_b200 import _lib
    from paper_2212_04540_b200 import functional as F
    s = torch.zeros(4, 10, device="cuda")
    for k in (0, -1):
        with pytest.raises(ValueError):
            F.topk_rows(s, k)
    # the K11 kernel itself takes 1 <= k <= 64; larger K ranks by a stable sort
    out = torch.empty((4, 65), dtype=torch.int32, device="cuda")
    st = _lib.load().kgq_topk_rows_f32(s.data_ptr(), 4, 10, 10, 65, out.data_ptr(), _lib.stream_ptr())
    assert st == _lib.KGQ_ERR_INVALID_ARG


@pytest.mark.parametrize("name", ["int", "gauss"])
def test_evaluate_matches_reference_golden(name):
    """train.evaluate on the GPU == kgact.train.evaluate.  The integer readout
    makes every fp32 score exact under any summation order (bit-exact ranking,
    many ties); the Gaussian one relies on cuBLAS and numpy agreeing on the
    ranking (d = 16, no near-ties at this size)."""
    from paper_2212_04540_b200.data import KgDataset
    from paper_2212_04540_b200.train import evaluate
    z = golden_io.load("eval")
    nu, ni = int(z["num_users"]), int(z["num_items"])
    readout = z[f"readout_{name}"]
    ne = readout.shape[0] - nu
    ds = KgDataset(nu, ni, ne, z["train"], np.zeros((0, 2), np.int32), z["test"],
                   np.zeros((0, 3), np.int32), 1)
    r = torch.from_numpy(readout).cuda()
    for k, want in zip(z["ks"], z[f"metrics_{name}"]):
        got = evaluate(ds, r, int(k))
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


def test_evaluate_duplicate_test_pairs_and_chunking():
    """Duplicate test pairs count once (the reference's ``set(test_pos[u])``)
    and the user chunking does not change the result (oracle.evaluate)."""
    from paper_2212_04540_b200.data import KgDataset
    from paper_2212_04540_b200.train import evaluate
    z = golden_io.load("eval")
    nu, ni = int(z["num_users"]), int(z["num_items"])
    readout = z["readout_int"]
    test = np.concatenate([z["test"], z["test"][::4]], 0)
    ds = KgDataset(nu, ni, readout.shape[0] - nu, z["train"], np.zeros((0, 2), np.int32), test,
                   np.zeros((0, 3), np.int32), 1)
    want = orc.evaluate(nu, ni, z["train"], test, readout, 20)
    r = torch.from_numpy(readout).cuda()
    for chunk in (None, 7, 64):
        np.testing.assert_allclose(evaluate(ds, r, 20, chunk=chunk), want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("d", [32, 64])
@pytest.mark.parametrize("k", [1, 7, 20, 32])
@pytest.mark.parametrize("n_items", [1, 130, 1000, 24915])
def test_score_topk_fused_matches_stable_argsort(d, k, n_items):
    """K12 (kgq_score_topk_f32) == s = U . I^T; s[train] = -inf;
    np.argsort(-s, kind="stable")[:k] (train.py:137-143).  Integer-valued
    embeddings make every score exact (ties by index decide the order); item
    rows with NaN give NaN scores (ranked last), an all-zero user ties every
    item at +-0."""
    from paper_2212_04540_b200 import functional as F
    rng = np.random.default_rng(d * 1000 + k * 17 + n_items)
    n_users = 300
    U = rng.integers(-3, 4, (n_users + 11, d)).astype(np.float32)
    U[5] = 0.0
    items = rng.integers(-3, 4, (n_items, d)).astype(np.float32)
    if n_items > 10:
        items[rng.integers(0, n_items, 3)] = np.nan
    users = np.sort(rng.choice(n_users + 11, n_users, replace=False)).astype(np.int64)
    tr_items, tr_start, tr_end = [], [], []
    for i in range(n_users):
        m = int(rng.integers(0, min(n_items, 40) + 1)) if i % 9 else min(n_items, 5 * k)
        its = np.sort(rng.choice(n_items, m, replace=False))
        tr_start.append(len(tr_items)); tr_items.extend(its.tolist()); tr_end.append(len(tr_items))
    s = U[users].astype(np.float64) @ items.astype(np.float64).T
    for i in range(n_users):
        s[i, tr_items[tr_start[i]:tr_end[i]]] = -np.inf
    want = _expect(s, k)
    dev = lambda a, t: torch.from_numpy(np.asarray(a, dtype=t)).cuda()
    got = F.score_topk(dev(U, np.float32), dev(users, np.int64), dev(items, np.float32),
                       dev(tr_items if tr_items else [0], np.int32), dev(tr_start, np.int64),
                       dev(tr_end, np.int64), k).cpu().numpy()
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("k", [5, 20])
def test_evaluate_fused_equals_score_block_path(k):
    """train.evaluate with K12 == the score-block path (cuBLAS scores + K11),
    on the BASELINE configs[0] dataset with an integer-valued d = 64 readout
    (exact scores under either summation order), and == oracle.evaluate."""
    from paper_2212_04540_b200 import data as D
    from paper_2212_04540_b200.train import evaluate
    ds = D.reference_dataset("default")
    rng = np.random.default_rng(k)
    readout = rng.integers(-2, 3, (ds.num_nodes, 64)).astype(np.float32)
    r = torch.from_numpy(readout).cuda()
    a = evaluate(ds, r, k, fused=True)
    b = evaluate(ds, r, k, fused=False)
    want = orc.evaluate(ds.num_users, ds.num_items, ds.train, ds.test, readout, k)
    np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    np.testing.assert_allclose(a, want, rtol=0, atol=1e-12)
