"""Host-side input formats (the caller side of the hot path) vs the reference."""
import numpy as np
import pytest

from paper_2212_04540_b200 import data as D
from tests import golden_io


def _c1():
    z = golden_io.load("c1")
    ds = D.KgDataset(int(z["num_users"]), int(z["num_items"]), int(z["num_entities"]), z["train"],
                     z["val"], z["test"], z["triples"], int(z["num_relations"]))
    return ds, z


def test_adjacency_bit_identical_to_reference():
    ds, z = _c1()
    indptr, indices, vals = D.adjacency_arrays(ds)
    assert np.array_equal(indptr, z["adj_indptr"])
    assert np.array_equal(indices, z["adj_indices"])
    assert np.array_equal(vals.view(np.uint32), z["adj_data"].view(np.uint32))
    t = golden_io.load("tape")
    assert t["indptr"][-1] == len(t["indices"])


def test_negatives_and_order_identical_to_reference():
    ds, z = _c1()
    rng = np.random.default_rng(0)
    trip = D.sample_negatives(ds, rng)
    order = rng.permutation(len(trip))
    assert np.array_equal(trip[order], z["epoch0_triples"])


def test_synthetic_shapes_and_partition():
    ds = D.synth_kg(D.SynthShape(500, 300, 1000, relations=5), seed=1)
    assert ds.train[:, 1].max() < 300 and ds.triples[:, 2].max() < 1000
    indptr, indices, vals = D.adjacency_arrays(ds)
    n = ds.num_nodes
    assert indptr[-1] == len(indices) and len(indptr) == n + 1
    # symmetric (bitwise)
    import scipy.sparse as sp
    a = sp.csr_matrix((vals, indices, indptr), shape=(n, n))
    assert (a != a.T).nnz == 0
    for w in (1, 2, 4, 8):
        cuts = D.partition_rows(indptr, w)
        assert cuts[0] == 0 and cuts[-1] == n and np.all(np.diff(cuts) >= 0)
        parts = [D.row_block(indptr, indices, vals, cuts[i], cuts[i + 1]) for i in range(w)]
        assert sum(len(p[1]) for p in parts) == len(indices)
        nnz = [len(p[1]) for p in parts]
        assert max(nnz) <= indptr[-1] / w + np.diff(indptr).max() + 1


def test_industry_generator_blocks_equal_adjacency():
    """The chunked device generator (industry.py) at a small shape: its row
    blocks, concatenated, are bit-identical to adjacency_arrays of the same
    dataset (data.py:230-266 semantics), and its equal-nnz cuts match
    partition_rows."""
    from paper_2212_04540_b200.industry import IndustryGraph, IndustryShape
    sh = IndustryShape(users=3000, items=1200, entities=9000, relations=7, groups=13,
                       interactions_per_user=15.0, attr_links_per_item=6.0, user_chunk=700, item_chunk=250)
    g = IndustryGraph(sh, seed=5, device="cpu")
    ds = g.dataset()
    ds.validate()
    ip, ix, vv = D.adjacency_arrays(ds)
    deg = g.degrees()
    assert np.array_equal(np.diff(ip), deg.numpy())
    for world in (1, 3):
        cuts = g.partition(deg, world)
        assert np.array_equal(cuts, D.partition_rows(ip, world))
        parts = [g.row_block(int(cuts[r]), int(cuts[r + 1]), deg) for r in range(world)]
        assert np.array_equal(np.concatenate([p[1].numpy() for p in parts]), ix)
        vcat = np.concatenate([p[2].numpy() for p in parts])
        assert np.array_equal(vcat.view(np.uint32), vv.view(np.uint32))
        for r, p in enumerate(parts):
            lo, hi = int(cuts[r]), int(cuts[r + 1])
            assert np.array_equal(p[0].numpy(), ip[lo:hi + 1] - ip[lo])


def test_compact_codec_roundtrip():
    ds = D.synth_kg(D.SynthShape(300, 200, 700, relations=6), seed=2)
    # reference order: splits grouped by user, triples lexsorted
    for name in ("train", "test"):
        a = getattr(ds, name)
        setattr(ds, name, a[np.lexsort((a[:, 1], a[:, 0]))])
    z = D.pack_dataset(ds)
    back = D.unpack_dataset(z)
    for k in ("train", "val", "test", "triples"):
        assert np.array_equal(getattr(back, k), getattr(ds, k)), k
    shuffled = ds.train[::-1].copy()
    ds.train = shuffled
    with pytest.raises(ValueError):
        D.pack_dataset(ds)


def test_reference_datasets_match_survey_counts():
    """datasets/*_seed0.npz are the reference generator's output (SURVEY.md
    8 C3/C4 probe counts: Amazon nnz 6,425,569 / train 579,759)."""
    ds = D.reference_dataset("amazon")
    assert (ds.num_users, ds.num_items, ds.num_entities) == (70679, 24915, 88572)
    assert len(ds.train) == 579759
    ip, _, _ = D.adjacency_arrays(ds)
    assert int(ip[-1]) == 6425569


def test_industry_referenced_by_others_matches_blocks():
    """The halo send side from one streaming pass equals, for each other rank,
    the distinct local rows that rank's CSR block references."""
    import torch
    from paper_2212_04540_b200.industry import IndustryGraph, IndustryShape
    sh = IndustryShape(users=2000, items=800, entities=6000, relations=5, groups=11,
                       interactions_per_user=12.0, attr_links_per_item=5.0, user_chunk=500, item_chunk=200)
    g = IndustryGraph(sh, seed=2, device="cpu")
    deg = g.degrees()
    W = 3
    cuts = g.partition(deg, W)
    blocks = [g.row_block(int(cuts[r]), int(cuts[r + 1]), deg) for r in range(W)]
    for R in range(W):
        lo, hi = int(cuts[R]), int(cuts[R + 1])
        got = g.referenced_by_others(lo, hi, cuts).tolist()
        for q in range(W):
            if q == R:
                assert got[q] == 0
                continue
            cols = blocks[q][1].long()
            want = torch.unique(cols[(cols >= lo) & (cols < hi)]).numel()
            assert got[q] == want, (R, q)
