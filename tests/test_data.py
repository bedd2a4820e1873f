"""Host-side input formats (the caller side of the hot path) vs the reference."""
import numpy as np

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
