"""On-disk formats (dataset directory TSV + sidecars, KGACTCK1 checkpoints)
against fixtures written and read by the reference itself
(tests/golden/make_formats_golden.py).  CPU only."""
import filecmp
import json
import os

import numpy as np
import pytest
import torch

from paper_2212_04540_b200 import formats as F
from paper_2212_04540_b200.model import ModelParams

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "formats")


@pytest.fixture(scope="module")
def exp():
    return np.load(os.path.join(GOLD, "expected.npz"))


def _check_ds(ds, exp, prefix):
    for k in ("train", "val", "test", "triples"):
        a = getattr(ds, k)
        b = exp[prefix + k]
        assert a.dtype == np.int32 and np.array_equal(a.reshape(b.shape), b), k
    assert [ds.num_users, ds.num_items, ds.num_entities] == exp[prefix + "sizes"].tolist()
    uv, ev, rv = json.loads(str(exp[prefix + "vocabs"]))
    assert ds.user_vocab == uv and ds.entity_vocab == ev and ds.relation_vocab == rv


@pytest.mark.parametrize("kcore,prefix", [(0, "synth_s3_"), (2, "synth_s3_k2_")])
def test_load_dataset_with_sidecars_matches_reference(exp, kcore, prefix):
    ds = F.load_dataset(os.path.join(GOLD, "synth"), seed=3, kcore=kcore)
    _check_ds(ds, exp, prefix)


def test_load_dataset_first_seen_order_matches_reference(exp):
    _check_ds(F.load_dataset(os.path.join(GOLD, "raw"), seed=5), exp, "raw_s5_")


def test_save_dataset_is_byte_identical(tmp_path):
    ds = F.load_dataset(os.path.join(GOLD, "synth"), seed=3)
    F.save_dataset(ds, str(tmp_path))
    names = sorted(os.listdir(os.path.join(GOLD, "synth")))
    assert sorted(os.listdir(tmp_path)) == names
    for n in names:
        assert filecmp.cmp(os.path.join(GOLD, "synth", n), os.path.join(tmp_path, n), shallow=False), n


def test_split_and_kcore_match_reference(exp):
    tr, va, te = F.split_interactions(exp["split_pairs"], seed=7)
    assert np.array_equal(tr, exp["split_train"]) and np.array_equal(va, exp["split_val"])
    assert np.array_equal(te, exp["split_test"])
    assert np.array_equal(F.kcore_filter(exp["split_pairs"], 3), exp["kcore3"])
    with pytest.raises(ValueError):
        F.kcore_filter(exp["split_pairs"], 0)


def test_checkpoint_reads_reference_file_and_writes_identical_bytes(exp, tmp_path):
    params, meta = F.load_checkpoint(os.path.join(GOLD, "ckpt.kgact"), device="cpu")
    names = list(params.as_dict())
    assert names == ["E0", "theta0", "theta1"]
    for k, v in params.as_dict().items():
        assert v.dtype == torch.float32
        assert np.array_equal(v.numpy(), exp["ckpt_" + k])
    assert json.dumps(meta, sort_keys=True) == str(exp["ckpt_meta"])
    out = tmp_path / "again.kgact"
    F.save_checkpoint(str(out), params, meta)
    assert out.read_bytes() == open(os.path.join(GOLD, "ckpt.kgact"), "rb").read()


def test_checkpoint_errors(tmp_path):
    bad = tmp_path / "bad"
    bad.write_bytes(b"NOTACKPT" + b"\0" * 16)
    with pytest.raises(F.CheckpointError):
        F.load_checkpoint(str(bad), device="cpu")
    good = open(os.path.join(GOLD, "ckpt.kgact"), "rb").read()
    trunc = tmp_path / "trunc"
    trunc.write_bytes(good[:-5])
    with pytest.raises(F.CheckpointError):
        F.load_checkpoint(str(trunc), device="cpu")
    assert issubclass(F.CheckpointError, ValueError)


def test_parse_errors(tmp_path):
    (tmp_path / "interactions.tsv").write_text("u1\ti1\nbroken line\n")
    with pytest.raises(F.ParseError):
        F.load_dataset(str(tmp_path), seed=0)
    (tmp_path / "interactions.tsv").write_text("u1\ti1\n")
    (tmp_path / "triples.tsv").write_text("i1\trel\n")
    with pytest.raises(F.ParseError):
        F.load_dataset(str(tmp_path), seed=0)


def test_generated_graph_roundtrip(tmp_path):
    """A generated (vocab-less) graph saves with the reference's default
    names and loads back to the same graph."""
    from paper_2212_04540_b200 import data
    ds = data.synth_kg(data.SynthShape(users=50, items=30, entities=90, relations=3,
                                       interactions_per_user=5.0), seed=1)
    F.save_dataset(ds, str(tmp_path))
    back = F.load_dataset(str(tmp_path), seed=0)
    assert (back.num_users, back.num_items, back.num_entities) == (ds.num_users, ds.num_items, ds.num_entities)
    assert np.array_equal(back.triples, ds.triples)
    key = lambda a: np.sort(a[:, 0].astype(np.int64) * 1000 + a[:, 1])
    allp = lambda d: np.concatenate([d.train, d.val, d.test])
    assert np.array_equal(key(allp(back)), key(allp(ds)))


def test_half_fraction_row_and_verification_args():
    """quantize.py:343-355 (deterministic) and the argument checks of
    quantizer_verification (raised before any device work)."""
    from paper_2212_04540_b200 import verification as V
    r = V.half_fraction_row(3, 10)
    assert r[0] == 0 and r[-1] == 3 and np.allclose(r[1:-1] % 1, 0.5)
    assert np.array_equal(r[1:-1], (np.arange(8) % 3) + 0.5)
    with pytest.raises(ValueError):
        V.quantizer_verification(n_rows=0)
    with pytest.raises(ValueError):
        V.quantizer_verification(dim=2)
