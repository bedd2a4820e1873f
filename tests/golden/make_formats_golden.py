"""Generate the on-disk-format fixtures in tests/golden/formats/ by running
the REFERENCE (kgact, read-only from /root/reference/pkg/src):

    python tests/golden/make_formats_golden.py

* synth/      -- kgact.data.save_dataset of a small synth_generate dataset
                 (TSV + the four vocabulary sidecars, data.py:413-436)
* raw/        -- hand-written interactions/triples TSV without sidecars
                 (string ids, a duplicate pair), the first-seen-order path
* ckpt.kgact  -- kgact.checkpoint.save_checkpoint of init_params (KGACTCK1)
* expected.npz -- what the reference's loaders return for those inputs
                 (load_dataset splits with two seeds and a k-core, the
                 vocabularies as JSON, split_interactions / kcore_filter on a
                 random pair list, the checkpoint arrays and meta)
"""
import json
import os
import shutil
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "formats")
sys.path.insert(0, "/root/reference/pkg/src")

from kgact import data as kd  # noqa: E402
from kgact.checkpoint import load_checkpoint, save_checkpoint  # noqa: E402
from kgact.model import ModelConfig, init_params  # noqa: E402

RAW_INTERACTIONS = """alice\tbook7
bob\tbook2
alice\tbook2
carol\tbook9
alice\tbook7
bob\tbook9
dave\tbook2
carol\tbook7
alice\tbook1
bob\tbook1
carol\tbook1
carol\tbook2
dave\tbook7
dave\tbook9
"""
RAW_TRIPLES = """book7\tauthor\tann
book2\tgenre\tscifi
book9\tauthor\tann
book1\tgenre\tdrama
ann\tborn_in\tparis
"""


def ds_arrays(prefix, ds):
    return {prefix + "train": ds.train, prefix + "val": ds.val, prefix + "test": ds.test,
            prefix + "triples": ds.triples,
            prefix + "sizes": np.array([ds.num_users, ds.num_items, ds.num_entities]),
            prefix + "vocabs": np.array(json.dumps([ds.user_vocab, ds.entity_vocab, ds.relation_vocab]))}


def main():
    if os.path.exists(OUT):
        shutil.rmtree(OUT)
    os.makedirs(OUT)
    spec = kd.parse_synth_spec("default,users=60,items=40,entities=120,relations=4,groups=4,"
                               "interactions_per_user=6,attr_links_per_item=2")
    ds = kd.synth_generate(spec, seed=2)
    kd.save_dataset(ds, os.path.join(OUT, "synth"))
    raw = os.path.join(OUT, "raw")
    os.makedirs(raw)
    with open(os.path.join(raw, "interactions.tsv"), "w") as fh:
        fh.write(RAW_INTERACTIONS)
    with open(os.path.join(raw, "triples.tsv"), "w") as fh:
        fh.write(RAW_TRIPLES)

    exp = {}
    exp.update(ds_arrays("synth_s3_", kd.load_dataset(os.path.join(OUT, "synth"), seed=3)))
    exp.update(ds_arrays("synth_s3_k2_", kd.load_dataset(os.path.join(OUT, "synth"), seed=3, kcore=2)))
    exp.update(ds_arrays("raw_s5_", kd.load_dataset(raw, seed=5)))
    rng = np.random.default_rng(11)
    pairs = np.unique(np.stack([rng.integers(0, 30, 400), rng.integers(0, 50, 400)], 1), axis=0)
    pairs = pairs[rng.permutation(len(pairs))].astype(np.int32)
    exp["split_pairs"] = pairs
    tr, va, te = kd.split_interactions(pairs, seed=7)
    exp.update(split_train=tr, split_val=va, split_test=te)
    exp["kcore3"] = kd.kcore_filter(pairs, 3)

    params = init_params(50, ModelConfig(layers=2, dim=8), seed=1)
    meta = {"epoch": 4, "bits": 2, "note": "golden", "recall@20": 0.125}
    save_checkpoint(os.path.join(OUT, "ckpt.kgact"), params, meta)
    back, meta2 = load_checkpoint(os.path.join(OUT, "ckpt.kgact"))
    for k, v in back.as_dict().items():
        exp["ckpt_" + k] = v
    exp["ckpt_meta"] = np.array(json.dumps(meta2, sort_keys=True))
    np.savez_compressed(os.path.join(OUT, "expected.npz"), **exp)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
