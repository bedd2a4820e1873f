"""Write the Last-FM- and Amazon-book-shaped datasets produced by the
REFERENCE generator (kgact.data.synth_generate, data.py:356-411, seed 0) with
the spec overrides of SURVEY.md 8(d), in the compact lossless codec of
``paper_2212_04540_b200.data.pack_dataset``.

Run in the build container (the only place /root/reference exists):

    python datasets/make_reference_datasets.py amazon lastfm

The reference generator is a Python loop (~3 min at Amazon shape, ~6-8 min at
Last-FM shape), so its output is committed; the GPU box reads these files and
never /root/reference.  ``data.reference_dataset(name)`` loads them.
"""
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(HERE))

from kgact.data import parse_synth_spec, synth_generate  # noqa: E402

from paper_2212_04540_b200 import data as D  # noqa: E402

SPECS = {
    "default": "default",     # the reference's acceptance-test dataset (test_acceptance.py:44-45)
    "amazon": "default,users=70679,items=24915,entities=88572,relations=39,"
              "interactions_per_user=12,attr_links_per_item=101.7",
    "lastfm": "default,users=23566,items=48123,entities=58266,relations=9,"
              "interactions_per_user=128.8,attr_links_per_item=8.66",
}


def main(names):
    for name in names:
        t0 = time.time()
        ref = synth_generate(parse_synth_spec(SPECS[name]), seed=0)
        ds = D.KgDataset(ref.num_users, ref.num_items, ref.num_entities, ref.train, ref.val, ref.test,
                         ref.triples, len(ref.relation_vocab))
        path = os.path.join(HERE, f"{name}_seed0.npz")
        D.save_compact(ds, path)
        back = D.load_compact(path)
        for k in ("train", "val", "test", "triples"):
            assert (getattr(back, k) == getattr(ref, k)).all(), k
        print(f"{name}: {time.time() - t0:.0f}s, train {len(ref.train)}, test {len(ref.test)}, "
              f"triples {len(ref.triples)} -> {os.path.getsize(path) / 1e6:.2f} MB", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SPECS))
