"""Golden fixture for the Top-K evaluation (kgact/train.py:108-160), written
by running the REFERENCE in the build container:

    python tests/golden/make_eval_golden.py

A small reference-generated KG and two readouts: small integers (d = 8, every
score exact in fp32 whatever the summation order, many ties -> exercises the
index tie-break) and Gaussian fp32.  Stores kgact.train.evaluate's
(recall, ndcg) for k in KS.  Nothing at test time reads /root/reference."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from kgact.data import parse_synth_spec, synth_generate  # noqa: E402
from kgact.train import evaluate  # noqa: E402

KS = (1, 5, 20, 40)


def main():
    ds = synth_generate(parse_synth_spec("default,users=300,items=150,entities=400,relations=4,groups=6"), seed=3)
    rng = np.random.default_rng(11)
    readouts = {
        "int": rng.integers(-2, 3, size=(ds.num_nodes, 8)).astype(np.float32),
        "gauss": rng.standard_normal((ds.num_nodes, 16)).astype(np.float32),
    }
    out = {"num_users": ds.num_users, "num_items": ds.num_items, "train": ds.train, "test": ds.test,
           "ks": np.array(KS)}
    for name, r in readouts.items():
        out[f"readout_{name}"] = r
        out[f"metrics_{name}"] = np.array([evaluate(ds, r, k) for k in KS], dtype=np.float64)
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **out)
    print({k: v.tolist() for k, v in out.items() if k.startswith("metrics")})


if __name__ == "__main__":
    main()
